TAG=${TAG:-r2qq}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${TAG}_gputest.log 2>&1
tail -4 gpurun_out/${TAG}_gputest.log | cut -c1-300
python -c "import __graft_entry__; __graft_entry__.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/bench_$TAG.json
