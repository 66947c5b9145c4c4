TAG=r2bb
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
tail -4 gpurun_out/${TAG}_gputest.log
python -c "import __graft_entry__; __graft_entry__.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cut -c1-300 gpurun_out/bench_$TAG.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python tools/p_sweep.py --out gpurun_out/p_sweep_$TAG.json > gpurun_out/p_sweep_$TAG.log 2>&1; tail -2 gpurun_out/p_sweep_$TAG.log | cut -c1-200
bash tools/scratch/gpu_ncu.sh $TAG
