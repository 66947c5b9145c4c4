set -x
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2a_build.log 2>&1
python tools/fp64_peak.py > gpurun_out/r2a_fp64.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_gputest.log 2>&1
tail -5 gpurun_out/r2a_gputest.log
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
cat gpurun_out/r2a_bench.json
