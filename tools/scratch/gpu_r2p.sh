python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2p_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2p_gputest.log 2>&1
tail -8 gpurun_out/r2p_gputest.log
python tools/p_sweep.py --out gpurun_out/r2p_psweep.json > gpurun_out/r2p_psweep.log 2>&1
cat gpurun_out/r2p_psweep.log | cut -c1-200
python bench.py --steps 20 --warmup 3 > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
cat gpurun_out/r2p_bench.json | cut -c1-600
