python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2q_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_loopback.py -q -p no:cacheprovider -x > gpurun_out/r2q_loop.log 2>&1
tail -3 gpurun_out/r2q_loop.log
