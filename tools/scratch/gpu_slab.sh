TAG=${TAG:-r2d1}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernel_families.py tests/test_gpu_loopback.py -q -p no:cacheprovider > gpurun_out/${TAG}_test.log 2>&1
tail -15 gpurun_out/${TAG}_test.log | cut -c1-300
