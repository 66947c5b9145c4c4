TAG=${TAG:-r2s1}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7_operator_parity" > gpurun_out/${TAG}_test.log 2>&1
tail -3 gpurun_out/${TAG}_test.log | cut -c1-300
python tools/op_time.py --ops v7,big --cases cfg3:16,cfg3:17,cfg3:20,cfg3:24 --reps 10 > gpurun_out/${TAG}_optime.log 2>&1
grep '^{' gpurun_out/${TAG}_optime.log | cut -c1-95
