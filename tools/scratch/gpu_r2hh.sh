python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2hh_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" > gpurun_out/r2hh_test.log 2>&1
tail -25 gpurun_out/r2hh_test.log | cut -c1-300
python tools/op_time.py --ops v7,v3 --cases cfg5,cfg3:8 --reps 10 > gpurun_out/r2hh_optime.log 2>&1
cut -c1-150 gpurun_out/r2hh_optime.log
SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/r2hh_ncu.csv 2>&1
grep -E "k_v7" gpurun_out/r2hh_ncu.csv | tail -24 | cut -c1-220
