TAG=${TAG:-r2g1}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernel_families.py tests/test_gpu_loopback.py -q -p no:cacheprovider > gpurun_out/${TAG}_test.log 2>&1
tail -3 gpurun_out/${TAG}_test.log | cut -c1-300
python tools/op_time.py --ops v7 --cases ${CASES:-cfg5,cfg3:3,cfg3:4,cfg3:8,cfg3:12,cfg3:16} --reps 10 > gpurun_out/${TAG}_optime.log 2>&1
grep '^{' gpurun_out/${TAG}_optime.log | cut -c1-95
SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu.csv 2>&1
grep -E "k_v7_(lines|assemble|faces)" gpurun_out/${TAG}_ncu.csv | tail -15 | awk -F'","' '{print $5, $13, $15}' | cut -c1-120
python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench.json
