TAG=${TAG:-r2mm}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" > gpurun_out/${TAG}_test.log 2>&1
tail -2 gpurun_out/${TAG}_test.log | cut -c1-300
for S in 1 2; do
SC_V7_STAGES=$S python tools/op_time.py --ops v7 --cases ${CASES:-cfg5,cfg3:8} --reps 10 > gpurun_out/${TAG}_optime_s$S.log 2>&1
echo "stages $S"; grep '^{' gpurun_out/${TAG}_optime_s$S.log | cut -c1-110
SC_V7_STAGES=$S SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu_s$S.csv 2>&1
grep -E "k_v7_(lines|assemble)" gpurun_out/${TAG}_ncu_s$S.csv | tail -10 | awk -F'","' '{print $5, $13, $15}' | cut -c1-150
done
