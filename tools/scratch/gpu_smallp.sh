python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/sp_build.log 2>&1
for p in 12 16; do
SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg3:$p --reps 1 > gpurun_out/sp_ncu_$p.csv 2>&1
echo "p=$p"; grep -E "k_v7_(lines|assemble)" gpurun_out/sp_ncu_$p.csv | tail -12 | awk -F'","' '{print $5, $13, $15}' | cut -c1-120
done
