python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/exp2_build.log 2>&1
for E in none store; do
SC_V7_EXP=$E SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/exp2_$E.csv 2>&1
echo "exp $E"; grep -E "k_v7_lines" gpurun_out/exp2_$E.csv | awk -F'","' '{print $13, $15}' | cut -c1-80 | tail -4
done
