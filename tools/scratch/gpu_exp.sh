python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/exp_build.log 2>&1
for E in none; do
SC_V7_EXP=$E SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5,cfg3:4 --reps 1 > gpurun_out/exp_$E.csv 2>&1
echo "exp $E"; grep -E "k_v7_assemble" gpurun_out/exp_$E.csv | awk -F'","' '{print $13, $15}' | cut -c1-80 | sed -n '1,3p;10,12p'
done
