python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2s_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s_gputest.log 2>&1
tail -4 gpurun_out/r2s_gputest.log
python tools/op_time.py --ops v3,v6 --cases cfg5,cfg3:8 --reps 10 > gpurun_out/r2s_optime.log 2>&1
cut -c1-160 gpurun_out/r2s_optime.log
for op in v3 v6; do
SC_OP=$op timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_${op}_r2s python tools/op_time.py --ops $op --cases cfg5 --reps 2 > gpurun_out/r2s_ncu_$op.log 2>&1
tail -1 gpurun_out/r2s_ncu_$op.log
done
python bench.py --steps 20 --warmup 3 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
cut -c1-400 gpurun_out/r2s_bench.json
