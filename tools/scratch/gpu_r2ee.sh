python -c "import __graft_entry__; __graft_entry__.build()" > /dev/null 2>&1
SC_OP=v7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_v7 -s 8 -c 3 -o gpurun_out/prof_v7_r2gg python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/r2gg_ncu.log 2>&1
tail -2 gpurun_out/r2gg_ncu.log
