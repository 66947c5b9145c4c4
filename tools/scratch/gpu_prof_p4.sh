python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/p4_build.log 2>&1
SC_OP=v7 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_v7_assemble" -s 1 -c 1 -o gpurun_out/prof_p4 python tools/op_time.py --ops v7 --cases cfg3:4 --reps 1 > gpurun_out/p4_ncu.log 2>&1; echo "ncu rc=$?"
