TAG=${TAG:-r2ll}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
SC_OP=v7 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_v7_(cond|assemble)" -s 2 -c 2 -o gpurun_out/prof_v7_${TAG} python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu_v7.log 2>&1; echo "ncu v7 rc=$?"
tail -3 gpurun_out/${TAG}_ncu_v7.log
