python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2o_build.log 2>&1
SC_OP=v6 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "operator_parity_nodal or multitile or zsegments or slab_rank or bitwise or pcg_parity_manufactured or pcg_parity_multitile or symmetry or cfg5_full" > gpurun_out/r2o_gputest.log 2>&1
tail -3 gpurun_out/r2o_gputest.log
python tools/op_time.py --ops v6 --cases cfg5,cfg3:8,p7:85,p6:99,p5:119,cfg3:4 --reps 10 > gpurun_out/r2o_optime.log 2>&1
cat gpurun_out/r2o_optime.log | cut -c1-120
python tools/op_time.py --ops v6 --cases cfg5 --reps 3 > gpurun_out/r2o_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_apply_v6 -s 2 -c 1 -o gpurun_out/prof_v6_r2o python tools/op_time.py --ops v6 --cases cfg5 --reps 3 > gpurun_out/r2o_ncu.log 2>&1
tail -2 gpurun_out/r2o_ncu.log
