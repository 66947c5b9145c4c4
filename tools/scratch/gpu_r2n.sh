python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2n_build.log 2>&1
SC_OP=v6 SC_V6_H=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "operator_parity_nodal or multitile or zsegments or slab_rank or bitwise or pcg_parity or symmetry or cfg5_full" > gpurun_out/r2n_gputest.log 2>&1
tail -3 gpurun_out/r2n_gputest.log
for H in 4 8; do SC_V6_H=$H python tools/op_time.py --ops v6 --cases cfg5,cfg3:8,p7:85,p6:99,p5:119,cfg3:4 --reps 10 > gpurun_out/r2n_optime_h$H.log 2>&1; done
cat gpurun_out/r2n_optime_h*.log | cut -c1-120
SC_V6_H=8 python tools/op_time.py --ops v6 --cases cfg5 --reps 3 > gpurun_out/r2n_plain.log 2>&1 && \
SC_V6_H=8 ncu --set full --clock-control none --import-source on -k regex:k_apply_v6 -s 2 -c 1 -o gpurun_out/prof_v6_r2n python tools/op_time.py --ops v6 --cases cfg5 --reps 3 > gpurun_out/r2n_ncu.log 2>&1
tail -2 gpurun_out/r2n_ncu.log
