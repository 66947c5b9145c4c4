python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2z_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "p2 or nodal or multitile or cfg3_full_size and 2 or repeatable or zseg or pcg_parity_multitile" > gpurun_out/r2z_test.log 2>&1
tail -6 gpurun_out/r2z_test.log
python tools/op_time.py --ops v3 --cases cfg3:2 --reps 10 > gpurun_out/r2z_optime.log 2>&1
SC_P2_COLOUR=1 python tools/op_time.py --ops v3 --cases cfg3:2 --reps 10 >> gpurun_out/r2z_optime.log 2>&1
cut -c1-150 gpurun_out/r2z_optime.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_p2s -s 2 -c 1 -o gpurun_out/prof_p2s_r2z python tools/op_time.py --ops v3 --cases cfg3:2 --reps 2 > gpurun_out/r2z_ncu.log 2>&1
tail -1 gpurun_out/r2z_ncu.log
