python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2v_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider > gpurun_out/r2v_fam.log 2>&1
tail -3 gpurun_out/r2v_fam.log
python tools/op_time.py --ops v3,v6 --cases cfg5,cfg3:8,p7:85,p6:99,p5:119 --reps 10 > gpurun_out/r2v_optime.log 2>&1
cut -c1-140 gpurun_out/r2v_optime.log
SC_OP=v6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_v6_r2v python tools/op_time.py --ops v6 --cases cfg5 --reps 2 > gpurun_out/r2v_ncu.log 2>&1
tail -1 gpurun_out/r2v_ncu.log
