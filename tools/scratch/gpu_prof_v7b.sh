TAG=${TAG:-r2oo}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" > gpurun_out/${TAG}_test.log 2>&1
tail -2 gpurun_out/${TAG}_test.log | cut -c1-300
SC_OP=v7 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_v7_(lines|cond|assemble)" -s 2 -c 2 -o gpurun_out/prof_v7_${TAG} python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu_v7.log 2>&1; echo "ncu v7 rc=$?"
