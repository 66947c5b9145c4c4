python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2r_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "e4 or e3" > gpurun_out/r2r_e4test.log 2>&1
timeout 1500 python tools/e3_study.py --out gpurun_out/e3_r2.json > gpurun_out/r2r_e3.log 2>&1
timeout 1500 python tools/e3_study.py --ps 16 --alphas 1 --ns 2,4,8,16,24,32 --reps 3 --out gpurun_out/e4_r2.json > gpurun_out/r2r_e4.log 2>&1
tail -3 gpurun_out/r2r_e4test.log; tail -2 gpurun_out/r2r_e3.log; tail -2 gpurun_out/r2r_e4.log
