python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2u_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider > gpurun_out/r2u_vartest.log 2>&1
tail -15 gpurun_out/r2u_vartest.log
timeout 1200 python tools/e3_study.py --ps 2,4,8,12,16 --solvers uc,dc,bc,bt --reps 3 --out gpurun_out/e3_solvers_r2u.json > gpurun_out/r2u_e3.log 2>&1
tail -2 gpurun_out/r2u_e3.log | cut -c1-1500
