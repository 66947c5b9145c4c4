python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider -x > gpurun_out/r2t_vartest.log 2>&1
tail -15 gpurun_out/r2t_vartest.log
timeout 900 python tools/variants_sweep.py --out gpurun_out/variants_r2t.json > gpurun_out/r2t_sweep.log 2>&1
tail -3 gpurun_out/r2t_sweep.log | cut -c1-300
