python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2w_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py tests/test_gpu_loopback.py -q -p no:cacheprovider -x > gpurun_out/r2w_fam.log 2>&1
tail -15 gpurun_out/r2w_fam.log
for cfg in "v3:1" "v6:0" "v6:1"; do op=${cfg%%:*}; fd=${cfg##*:};
SC_OP=$op SC_FUSED_DIR=$fd timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_bench_${op}_$fd.json 2> gpurun_out/r2w_bench_${op}_$fd.err
python -c "import json;d=json.load(open('gpurun_out/r2w_bench_${op}_$fd.json'));print('$op fd=$fd', d['ms_per_step'], d['value'], d['operator'], d['roofline']['kernel_ms'], d['gpu_launches'])"
done
