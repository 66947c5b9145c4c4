TAG=${TAG:-r2c1}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" > gpurun_out/${TAG}_test.log 2>&1
tail -3 gpurun_out/${TAG}_test.log | cut -c1-300
python tools/op_time.py --ops v7,big --cases cfg3:9,cfg3:10,cfg3:12,cfg3:14,cfg3:16,cfg5 --reps 10 > gpurun_out/${TAG}_optime.log 2>&1
python - <<'PY'
import json,os
for l in open(f"gpurun_out/{os.environ.get('TAG','r2c1')}_optime.log"):
    if l.startswith('{'):
        d=json.loads(l); print(d['case'],d['op'],round(d['ms'],3),round(d['hbm_frac'],3))
PY
