TAG=${TAG:-r2jj}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" > gpurun_out/${TAG}_test.log 2>&1
tail -5 gpurun_out/${TAG}_test.log | cut -c1-300
python tools/op_time.py --ops v7 --cases cfg5,cfg3:3,cfg3:4,cfg3:5,cfg3:6,cfg3:7,cfg3:8 --reps 10 > gpurun_out/${TAG}_optime.log 2>&1
python - <<'PY'
import json,os
for l in open(f"gpurun_out/{os.environ.get('TAG','r2jj')}_optime.log"):
    if l.startswith('{'):
        d=json.loads(l); print(d['case'],d['op'],round(d['ms'],3),round(d['hbm_frac'],3))
PY
SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu.csv 2>&1
grep -E "k_v7" gpurun_out/${TAG}_ncu.csv | tail -12 | cut -c1-250
