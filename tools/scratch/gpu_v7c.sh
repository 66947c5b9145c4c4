TAG=${TAG:-r2nn}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" -x > gpurun_out/${TAG}_test.log 2>&1
tail -3 gpurun_out/${TAG}_test.log | cut -c1-400
for A in lines class; do
SC_V7_A=$A python tools/op_time.py --ops v7 --cases ${CASES:-cfg5,cfg3:3,cfg3:4,cfg3:5,cfg3:6,cfg3:7,cfg3:8} --reps 10 > gpurun_out/${TAG}_optime_$A.log 2>&1
echo "A=$A"; python - $A <<'PY'
import json,os,sys
for l in open(f"gpurun_out/{os.environ.get('TAG')}_optime_{sys.argv[1]}.log"):
    if l.startswith('{'):
        d=json.loads(l); print(d['case'],d['op'],round(d['ms'],3),round(d['hbm_frac'],3))
PY
done
SC_OP=v7 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active --clock-control none --csv python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu.csv 2>&1
grep -E "k_v7_(lines|assemble)" gpurun_out/${TAG}_ncu.csv | tail -12 | awk -F'","' '{print $5, $13, $15}' | cut -c1-150
