TAG=${TAG:-r2f1}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
SC_V7_OVERLAP=1 timeout 900 python -m pytest tests/test_gpu_kernel_families.py -q -p no:cacheprovider -k "v7" > gpurun_out/${TAG}_test.log 2>&1
tail -1 gpurun_out/${TAG}_test.log | cut -c1-300
for O in 0 1; do
SC_V7_OVERLAP=$O python tools/op_time.py --ops v7 --cases cfg5,cfg3:4,cfg3:8,cfg3:12 --reps 10 > gpurun_out/${TAG}_optime_o$O.log 2>&1
echo "overlap $O"; grep '^{' gpurun_out/${TAG}_optime_o$O.log | cut -c1-95
done
SC_V7_OVERLAP=1 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/${TAG}_bench.json
