TAG=r2ii
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
python tools/op_time.py --ops v7,v6,v3,rw --cases cfg5,cfg3:3,cfg3:4,cfg3:5,cfg3:6,cfg3:7,cfg3:8 --reps 10 > gpurun_out/${TAG}_optime.log 2>&1
cut -c1-160 gpurun_out/${TAG}_optime.log | grep case
SC_OP=v7 python bench.py --no-cpu > gpurun_out/${TAG}_bench_v7.json 2> gpurun_out/${TAG}_bench_v7.err; echo "bench v7 rc=$?"; cut -c1-400 gpurun_out/${TAG}_bench_v7.json
SC_OP=v7 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_v7 -c 12 -o gpurun_out/prof_v7_${TAG} python tools/op_time.py --ops v7 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu_v7.log 2>&1; echo "ncu v7 rc=$?"
SC_OP=v3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_v3_${TAG} python tools/op_time.py --ops v3 --cases cfg5 --reps 1 > gpurun_out/${TAG}_ncu_v3.log 2>&1; echo "ncu v3 rc=$?"
