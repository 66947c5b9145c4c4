python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2g_build.log 2>&1
python tools/op_time.py --ops v5,v3,rw --cases p3:198,cfg3:4,p5:119,p6:99,p7:85,cfg3:8 --reps 10 --out gpurun_out/r2g_optime.json > gpurun_out/r2g_optime.log 2>&1
cat gpurun_out/r2g_optime.log
