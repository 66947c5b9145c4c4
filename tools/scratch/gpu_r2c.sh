python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/r2c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "operator_parity_nodal or multitile or zsegments or slab_rank or bitwise or pcg_parity_manufactured or symmetry or small_grid_switch" > gpurun_out/r2c_gputest.log 2>&1
tail -15 gpurun_out/r2c_gputest.log
timeout 600 python tools/op_time.py --ops v5,v3 --cases cfg5,cfg3:8,cfg3:4 --out gpurun_out/r2c_optime.json > gpurun_out/r2c_optime.log 2>&1
cat gpurun_out/r2c_optime.log | tail -12
