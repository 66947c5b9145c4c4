# end-of-milestone run: GPU tests, smoke, bench (+ reference arm), p sweep, ncu launch list + full capture
TAG=${TAG:-r2a1}
python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
tail -3 gpurun_out/${TAG}_gputest.log | cut -c1-300
python -c "import __graft_entry__; __graft_entry__.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cut -c1-300 gpurun_out/bench_$TAG.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python tools/p_sweep.py --out gpurun_out/p_sweep_$TAG.json > gpurun_out/p_sweep_$TAG.log 2>&1; tail -2 gpurun_out/p_sweep_$TAG.log | cut -c1-200
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_v7_(lines|assemble)" -s 2 -c 2 -o gpurun_out/prof_cfg5_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
