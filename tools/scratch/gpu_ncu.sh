mkdir -p gpurun_out
TAG=${1:-r1f}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_apply_col -s 1 -c 1 -o gpurun_out/prof_cfg5_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo rc=$?
tail -2 gpurun_out/plain_$TAG.log gpurun_out/ncu_full_$TAG.log
