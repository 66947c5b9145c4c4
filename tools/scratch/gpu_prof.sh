mkdir -p gpurun_out
python tools/prof_apply.py --p 8 --n 32 --reps 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_apply_col -s 1 -c 1 -o gpurun_out/prof_v3g python tools/prof_apply.py --p 8 --n 32 --reps 2 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/plain.log gpurun_out/ncu.log
