mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for n in 32 128; do timeout 120 python tools/prof_apply.py --p 8 --n $n --reps 5 2>&1 | tail -1; done
for p in 2 4 6; do timeout 120 python tools/prof_apply.py --p $p --n 64 --reps 5 2>&1 | tail -1; done
bash tools/gpu_phase.sh
