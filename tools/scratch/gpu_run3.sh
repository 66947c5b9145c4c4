python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for n in 32 128; do timeout 120 python tools/prof_apply.py --p 8 --n $n --reps 5 2>&1 | tail -1; done
bash tools/gpu_abl.sh
