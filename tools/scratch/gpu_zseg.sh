# operator time at cfg5 (p=8, 128^3) and cfg3 points for forced z-segment counts
python -c "import __graft_entry__; __graft_entry__.build()"
for S in 1 2 3 4; do
  echo "== SC_ZSEG=$S cfg5"; SC_ZSEG=$S python tools/prof_apply.py --p 8 --n 128 --reps 10 | tail -1
done
echo "== auto cfg5"; python tools/prof_apply.py --p 8 --n 128 --reps 10 | tail -1
python tools/p_sweep.py --ps 2,4,8 --reps 10 --out gpurun_out/p_sweep_r1d.json 2>&1 | tail -3
