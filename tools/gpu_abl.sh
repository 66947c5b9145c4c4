python -m pytest tests -m gpu -x -q 2>&1 | tail -2
echo base; python tools/prof_apply.py --p 8 --n 32 --reps 5 | tail -1
python tools/prof_apply.py --p 8 --n 128 --reps 3 | tail -1
for e in 21 22 23 24 25 26; do echo "EXP $e"; for n in 32 128; do SC_LIB_PATH=exp_lib/exp$e/libsc.so SC_LIBDIR=exp_lib/exp$e SC_EXP=$e python tools/prof_apply.py --p 8 --n $n --reps 3 | tail -1; done; done
