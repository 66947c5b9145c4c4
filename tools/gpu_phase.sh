export SC_EXP=9 SC_LIBDIR=/tmp/exp9 SC_LIB_PATH=/tmp/exp9/libsc.so
python -c "from paper_1601_08179_b200 import build as b; b.build()" > /dev/null
python tools/prof_apply.py --p 8 --n 128 --reps 2 | tail -1
python tools/phase_exp.py 128
