export SC_EXP=9 SC_LIBDIR=exp_lib/exp9 SC_LIB_PATH=exp_lib/exp9/libsc.so
python tools/prof_apply.py --p 8 --n ${1:-32} --reps 2 | tail -1
python tools/phase_exp.py ${1:-32}
