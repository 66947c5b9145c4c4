echo base; python tools/prof_apply.py --p 8 --n 32 --reps 5 | tail -1
for e in ${@:-21 22 23 24 25 30 31 32}; do echo "EXP $e"; SC_LIB_PATH=exp_lib/exp$e/libsc.so SC_LIBDIR=exp_lib/exp$e SC_EXP=$e python tools/prof_apply.py --p 8 --n 32 --reps 5 | tail -1; done
