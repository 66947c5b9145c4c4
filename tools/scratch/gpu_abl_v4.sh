# v4 ablations (timing only; ablated builds give wrong results): 40 no Newton, 41 no reciprocal,
# 42 no Qy transpose.  Libraries prebuilt under exp_lib/exp<E>/.
for pn in "12 50" "16 37" "20 30" "24 25" "32 19"; do
  set -- $pn
  echo "p=$1 base"; python tools/prof_apply.py --p $1 --n $2 --reps 5 | tail -1
  for e in ${EXPS:-40 41 42}; do
    echo "p=$1 EXP $e"; SC_LIB_PATH=exp_lib/exp$e/libsc.so python tools/prof_apply.py --p $1 --n $2 --reps 5 | tail -1
  done
done
