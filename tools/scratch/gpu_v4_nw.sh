# v4 warps-per-CTA variants for 9 <= n_I <= 14 (prebuilt under exp_lib/nw<mode>/)
for pn in "10 59" "11 54" "12 50" "13 46" "14 42" "15 40"; do
  set -- $pn
  echo "p=$1 base $(python tools/prof_apply.py --p $1 --n $2 --reps 5 | tail -1)"
  for v in nw1 nw2; do
    echo "p=$1 $v $(SC_LIB_PATH=exp_lib/$v/libsc.so python tools/prof_apply.py --p $1 --n $2 --reps 5 | tail -1)"
  done
done
for v in nw1 nw2; do
  echo "tests $v: $(SC_LIB_PATH=exp_lib/$v/libsc.so python -m pytest tests -m gpu -x -q -k 'big or nonuniform or bitwise' 2>&1 | tail -1)"
done
