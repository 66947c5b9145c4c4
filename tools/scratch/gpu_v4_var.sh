# v4 variants (prebuilt under exp_lib/<name>/): timing at cfg3 sizes, p = 9..32
for pn in "9 66" "12 50" "16 37" "20 30" "24 25" "32 19"; do
  set -- $pn
  echo "p=$1 base"; python tools/prof_apply.py --p $1 --n $2 --reps 5 | tail -1
  for v in ${VARS:-v4b v4c v4d}; do
    echo "p=$1 $v"; SC_LIB_PATH=exp_lib/$v/libsc.so python tools/prof_apply.py --p $1 --n $2 --reps 5 | tail -1
  done
done
