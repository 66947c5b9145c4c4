# ablations at cfg5 size (timing only; ablated builds give wrong results)
python -c "import paper_1601_08179_b200.build as b; b.build()"
echo base; python tools/prof_apply.py --p 8 --n 128 --reps 5 | tail -1
for e in ${@:-24 27}; do
  export SC_LIB_PATH=exp_lib/exp$e/libsc.so SC_LIBDIR=exp_lib/exp$e SC_EXP=$e
  python -c "import paper_1601_08179_b200.build as b; b.build()"
  echo "EXP $e"; python tools/prof_apply.py --p 8 --n 128 --reps 5 | tail -1
done
