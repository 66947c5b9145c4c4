# per-phase cycle split at small p (SC_EXP=9 build): tools/gpu_phase2.sh
set -e
export SC_EXP=9 SC_LIBDIR=exp_lib/exp9 SC_LIB_PATH=exp_lib/exp9/libsc.so
python -c "import paper_1601_08179_b200.build as b; b.build()"
for pn in "2 128" "4 96" "8 32"; do
  set -- $pn
  echo "== p=$1 n=$2"
  python tools/phase_exp.py $2 $1
done
