# per-phase cycle split of the v3 operator at cfg5 size (SC_EXP=9 build)
set -e
export SC_EXP=9 SC_LIBDIR=exp_lib/exp9 SC_LIB_PATH=exp_lib/exp9/libsc.so
python -c "import paper_1601_08179_b200.build as b; b.build()"
python tools/phase_exp.py ${1:-128} ${2:-8}
