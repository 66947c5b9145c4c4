mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; tail -3 gpurun_out/bench_r1c.err
cat gpurun_out/bench_r1c.json
for e in 9 1 2 3 4 6; do
 SC_EXP=$e SC_LIBDIR=/tmp/exp$e python -c "from paper_1601_08179_b200 import build as b; b.build()" >/dev/null 2>&1
 echo "EXP $e"; SC_EXP=$e SC_LIBDIR=/tmp/exp$e SC_LIB_PATH=/tmp/exp$e/libsc.so timeout 120 python tools/prof_apply.py --p 8 --n 128 --reps 3 2>&1 | tail -1
 if [ $e = 9 ]; then SC_EXP=9 SC_LIBDIR=/tmp/exp9 SC_LIB_PATH=/tmp/exp9/libsc.so timeout 120 python tools/phase_exp.py 2>&1 | tail -10; fi
done
