python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/z_build.log 2>&1
for Z in 8 16 32 64 128; do
SC_V7_Z=$Z python tools/op_time.py --ops v7 --cases cfg5 --reps 10 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('Z=$Z', round(d['ms'],3))"
done
