python -c "import __graft_entry__; __graft_entry__.build()" > /dev/null 2>&1
for mb in 3 4 5 6 8; do
SC_LIB_PATH=/root/repo/exp_lib/mb$mb/libsc.so python tools/op_time.py --ops v3 --cases cfg3:2 --reps 20 2>&1 | cut -c1-110 | sed "s/^/mb=$mb /"
done
