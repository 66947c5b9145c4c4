# ncu source-level capture of the tile-column operator at a given p / n (one launch)
mkdir -p gpurun_out
P=${1:-4}; N=${2:-96}
python tools/prof_apply.py --p $P --n $N --reps 2 > gpurun_out/plain_p$P.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_apply -s 1 -c 1 -o gpurun_out/prof_p$P \
  python tools/prof_apply.py --p $P --n $N --reps 2 > gpurun_out/ncu_p$P.log 2>&1
tail -1 gpurun_out/plain_p$P.log
