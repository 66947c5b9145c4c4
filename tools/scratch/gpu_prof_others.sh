# ncu captures of the non-cfg5 operator kernels at cfg3 sizes (one colour launch each)
mkdir -p gpurun_out
TAG=${1:-r1p}
for spec in "2 297 k_apply_p2" "4 148 k_apply_rw" "16 37 k_apply_big" "32 19 k_apply_big"; do
  set -- $spec
  python tools/prof_apply.py --p $1 --n $2 --reps 2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 8 -c 1 -o gpurun_out/prof_${TAG}_p$1 \
    python tools/prof_apply.py --p $1 --n $2 --reps 2 > gpurun_out/ncu_${TAG}_p$1.log 2>&1
  echo "p=$1 rc=$?"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:$3 -c 8 --csv \
    python tools/prof_apply.py --p $1 --n $2 --reps 1 > gpurun_out/traffic_${TAG}_p$1.csv 2>&1
done
