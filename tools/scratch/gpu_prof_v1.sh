# ncu capture of the one-CTA-per-element kernel (p > 8) at cfg3 sizes
mkdir -p gpurun_out
for pn in "32 19" "16 37"; do
  set -- $pn
  python tools/prof_apply.py --p $1 --n $2 --reps 2 > gpurun_out/plain_v1_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_apply_v1 -s 1 -c 1 -o gpurun_out/prof_v1_p$1 \
    python tools/prof_apply.py --p $1 --n $2 --reps 2 > gpurun_out/ncu_v1_$1.log 2>&1
  tail -1 gpurun_out/plain_v1_$1.log
done
