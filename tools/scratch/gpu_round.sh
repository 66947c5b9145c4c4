# round bench + profiles: default bench line, reference arm, ncu launch list + full capture
mkdir -p gpurun_out
TAG=${1:-r1g}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref_$TAG.json
bash tools/gpu_ncu.sh $TAG
