python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/c4_build.log 2>&1
timeout 1200 python tools/cfg4_aniso.py --out gpurun_out/cfg4_r2.json > gpurun_out/cfg4_r2.log 2>&1; echo "cfg4 rc=$?"; tail -5 gpurun_out/cfg4_r2.log | cut -c1-200
timeout 1200 python tools/e3_study.py --ps 16 --alphas 1 --ns 2,4,8,16,32 --reps 3 --out gpurun_out/e4_r2b.json > gpurun_out/e4_r2b.log 2>&1; echo "e4 rc=$?"; tail -6 gpurun_out/e4_r2b.log | cut -c1-200
timeout 600 python tools/cfg12.py > gpurun_out/cfg12_r2.log 2>&1; echo "cfg12 rc=$?"; tail -4 gpurun_out/cfg12_r2.log | cut -c1-200
