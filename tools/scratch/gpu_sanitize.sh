python -c "import __graft_entry__; __graft_entry__.build()" > gpurun_out/san_build.log 2>&1
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/scratch/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard" gpurun_out/sanitize_$tool.log | head -5
done
