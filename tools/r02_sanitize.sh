#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s}
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_factor.py > gpurun_out/${T}_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/${T}_${tool}.log
done
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_factor.py box > gpurun_out/${T}_racecheck_box.log 2>&1
echo "exit $?" >> gpurun_out/${T}_racecheck_box.log
