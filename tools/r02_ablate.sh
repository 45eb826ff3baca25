#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02o}
for a in none 4 2,3 1 2,3,4; do
  if [ $a = none ]; then unset H2G_ABLATE_LANES; else export H2G_ABLATE_LANES=$a; fi
  timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_ablate_${a}.json 2>&1
done
