#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s}
for v in base t256 t128; do
  if [ $v != base ]; then export H2G_LIB_PATH=$PWD/paper_2502_02395_b200/libh2ulv_b200_$v.so; fi
  timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_$v.json 2> gpurun_out/${T}_bench_$v.err
done
