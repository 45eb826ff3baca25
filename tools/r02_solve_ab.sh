#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02m}
for v in base ab; do
  if [ $v = ab ]; then export H2G_LIB_PATH=$PWD/paper_2502_02395_b200/libh2ulv_b200_ab.so; fi
  timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_$v.json 2> gpurun_out/${T}_bench_$v.err
done
for v in 0 1; do
  for nb in 1 16 444 4096; do ./tools/microbench/diag_trace_v$v $nb | tail -1; done > gpurun_out/${T}_diag_trace_v$v.txt 2>&1
done
