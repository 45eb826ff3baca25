#!/bin/bash
# One GPU session: tests, bench, ncu launch list and a full capture of the top kernel.
# Usage (via gpurun): bash tools/gpu_round.sh <tag> [config]
set -x
TAG=${1:-r01}
CFG=${2:-c2}
OUT=gpurun_out
mkdir -p $OUT
nproc > $OUT/${TAG}_nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_gpu.txt
timeout 900 python bench.py --config $CFG > $OUT/${TAG}_bench_${CFG}.json 2> $OUT/${TAG}_bench_${CFG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_${CFG}.csv \
  python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/${TAG}_ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_grouped -s 40 -c 3 \
  -o $OUT/${TAG}_gemm_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > $OUT/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_potrf -s 10 -c 2 \
  -o $OUT/${TAG}_panel_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > $OUT/${TAG}_ncu_panel.log 2>&1
ls -la $OUT
