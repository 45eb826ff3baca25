#!/bin/bash
# Factorization-only profiling (construct runs outside the profiled range):
#   launch list of ONE factorization, ncu --set full of the first GEMM launches
#   (leaf diag_mul1 NN / diag_mul2 TN / first panel TRSM+update NT) and of the
#   DIAG kernel, per-step CUDA-event dump of the bench.
# Usage (via gpurun): bash tools/gpu_profile.sh <tag> [config]
set -x
TAG=${1:-r01}
CFG=${2:-c2}
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none --profile-from-start off"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/${TAG}_factor_launches_${CFG}.csv \
  python tools/profile_factor.py $CFG 1 > $OUT/${TAG}_factor_launches.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:gemm_grouped -c 4 -o $OUT/${TAG}_factor_gemm_${CFG} -f \
  python tools/profile_factor.py $CFG 1 > $OUT/${TAG}_factor_gemm.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:potrf_diag -c 1 -o $OUT/${TAG}_factor_diag_${CFG} -f \
  python tools/profile_factor.py $CFG 1 > $OUT/${TAG}_factor_diag.log 2>&1
BENCH_DUMP=$OUT/${TAG}_steps_${CFG}.json timeout 900 python bench.py --config $CFG --steps 20 --e2e-steps 1 --no-cpu-baseline \
  > $OUT/${TAG}_bench_dump_${CFG}.json 2> $OUT/${TAG}_bench_dump.err
ls -la $OUT
