#!/bin/bash
# Factorization-only profiling (construct runs outside the profiled range):
#   launch list of ONE factorization, ncu --set full of the first GEMM launches
#   and of the panel / row-solve kernels.
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
for K in chol_diag chol_rows trsm_rows; do
timeout 600 $NCU --set full --import-source on -k regex:$K -c 1 -o $OUT/${TAG}_factor_${K}_${CFG} -f \
  python tools/profile_factor.py $CFG 1 > $OUT/${TAG}_factor_${K}.log 2>&1
done
ls -la $OUT
