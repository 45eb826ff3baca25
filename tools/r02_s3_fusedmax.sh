#!/bin/bash
# one-launch panel step threshold (static per process: one bench per value)
mkdir -p gpurun_out
T=${1:-r02s3v}
for v in 128 256 512; do
  H2G_PANEL_FUSED_MAX=$v timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_fm$v.json 2> gpurun_out/${T}_fm$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/${T}_fm$v.json').read().strip().splitlines()[-1]); print('fused_max $v', round(d['ms_per_step'],3))"
done
