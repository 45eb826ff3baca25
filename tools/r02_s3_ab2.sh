#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3o}
timeout 1200 python tools/ab_once.py m1 base "H2G_WY_CFG=2,,,7" "H2G_WY_CFG=9,,,7" "H2G_WY_CFG=,9,9,7" "H2G_TILE32_ALL=2.0;H2G_GEMM_SPLIT=2.0" "H2G_TILE32_ALL=1.25;H2G_GEMM_SPLIT=1.25" "H2G_CHOL_BOX_MIN=2048" > gpurun_out/${T}_ab.txt 2>&1
grep '^\[' gpurun_out/${T}_ab.txt
timeout 1500 python bench.py --gpus 1 --steps 10 --warmup 3 --e2e-steps 4 --no-exact-residual > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['seconds_per_step'], d['cpu_baseline']['value'])"
