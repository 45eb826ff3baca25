#!/bin/bash
# block API + factor tests, staged reference suite, M1 per-step dump, default bench
mkdir -p gpurun_out
T=${1:-r02e}
timeout 900 python -m pytest tests/test_gpu_block_api.py tests/test_gpu_factor_solve.py -x -q > gpurun_out/${T}_pytest_new.log 2>&1
timeout 1200 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_m1.json timeout 1200 python bench.py --steps 5 --e2e-steps 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
