#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02u}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
timeout 600 python bench.py --steps 10 --e2e-steps 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
H2G_SOLVE_EXPLICIT_MAX=0 timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_noexpl.json 2> gpurun_out/${T}_bench_noexpl.err
timeout 600 python bench.py --config c2 --steps 10 --e2e-steps 3 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
