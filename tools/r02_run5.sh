#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02h}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_m1.json timeout 600 python bench.py --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
H2G_CHOL_BOX_MIN=100000 timeout 600 python bench.py --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_nobox.json 2> gpurun_out/${T}_bench_nobox.err
BENCH_DUMP=gpurun_out/${T}_steps_c2.json timeout 600 python bench.py --config c2 --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
