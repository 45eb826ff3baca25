#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02y}
timeout 900 python -m pytest tests/test_gpu_construct.py -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_m1.json timeout 600 python bench.py --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
H2G_WY=0 timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_nowy.json 2> gpurun_out/${T}_bench_nowy.err
H2G_WY_RATIO=0.8 timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_wy08.json 2> gpurun_out/${T}_bench_wy08.err
timeout 600 python bench.py --config c2 --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
