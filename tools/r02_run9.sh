#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02p}
timeout 900 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_construct.py tests/test_gpu_storage.py -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_m1.json timeout 600 python bench.py --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
H2G_CHOL_BOX_MIN=100000 timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_nobox.json 2> gpurun_out/${T}_bench_nobox.err
H2G_CHOL_BOX_MIN=1024 timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_box1024.json 2> gpurun_out/${T}_bench_box1024.err
H2G_ABLATE_LANES=2,3,4 timeout 600 python bench.py --steps 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_ablate234.json 2>&1
