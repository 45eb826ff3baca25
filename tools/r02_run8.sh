#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02m}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factor_solve.py tests/test_gpu_block_api.py -x -q > gpurun_out/${T}_pytest.log 2>&1
bash tools/r02_solve_ab.sh ${T}
