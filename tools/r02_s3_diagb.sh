#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3s}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factor_solve.py tests/test_gpu_construct.py tests/test_gpu_block_api.py -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
timeout 900 python tools/ab_once.py m1 base > gpurun_out/${T}_ab_m1.txt 2>&1; grep '^\[' gpurun_out/${T}_ab_m1.txt
timeout 600 python tools/ab_once.py c2 base > gpurun_out/${T}_ab_c2.txt 2>&1; grep '^\[' gpurun_out/${T}_ab_c2.txt
timeout 600 python tools/ab_once.py c3 base > gpurun_out/${T}_ab_c3.txt 2>&1; grep '^\[' gpurun_out/${T}_ab_c3.txt
