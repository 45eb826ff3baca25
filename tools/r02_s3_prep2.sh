#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3j}
timeout 900 python -m pytest tests/test_gpu_block_api.py tests/test_gpu_factor_solve.py tests/test_gpu_storage.py -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
timeout 600 python tools/prepare_probe.py m1 > gpurun_out/${T}_prepare.txt 2>&1
tail -12 gpurun_out/${T}_prepare.txt
timeout 900 python tools/e2e_phases.py m1 > gpurun_out/${T}_e2e.txt 2>&1; head -4 gpurun_out/${T}_e2e.txt
