#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3i}
timeout 600 python tools/prepare_probe.py m1 > gpurun_out/${T}_prepare.txt 2>&1
cat gpurun_out/${T}_prepare.txt | tail -22
timeout 900 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py tests/test_distributed.py -x -q -m gpu > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
timeout 900 python tools/e2e_phases.py m1 > gpurun_out/${T}_e2e.txt 2>&1; head -4 gpurun_out/${T}_e2e.txt
