#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3l}
timeout 900 python -m pytest tests/test_gpu_construct.py tests/test_gpu_factor_solve.py tests/test_gpu_storage.py -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -30 gpurun_out/${T}_pytest.log | grep -v '^\s*$' | tail -25
timeout 900 python tools/e2e_phases.py m1 > gpurun_out/${T}_e2e.txt 2>&1; head -6 gpurun_out/${T}_e2e.txt; tail -3 gpurun_out/${T}_e2e.txt
