#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3z}
timeout 1200 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_construct.py tests/test_gpu_storage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
timeout 600 python tools/sanitize_factor.py wy > gpurun_out/${T}_wyfunc.log 2>&1; tail -5 gpurun_out/${T}_wyfunc.log
timeout 900 python tools/e2e_phases.py m1 > gpurun_out/${T}_e2e.txt 2>&1; head -4 gpurun_out/${T}_e2e.txt
timeout 1500 python bench.py --gpus 1 --steps 10 --warmup 3 --e2e-steps 4 --no-exact-residual > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['seconds_per_step'], d['config']['residual'])"
