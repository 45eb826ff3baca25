#!/bin/bash
# e2e upload restructure: host-H2 tests + M1 e2e
mkdir -p gpurun_out
T=${1:-r02s3e}
timeout 900 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py tests/test_gpu_construct.py -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 6 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --e2e-steps 6 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench_c2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
