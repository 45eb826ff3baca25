#!/bin/bash
# split-K tests + A/B of split-K and WY tile configs at M1
mkdir -p gpurun_out
T=${1:-r02s3d}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factor_solve.py -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual"
timeout 600 $B > gpurun_out/${T}_default.json 2> gpurun_out/${T}_default.err
H2G_SPLITK=1 timeout 600 $B > gpurun_out/${T}_nosplit.json 2> gpurun_out/${T}_nosplit.err
H2G_WY_CFG=",,,2" timeout 600 $B > gpurun_out/${T}_k3cfg2.json 2> gpurun_out/${T}_k3cfg2.err
H2G_CHOL_BOX_V=1 timeout 600 $B > gpurun_out/${T}_boxv.json 2> gpurun_out/${T}_boxv.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
H2G_SPLITK=1 timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_c2_nosplit.json 2> gpurun_out/${T}_c2_nosplit.err
for f in default nosplit k3cfg2 boxv c2 c2_nosplit; do python -c "
import json,sys;d=json.loads(open('gpurun_out/${T}_'+sys.argv[1]+'.json').read().strip().splitlines()[-1]); print(sys.argv[1], round(d['ms_per_step'],3), d['config']['residual'])" $f; done
