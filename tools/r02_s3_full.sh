#!/bin/bash
# full validation after the compact-WY transform + default bench + ncu of the new leaf GEMMs
mkdir -p gpurun_out
T=${1:-r02s3c}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --config c3 --steps 10 --e2e-steps 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --set full --import-source on -k regex:gemm_grouped --launch-skip 6 --launch-count 1 -o gpurun_out/${T}_k3_m1 -f python tools/profile_factor.py m1 1 > gpurun_out/${T}_k3.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:gemm_grouped --launch-skip 0 --launch-count 1 -o gpurun_out/${T}_k1_m1 -f python tools/profile_factor.py m1 1 > gpurun_out/${T}_k1.log 2>&1
