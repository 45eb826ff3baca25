#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02x}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_SHARE_GPU=1 BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/${T}_dist2_gloo_c2.json 2> gpurun_out/${T}_dist2_gloo_c2.err
