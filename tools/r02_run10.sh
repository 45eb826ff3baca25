#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02q}
timeout 900 python -m pytest tests/test_gpu_factor_solve.py tests/test_distributed.py tests/test_gpu_kernels.py -x -q > gpurun_out/${T}_pytest.log 2>&1
for sp in 1.5 0; do
  H2G_GEMM_SPLIT=$sp timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_split$sp.json 2> gpurun_out/${T}_bench_split$sp.err
  H2G_GEMM_SPLIT=$sp timeout 600 python bench.py --config c2 --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_c2_split$sp.json 2> gpurun_out/${T}_bench_c2_split$sp.err
done
