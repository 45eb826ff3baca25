#!/bin/bash
# fused per-box Cholesky: parity tests, then M1 A/B over the box-count threshold
mkdir -p gpurun_out
T=${1:-r02g}
timeout 900 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py -x -q > gpurun_out/${T}_pytest.log 2>&1
for m in 100000 1024 512 256; do
  H2G_CHOL_BOX_MIN=$m BENCH_DUMP=gpurun_out/${T}_steps_box$m.json timeout 600 python bench.py --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_box$m.json 2> gpurun_out/${T}_bench_box$m.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${T}_solve_launches.csv python tools/profile_solve.py m1 > gpurun_out/${T}_solve_prof.log 2>&1
