#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02t}
timeout 900 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py tests/test_gpu_construct.py -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python bench.py --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${T}_solve_launches.csv python tools/profile_solve.py m1 > gpurun_out/${T}_solve_prof.log 2>&1
