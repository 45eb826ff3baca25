#!/bin/bash
# Round-2 first GPU session: tests, C2/M1 bench with per-step dumps, oracle timing at M1.
mkdir -p gpurun_out
T=r02a
nproc > gpurun_out/${T}_nproc.txt; free -g >> gpurun_out/${T}_nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_m1.json timeout 1500 python bench.py --config m1 --steps 10 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${T}_bench_m1.json 2> gpurun_out/${T}_bench_m1.err
BENCH_DUMP=gpurun_out/${T}_steps_c2.json timeout 900 python bench.py --config c2 --steps 20 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 1200 python tools/oracle_time.py m1 1 8 16 > gpurun_out/${T}_oracle_m1.txt 2>&1
