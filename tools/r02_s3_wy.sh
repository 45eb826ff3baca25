#!/bin/bash
# compact-WY diag transform: GPU tests + M1 bench A/B
mkdir -p gpurun_out
T=${1:-r02s3b}
timeout 600 python -m pytest tests/test_gpu_construct.py -x -q -k "compact_wy or c1_construct or yukawa or many_boxes" > gpurun_out/${T}_pytest_wy.log 2>&1
tail -30 gpurun_out/${T}_pytest_wy.log
timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench_wy.json 2> gpurun_out/${T}_bench_wy.err
tail -3 gpurun_out/${T}_bench_wy.err
H2G_WY=0 timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench_dense.json 2> gpurun_out/${T}_bench_dense.err
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${T}_launches_m1.csv python tools/profile_factor.py m1 1 > gpurun_out/${T}_pf.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches_m1.csv > gpurun_out/${T}_launches_m1.txt 2>&1
