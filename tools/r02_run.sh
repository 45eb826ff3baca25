#!/bin/bash
# Round-2 GPU session: gpu tests, default bench (driver's command), reference arm, launch list.
mkdir -p gpurun_out
T=${1:-r02d}
nproc > gpurun_out/${T}_host.txt; free -g >> gpurun_out/${T}_host.txt; nvidia-smi >> gpurun_out/${T}_host.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
s=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench wall $(( $(date +%s) - s ))" > gpurun_out/${T}_wall.txt
s=$(date +%s); timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "ref wall $(( $(date +%s) - s ))" >> gpurun_out/${T}_wall.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
