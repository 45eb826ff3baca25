#!/bin/bash
# default bench (driver's command line) + the reference arm, wall times
mkdir -p gpurun_out
T=${1:-r02c}
s=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench wall $(( $(date +%s) - s ))" > gpurun_out/${T}_wall.txt
s=$(date +%s); timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "ref wall $(( $(date +%s) - s ))" >> gpurun_out/${T}_wall.txt
