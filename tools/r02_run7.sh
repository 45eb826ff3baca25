#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02k}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --config c4 --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 900 python bench.py --config m2 --steps 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_m2.json 2> gpurun_out/${T}_bench_m2.err
