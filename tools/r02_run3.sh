#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02f}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 1200 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
timeout 900 python bench.py --steps 10 --e2e-steps 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
