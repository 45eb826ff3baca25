#!/bin/bash
# session-3 re-entry check: GPU suite, smoke, default bench
mkdir -p gpurun_out
T=${1:-r02s3a}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
