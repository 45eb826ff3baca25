#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3y}
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
timeout 900 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
tail -3 gpurun_out/${T}_refsuite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
bash tools/r02_sanitize.sh ${T} > gpurun_out/${T}_sanitize.out 2>&1; tail -5 gpurun_out/${T}_sanitize.out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_factor.py wy > gpurun_out/${T}_memcheck_wy.log 2>&1; echo "exit $?" >> gpurun_out/${T}_memcheck_wy.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_factor.py wy > gpurun_out/${T}_racecheck_wy.log 2>&1; echo "exit $?" >> gpurun_out/${T}_racecheck_wy.log
tail -4 gpurun_out/${T}_memcheck_wy.log gpurun_out/${T}_racecheck_wy.log
