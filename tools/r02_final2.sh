#!/bin/bash
# full validation + the driver's commands + solve kernel captures
mkdir -p gpurun_out
T=${1:-r02f2}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${T}_solve_launches_m1.csv python tools/profile_solve.py m1 > gpurun_out/${T}_s1.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:xform -c 2 -o gpurun_out/${T}_xform_m1 -f python tools/profile_solve.py m1 > gpurun_out/${T}_s2.log 2>&1
