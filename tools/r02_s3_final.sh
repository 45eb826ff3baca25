#!/bin/bash
# session-3 final-style run: the driver's commands + configs + launch list
mkdir -p gpurun_out
T=${1:-r02s3n}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
timeout 900 python bench.py --config c3 --steps 10 --e2e-steps 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 python bench.py --config c2 --steps 20 --e2e-steps 3 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 600 python bench.py --config c1 --steps 10 --e2e-steps 3 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${T}_launches_m1.csv python tools/profile_factor.py m1 1 > gpurun_out/${T}_pf.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches_m1.csv > gpurun_out/${T}_launches_m1.txt 2>&1
timeout 900 python tools/ablate_once.py m1 > gpurun_out/${T}_ablate.txt 2>&1
