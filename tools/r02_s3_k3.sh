#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3f}
timeout 900 python -m pytest tests/test_gpu_construct.py tests/test_gpu_kernels.py -x -q -k "compact_wy or gemm or c1_construct" > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['config']['residual'])"
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${T}_launches_m1.csv python tools/profile_factor.py m1 1 > gpurun_out/${T}_pf.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches_m1.csv > gpurun_out/${T}_launches_m1.txt 2>&1
head -12 gpurun_out/${T}_launches_m1.txt
