#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3as}
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${T}_launches_m1.csv python tools/profile_factor.py m1 1 > gpurun_out/${T}_pf.log 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches_m1.csv > gpurun_out/${T}_launches_m1.txt 2>&1
timeout 900 $NCU --set full --import-source on -k regex:gemm_grouped --launch-skip 6 --launch-count 1 -o gpurun_out/${T}_k3_m1 -f python tools/profile_factor.py m1 1 > gpurun_out/${T}_k3.log 2>&1
head -8 gpurun_out/${T}_launches_m1.txt
