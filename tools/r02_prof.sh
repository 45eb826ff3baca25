#!/bin/bash
# sanitizers + M1 launch list + ncu full captures of the new / dominant kernels
mkdir -p gpurun_out
T=${1:-r02l}
bash tools/r02_sanitize.sh ${T}
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${T}_factor_launches_m1.csv python tools/profile_factor.py m1 1 > gpurun_out/${T}_f1.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:chol_box -c 1 -o gpurun_out/${T}_chol_box_m1 -f python tools/profile_factor.py m1 1 > gpurun_out/${T}_f2.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:gemm_grouped -c 2 -o gpurun_out/${T}_gemm_m1 -f python tools/profile_factor.py m1 1 > gpurun_out/${T}_f3.log 2>&1
