#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02g1}
H2G_LIB_PATH=$PWD/paper_2502_02395_b200/libh2ulv_b200_s3.so timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_s3.json 2> gpurun_out/${T}_bench_s3.err
timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_s2.json 2> gpurun_out/${T}_bench_s2.err
timeout 900 python bench.py --config c3 --steps 10 --e2e-steps 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 python bench.py --config c1 --steps 10 --e2e-steps 3 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 900 python bench.py --config c2 --steps 20 --e2e-steps 3 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
