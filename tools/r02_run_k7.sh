set -x
T=r02k7
timeout 1800 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py tests/test_distributed.py tests/test_gpu_block_api.py tests/test_gpu_construct.py -x -q > gpurun_out/${T}_pytest.log 2>&1
for v in base xn64; do
  if [ $v != base ]; then export H2G_LIB_PATH=$PWD/paper_2502_02395_b200/libh2ulv_b200_$v.so; fi
  timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench_$v.json 2> gpurun_out/${T}_bench_$v.err
done
unset H2G_LIB_PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${T}_solve_launches.csv python tools/profile_solve.py m1 > gpurun_out/${T}_solve_prof.log 2>&1
