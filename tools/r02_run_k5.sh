set -x
T=r02k5
timeout 1800 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py tests/test_distributed.py -x -q > gpurun_out/${T}_pytest.log 2>&1
for v in "592 592" "592 0" "296 592" "1184 592" "1184 1184"; do
  set -- $v
  H2G_GEMV_BALANCE=$1 H2G_XFORM_MIN_CTAS=$2 timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench_$1_$2.json 2> gpurun_out/${T}_bench_$1_$2.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${T}_solve_launches.csv python tools/profile_solve.py m1 > gpurun_out/${T}_solve_prof.log 2>&1
