set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02k3_pytest.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exact-residual > gpurun_out/r02k3_bench_m1.json 2> gpurun_out/r02k3_bench_m1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02k3_solve_launches.csv python tools/profile_solve.py m1 > gpurun_out/r02k3_solve_prof.log 2>&1
