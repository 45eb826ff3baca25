set -x
T=r02k9
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${T}_solve_launches.csv python tools/profile_solve.py m1 > gpurun_out/${T}_solve_prof.log 2>&1
