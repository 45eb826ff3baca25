# GPU tests, C2 and M1 benches with per-step dumps, e2e breakdown
mkdir -p gpurun_out
T=${1:-r01}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_c2.json timeout 900 python bench.py --config c2 --steps 20 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 600 python tools/e2e_profile.py c2 > gpurun_out/${T}_e2e_c2.txt 2>&1
if [ "$2" = "m1" ]; then
BENCH_DUMP=gpurun_out/${T}_steps_m1.json timeout 1500 python bench.py --config m1 --steps 5 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_m1.json 2> gpurun_out/${T}_bench_m1.err
fi
