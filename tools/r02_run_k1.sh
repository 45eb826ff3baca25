set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02k1_pytest.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exact-residual > gpurun_out/r02k1_bench_m1.json 2> gpurun_out/r02k1_bench_m1.err
