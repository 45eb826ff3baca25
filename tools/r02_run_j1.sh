set -x
timeout 900 python -m pytest tests/test_gpu_direct.py -x -q > gpurun_out/r02j1_pytest.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r02j1_bench_m1.json 2> gpurun_out/r02j1_bench_m1.err
timeout 2400 python bench.py --config m4 --steps 5 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02j1_bench_m4.json 2> gpurun_out/r02j1_bench_m4.err
