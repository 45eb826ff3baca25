set -x
timeout 600 python -m pytest tests/test_gpu_construct.py -x -q > gpurun_out/r02i1_pytest.log 2>&1
timeout 600 python tools/e2e_phases.py m1 > gpurun_out/r02i1_phases.log 2>&1
timeout 2400 python bench.py --config m4 --steps 5 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02i1_bench_m4.json 2> gpurun_out/r02i1_bench_m4.err
