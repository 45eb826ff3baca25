# microbenchmarks of the panel kernels + GPU tests + C2 bench (per-step dump)
mkdir -p gpurun_out
T=${1:-r01}
for bs in 0 2; do
  for args in "1 256 64" "256 256 64" "256 256 0" "4096 256 64" "2 900 256"; do
    echo "== bs $bs args $args"
    ./tools/microbench/panel_bench_bs$bs $args | tail -6
  done
done > gpurun_out/${T}_panel_bench.txt 2>&1
./tools/microbench/diag_bench 256 >> gpurun_out/${T}_panel_bench.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
BENCH_DUMP=gpurun_out/${T}_steps_c2.json timeout 900 python bench.py --config c2 --steps 20 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
