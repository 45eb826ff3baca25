set -x
T=r02k10
BENCH_DUMP=gpurun_out/${T}_dump_m1.json timeout 600 python bench.py --steps 3 --e2e-steps 0 --no-cpu-baseline --no-exact-residual > gpurun_out/${T}_bench_dump.json 2> gpurun_out/${T}_bench_dump.err
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c --steps 10 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
