# End-of-round evidence for profiles/: the default bench line, its ncu launch list,
# and a full ncu capture of the dominant GEMM launch of one factorization.
mkdir -p gpurun_out
T=${1:-r01}
timeout 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench_default.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_ncu_launch_run.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
NCU="ncu --clock-control none --profile-from-start off"
for K in chol_panel_fused trsm_rows chol_diag; do
  timeout 600 $NCU --set full --import-source on -k regex:$K -c 1 -o gpurun_out/${T}_factor_${K}_c2 -f \
    python tools/profile_factor.py c2 1 > gpurun_out/${T}_factor_${K}.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
