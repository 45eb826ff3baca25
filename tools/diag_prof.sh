mkdir -p gpurun_out
./tools/microbench/fp64_latency > gpurun_out/r01h_fp64_latency.txt 2>&1
for bs in 2 4; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:potrf_diag -s 2 -c 1 -o gpurun_out/r01h_diag_bs$bs -f ./tools/microbench/panel_bench_bs$bs 148 256 64 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:chol_panel -s 2 -c 1 -o gpurun_out/r01h_cpanel_bs$bs -f ./tools/microbench/panel_bench_bs$bs 148 256 64 > /dev/null 2>&1
done
ls gpurun_out
