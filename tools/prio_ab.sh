mkdir -p gpurun_out
T=${1:-r01}
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
for P in 1 0; do
  echo "== H2G_LANE_PRIORITY=$P"
  H2G_LANE_PRIORITY=$P timeout 600 python tools/ablate.py c2 20 2>&1 | grep ablate
done > gpurun_out/${T}_prio_c2.txt 2>&1
