# critical-path ablation: graph time of the factorization with lanes turned into NOPs (results invalid)
mkdir -p gpurun_out
T=${1:-r01}; CFG=${2:-c2}
for L in "" "1" "2" "3" "4" "3,4" "1,2,3,4"; do
  echo "== ablate lanes [$L]"
  H2G_ABLATE_LANES=$L timeout 900 python bench.py --config $CFG --steps 20 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done > gpurun_out/${T}_ablate_${CFG}.txt 2>&1
