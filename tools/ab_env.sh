# A/B of an environment knob on the default (C2) and M1 factorization time.
# Usage: bash tools/ab_env.sh TAG VAR "v1 v2" [m1]
mkdir -p gpurun_out
T=$1; VAR=$2; VALS=$3
for rep in 1 2; do
  for V in $VALS; do
    for C in c2 $4; do
      S=20; [ $C = m1 ] && S=5
      echo "$VAR=$V $C $(env $VAR=$V timeout 900 python bench.py --config $C --steps $S --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['residual'])")"
    done
  done
done > gpurun_out/${T}_ab.txt 2>&1
