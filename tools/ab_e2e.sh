# A/B of upload knobs on the C2 end-to-end time (public API, host H2Matrix in, solution out)
mkdir -p gpurun_out
T=$1
for rep in 1 2; do
  for TH in 8 12 16; do
    for CH in 524288 2097152; do
      echo "threads=$TH chunk=$CH $(H2G_UPLOAD_THREADS=$TH H2G_UPLOAD_CHUNK=$CH timeout 900 python bench.py --config c2 --steps 5 --e2e-steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['seconds_per_step']*1e3,2), 'ms', d['ms_per_step'])")"
    done
  done
done > gpurun_out/${T}_ab_e2e.txt 2>&1
