set -x
T=r02k12
bash tools/r02_sanitize.sh ${T}
timeout 900 ncu --clock-control none --profile-from-start off --set full --import-source on -k regex:xform_n --launch-skip 6 -c 1 -o gpurun_out/${T}_xform_n_m1 -f python tools/profile_solve.py m1 > gpurun_out/${T}_s2.log 2>&1
timeout 900 python bench.py --steps 10 --e2e-steps 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
