set -x
T=r02k11
timeout 1800 python -m pytest tests/test_gpu_factor_solve.py tests/test_gpu_storage.py tests/test_distributed.py -x -q > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
timeout 900 ncu --clock-control none --profile-from-start off --set full --import-source on -k regex:xform_n -c 1 -o gpurun_out/${T}_xform_n_m1 -f python tools/profile_solve.py m1 > gpurun_out/${T}_s2.log 2>&1
nproc > gpurun_out/${T}_nproc.txt
