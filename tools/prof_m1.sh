OUT=gpurun_out; mkdir -p $OUT
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --set full --import-source on -k regex:chol_diag -s 1 -c 1 -o $OUT/r01bc_chol_diag_m1 -f python tools/profile_factor.py m1 1 > $OUT/r01bc_1.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:trsm_rows -c 1 -o $OUT/r01bc_trsm_rows_m1 -f python tools/profile_factor.py m1 1 > $OUT/r01bc_2.log 2>&1
