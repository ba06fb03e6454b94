mkdir -p gpurun_out
python scripts/diag_power.py cublas 2>&1 | tail -1
python scripts/diag_power.py product 2>&1 | grep label
for f in no_epilogue no_b_load no_a_load; do AMS_LIBRARY=diag_lib/libams_diag_ams_diag_$f.so python scripts/diag_power.py $f 2>&1 | grep label; done
python scripts/diag_power.py product 2>&1 | grep label
