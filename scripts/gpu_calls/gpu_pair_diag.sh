TIME=1 timeout 300 python scripts/scan_pair_calls.py
AMS_LIBRARY=diag_lib/libams_diag_ams_diag_no_epilogue.so TIME=1 timeout 300 python scripts/scan_pair_calls.py
