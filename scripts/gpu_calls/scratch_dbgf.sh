# scratch (a temporary build with AMS_DBGF switches in match_scan_kernel, not kept): bit 0
# compiled the MMA issue out, bit 1 the query-operand loads; C3 pool per-call times
set -x
for f in 0 1 3; do
  AMS_DBGF=$f python scripts/one_call.py c3 --nq 200 --k 8 --calls 9 2>&1 | grep "^c3"
  AMS_DBGF=$f python scripts/one_call.py c3 --nq 144 --k 8 --calls 9 2>&1 | grep "^c3"
done
for f in 0 1; do AMS_DBGF=$f python scripts/one_call.py c3 --nq 64 --calls 9 2>&1 | grep "^c3"; done
