# C3 batch (16384 queries) through the gate-first path: timeline (regression check)
set -x
timeout 400 python scripts/one_call.py c3 --nq 16384 --gate-first --calls 5 --timeline 2>&1 | grep -v "_warn" | head -12
timeout 400 python scripts/one_call.py c3 --nq 16384 --auto --calls 5 --timeline 2>&1 | grep -v "_warn" | head -12
