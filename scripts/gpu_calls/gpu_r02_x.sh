# scratch (temporary env switch AMS_XQ = the largest binned batch): binned vs block kernel at 512..2048 queries
set -x
for nq in 384 512 768 1024 2048; do
  AMS_XQ=100000 python scripts/one_call.py c3 --nq $nq --gate-first --calls 7 2>&1 | grep "^c3"
  AMS_XQ=16 python scripts/one_call.py c3 --nq $nq --gate-first --calls 7 2>&1 | grep "^c3"
done
for nq in 256 512 1024; do
  AMS_XQ=100000 python scripts/one_call.py c5 --nq $nq --gate-first --calls 7 2>&1 | grep "^c5"
  AMS_XQ=16 python scripts/one_call.py c5 --nq $nq --gate-first --calls 7 2>&1 | grep "^c5"
done
