# scratch (a temporary AMS_XST cap on the CTA-pair stage count, not kept): is the pair
# kernel's time sensitive to its stage count?  C3 pool, 129 / 200 queries, k = 8
set -x
for st in 6 5 4 3; do
  AMS_XST=$st python scripts/one_call.py c3 --nq 129 --k 8 --calls 9 2>&1 | grep "^c3"
  AMS_XST=$st python scripts/one_call.py c3 --nq 200 --k 8 --calls 9 2>&1 | grep "^c3"
done
