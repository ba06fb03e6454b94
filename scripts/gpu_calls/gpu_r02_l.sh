# in-stream timelines of small-batch calls: kernel durations and inter-kernel gaps
set -x
for args in "c3 --nq 64 --gamma inf" "c3 --nq 64" "c3 --nq 200 --k 8" "c3 --nq 1" "c1 --nq 64" "c4 --nq 64 --gamma inf"; do
  timeout 300 python scripts/one_call.py $args --calls 5 --timeline
done
