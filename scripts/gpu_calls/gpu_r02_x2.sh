# scratch (temporary env switch AMS_XQ = the largest binned batch): the windowed snapshot kernel
# for > 1024 queries vs the block kernel over the 2-D order; then the gate-first tests
set -x
timeout 900 python -m pytest tests/test_gpu_gate_first.py -x -q 2>&1 | tail -2
for nq in 1024 2048 4096 16384; do
  AMS_XQ=100000 python scripts/one_call.py c3 --nq $nq --gate-first --calls 7 2>&1 | grep "^c3"
  AMS_XQ=16 python scripts/one_call.py c3 --nq $nq --gate-first --calls 7 2>&1 | grep "^c3"
done
for nq in 2048 8192; do
  AMS_XQ=100000 python scripts/one_call.py c5 --nq $nq --gate-first --calls 5 2>&1 | grep "^c5"
  AMS_XQ=16 python scripts/one_call.py c5 --nq $nq --gate-first --calls 5 2>&1 | grep "^c5"
done
