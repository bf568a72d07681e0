# trace kernel: shared-memory carveout / resident-block sweep (L1 capacity for the hash gathers)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_tail.txt
for c in "" 50 58 72 86; do for b in "" 7 6; do
  env ${c:+LSNIF_TRACE_CARVEOUT=$c} ${b:+LSNIF_TRACE_BLOCKS=$b} timeout 300 python scripts/trace_tune.py 16 2>&1 | grep '^{' >> gpurun_out/tune.jsonl
done; done
