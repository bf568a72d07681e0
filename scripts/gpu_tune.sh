# A/B: trace kernel variants (scratch_so/*.so) x drain thresholds
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for so in scratch_so/*.so; do
  LSNIF_LIB=$PWD/$so timeout 300 python scripts/trace_tune.py ${DRAINS:-8,12,16,20,24} 2>&1 | grep '^{' >> gpurun_out/tune.jsonl
done
