# A/B: GPU suite + trace_tune over scratch_so/*.so (two rounds)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1 > gpurun_out/tl2.txt
rm -f gpurun_out/tune.jsonl
for i in 1 2; do for so in scratch_so/*.so; do LSNIF_LIB=$PWD/$so timeout 300 python scripts/trace_tune.py 16 2>&1 | grep "^{" >> gpurun_out/tune.jsonl; done; done
