# A/B: GPU suite + trace_tune on base.so vs new.so (two rounds)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1 > gpurun_out/tl2.txt
rm -f gpurun_out/tune.jsonl
for i in 1 2; do for so in base new; do LSNIF_LIB=$PWD/scratch_so/$so.so timeout 300 python scripts/trace_tune.py 16 2>&1 | grep "^{" >> gpurun_out/tune.jsonl; done; done
