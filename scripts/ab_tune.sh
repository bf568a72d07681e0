for w in c2 shadow; do echo "== $w"; LSNIF_LIB=$PWD/scratch_so/tl2.so python scripts/mlp_timeline.py $w 2>&1 | head -2; done > gpurun_out/tl2.txt
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1 >> gpurun_out/tl2.txt
rm -f gpurun_out/tune.jsonl
for i in 1 2; do for so in base new; do LSNIF_LIB=$PWD/scratch_so/$so.so timeout 300 python scripts/trace_tune.py 16 2>&1 | grep "^{" >> gpurun_out/tune.jsonl; done; done
