# A/B of library builds with the parity tests run against EACH variant:
# for every ab/*.so, the bit-exact parity tests through LSNIF_LIB, then
# device time per query (scripts/trace_tune.py) for each build and the
# in-tree one. Usage: bash scripts/gpu_ab_var.sh TAG [pytest -k expr]
TAG=${1:-ab}
mkdir -p gpurun_out
for lib in ab/*.so; do
  echo "== $lib" | tee -a gpurun_out/${TAG}_tests.log
  LSNIF_LIB=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_sweep.py -q -x -m gpu ${2:+-k "$2"} 2>&1 | tail -4 | tee -a gpurun_out/${TAG}_tests.log
done
for rep in 1 2; do
for lib in ab/*.so paper_2504_21627_b200/liblsnif_gpu.so; do
  LSNIF_LIB=$PWD/$lib timeout 600 python scripts/trace_tune.py 16 2>&1 | grep '^{' >> gpurun_out/${TAG}_tune.jsonl
done
done
python - <<'PY' "$TAG"
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}_tune.jsonl"):
    r = json.loads(l)
    print(f"{r['lib']:22s} {r['set']:9s} trace {r['trace_ms']*1e3:8.1f} us  mlp {r['mlp_ms']*1e3:7.1f} us  query {r['query_ms']*1e3:8.1f} us")
PY
