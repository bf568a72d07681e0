# Device time per query (scripts/trace_tune.py) of the in-tree build under
# each value of an environment switch. Usage: bash scripts/gpu_ab_env.sh TAG VAR v1 [v2 ...]
TAG=$1; VAR=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  env $VAR=$v timeout 600 python scripts/trace_tune.py 16 2>&1 | grep '^{' | sed "s/^{/{\"$VAR\": \"$v\", /" >> gpurun_out/${TAG}_env.jsonl
done
python - "$TAG" "$VAR" <<'PY'
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}_env.jsonl"):
    r = json.loads(l)
    print(f"{sys.argv[2]}={r[sys.argv[2]]:4s} {r['set']:9s} trace {r['trace_ms']*1e3:8.1f} us  bin {r.get('bin_ms',0)*1e3:6.1f} us  mlp {r['mlp_ms']*1e3:7.1f} us  query {r['query_ms']*1e3:8.1f} us")
PY
