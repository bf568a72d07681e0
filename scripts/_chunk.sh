for rep in 1 2; do for c in 23 24; do
LSNIF_CHUNK_LOG2=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print($c, '%.4g'%r['value'], '%.3f'%r['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in r['kernels'].items()})"
done; done
