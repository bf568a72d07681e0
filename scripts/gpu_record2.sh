# Round-2 record run: GPU tests, smoke, the default bench (C5) + its reference
# arm, and the secondary workloads. Usage: bash scripts/gpu_record2.sh TAG
TAG=${1:-rec}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -6 | tee gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py 2>gpurun_out/${TAG}_bench_c5.err | tail -1 > gpurun_out/${TAG}_bench_c5.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/${TAG}_bench_ref_c5.json
for w in c3 c2 c1 c4 render; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_bench_$w.json
done
for w in c5 c3 c2 c1 c4 render; do python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench_$w.json').read())
k=d.get('kernels', {}); print('$w', 'value %.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'ms/step %.3f'%d['ms_per_step'], {n: round(v['ms_per_step'], 3) for n, v in k.items()}, d['clocks'])
"; done
python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_ref_c5.json').read()); print('ref', d.get('value'), d.get('cpu_baseline', {}).get('cores'))"
