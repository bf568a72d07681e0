# Full GPU check: all -m gpu tests, smoke, default bench (C5) and C3/C2 lines.
# Usage: bash scripts/gpu_full.sh TAG
TAG=${1:-full}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -6 | tee gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py 2>gpurun_out/${TAG}_bench_c5.err | tail -1 > gpurun_out/${TAG}_bench_c5.json
timeout 600 python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_bench_c3.json
timeout 600 python bench.py --workload c2 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_bench_c2.json
for w in c5 c3 c2; do python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench_$w.json').read())
k=d['kernels']; print('$w', 'value %.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'trace %.3f ms'%k['trace_encode_kernel']['ms_per_step'], 'mlp %.3f ms %.0f TF/s'%(k['mlp_tc_kernel']['ms_per_step'], k['mlp_tc_kernel']['tflops']), 'clk', d['clocks'])
"; done
