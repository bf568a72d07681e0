# Quick iteration: GPU parity tests + C2/C3 bench (no ncu)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c2.log
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c3.log
./examples/query_cpp tests/golden/teapot_seed0.lsnif
