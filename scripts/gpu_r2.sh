# Round-2 GPU session: GPU tests, smoke, the default bench (C5) + the reference
# arm, secondary lines. Usage: bash scripts/gpu_r2.sh [tag]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"; df -h /dev/shm | tail -1; free -g | head -2
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 | tee gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py 2>gpurun_out/${TAG}_bench_c5.err | tail -1 | tee gpurun_out/${TAG}_bench_c5.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 | tee gpurun_out/${TAG}_bench_ref_c5.json
timeout 600 python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/${TAG}_bench_c3.json
timeout 600 python bench.py --workload c2 2>&1 | tail -1 | tee gpurun_out/${TAG}_bench_c2.json
tail -5 gpurun_out/${TAG}_bench_c5.err
