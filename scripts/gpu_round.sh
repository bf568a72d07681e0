# One GPU session: tests, smoke, bench, ncu launch list + full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_c2.log
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -2 | tee gpurun_out/bench_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 4 -c 1 -o gpurun_out/prof_trace_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 4 -c 1 -o gpurun_out/prof_mlp_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_mlp.log 2>&1
ls -la gpurun_out
