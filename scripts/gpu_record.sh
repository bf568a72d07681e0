# Full record: tests, smoke, default bench (with CPU baseline), C3/C4/C1 bench lines,
# ncu launch list and full captures of both kernels (C2), traffic summary.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_c2.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 | tee gpurun_out/bench_ref_c2.json
timeout 600 python bench.py --workload c3 --steps 10 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c4 --steps 10 2>&1 | tail -1 | tee gpurun_out/bench_c4.json
timeout 600 python bench.py --workload c1 --steps 20 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c1.json
timeout 600 python bench.py --workload render --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_render.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 2 -c 1 -o gpurun_out/prof_trace_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 -o gpurun_out/prof_mlp_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_mlp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 2 -c 1 -o gpurun_out/prof_trace_c3 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trace_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 -o gpurun_out/prof_mlp_c3 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_mlp_c3.log 2>&1
# per-ray kernel metrics for the auxiliary rooflines (profiles/kernel_metrics_<w>.json)
M=$(python scripts/metrics_probe.py metrics)
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"trace_encode|mlp_tc" --launch-skip 6 --log-file gpurun_out/metrics_c2.csv python scripts/metrics_probe.py run c2 gpurun_out/metrics_rays_c2.json > gpurun_out/metrics_c2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"trace_encode|mlp_tc" --launch-skip 2 --log-file gpurun_out/metrics_c3.csv python scripts/metrics_probe.py run c3 gpurun_out/metrics_rays_c3.json > gpurun_out/metrics_c3.log 2>&1
ls gpurun_out
