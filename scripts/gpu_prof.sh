# ncu full captures of both kernels on a workload ($1 = c2|c3)
set -x
W=${1:-c3}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 -o gpurun_out/prof_mlp_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_mlp_$W.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 2 -c 1 -o gpurun_out/prof_trace_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trace_$W.log 2>&1
ls gpurun_out
