# ncu --set full captures (source-mapped) of the trace and MLP kernels on C3
# (one launch each, after warm-up launches). Usage: bash scripts/gpu_prof_c3.sh TAG [workload]
TAG=${1:-r2}
W=${2:-c3}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG}_trace_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_trace_$W.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG}_mlp_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_mlp_$W.log 2>&1
ls -la gpurun_out
