set -x
mkdir -p gpurun_out
for W in c2 c3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 2 -c 1 -o gpurun_out/prof_trace_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trace_$W.log 2>&1
done
