# ncu --set full (source-mapped) of one mlp_tc_kernel launch per workload.
# Usage: bash scripts/gpu_prof_mlp2.sh TAG w1 [w2 ...]
TAG=$1; shift
mkdir -p gpurun_out
for W in "$@"; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG}_mlp_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_mlp_$W.log 2>&1
done
ls gpurun_out | grep $TAG
