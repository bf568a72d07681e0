# Round-2 record profiles: ncu --set full of one trace and one MLP launch on
# the headline workload (C5) and on C3, the launch list of a default bench
# run, and the SASS census. Usage: bash scripts/gpu_prof_r2.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
for W in c5 c3; do
  EXTRA=""
  [ $W = c5 ] && EXTRA="--rays 16777216"  # a 16.8M-ray C5 frame: same launches, fewer of them
  for K in trace_encode_kernel mlp_tc_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/${TAG}_${K%%_*}_$W python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline \
      $EXTRA > gpurun_out/${TAG}_ncu_${K%%_*}_$W.log 2>&1
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  --rays 16777216 > gpurun_out/${TAG}_launches_c5.log 2>&1
ls gpurun_out | grep $TAG
