# Multi-rank logic on one GPU (gloo, both ranks on cuda:0) + reference arm under torchrun
set -x
mkdir -p gpurun_out
export LSNIF_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -v "^W1\|OMP" | tail -3 | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --workload c5 --no-cpu-baseline 2>&1 | grep -v "^W1\|OMP" | tail -3 | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 2>&1 | tail -2 | cut -c1-800
unset LSNIF_DIST_BACKEND
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_encode_kernel -s 2 -c 1 -o gpurun_out/prof_trace_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trace_c2.log 2>&1
