#!/bin/bash
# multi-GPU bench lines on all visible GPUs (run under gpurun --gpus N)
N=$(python -c "import torch; print(torch.cuda.device_count())")
mkdir -p gpurun_out/m
for c in c2 c4 c5; do
  steps=20; [ $c = c5 ] && steps=10
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps $steps --warmup 3 --config $c \
    > gpurun_out/m/bench_${c}_${N}gpu.json 2> gpurun_out/m/bench_${c}_${N}gpu.err
  echo "$c: $(head -c 200 gpurun_out/m/bench_${c}_${N}gpu.json)"
done
