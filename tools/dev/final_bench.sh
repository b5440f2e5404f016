#!/bin/bash
# Round-end bench set on one 4-GPU box: 1/2/4 GPUs + the reference arm
mkdir -p gpurun_out/final
timeout 400 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2951$n bench.py --gpus $n > gpurun_out/final/bench_n$n.json 2> gpurun_out/final/bench_n$n.err
done
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
