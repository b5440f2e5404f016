#!/bin/bash
# dev: NCCL algorithm choice for the case-2 B gather at 4 GPUs (BT_PHASES timeline)
for a in default Ring NVLS; do
  if [ "$a" = default ]; then unset NCCL_ALGO; else export NCCL_ALGO=$a; fi
  echo "== NCCL_ALGO=$a"
  BT_PHASES=1 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING,INIT timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/nccl_$a.log 2>&1
  grep "bt-gather" gpurun_out/nccl_$a.log | tail -3
  tail -1 gpurun_out/nccl_$a.log | cut -c1-160
done
