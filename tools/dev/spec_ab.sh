#!/bin/bash
# dev: case-2 B gather, exact vs speculative capacities, 2 and 4 GPUs (bench.py)
for n in 4 2; do
  for sp in 0 1 0 1; do
    BT_GATHER_SPEC=$sp timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n spec=$sp', d['ms_per_step'], d['value'])"
  done
done
