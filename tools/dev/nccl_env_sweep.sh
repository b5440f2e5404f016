#!/bin/bash
# dev: NCCL channel/protocol settings for the case-2 B gather at 4 GPUs
run() {
  env "$@" BT_PHASES=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/nenv.log 2>&1
  echo "== $*: $(tail -1 gpurun_out/nenv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])")"
  grep "bt-gather" gpurun_out/nenv.log | sed -n 8,9p
}
run X=1
run NCCL_MIN_NCHANNELS=32
run NCCL_PROTO=Simple
run NCCL_MIN_NCHANNELS=32 NCCL_PROTO=Simple
run NCCL_NTHREADS=512
