#!/bin/bash
# Round-end verification + measurement set on one 4-GPU box: GPU tests, smoke,
# then tools/final_measure.sh (bench 1/2/4 + reference arm, c2-c5, ncu), then
# c3 through case 1 on 2 and 4 GPUs.
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
bash tools/final_measure.sh > gpurun_out/final/measure.log 2>&1
for n in 2 4; do for o in 0.1 0.5; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2953$n tools/run_c3_dist.py --occ $o --steps 5 --check > gpurun_out/final/c3_case1_${n}gpu_$o.json 2>&1
done; done
