#!/bin/bash
# Round-end measurement set on one box (4 GPUs): bench 1/2/4 GPUs + reference
# arm, configs c2-c5, then the ncu launch list and one full capture of the
# numeric kernel of the bench (single GPU, after the plain run exited 0).
set -x
mkdir -p gpurun_out/final
nvidia-smi -L > gpurun_out/final/smi.txt
timeout 400 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2951$n bench.py --gpus $n > gpurun_out/final/bench_n$n.json 2> gpurun_out/final/bench_n$n.err
done
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
for c in c2 c3 c4; do timeout 400 python tools/run_config.py $c > gpurun_out/final/config_$c.json 2>&1; done
timeout 600 python tools/run_config.py c3 --occ 0.5 > gpurun_out/final/config_c3_occ0.5.json 2>&1
timeout 900 python tools/run_c5.py > gpurun_out/final/config_c5_1gpu.json 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29519 tools/run_c5.py --cannon > gpurun_out/final/config_c5_cannon4.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_smm_dmma -s 4 -c 1 \
  -o gpurun_out/final/prof_bench_dmma python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/final/ncu_full.log 2>&1
