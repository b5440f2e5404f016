#!/bin/bash
# Round-2 measurement set on one B200 (outputs under gpurun_out/r02/; the
# summaries worth keeping are copied to profiles/r02/).
mkdir -p gpurun_out/r02
python bench.py > gpurun_out/r02/bench_n1.json 2> gpurun_out/r02/bench_n1.err
for c in c1 c2 c4 tiny5 big64 big40; do python tools/run_config.py $c --steps 7 | tail -1 > gpurun_out/r02/config_$c.json; done
for o in 0.10 0.50; do python tools/run_config.py c3 --occ $o --steps 5 | tail -1 > gpurun_out/r02/config_c3_$o.json; done
python tools/run_c4_contract.py --steps 5 > gpurun_out/r02/c4_contract.json
python tools/run_c5.py --steps 2 > gpurun_out/r02/c5_1gpu.json 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r02/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_smm_dmma -s 4 -c 1 \
    -o gpurun_out/r02/ncu_bench_dmma python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
ls gpurun_out/r02
