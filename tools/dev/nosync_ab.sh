#!/bin/bash
# dev: exact two-pass multiply vs the bounded single pass (BT_NOSYNC), with and
# without the nvidia-smi clock sampler
for smi in 1 0; do
for ns in 0 1; do
  echo "== BT_NOSYNC=$ns no_smi=$smi"
  if [ $smi = 1 ]; then export BT_BENCH_NO_SMI=1; else unset BT_BENCH_NO_SMI; fi
  BT_NOSYNC=$ns BT_BENCH_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --steps 8 2>&1 | grep "rank 0\|metric" | cut -c 1-200
done
done
