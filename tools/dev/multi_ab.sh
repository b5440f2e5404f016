#!/bin/bash
# dev: per-class kernels vs one MULTI launch (BT_MULTI) on the mixed-size configs
for m in 0 1 0 1; do
  for c in c2 c4; do
    echo "BT_MULTI=$m $c $(BT_MULTI=$m timeout 300 python tools/run_config.py $c --no-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'])")"
  done
done
