#!/bin/bash
# dev: ring depth (BT_STAGES) sweep of the numeric phase on c3 / c4
for c in c4 c3; do
  for s in 1 2; do
    echo "$c stages=$s"; BT_STAGES=$s timeout 300 python tools/run_config.py $c --no-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'], d['numeric_tflops'])"
  done
done
