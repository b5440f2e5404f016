#!/bin/bash
# dev: ring depth / warps sweep on c2 (small mixed blocks, latency bound)
for v in "0 24" "4 24" "4 12" "4 8" "2 12"; do
  set -- $v
  echo "== BT_STAGES=$1 BT_WARPS_PER_SM=$2"
  BT_STAGES=$1 BT_WARPS_PER_SM=$2 timeout 300 python tools/run_config.py c2 --no-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'])"
done
