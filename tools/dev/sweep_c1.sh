#!/bin/bash
# dev sweep of numeric-kernel launch knobs on config 1
for cfg in "8 2" "8 3" "12 2" "8 4" "16 2"; do
  set -- $cfg
  echo "== BT_WARPS_PER_SM=$1 BT_STAGES=$2"
  BT_WARPS_PER_SM=$1 BT_STAGES=$2 python tools/quick_c1.py 2>&1 | tail -2
done
