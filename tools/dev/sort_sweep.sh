#!/bin/bash
# dev: fill-pass emission threshold sweep (BT_SORT_MIN) on c1 and c2
for t in 48 16 4 0; do
  echo "sort_min=$t c1"; BT_SORT_MIN=$t BT_PHASES=1 timeout 300 python tools/quick_c1.py 2>&1 | tail -2
  echo "sort_min=$t c2"; BT_SORT_MIN=$t timeout 300 python tools/run_config.py c2 --no-check 2>&1 | tail -1 | cut -c 150-400
done
