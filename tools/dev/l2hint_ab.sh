#!/bin/bash
# dev: L2 cache hints on the stage copies (BT_L2_HINTS) x column bands (BT_BANDS), c1
for b in 2 4; do for h in 0 1; do
  echo "bands=$b hints=$h $(BT_BANDS=$b BT_L2_HINTS=$h timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'])")"
done; done
