#!/bin/bash
# dev: numeric-phase sweep over the column-band count (BT_BANDS) on c1 and c5-like shapes
for b in 1 2 3 4; do
  echo "bands=$b c1"; BT_BANDS=$b timeout 300 python tools/quick_c1.py 23 400 0.1 2>&1 | tail -2
done
for b in 1 2 4; do
  echo "bands=$b 32x32 nb=600 occ .2"; BT_BANDS=$b timeout 300 python tools/quick_c1.py 32 600 0.2 2>&1 | tail -1
done
