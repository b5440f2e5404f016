#!/bin/bash
# dev: A/B two builds of libbtcuda (BT_LIB) on c1 (quick_c1) and c5-like shapes
for lib in "$@"; do
  echo "== $lib"
  BT_LIB=$lib timeout 300 python tools/quick_c1.py 2>&1 | tail -2
  BT_LIB=$lib timeout 300 python tools/quick_c1.py 32 600 0.2 2>&1 | tail -1
done
