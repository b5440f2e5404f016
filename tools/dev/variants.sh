#!/bin/bash
# dev: numeric-kernel variants on config 1
for ktr in 3 0; do
  for s in 1 2; do
    echo "== KTR=$ktr stages=$s"
    BT_KTR=$ktr BT_STAGES=$s python tools/quick_c1.py 2>&1 | tail -1
  done
done
