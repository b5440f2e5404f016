#!/bin/bash
# dev: whole-product stages vs the k-tile ring (BT_KT_RING / BT_KT_SLOTS)
BT_KT_RING=1 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for v in "0 0" "1 3" "1 4" "1 6"; do
  set -- $v
  echo "== ring=$1 slots=$2"
  BT_KT_RING=$1 BT_KT_SLOTS=$2 timeout 300 python tools/quick_c1.py 2>&1 | tail -1
  BT_KT_RING=$1 BT_KT_SLOTS=$2 timeout 300 python tools/quick_c1.py 32 600 0.2 2>&1 | tail -1
  for c in c3 c4; do
    BT_KT_RING=$1 BT_KT_SLOTS=$2 timeout 300 python tools/run_config.py $c --no-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_median'], d['numeric_ms'], d['numeric_tflops'])"
  done
done
