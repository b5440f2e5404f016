#!/bin/bash
# dev: K-panel count on c3 (BT_KPANELS; 0 = heuristic)
for occ in 0.1 0.5; do
  for p in 0 1 4 16 32; do
    echo "c3 occ=$occ panels=$p $(BT_KPANELS=$p timeout 300 python tools/run_config.py c3 --occ $occ 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'], d['numeric_tflops'])")"
  done
done
