#!/bin/bash
# dev: tile height for tall blocks (BT_TALL_ROWS) on c4
for t in 32 24; do
  echo "c4 tall_rows=$t"; BT_TALL_ROWS=$t timeout 300 python tools/run_config.py c4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'], d['numeric_tflops'], d.get('max_frob_rel'))"
done
