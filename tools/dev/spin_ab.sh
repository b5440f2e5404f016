#!/bin/bash
# dev: blocking vs polling host waits in the multiply (BT_SPIN_SYNC), c1 bench + host probe
for sp in 0 1 0 1; do
  echo "== BT_SPIN_SYNC=$sp"
  BT_SPIN_SYNC=$sp timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
  BT_SPIN_SYNC=$sp timeout 300 python tools/host_probe.py 2>&1 | tail -2
done
