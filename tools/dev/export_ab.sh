#!/bin/bash
# dev: D2H streams of the chunked export (BT_EXPORT_STREAMS) on the c1 e2e probe
for n in 1 2 4 1 2 4; do
  echo "== BT_EXPORT_STREAMS=$n"; BT_EXPORT_STREAMS=$n timeout 300 python tools/e2e_probe.py 2>&1 | grep putA | tail -2
done
