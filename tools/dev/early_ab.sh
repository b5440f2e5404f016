#!/bin/bash
# dev: early stage release (copy of the next product issued before the last k tile's DMMAs)
for lib in late early late early; do
  echo "== $lib"
  BT_LIB=_bisect/$lib.so timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 bench', d['ms_per_step'], d['roofline']['achieved'])"
  BT_LIB=_bisect/$lib.so timeout 300 python tools/quick_c1.py 32 600 0.2 2>&1 | tail -1 | cut -c 1-90
  for c in c2 c3 c4; do echo "$c $(BT_LIB=_bisect/$lib.so timeout 300 python tools/run_config.py $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'])")"; done
done
