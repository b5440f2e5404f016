#!/bin/bash
# dev: warps per CTA of the numeric kernel (w4: 4 x 5 = 20 warps/SM, w3: 3 x 7 = 21)
for lib in w4 w3 w4 w3; do
  echo "== $lib"
  BT_LIB=_bisect/$lib.so timeout 300 python tools/quick_c1.py 2>&1 | tail -1
  BT_LIB=_bisect/$lib.so timeout 300 python tools/quick_c1.py 32 600 0.2 2>&1 | tail -1
  for c in c2 c3 c4; do echo "$c $(BT_LIB=_bisect/$lib.so timeout 300 python tools/run_config.py $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_median'], d['numeric_ms'])")"; done
done
