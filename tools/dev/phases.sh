# usage: phases.sh CONFIG "ENV=.. ENV=.." ... -- median symbolic/numeric phases per variant
c=$1; shift
for v in "$@"; do
  env $v BT_PHASES=1 python tools/run_config.py $c --steps 7 > /tmp/o.txt 2>&1
  python - "$v" "$c" <<'PY'
import sys, re, json, statistics
t = open('/tmp/o.txt').read()
ph = re.findall(r'pass1\+scan ([\d.]+) us \| host sync gap ([\d.]+) us \| fill ([\d.]+) us \| pre-numeric ([\d.]+) us \| numeric ([\d.]+) us \| total ([\d.]+) us', t)[2:]
j = json.loads(t.strip().splitlines()[-1])
med = lambda i: statistics.median(float(p[i]) for p in ph)
print(f"{sys.argv[2]} [{sys.argv[1]:28s}] pass1 {med(0):7.1f} gap {med(1):5.1f} fill {med(2):7.1f} pre {med(3):5.1f} numeric {med(4):8.1f} total {med(5):8.1f} us  step {j['ms_median']} ms")
PY
done
