#!/bin/bash
# Per-kernel launch list (ncu, cold, serialised) of one frame: scripts/launch_list.sh CFG OUT.csv [bwd]
cfg=$1; out=$2; shift 2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" python scripts/one_frame.py "$cfg" "$@" > /dev/null 2>&1
python - "$out" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[vi].replace(',', '')) * {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}[r[ui]]
    k = r[ki].split('(')[0][:60]
    n, t = agg.get(k, (0, 0.0)); agg[k] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f'{t/1e3:9.3f} ms {100*t/tot:5.1f}% x{n:<4d} {k}')
print(f'{tot/1e3:9.3f} ms total')
PY
