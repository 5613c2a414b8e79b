"""Per-launch table of the factor-solve kernels from an ncu --csv launch list (last sweep)."""
import sys
sys.path.insert(0, __file__.rsplit('/', 2)[0] + '/profiles')
from parse_launches import load

items = load(sys.argv[1])
nsweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = len(items) // nsweeps
tot = 0.0
agg = {}
for it in items[-n:]:
    t = it['gpu__time_duration.sum'] / 1e3
    b = (it.get('dram__bytes_read.sum', 0) + it.get('dram__bytes_write.sum', 0)) / 1e6
    k = it['name'].split('::')[-1]
    tot += t
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1; a[1] += t; a[2] += b
    if '-v' in sys.argv:
        print(f"{k:22s} {it['grid']:>14s} {t:8.1f}us {b:9.1f}MB {b / t:6.2f}TB/s")
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:22s} {c:4d} {t:9.1f}us {b:9.1f}MB {b / t:6.2f}TB/s")
print(f"total {tot:.1f} us per sweep (serialised, cold)")
