"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    byid = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = byid.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]].split("(")[0].replace("void ", ""),
                                          "grid": r[ix["Grid Size"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return list(byid.values())


if __name__ == "__main__":
    items = load(sys.argv[1])
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for it in items:
        t = tot[it["name"]]
        t[0] += 1
        t[1] += it.get("gpu__time_duration.sum", 0) / 1e3
        t[2] += (it.get("dram__bytes_read.sum", 0) + it.get("dram__bytes_write.sum", 0)) / 1e6
    allt = sum(v[1] for v in tot.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'MB':>10s} {'TB/s':>8s}")
    for k, (n, us, mb) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:28]:28s} {n:8d} {us:10.1f} {us / allt:6.1%} {mb:10.1f} {mb / us * 1e3 / 1e3 if us else 0:8.1f}")
