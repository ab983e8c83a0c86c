"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if r[0] == "ID")
    H = rows[hdr]
    agg = collections.defaultdict(lambda: [0, 0.0, set()])
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        d = dict(zip(H, r))
        name = d["Kernel Name"].split("(")[0].split("::")[-1].replace("void ", "")
        v = float(d["Metric Value"]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        a = agg[name]
        a[0] += 1
        a[1] += v
        a[2].add(d["Grid Size"])
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    print(f"{n} launches, {tot:.1f} us total (ncu: serialised, cold-cache)")
    for k, (c, t, grids) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:42s} n={c:5d} total={t:10.1f}us avg={t / c:8.2f}us share={t / tot:6.1%} grids={sorted(grids)[:3]}")


if __name__ == "__main__":
    main(sys.argv[1])
