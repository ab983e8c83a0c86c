"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv):
per kernel name the launch count, total / average duration, share of the listed time and, when captured,
the DRAM bytes per launch.  ncu serialises launches and runs them cold, so the absolute times are not bench
numbers; the kernels' shares are what compares with the bench's probes.

    python profiles/launch_summary.py launches.csv [out.json]
"""
import collections
import csv
import json
import sys

TIME_SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTE_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if r[0] == "ID")
    H = rows[hdr]
    launches = collections.defaultdict(dict)  # launch id -> metrics
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        d = dict(zip(H, r))
        rec = launches[d["ID"]]
        rec["name"] = d["Kernel Name"].split("(")[0].split("::")[-1].replace("void ", "")
        rec["grid"] = d["Grid Size"]
        m, u = d["Metric Name"], d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            rec["us"] = v * TIME_SCALE.get(u, 1.0)
        elif m.startswith("dram__bytes"):
            rec["bytes"] = rec.get("bytes", 0.0) + v * BYTE_SCALE.get(u, 1.0)
    agg = collections.defaultdict(lambda: {"n": 0, "us": 0.0, "bytes": 0.0, "grids": set()})
    for rec in launches.values():
        if "us" not in rec:
            continue
        a = agg[rec["name"]]
        a["n"] += 1
        a["us"] += rec["us"]
        a["bytes"] += rec.get("bytes", 0.0)
        a["grids"].add(rec["grid"])
    tot = sum(a["us"] for a in agg.values())
    out = {"launches": sum(a["n"] for a in agg.values()), "total_us": tot, "kernels": {}}
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        out["kernels"][k] = {"launches": a["n"], "total_us": a["us"], "avg_us": a["us"] / a["n"],
                             "share": a["us"] / tot if tot else 0.0,
                             "dram_bytes_per_launch": a["bytes"] / a["n"] if a["bytes"] else None,
                             "grids": sorted(a["grids"])[:3]}
    return out


def main(path, out=None):
    s = summarise(path)
    print(f"{s['launches']} launches, {s['total_us']:.1f} us total (ncu: serialised, cold-cache)")
    for k, a in s["kernels"].items():
        b = f" dram/launch={a['dram_bytes_per_launch'] / 1e6:.2f}MB" if a["dram_bytes_per_launch"] else ""
        print(f"{k:42s} n={a['launches']:5d} avg={a['avg_us']:8.2f}us share={a['share']:6.1%}{b} grids={a['grids']}")
    if out:
        json.dump(s, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:3])
