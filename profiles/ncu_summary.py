"""Summarise ncu --set full reports: per kernel launch, duration, DRAM bytes,
DRAM / L2 throughput, SM activity, achieved occupancy.

    python profiles/ncu_summary.py out.json report1.ncu-rep [report2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_active.avg": "sm_active_cycles_avg",
    "sm__cycles_active.max": "sm_active_cycles_max",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pipe_active_pct",
}
UNIT_SCALE = {"us": 1.0, "usecond": 1.0, "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            if k not in d:
                continue
            try:
                v = float(d[k])
            except ValueError:
                continue
            unit = u.get(k, "")
            if name == "duration_us":
                v *= UNIT_SCALE.get(unit, 1.0)
            elif "bytes" in name and unit in UNIT_SCALE:
                v *= UNIT_SCALE[unit]
            rec[name] = v
        if "duration_us" in rec and "dram_read_bytes" in rec:
            rec["dram_gbs"] = (rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0)) / (rec["duration_us"] * 1e3)
        res.append(rec)
    return res


if __name__ == "__main__":
    out = {rep.split("/")[-1]: summarise(rep) for rep in sys.argv[2:]}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    for rep, recs in out.items():
        for r in recs:
            print(rep, r["kernel"][:48], {k: round(v, 2) for k, v in r.items() if isinstance(v, float)})
