#!/usr/bin/env python
"""Faster-MoA tree request benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl b200|reference]

One *step* = one tree-MoA request (run_query, orchestrator.cpp:130-295) of the
configured workload, sample index = step % 24 (the preset's 24 repetitions,
config.cpp:230).  `value` = agent tokens/s = output tokens of invoked,
unpruned agents / device-event time (first tick -> last completion), summed
over the K timed requests; L2 is flushed (256 MiB write) between requests,
outside each request's events.  `e2e` = the same metric through the C-ABI call
with host buffers (prompt synthesis, row upload, result read-back) on the host
wall clock.  Multi-GPU (torchrun): each rank serves its own requests
(replicas), value = all ranks' tokens / max rank time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tree_moa_agent_tokens_per_s"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-baseline-s", type=float, default=15.0, help="CPU sample budget (seconds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--placement", default="replicas", choices=["replicas", "tree"],
                    help="N>1: independent replicas (weak scaling) or one request tree-partitioned over the ranks")
    ap.add_argument("--profile-only", action="store_true", help="run steps without JSON (for ncu)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary 1B-agent (C2) decode measurement reported beside the headline")
    ap.add_argument("--secondary-out", type=int, default=128, help="C2 output tokens per agent for the secondary run")
    ap.add_argument("--no-timeline", action="store_true", help="skip the in-graph tick timeline (chain stamps)")
    ap.add_argument("--concurrency", default="4,8",
                    help="continuous-batching sweep reported beside the headline (comma list; '' to skip)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.stop = device, [], threading.Event()

    def _loop(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 7:
                    self.rows.append(vals)
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return j["hbm_gbs"], j["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


def roofline(probes, hbm_gbs, src, cfg_name="C1"):
    """Dominant kernel (largest share of probed time): algorithmic bytes per
    launch / average launch duration, against the measured HBM copy peak.
    `traffic` = DRAM bytes per launch of that kernel from the committed ncu
    --set full capture of this config (profiles/ncu_traffic.json)."""
    kind, v = max(probes.items(), key=lambda kv: kv[1]["ms"])
    if v["launches"] == 0:
        return None
    achieved = v["bytes"] / (v["ms"] / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(cfg_name, {}).get(kind)
    return {"kernel": kind, "bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
            "frac": achieved / hbm_gbs, "traffic": traffic, "peak_source": src,
            "bytes_per_launch": v["bytes"] / v["launches"], "avg_us": 1e3 * v["ms"] / v["launches"],
            "share_of_probed_time": v["ms"] / max(1e-12, sum(p["ms"] for p in probes.values()))}


def secondary_c2(args, hbm, src, local):
    """The headline C1 agents are tiny (34 MB of weights, latency-bound); the
    HBM roofline of the decode path is only visible at the ~1B shape.  One
    C2-shaped request (tree 8-2-1 of ~1B agents, `--secondary-out` tokens per
    agent) is timed with device events like the headline, then replayed with
    kernel probes: per-kernel achieved GB/s against the measured HBM peak."""
    import torch
    from paper_2512_18126_b200 import capi
    from paper_2512_18126_b200.configs import C2
    cfg = dict(C2, out_len=[args.secondary_out] * 3)
    eng, qc = capi.engine_for(cfg, device=local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    eng.run_query(qc, sample=0, resolve=False, detail=False)  # warm-up (graph capture)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    r = eng.run_query(qc, sample=1, resolve=False, detail=False)
    fwd_gb = r["weight_bytes"] / 1e9
    out = {"config": {"workload": cfg["workload"].replace("greedy 512", f"greedy {args.secondary_out}"),
                      "name": "C2", "models": {t: m["shape"] for t, m in cfg["models"].items()}},
           "value": r["tokens"] / (r["e2e_ms"] / 1e3), "unit": UNIT, "e2e_ms": r["e2e_ms"], "ticks": r["ticks"],
           "forwards": r["forwards"], "ms_per_forward": r["e2e_ms"] / max(1, r["forwards"]),
           "weight_gb_per_forward": fwd_gb / max(1, r["forwards"]),
           "weight_stream_gbs": fwd_gb / (r["e2e_ms"] / 1e3),
           "weight_stream_frac": fwd_gb / (r["e2e_ms"] / 1e3) / hbm}
    eng.probe(True)
    eng.run_query(qc, sample=1, resolve=False, detail=False)
    probes = eng.probe_stats()
    eng.probe(False)
    out["kernels"] = {k: {"launches": v["launches"], "avg_us": 1e3 * v["ms"] / max(1, v["launches"]),
                          "gbs": v["bytes"] / max(1e-12, v["ms"] / 1e3) / 1e9,
                          "frac_hbm": v["bytes"] / max(1e-12, v["ms"] / 1e3) / 1e9 / hbm}
                      for k, v in probes.items() if v["launches"]}
    out["roofline"] = roofline(probes, hbm, src, "C2")
    out["note"] = ("kernels: CUDA events around every launch (graphs bypassed, so launch gaps are inside "
                   "each kernel's time); weight_stream_frac: whole-forward weight bytes / device time")
    eng.close()
    return out


def concurrency_sweep(cfg, levels, local):
    """Continuous batching: B independent requests of the same config served
    concurrently by one engine (moa_run_batch).  Throughput = all requests'
    agent tokens / the batch's device time; latency = each request's own
    first-tick -> last-completion time.  Reported beside the single-request
    headline (which matches the reference's one-request-at-a-time
    run_repetitions, orchestrator.cpp:297-302)."""
    import torch
    from paper_2512_18126_b200 import capi
    out = []
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for b in levels:
        eng, qc = capi.engine_for(cfg, device=local, concurrency=b)
        eng.run_batch(qc, list(range(b)), resolve=False, detail=False)  # warm-up (graph capture)
        flush.fill_(2.0)
        torch.cuda.synchronize()
        rs = eng.run_batch(qc, [b + i for i in range(b)], resolve=False, detail=False)
        eng.close()
        batch_ms = max(r["e2e_ms"] for r in rs)
        lat = sorted(r["e2e_ms"] for r in rs)
        out.append({"concurrent_requests": b, "value": sum(r["tokens"] for r in rs) / (batch_ms / 1e3), "unit": UNIT,
                    "batch_ms": batch_ms, "p50_ms_per_request": lat[len(lat) // 2], "ticks": rs[0]["ticks"]})
    return out


def cpu_baseline(cfg, budget_s):
    """The oracle (numpy transformer + reference-semantics orchestration) on
    a bounded sample of the same workload, all host cores."""
    import numpy as np  # noqa: F401

    from oracle.configs import models_of, run_config
    from oracle.orchestrator import run_query
    rc = run_config(cfg)
    ms = models_of(cfg, 1024)
    t0, toks, n = time.perf_counter(), 0, 0
    while True:
        r = run_query(rc, ms, n % 24)
        toks += r["tokens"]
        n += 1
        if time.perf_counter() - t0 > budget_s or n >= 24:
            break
    dt = time.perf_counter() - t0
    return {"value": toks / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{n} {cfg['name']} requests (samples 0..{n - 1}), oracle/orchestrator.py + numpy fp32 "
                      f"transformer, {os.cpu_count()} host threads", "seconds": dt, "tokens": toks}


def reference_simulator_time(cfg, reps=24):
    """Wall time of the reference's own run_repetitions (the virtual-time
    simulator, oracle/_ref) on the same tree shape -- context only."""
    lib = ROOT / "oracle" / "_ref" / "libmoaref.so"
    if not lib.exists():
        return None
    import ctypes
    L = ctypes.CDLL(str(lib))
    L.moaref_call.restype = ctypes.c_char_p
    t = cfg["topology"]
    req = {"cmd": "time_run_query", "topology": t, "reps": reps,
           "profiles": {tag: {"output_len": cfg["out_len"][0] if isinstance(cfg["out_len"][0], int) else 64}
                        for tag in cfg["models"]},
           "assign": cfg["assign"], "mode": cfg["mode"], "early_exit": cfg["early_exit"],
           "chunk_size": cfg["chunk_size"], "seed": cfg["seed"]}
    r = json.loads(L.moaref_call(json.dumps(req).encode()))
    if "seconds" not in r:
        return None
    return {"seconds_per_request": r["seconds"] / reps, "reps": reps, "cores": 1,
            "note": "reference SimWorld (virtual-time, no model compute), orchestrator.cpp:297-302"}


def run_reference_arm(args, cfg, rank, world):
    if rank != 0:
        return
    tree = world > 1 and args.placement == "tree"
    steps = []
    from oracle.configs import models_of, run_config
    from oracle.orchestrator import run_query
    rc, ms = run_config(cfg), models_of(cfg, 1024)
    for i in range(args.warmup):
        run_query(rc, ms, i % 24)
    t_all = time.perf_counter()
    toks = 0
    for i in range(args.steps):
        t0 = time.perf_counter()
        r = run_query(rc, ms, i % 24)
        steps.append(time.perf_counter() - t0)
        toks += r["tokens"]
    dt = time.perf_counter() - t_all
    value = toks / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "p50_ms_per_request": 1e3 * statistics.median(steps), "higher_is_better": True,
            "scaling": "strong" if tree else "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "name": cfg["name"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{args.steps} {cfg['name']} requests through oracle/ (numpy fp32 "
                                       f"transformer agents + reference-semantics orchestration)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    sim = reference_simulator_time(cfg)
    if sim:
        line["reference_simulator"] = sim
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    from paper_2512_18126_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    from paper_2512_18126_b200 import capi

    eng, qc = capi.engine_for(cfg, device=local)
    tree = world > 1 and args.placement == "tree"
    if tree:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(capi.nccl_unique_id()), dtype=torch.uint8))
        pg.broadcast(uid, 0)
        eng.attach_comm(bytes(uid.cpu().numpy()), rank, world)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def sample_of(i):  # tree mode: every rank serves the same request
        return (i if tree else rank * 1000 + i) % 24

    def one(i, detail=False):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        return eng.run_query(qc, sample=sample_of(i), resolve=detail, detail=detail)

    for i in range(args.warmup):
        one(i)
    if args.profile_only:
        for i in range(args.steps):
            one(i)
        return
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    dev_ms, toks, per_req, rows, fwd, wbytes, host_ms = 0.0, 0, [], 0, 0, 0.0, 0.0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            s = one(i)
            host_ms += s["host_ms"]
            dev_ms += s["e2e_ms"]
            per_req.append(s["e2e_ms"])
            toks += s["tokens"]
            rows += s["rows"]
            fwd += s["forwards"]
            wbytes += s["weight_bytes"]
    torch.cuda.synchronize()
    # e2e: through the C-ABI with host buffers (resolve = copy results back)
    e2e_wall, e2e_toks, h2d, d2h = 0.0, 0, 0, 0
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = eng.run_query(qc, sample=sample_of(i), resolve=True, detail=True)
        e2e_wall += time.perf_counter() - t0
        e2e_toks += r["tokens"]
        h2d += r["rows"] * 16
        d2h += sum(4 * len(a["prompt"]) + 12 * len(a["output"]) for a in r["agents"].values())
    # kernel probes: CUDA events around every forward kernel while the same
    # K requests replay (graphs bypassed during this pass only)
    eng.probe(True)
    n_ee_launches = 0
    for i in range(args.steps):
        r = one(i, detail=True)
        n_ee_launches += sum(4 + (e["outputs"] > 1) for e in r["metricq"] if e["evaluated"])
    probes = eng.probe_stats()
    eng.probe(False)
    # in-graph tick timeline of one more (untimed) request: per-CTA %globaltimer
    # stamps of the decode chain (chain.py) -- the probes above bypass the graphs
    timeline = None
    if rank == 0 and not args.no_timeline:
        from paper_2512_18126_b200 import chain
        try:
            timeline = chain.request_timeline(eng, qc, sample_of(0))
        except Exception as e:  # diagnostics only
            timeline = {"error": str(e)}
    if pg:
        t = torch.tensor([dev_ms, e2e_wall * 1e3, toks, e2e_toks], dtype=torch.float64, device="cuda")
        mx = t.clone()
        pg.all_reduce(mx, op=pg.ReduceOp.MAX)
        sm = t.clone()
        pg.all_reduce(sm, op=pg.ReduceOp.SUM)
        dev_ms_max, e2e_ms_max, toks_all, e2e_toks_all = mx[0].item(), mx[1].item(), sm[2].item(), sm[3].item()
        if tree:  # one request shared by all ranks: count its tokens once
            toks_all, e2e_toks_all = toks, e2e_toks
    else:
        dev_ms_max, e2e_ms_max, toks_all, e2e_toks_all = dev_ms, e2e_wall * 1e3, toks, e2e_toks
    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return
    hbm, tf, src = peaks()
    value = toks_all / (dev_ms_max / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
        "p50_ms_per_request": statistics.median(per_req), "higher_is_better": True,
        "scaling": "strong" if tree else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": cfg["workload"], "name": cfg["name"], "l2": "flushed (256 MiB write) between requests",
                   "models": {t: m["shape"] for t, m in cfg["models"].items()}, "parallelism": f"tree{world}" if tree else f"replicas{world}"},
        "e2e": {"value": e2e_toks_all / (e2e_ms_max / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": int(sum(v["launches"] for v in probes.values()) + n_ee_launches),
        "roofline": roofline(probes, hbm, src, cfg["name"]),
        "kernels": {k: {"launches": v["launches"], "ms_per_request": v["ms"] / args.steps,
                        "avg_us": 1e3 * v["ms"] / max(1, v["launches"]),
                        "gbs": v["bytes"] / max(1e-12, v["ms"] / 1e3) / 1e9} for k, v in probes.items()},
        "tick_timeline": timeline,
        "clocks": clk.summary(),
        "peaks": {"hbm_gbs": hbm, "bf16_tflops": tf, "source": src},
        "engine": {"rows_per_request": rows / args.steps, "forwards_per_request": fwd / args.steps,
                   "host_ms_per_request": host_ms / args.steps,
                   "weight_gb_per_request": wbytes / args.steps / 1e9,
                   "weight_stream_gbs": wbytes / (dev_ms / 1e3) / 1e9},
    }
    eng.close()  # the headline engine; the extra measurements build their own
    if not args.no_secondary and args.config != "C2":
        line["secondary"] = secondary_c2(args, hbm, src, local)
    levels = [int(x) for x in args.concurrency.split(",") if x.strip()]
    if levels and not tree:
        line["concurrency"] = concurrency_sweep(cfg, levels, local)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_baseline_s)
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
