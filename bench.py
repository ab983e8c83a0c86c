#!/usr/bin/env python
"""Faster-MoA tree request benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl b200|reference]

One *step* = one tree-MoA request (run_query, orchestrator.cpp:130-295) of the
configured workload (default C3: tree 8-2-1 of heterogeneous 1B/8B agents,
2048-token leaf prompts, 512 greedy tokens per agent -- the largest BASELINE
config that fits one GPU), sample index = step % 24 (the preset's 24
repetitions, config.cpp:230).

* `value` = agent tokens/s = output tokens of invoked, unpruned agents /
  device-event time (first tick -> last completion), summed over the K timed
  requests; L2 flushed (256 MiB write) before every request, outside its events.
* `e2e` = the same requests timed on the host wall clock around the C-ABI call
  (`moa_run_query` with host buffers: prompt synthesis, row uploads, the
  results copied back to host memory).
* `roofline` = the dominant decode kernel (CUDA events around every launch on
  the launching stream, graphs bypassed, one or two extra requests), its
  algorithmic bytes per launch / average launch time against the measured
  HBM peak; `roofline_prefill` the same for the dominant prefill kernel
  against the bf16 tensor peak.
* N > 1: without torchrun in the environment the script re-launches itself
  under `torch.distributed.run` with N ranks (NCCL_DEBUG=INFO).  Default
  placement for N > 1 is `tree` (one request partitioned along the tree,
  DESIGN.md §9, scaling "strong"); `--placement replicas` serves independent
  requests per rank (scaling "weak").  Device time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-baseline-s", type=float, default=12.0, help="CPU sample budget (seconds of timed work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--placement", default=None, choices=["replicas", "tree"],
                    help="N>1: one request tree-partitioned over the ranks (default) or independent replicas")
    ap.add_argument("--probe-steps", type=int, default=2, help="requests replayed with per-kernel probes")
    ap.add_argument("--profile-only", action="store_true", help="run steps without JSON (for ncu)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary configs (C1 with early exit, C2 at 512 tokens) reported beside the headline")
    ap.add_argument("--no-timeline", action="store_true",
                    help="skip the in-graph tick timeline (chain stamps) of one extra request")
    ap.add_argument("--concurrency", default="4,8",
                    help="continuous-batching sweep on C1 reported beside the headline (comma list; '' to skip)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU: exercise the N-rank launcher and the cross-rank reductions (gloo), no GPU work")
    return ap.parse_args(argv)


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`bench.py --gpus N` outside torchrun: one rank per GPU under
    torch.distributed.run (same flags), NCCL_DEBUG=INFO so the communicator
    size is visible in the log."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


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
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


PREFILL_KINDS = ("attn_prefill", "pf_qkv", "pf_o_proj", "pf_gate_up", "pf_down")


def kernel_table(probes, hbm, tf, n_req):
    out = {}
    for k, v in probes.items():
        if not v["launches"]:
            continue
        s = v["ms"] / 1e3
        out[k] = {"launches": v["launches"], "ms_per_request": v["ms"] / n_req, "avg_us": 1e6 * s / v["launches"],
                  "gbs": v["bytes"] / s / 1e9, "frac_hbm": v["bytes"] / s / 1e9 / hbm,
                  "tflops": v["flops"] / s / 1e12, "frac_tensor": v["flops"] / s / 1e12 / tf}
    return out


def roofline(probes, hbm, tf, src, cfg_name, prefill=False):
    """Dominant kernel of the regime (largest share of probed time): its
    algorithmic bytes (decode, HBM-bound) or flops (prefill, tensor-bound) per
    launch / average launch duration.  `traffic` = DRAM bytes per launch of
    that kernel from the committed ncu --set full capture
    (profiles/ncu_traffic.json), else null."""
    pool = {k: v for k, v in probes.items() if (k in PREFILL_KINDS) == prefill and v["launches"]}
    if not pool:
        return None
    kind, v = max(pool.items(), key=lambda kv: kv[1]["ms"])
    s = v["ms"] / 1e3
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(cfg_name, {}).get(kind)
    share = v["ms"] / max(1e-12, sum(p["ms"] for p in probes.values()))
    common = {"kernel": kind, "peak_source": src, "avg_us": 1e6 * s / v["launches"], "launches": v["launches"],
              "share_of_probed_time": share, "traffic": traffic}
    if prefill:
        a = v["flops"] / s / 1e12
        return {"bound": "tensor", "achieved": a, "peak": tf, "unit": "TFLOP/s", "frac": a / tf,
                "flops_per_launch": v["flops"] / v["launches"], **common}
    a = v["bytes"] / s / 1e9
    return {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm,
            "bytes_per_launch": v["bytes"] / v["launches"], **common}


def in_graph_roofline(gu, cfg, hbm):
    """The dominant decode kernel inside the graphs, with PDL overlap: per-CTA
    %globaltimer stamps of one request, the gate/up launches of its last phase
    (the root decoding alone, one row): each launch's incremental time (its
    last CTA's end minus the previous launch's end) against its algorithmic
    bytes."""
    from paper_2512_18126_b200.configs import agent_tag
    if not gu:
        return None
    depth = len(cfg["topology"]["widths"])
    shape = cfg["models"][agent_tag(cfg, depth, 0)]["shape"]
    D, F = {"tiny": (256, 1024), "1b": (2048, 8192), "8b": (4096, 14336)}[shape]
    us = statistics.median(gu)
    byts = 2.0 * (2 * F) * D + 4.0 * D + 2.0 * F  # weights + one row in / out
    a = byts / (us * 1e-6) / 1e9
    return {"bound": "hbm", "kernel": "gate_up", "rows": 1, "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm,
            "bytes_per_launch": byts, "incremental_us": us, "launches": len(gu),
            "source": "per-CTA %globaltimer stamps of one request's root-decode ticks (graphs and PDL as in the "
                      "timed region): launch end minus the previous launch's end"}


def probe_requests(eng, qc, samples):
    """Replay requests with CUDA events around every forward kernel."""
    eng.probe(True)
    launches_ee = 0
    for s in samples:
        r = eng.run_query(qc, sample=s, resolve=False, detail=True)
        launches_ee += sum(4 + (e["outputs"] > 1) for e in r["metricq"] if e["evaluated"])
    probes = eng.probe_stats()
    eng.probe(False)
    return probes, launches_ee


def secondary(name, out_len, hbm, tf, src, local, requests=2, probe=True):
    """A smaller BASELINE config measured the headline's way (device events,
    L2 flushed), reported beside the headline."""
    import torch
    from paper_2512_18126_b200 import capi
    from paper_2512_18126_b200.configs import CONFIGS
    cfg = dict(CONFIGS[name])
    if out_len:
        cfg["out_len"] = [out_len] * len(cfg["out_len"])
    eng, qc = capi.engine_for(cfg, device=local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    eng.run_query(qc, sample=0, resolve=False, detail=False)  # warm-up (graph capture)
    ms, toks, fwd, wb = [], 0, 0, 0.0
    for i in range(requests):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        r = eng.run_query(qc, sample=1 + i, resolve=False, detail=False)
        ms.append(r["e2e_ms"])
        toks += r["tokens"]
        fwd += r["forwards"]
        wb += r["weight_bytes"]
    out = {"config": {"workload": cfg["workload"], "name": name,
                      "models": {t: m["shape"] for t, m in cfg["models"].items()}},
           "value": toks / (sum(ms) / 1e3), "unit": UNIT, "p50_ms_per_request": statistics.median(ms),
           "requests": requests, "ms_per_forward": sum(ms) / max(1, fwd),
           "weight_stream_gbs": wb / 1e9 / (sum(ms) / 1e3), "weight_stream_frac": wb / 1e9 / (sum(ms) / 1e3) / hbm}
    if probe:
        probes, _ = probe_requests(eng, qc, [1])
        out["kernels"] = kernel_table(probes, hbm, tf, 1)
        out["roofline"] = roofline(probes, hbm, tf, src, name)
    eng.close()
    return out


def concurrency_sweep(name, levels, local):
    """Continuous batching: B independent requests of the same config served
    concurrently by one engine (moa_run_batch).  Throughput = all requests'
    agent tokens / the batch's device time; latency = each request's own
    first-tick -> last-completion time."""
    import torch
    from paper_2512_18126_b200 import capi
    from paper_2512_18126_b200.configs import CONFIGS
    cfg = CONFIGS[name]
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
        out.append({"config": name, "concurrent_requests": b, "value": sum(r["tokens"] for r in rs) / (batch_ms / 1e3),
                    "unit": UNIT, "batch_ms": batch_ms, "p50_ms_per_request": lat[len(lat) // 2]})
    return out


# ---------------------------------------------------------------------------
# CPU side: the oracle port (oracle/ -- test infrastructure; only this arm and
# cpu_baseline execute it).

def _small_configs():
    return {"C0", "C1", "C1U", "C1H", "C4-tree", "C4-dense"}


class CpuSlice:
    """Bounded CPU sample of a 1B/8B workload: the first leaf agent whose
    model the host can hold in fp32 (the 8B shape needs 29 GB, so 1B) gets
    its real leaf prompt prefilled once (untimed setup, reported), then each
    sample decodes greedy tokens at that context through the oracle's numpy
    transformer on all host threads.  Agent tokens/s of the slice."""

    def __init__(self, cfg):
        import numpy as np  # noqa: F401
        from oracle.model import CpuModel, make_spec
        from oracle.rng import hash_combine, synth_tokens
        from paper_2512_18126_b200.configs import agent_tag
        t = cfg["topology"]
        pos = next(p for p in range(t["widths"][0])
                   if cfg["models"][agent_tag(cfg, 1, p)]["shape"] != "8b")
        tag = agent_tag(cfg, 1, pos)
        m = cfg["models"][tag]
        ss = hash_combine(cfg["seed"], 0)
        prompt = synth_tokens(ss, f"leaf_prefix:1:{pos}", cfg["leaf_prefix_tokens"]) + \
            synth_tokens(ss, "query", cfg["query_tokens"])
        t0 = time.perf_counter()
        self.model = CpuModel(make_spec(tag, m["shape"], seed=m.get("seed", 0)), len(prompt) + 1024)
        self.init_s = time.perf_counter() - t0
        self.kv = self.model.new_kv()
        t0 = time.perf_counter()
        lg = self.model.forward([(self.kv, i, int(x)) for i, x in enumerate(prompt)], [False] * (len(prompt) - 1) + [True])
        self.prefill_s = time.perf_counter() - t0
        self.pos, self.tok = len(prompt), int(lg[0].argmax())
        self.desc = (f"agent 1:{pos} ({m['shape']}) of {cfg['name']}: greedy decode at its {len(prompt)}-token "
                     f"leaf-prompt context (prompt prefilled once, untimed: {self.prefill_s:.1f} s = "
                     f"{len(prompt) / self.prefill_s:.0f} prompt tokens/s)")

    def decode(self, n):
        t0 = time.perf_counter()
        for _ in range(n):
            lg = self.model.forward([(self.kv, self.pos, self.tok)], [True])
            self.pos, self.tok = self.pos + 1, int(lg[0].argmax())
        return time.perf_counter() - t0


def cpu_baseline(cfg, budget_s):
    """The oracle on a bounded sample of the same workload, all host cores."""
    cores = os.cpu_count()
    if cfg["name"] in _small_configs():
        from oracle.configs import models_of, run_config
        from oracle.orchestrator import run_query
        rc, ms = run_config(cfg), models_of(cfg, 1024)
        t0, toks, n = time.perf_counter(), 0, 0
        while True:
            toks += run_query(rc, ms, n % 24)["tokens"]
            n += 1
            if time.perf_counter() - t0 > budget_s or n >= 24:
                break
        dt = time.perf_counter() - t0
        return {"value": toks / dt, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"{n} {cfg['name']} requests (samples 0..{n - 1}), oracle/orchestrator.py + numpy fp32 "
                          f"transformer, {cores} host threads", "seconds": dt, "tokens": toks}
    sl = CpuSlice(cfg)
    dt, toks = 0.0, 0
    while dt < budget_s and toks < 512:
        dt += sl.decode(4)
        toks += 4
    return {"value": toks / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{toks} tokens of {sl.desc}; oracle/model.py numpy fp32, {cores} host threads",
            "seconds": dt, "tokens": toks, "setup_s": sl.init_s + sl.prefill_s}


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
    ol = cfg["out_len"][0]
    req = {"cmd": "time_run_query", "topology": t, "reps": reps,
           "profiles": {tag: {"output_len": ol if isinstance(ol, int) else 64} for tag in cfg["models"]},
           "assign": cfg["assign"], "mode": cfg["mode"], "early_exit": cfg["early_exit"],
           "chunk_size": cfg["chunk_size"], "seed": cfg["seed"]}
    r = json.loads(L.moaref_call(json.dumps(req).encode()))
    if "seconds" not in r:
        return None
    return {"seconds_per_request": r["seconds"] / reps, "reps": reps, "cores": 1,
            "note": "reference SimWorld (virtual-time, no model compute), orchestrator.cpp:297-302"}


def run_reference_arm(args, cfg, rank, world):
    """The reference path's CPU implementation on the host cores: the oracle
    port (the reference itself has no model compute).  Small
    configs: whole requests; 1B/8B configs: the bounded decode slice per step."""
    if rank != 0:
        return
    tree = world > 1 and (args.placement or "tree") == "tree"
    steps, toks = [], 0
    cores = os.cpu_count()
    if cfg["name"] in _small_configs():
        from oracle.configs import models_of, run_config
        from oracle.orchestrator import run_query
        rc, ms = run_config(cfg), models_of(cfg, 1024)
        for i in range(args.warmup):
            run_query(rc, ms, i % 24)
        for i in range(args.steps):
            t0 = time.perf_counter()
            toks += run_query(rc, ms, i % 24)["tokens"]
            steps.append(time.perf_counter() - t0)
        sample = (f"{args.steps} {cfg['name']} requests through oracle/ (numpy fp32 transformer agents + "
                  f"reference-semantics orchestration)")
        per_step = None
    else:
        sl = CpuSlice(cfg)
        per_step = 8
        for _ in range(args.warmup):
            sl.decode(per_step)
        for _ in range(args.steps):
            steps.append(sl.decode(per_step))
            toks += per_step
        sample = f"per step {per_step} tokens of {sl.desc}; oracle/model.py numpy fp32, {cores} host threads"
    dt = sum(steps)
    value = toks / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "p50_ms_per_request": 1e3 * statistics.median(steps), "higher_is_better": True,
            "scaling": "strong" if tree else "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "name": cfg["name"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if per_step:
        line["tokens_per_step"] = per_step
    sim = reference_simulator_time(cfg)
    if sim:
        line["reference_simulator"] = sim
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def reduce_over_ranks(pg, device, dev_ms, e2e_ms, toks, e2e_toks, tree):
    """Max of the times, sum of the tokens over ranks (tree placement: one
    request shared by all ranks, its tokens counted once)."""
    if pg is None:
        return dev_ms, e2e_ms, toks, e2e_toks
    import torch
    t = torch.tensor([dev_ms, e2e_ms, toks, e2e_toks], dtype=torch.float64, device=device)
    mx, sm = t.clone(), t.clone()
    pg.all_reduce(mx, op=pg.ReduceOp.MAX)
    pg.all_reduce(sm, op=pg.ReduceOp.SUM)
    if tree:
        return mx[0].item(), mx[1].item(), toks, e2e_toks
    return mx[0].item(), mx[1].item(), sm[2].item(), sm[3].item()


def dry_run(args, rank, world):
    """CPU check of the multi-rank plumbing (gloo): barrier, id broadcast,
    max/sum reductions and the rank-0 line."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid.copy_(torch.arange(128, dtype=torch.uint8))
    dist.broadcast(uid, 0)
    assert int(uid[5]) == 5
    dist.barrier()
    tree = world > 1 and (args.placement or "tree") == "tree"
    dev_ms, e2e_ms, toks, e2e_toks = reduce_over_ranks(dist, "cpu", 100.0 + rank, 110.0 + rank, 1000, 1000, tree)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": toks / (dev_ms / 1e3), "unit": UNIT, "n_gpus": world,
                          "dry_run": True, "scaling": "strong" if tree else "weak", "dev_ms_max": dev_ms,
                          "e2e_ms_max": e2e_ms, "tokens": toks}), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.dry_run:
        dry_run(args, rank, world)
        return
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

    tree = world > 1 and (args.placement or "tree") == "tree"
    eng, qc = capi.engine_for(cfg, device=local)
    if tree:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(capi.nccl_unique_id()), dtype=torch.uint8))
        pg.broadcast(uid, 0)
        eng.attach_comm(bytes(uid.cpu().numpy()), rank, world)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def sample_of(i):  # tree mode: every rank serves the same request
        return (i if tree else rank * 1000 + i) % 24

    def one(i, resolve):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = eng.run_query(qc, sample=sample_of(i), resolve=resolve, detail=resolve)
        return r, time.perf_counter() - t0

    for i in range(args.warmup):
        one(i, False)
    if args.profile_only:
        for i in range(args.steps):
            one(i, False)
        return
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    # Timed requests.  Each is one C-ABI call with host buffers (resolve: the
    # outputs and prompts are copied back), so the same K requests give both
    # numbers: value from the device events inside the request (first tick ->
    # last completion), e2e from the host wall clock around the call.
    dev_ms, toks, per_req, rows, fwd, wbytes, host_ms, wait_ms = 0.0, 0, [], 0, 0, 0.0, 0.0, 0.0
    e2e_s, h2d, d2h = 0.0, 0, 0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            r, wall = one(i, True)
            e2e_s += wall
            dev_ms += r["e2e_ms"]
            per_req.append(r["e2e_ms"])
            toks += r["tokens"]
            rows += r["rows"]
            fwd += r["forwards"]
            wbytes += r["weight_bytes"]
            host_ms += r["host_ms"]
            wait_ms += r["host_wait_ms"]
            h2d += r["rows"] * 16  # row descriptors uploaded per tick (moa RowDesc, 16 B)
            d2h += sum(4 * len(a["prompt"]) + 12 * len(a["output"]) for a in r["agents"].values())
    torch.cuda.synchronize()
    # kernel probes: CUDA events around every forward kernel while a few of
    # the same requests replay (graphs bypassed during this pass only)
    npr = max(1, min(args.probe_steps, args.steps))
    probes, n_ee_launches = probe_requests(eng, qc, [sample_of(i) for i in range(npr)])
    timeline, gu_inc = None, []
    if rank == 0 and not args.no_timeline:
        from paper_2512_18126_b200 import chain
        try:
            recs, e2e_st = chain.collect(eng, qc, sample_of(0))
            timeline = chain.timeline(chain.ticks(recs))
            from paper_2512_18126_b200.configs import agent_tag
            root_shape = cfg["models"][agent_tag(cfg, len(cfg["topology"]["widths"]), 0)]["shape"]
            d_root = {"tiny": 256, "1b": 2048, "8b": 4096}[root_shape]
            gu_inc = chain.launch_increments(recs, f"gemv_tc(swiglu,K={d_root})")
        except Exception as e:  # diagnostics only
            timeline = {"error": str(e)}
    dev_ms_max, e2e_ms_max, toks_all, e2e_toks_all = reduce_over_ranks(pg, "cuda", dev_ms, e2e_s * 1e3, toks, toks,
                                                                       tree)
    if rank != 0:
        eng.close()
        if pg:
            pg.destroy_process_group()
        return
    hbm, tf, src = peaks()
    value = toks_all / (dev_ms_max / 1e3)
    launches_per_req = sum(v["launches"] for v in probes.values()) / npr + n_ee_launches / npr
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
        "p50_ms_per_request": statistics.median(per_req), "higher_is_better": True,
        "scaling": "strong" if tree else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": cfg["workload"], "name": cfg["name"], "l2": "flushed (256 MiB write) before every request",
                   "models": {t: m["shape"] for t, m in cfg["models"].items()},
                   "parallelism": f"tree{world}" if tree else f"replicas{world}"},
        "e2e": {"value": e2e_toks_all / (e2e_ms_max / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": int(round(launches_per_req * args.steps)),
        "roofline": roofline(probes, hbm, tf, src, cfg["name"]),
        "roofline_prefill": roofline(probes, hbm, tf, src, cfg["name"], prefill=True),
        "kernels": kernel_table(probes, hbm, tf, npr),
        "clocks": clk.summary(),
        "peaks": {"hbm_gbs": hbm, "bf16_tflops": tf, "source": src},
        "engine": {"rows_per_request": rows / args.steps, "forwards_per_request": fwd / args.steps,
                   "host_ms_per_request": host_ms / args.steps, "host_wait_ms_per_request": wait_ms / args.steps,
                   "weight_gb_per_request": wbytes / args.steps / 1e9,
                   "weight_stream_gbs": wbytes / (dev_ms / 1e3) / 1e9,
                   "weight_stream_frac": wbytes / (dev_ms / 1e3) / 1e9 / hbm},
        "probe_note": (f"kernels/roofline: {npr} request(s) replayed with CUDA events around every launch (graphs "
                       "bypassed, so no programmatic-dependent-launch overlap); weight_stream_frac: weight bytes of "
                       "every forward / device time"),
    }
    if timeline:
        line["tick_timeline"] = timeline
    rig = in_graph_roofline(gu_inc, cfg, hbm)
    if rig:
        line["roofline_in_graph"] = rig
    eng.close()  # the headline engine; the extra measurements build their own
    if not args.no_secondary and world == 1:
        sec = []
        if cfg["name"] != "C1":
            sec.append(secondary("C1", None, hbm, tf, src, local, requests=8, probe=False))
        if cfg["name"] != "C2":
            sec.append(secondary("C2", 512, hbm, tf, src, local, requests=2))
        line["secondary"] = sec
        levels = [int(x) for x in args.concurrency.split(",") if x.strip()]
        if levels:
            line["concurrency"] = concurrency_sweep("C1", levels, local)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_baseline_s)
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
