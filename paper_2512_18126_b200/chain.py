"""Decode-tick timeline from in-kernel %globaltimer stamps (csrc/kernels/stamp.cuh).

With a stamp buffer attached (`moa_k_chain_stamp`), every CTA of the decode
chain's kernels (SIMT GEMV, fused QKV+attention, LM head) records its entry,
the release of its programmatic-dependent-launch wait, intermediate phases
and its end, and publishes them with one atomic when it finishes.  This
module runs one request with stamps on and reduces the records to a per-tick
timeline: for each kernel position of a tick, when its first CTA started,
when its last CTA was released from the PDL wait, and when its last CTA
ended -- the in-graph view the per-kernel CUDA-event probes (which bypass the
graphs) cannot give.  Diagnostics only: not on the product path.
"""
from __future__ import annotations

import collections

import numpy as np

from . import capi

NAMES = {0x11010: "o_proj", 0x12010: "gate_up", 0x11040: "down", 0x13010: "qkv",
         0x20000: "qkv_attn", 0x20001: "qkv_attn+embed", 0x30000: "lm_head"}


def _name(tag):
    if tag in NAMES:
        return NAMES[tag]
    if tag >> 16 == 1:
        return f"gemv(epi={(tag >> 12) & 15},K={16 * (tag & 0xfff)})"
    if tag >> 16 == 5:
        epi = {0: "f32", 1: "residual", 2: "swiglu", 3: "qkv"}.get((tag >> 12) & 15, "?")
        return f"gemv_tc({epi},K={16 * (tag & 0xfff)})"
    if tag == 0x60001:
        return "attn_decode_tma"
    if tag >> 16 == 6:
        return "attention"
    if tag >> 16 == 7:
        return "rmsnorm"
    if tag == 0x80001:
        return "attn_prefill_tc"
    return hex(tag)


def collect(eng, qc, sample=0, cap=1 << 25):
    """Run one request with chain stamps on; returns (records [n, 4] = tag, phase, cta, ns), e2e_ms."""
    import torch
    buf = torch.zeros(2 + 2 * cap, dtype=torch.int64, device="cuda")
    capi.check(capi.lib().moa_k_chain_stamp(buf.data_ptr()))
    try:
        r = eng.run_query(qc, sample=sample, resolve=False, detail=False)
        torch.cuda.synchronize()
    finally:
        capi.lib().moa_k_chain_stamp(0)
    n = min(int(buf[0].item()), cap)
    rec = buf[2:2 + 2 * n].view(-1, 2).cpu().numpy().astype(np.uint64)
    meta, t = rec[:, 0], rec[:, 1].astype(np.int64)
    out = np.stack([(meta >> np.uint64(32)).astype(np.int64), ((meta >> np.uint64(24)) & np.uint64(0xff)).astype(np.int64),
                    (meta & np.uint64(0xffffff)).astype(np.int64), t - t.min()], axis=1)
    return out, r["e2e_ms"]


def ticks(records):
    """Group stamps into kernel launches (per tag, entry stamps split at > 8 us
    gaps) and launches into ticks (each ends with an LM head)."""
    tag, phase, t = records[:, 0], records[:, 1], records[:, 3]
    inst = []
    for tg in np.unique(tag):
        e = np.sort(t[(tag == tg) & (phase == 0)])
        if len(e) == 0:
            continue
        for s in np.split(e, np.where(np.diff(e) > 8000)[0] + 1):
            inst.append(dict(tag=int(tg), t0=int(s.min()), ph=collections.defaultdict(list)))
    inst.sort(key=lambda d: d["t0"])
    by_tag = collections.defaultdict(list)
    for k, d in enumerate(inst):
        by_tag[d["tag"]].append(k)
    for tg, ks in by_tag.items():
        t0s = np.array([inst[k]["t0"] for k in ks])
        m = tag == tg
        for tt, ph in zip(t[m], phase[m]):
            j = np.searchsorted(t0s, tt, side="right") - 1
            if j >= 0:
                inst[ks[j]]["ph"][int(ph)].append(int(tt))
    out, cur = [], []
    for d in inst:
        cur.append(d)
        if d["tag"] == 0x30000:
            out.append(cur)
            cur = []
    return out


def _end(d):
    """Last stamp of a launch (its end stamp when every CTA reached it)."""
    return max(max(v) for v in d["ph"].values() if v)


def timeline(tick_list, first_frac=0.75):
    """Median timeline over the ticks of the request's last phase (single
    agent decoding), in microseconds from the tick's first kernel entry."""
    sel = tick_list[int(len(tick_list) * first_frac):-1]
    if not sel:
        return None
    L = collections.Counter(len(x) for x in sel).most_common(1)[0][0]
    sel = [x for x in sel if len(x) == L]
    if len(sel) < 2:
        return None
    rows = []
    for pos in range(L):
        v = collections.defaultdict(list)
        for tk in sel:
            d, base = tk[pos], tk[0]["t0"]
            v["start"].append(d["t0"] - base)
            v["release"].append(max(d["ph"][1]) - base if d["ph"][1] else np.nan)
            v["end"].append(_end(d) - base)
        med = {k: float(np.nanmedian(x)) / 1e3 for k, x in v.items()}
        rows.append({"kernel": _name(sel[0][pos]["tag"]), "start_us": round(med["start"], 2),
                     "release_us": round(med["release"], 2), "end_us": round(med["end"], 2),
                     "release_to_end_us": round(med["end"] - med["release"], 2)})
    tick_us = float(np.median([_end(tk[-1]) - tk[0]["t0"] for tk in sel])) / 1e3
    gap_us = float(np.median([sel[i + 1][0]["t0"] - _end(sel[i][-1]) for i in range(len(sel) - 1)])) / 1e3
    return {"ticks_analysed": len(sel), "kernels_per_tick": L, "tick_us": round(tick_us, 2),
            "gap_to_next_tick_us": round(gap_us, 2), "kernels": rows}


def request_timeline(eng, qc, sample=0, first_frac=0.75):
    recs, e2e = collect(eng, qc, sample)
    tl = timeline(ticks(recs), first_frac)
    if tl is not None:
        tl["stamped_request_e2e_ms"] = round(e2e, 3)
    return tl


def launch_increments(records, prefix, last_frac=0.25, gap_ns=8000):
    """In-graph time of each launch of the kernels named `prefix...` in the
    last `last_frac` of the request: its last CTA's end minus the previous
    launch's (any kernel's) end -- the launch's share of the serial chain,
    programmatic-dependent-launch overlap included.  Returns microseconds."""
    tag, phase, t = records[:, 0], records[:, 1], records[:, 3]
    inst = []  # (end, is_target)
    for tg in np.unique(tag):
        e = np.sort(t[(tag == tg) & (phase == 0)])
        if len(e) == 0:
            continue
        ends = np.sort(t[(tag == tg) & (phase == 2)])
        starts = [g.min() for g in np.split(e, np.where(np.diff(e) > gap_ns)[0] + 1)] + [np.inf]
        target = _name(int(tg)).startswith(prefix)
        for j in range(len(starts) - 1):
            w = ends[(ends >= starts[j]) & (ends < starts[j + 1])]
            if len(w):
                inst.append((int(w.max()), target))
    inst.sort()
    if len(inst) < 3:
        return []
    t0 = inst[0][0] + (inst[-1][0] - inst[0][0]) * (1.0 - last_frac)
    return [(inst[i][0] - inst[i - 1][0]) / 1e3 for i in range(1, len(inst)) if inst[i][1] and inst[i][0] >= t0]
