"""The paper's headline comparisons measured on the GPU engine (SURVEY.md §8f
row 2): the four-setting ablation of run_ablation (orchestrator.cpp:451-521)
and the second-layer schedule study of run_second_layer_study
(orchestrator.cpp:532-578), with device-event latencies instead of the
reference's virtual time.

    python -m paper_2512_18126_b200.ablation [--base C1] [--samples 8] [--json out.json]

Ablation settings on the base tree config (same agents, same prompts):
all-to-all (same widths, sequential P/D, no early exit) -> tree (sequential
P/D) -> tree+overlap (incremental prefill overlap) -> tree+overlap+ee.  Each
row: mean / p50 / p95 e2e and the mean of per-sample ratios to all-to-all
(the reference's normalisation).  Second-layer study: P precursors -> one
aggregator, precursor outputs ~U(out_min, out_max), in each schedule mode.
"""
from __future__ import annotations

import argparse
import copy
import json
import statistics

from . import capi
from .configs import CONFIGS

MODES = ("sequential-pd", "dp-only", "dp-chunked-prefill", "incremental-overlap")


def _pct(xs, p):
    xs = sorted(xs)
    k = (len(xs) - 1) * p
    lo = int(k)
    hi = min(lo + 1, len(xs) - 1)
    return xs[lo] + (xs[hi] - xs[lo]) * (k - lo)  # linear interpolation (orchestrator.cpp:306-314)


def _latencies(cfg, samples, device):
    eng, qc = capi.engine_for(cfg, device=device)
    try:
        eng.run_query(qc, sample=samples[0], resolve=False, detail=False)  # warm-up: graph capture
        out = []
        for s in samples:
            r = eng.run_query(qc, sample=s, resolve=False, detail=False)
            out.append((r["e2e_ms"], r["tokens"]))
        return out
    finally:
        eng.close()


def run_ablation(base: dict, samples: int = 8, device: int = 0) -> list[dict]:
    widths = base["topology"]["widths"]
    settings = [
        ("all-to-all", dict(copy.deepcopy(base), topology=dict(kind="all_to_all", widths=widths),
                            mode="sequential-pd", early_exit=False)),
        ("tree", dict(copy.deepcopy(base), mode="sequential-pd", early_exit=False)),
        ("tree+overlap", dict(copy.deepcopy(base), mode="incremental-overlap", early_exit=False)),
        ("tree+overlap+ee", dict(copy.deepcopy(base), mode="incremental-overlap", early_exit=True)),
    ]
    idx = list(range(samples))
    res = [(name, _latencies(cfg, idx, device)) for name, cfg in settings]
    base_e2e = [e for e, _ in res[0][1]]
    rows = []
    for name, lat in res:
        e2e = [e for e, _ in lat]
        rows.append({"setting": name, "samples": samples, "mean_e2e_ms": statistics.fmean(e2e),
                     "p50_e2e_ms": _pct(e2e, 0.5), "p95_e2e_ms": _pct(e2e, 0.95),
                     "normalized_mean": statistics.fmean(e / b for e, b in zip(e2e, base_e2e)),
                     "mean_tokens": statistics.fmean(t for _, t in lat),
                     "tokens_per_s": sum(t for _, t in lat) / (sum(e2e) / 1e3)})
    return rows


def run_second_layer_study(base: dict, precursors: int = 4, out_min: int = 16, out_max: int = 96,
                           samples: int = 8, device: int = 0) -> list[dict]:
    cfg0 = dict(copy.deepcopy(base), topology=dict(kind="tree", widths=[precursors, 1], branching=[precursors]),
                assign=[base["assign"][0], base["assign"][-1]], out_len=[[out_min, out_max], base["out_len"][-1]],
                early_exit=False)
    rows, seq = [], None
    for mode in MODES:
        lat = _latencies(dict(cfg0, mode=mode), list(range(samples)), device)
        mean = statistics.fmean(e for e, _ in lat)
        seq = mean if seq is None else seq
        rows.append({"mode": mode, "mean_e2e_ms": mean, "normalized_vs_sequential": mean / seq})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", default="C1")
    ap.add_argument("--samples", type=int, default=8)
    ap.add_argument("--json", default=None)
    ap.add_argument("--out", type=int, default=None, help="override output tokens per agent")
    ap.add_argument("--query-tokens", type=int, default=None, help="override the shared query length")
    ap.add_argument("--no-second-layer", action="store_true", help="skip the second-layer schedule study")
    args = ap.parse_args()
    base = dict(CONFIGS[args.base])
    if args.out:
        base["out_len"] = [args.out] * len(base["out_len"])
    if args.query_tokens:
        base["query_tokens"] = args.query_tokens
    out = {"base": args.base, "overrides": {"out": args.out, "query_tokens": args.query_tokens}, "ablation": run_ablation(base, args.samples),
           "second_layer": [] if args.no_second_layer else run_second_layer_study(base, samples=args.samples)}
    for r in out["ablation"]:
        print(f"{r['setting']:18s} mean {r['mean_e2e_ms']:8.2f} ms  p50 {r['p50_e2e_ms']:8.2f}  p95 {r['p95_e2e_ms']:8.2f}"
              f"  normalized {r['normalized_mean']:.3f}  {r['mean_tokens']:.0f} tokens  {r['tokens_per_s']:.0f} tok/s")
    for r in out["second_layer"]:
        print(f"{r['mode']:20s} mean {r['mean_e2e_ms']:8.2f} ms  normalized {r['normalized_vs_sequential']:.3f}")
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
