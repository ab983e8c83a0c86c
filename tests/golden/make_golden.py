"""Regenerate tests/golden/*.json from the reference implementation itself.

    make -C oracle/ref && python tests/golden/make_golden.py

Runs in the dev container only (needs /root/reference, via oracle/_ref/
libmoaref.so built from the reference's own proj/core sources).  The fixtures
it writes are small and committed; the GPU box never reads the reference.
"""
from __future__ import annotations

import ctypes
import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from oracle.rng import synth_tokens  # noqa: E402

_L = ctypes.CDLL(str(ROOT / "oracle" / "_ref" / "libmoaref.so"))
_L.moaref_call.restype = ctypes.c_char_p


def ref(req: dict) -> dict:
    return json.loads(_L.moaref_call(json.dumps(req).encode()))


def dump(name, obj):
    (OUT / name).write_text(json.dumps(obj, separators=(",", ":")) + "\n")
    print("wrote", name)


def gen_rng():
    cases = []
    for seed in (0, 5, 2**63 + 11, 123456789):
        for label in ("query", "leaf_prefix:1:0", "ee:0", "outlen:2:1", ""):
            r = ref({"cmd": "rng", "seed": seed, "label": label, "n": 6})
            cases.append(dict(seed=seed, label=label, **r))
    dump("rng.json", cases)


TOPOS = [
    dict(kind="tree", widths=[4, 2, 1], branching=[2, 2]),
    dict(kind="tree", widths=[9, 3, 1], branching=[3, 3]),
    dict(kind="tree", widths=[8, 2, 1], branching=[4, 2]),
    dict(kind="tree", widths=[5, 2, 1], cluster_sizes=[[3, 2], [2]]),
    dict(kind="tree", widths=[1]),
    dict(kind="all_to_all", widths=[6, 6, 1]),
    dict(kind="all_to_all", widths=[3, 2]),
]
BAD_TOPOS = [
    dict(kind="tree", widths=[4, 3, 1], branching=[2, 3]),
    dict(kind="tree", widths=[4, 2], cluster_sizes=[[3, 2]]),
    dict(kind="tree", widths=[0, 1], branching=[1]),
    dict(kind="tree", widths=[4, 2, 1], branching=[2]),
]


def gen_topology():
    cases = []
    for t in TOPOS:
        if t["widths"] == [1]:
            t = dict(t, branching=[])
        cases.append(dict(spec=t, out=ref({"cmd": "topology", **t})))
    for t in BAD_TOPOS:
        cases.append(dict(spec=t, out=ref({"cmd": "topology", **t})))
    dump("topology.json", cases)


def random_plan_case(rng: random.Random, k: int):
    """One randomized slot-plan interleaving (the shape of test_router.cpp's
    300 random interleavings with prunes)."""
    n_slots = rng.randint(0, 4)
    prods = [f"1:{i}" for i in range(n_slots)]
    slots = [dict(precursor=p, separator=[9000 + 10 * i + j for j in range(rng.randint(0, 2))])
             for i, p in enumerate(prods)]
    prefix = list(range(100, 100 + rng.randint(0, 5)))
    suffix = list(range(200, 200 + rng.randint(0, 3)))
    incremental = rng.random() < 0.8
    remaining = {p: rng.randint(0, 5) for p in prods}
    emitted = {p: 0 for p in prods}
    alive = set(prods)
    events = [] if rng.random() < 0.2 else [dict(op="start")]
    started = bool(events)
    order_done = []
    for _ in range(60):
        live = [p for p in prods if p in alive and p not in order_done]
        if not live:
            break
        p = rng.choice(live)
        x = rng.random()
        if x < 0.55 and remaining[p] > 0:
            n = rng.randint(1, 3)
            toks = [int(p.split(":")[1]) * 1000 + emitted[p] + j for j in range(n)]
            emitted[p] += n
            remaining[p] -= 1
            events.append(dict(op="chunk", producer=p, tokens=toks))
        elif x < 0.85:
            events.append(dict(op="done", producer=p))
            order_done.append(p)
        else:
            events.append(dict(op="cancelled", producer=p))
            alive.discard(p)
        if not started and rng.random() < 0.3:
            events.append(dict(op="start"))
            started = True
    if not started:
        events.append(dict(op="start"))
    return dict(self="2:0", prefix=prefix, slots=slots, suffix=suffix, incremental=incremental, events=events)


def gen_slotplan():
    cases = []
    # the fixed shapes of test_router.cpp:67-263
    base = dict(self="2:0", prefix=[1, 2, 3], slots=[dict(precursor="1:0", separator=[7]),
                                                     dict(precursor="1:1", separator=[8])], suffix=[9, 9])
    fixed = [
        dict(base, incremental=True, events=[dict(op="start"), dict(op="chunk", producer="1:0", tokens=[10, 11]),
                                             dict(op="chunk", producer="1:1", tokens=[20]),
                                             dict(op="done", producer="1:0"), dict(op="done", producer="1:1")]),
        dict(base, incremental=False, events=[dict(op="start"), dict(op="chunk", producer="1:0", tokens=[10]),
                                              dict(op="done", producer="1:0"),
                                              dict(op="chunk", producer="1:1", tokens=[20, 21]),
                                              dict(op="done", producer="1:1")]),
        dict(base, incremental=True, events=[dict(op="start"), dict(op="chunk", producer="1:0", tokens=[10, 11]),
                                             dict(op="cancelled", producer="1:0"),
                                             dict(op="chunk", producer="1:1", tokens=[20]),
                                             dict(op="done", producer="1:1")]),
        dict(base, incremental=True, events=[dict(op="start"), dict(op="done", producer="1:0"),
                                             dict(op="cancelled", producer="1:0")]),
        dict(base, incremental=True, events=[dict(op="start"), dict(op="done", producer="1:0"),
                                             dict(op="done", producer="1:1"),
                                             dict(op="chunk", producer="1:1", tokens=[5])]),
    ]
    rng = random.Random(2512)
    rand = [random_plan_case(rng, k) for k in range(300)]
    for c in fixed + rand:
        cases.append(dict(case=c, out=ref({"cmd": "slotplan", **c})))
    dump("slotplan.json", cases)


def gen_mock_embed():
    cases = []
    for tokens, hidden, seed in (([1, 2, 3, 49999], 8, 0), ([7, 7, 7], 3, 42), ([0], 1, 9),
                                 (synth_tokens(3, "o", 64), 64, 0)):
        cases.append(dict(tokens=tokens, hidden=hidden, seed=seed,
                          embedding=ref({"cmd": "mock_embed", "tokens": tokens, "hidden": hidden,
                                         "seed": seed})["embedding"]))
    dump("mock_embed.json", cases)


def gen_metricq():
    cases = []
    rng = random.Random(7)
    for k in range(12):
        m = rng.randint(1, 4)
        n = rng.choice([1, 5, 32, 64])
        hidden = rng.choice([4, 16, 64])
        outs = [[rng.randrange(50000) for _ in range(n)] for _ in range(m)]
        lps = [[-abs(rng.gauss(1.0, 0.6)) for _ in range(n)] for _ in range(m)]
        req = dict(cmd="metricq", outputs=outs, logprobs=lps, hidden=hidden, seed=k, tau=0.7,
                   include_diagonal=(k % 3 != 0), rng_master=1000 + k, rng_label=f"ee:{k % 3}")
        cases.append(dict(req=req, out=ref(req)))
    # the worked pair of test_metricq.cpp:18-26 / :143-155 (explicit embeddings)
    req = dict(cmd="metricq", outputs=[[1, 2], [3, 4]], logprobs=[[-0.1, -0.3], [-0.1, -0.3]], hidden=2,
               embeddings=[[[1.0, 1.0], [1.0, -1.0]], [[1.0, 0.75], [0.0, 0.4375 ** 0.5]]])
    cases.append(dict(req=req, out=ref(req)))
    dump("metricq.json", cases)


SUMMARY_CASES = [
    dict(topology=dict(kind="tree", widths=[4, 2, 1], branching=[2, 2]), assign=[["leaf"], ["agg"], ["agg"]],
         profiles={"leaf": {"output_len": 64}, "agg": {"output_len": 64}}, early_exit=False, reps=6),
    dict(topology=dict(kind="tree", widths=[4, 2, 1], branching=[2, 2]), assign=[["leaf"], ["agg"], ["agg"]],
         profiles={"leaf": {"output_min": 24, "output_max": 96}, "agg": {"output_len": 64}}, early_exit=True,
         reps=8),
    dict(topology=dict(kind="tree", widths=[9, 3, 1], branching=[3, 3]), assign=[["4b", "8b", "32b"], ["agg"], ["root"]],
         profiles={"4b": {"output_min": 100, "output_max": 400}, "8b": {"output_len": 200},
                   "32b": {"output_len": 300, "prefill_rate": 2000.0}, "agg": {"output_len": 150},
                   "root": {"output_len": 120}},
         early_exit=True, ee_eval_latency=0.25, reps=6),
    dict(topology=dict(kind="tree", widths=[9, 3, 1], branching=[3, 3]), assign=[["leaf"], ["agg"], ["agg"]],
         profiles={"leaf": {"output_len": 64}, "agg": {"output_len": 64}}, early_exit=True, force_q=1.0, reps=3),
    dict(topology=dict(kind="all_to_all", widths=[6, 6, 1]), assign=[["leaf"], ["agg"], ["agg"]],
         profiles={"leaf": {"output_min": 30, "output_max": 90}, "agg": {"output_len": 64}}, early_exit=True,
         mode="sequential-pd", reps=5),
    dict(topology=dict(kind="tree", widths=[8, 2, 1], branching=[4, 2]), assign=[["leaf"], ["agg"], ["agg"]],
         profiles={"leaf": {"output_len": 512}, "agg": {"output_len": 512}}, early_exit=False, mode="dp-chunked-prefill",
         reps=4),
]


def gen_summary():
    """RunSummary of the reference's own run_repetitions (orchestrator.cpp:297-382)
    with the per-trace fields summarize reads."""
    cases = []
    for c in SUMMARY_CASES:
        req = {"cmd": "summarize", "chunk_size": 32, "seed": 7, **c}
        cases.append(dict(spec=c, out=ref(req)))
    dump("summary.json", cases)


def gen_outlen():
    """OutputLenDist::sample for every kind (agent.hpp:40-103), as run_query
    draws it (RngStream::derive(sample seed, "outlen:<agent>"))."""
    dists = [dict(kind="fixed", n=64), dict(kind="uniform", lo=24, hi=96), dict(kind="uniform", lo=7, hi=7),
             dict(kind="empirical", values=[16, 40, 24]), dict(kind="empirical", values=[5]),
             dict(kind="empirical", values=[1, 2, 3, 5, 8, 13, 21, 34])]
    cases = []
    for d in dists:
        for seed in (0, 3, 2**63 + 11):
            for agent in ("1:0", "1:3", "2:1"):
                cases.append(dict(dist=d, seed=seed, agent=agent,
                                  n=ref({"cmd": "outlen", "seed": seed, "agent": agent, "dist": d})["n"]))
    dump("outlen.json", cases)


if __name__ == "__main__":
    gen_outlen()
    gen_rng()
    gen_topology()
    gen_slotplan()
    gen_mock_embed()
    gen_metricq()
    gen_summary()
