"""Tree-partitioned engine on ONE GPU: two or three engines in
one process, one thread each, joined by the in-process loopback hub -- the
same per-tick message sequence the engine issues to NCCL across GPUs.  With
the batch-invariant GEMV path (gemv_only) every agent's tokens and logprobs do
not depend on which rows share its forward, so each rank must reproduce the
single-engine run bit for bit: outputs, schedule and MetricQ decisions."""
import threading

import pytest

from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import C0, C1U

pytestmark = pytest.mark.gpu


def _single(cfg, sample, gemv_only=True):
    eng, qc = capi.engine_for(cfg, gemv_only=gemv_only)
    try:
        return eng.run_query(qc, sample=sample)
    finally:
        eng.close()


def _partitioned(cfg, sample, world, gemv_only=True):
    hub = capi.LoopbackHub(world)
    engs = []
    for r in range(world):
        eng, qc = capi.engine_for(cfg, gemv_only=gemv_only)
        eng.attach_loopback(hub, r)
        engs.append(eng)
    out, err = [None] * world, []

    def run(r):
        try:
            out[r] = engs[r].run_query(qc, sample=sample)
        except Exception as e:  # surfaced below
            err.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "partitioned run hung"
    for e in engs:
        e.close()
    if err:
        raise err[0]
    return out


TREE9 = dict(kind="tree", widths=[9, 3, 1], branching=[3, 3])


def _holds(cfg, owner, rank, k):
    """Whether `rank` holds agent k's outputs after a partitioned run: its own
    agents, and the chunks it receives -- every agent's with an early-exit
    gate (all ranks evaluate it), else those of its agents' precursors, and
    everything on rank 0 (which resolves the request)."""
    from oracle.configs import topology_of
    from oracle.topology import aid
    topo = topology_of(cfg["topology"])
    if owner[k] == rank or rank == 0 or (cfg["early_exit"] and topo.depth > 1):
        return True
    return any(owner[aid(c)] == rank for c in topo.agents() if k in [aid(p) for p in topo.precursors(c)])


def _holds_prompt(cfg, owner, rank, k):
    """A dependent agent's literal prompt resolves on `rank` when every
    precursor's chunks reached it."""
    from oracle.configs import topology_of
    from oracle.topology import aid, parse_aid
    topo = topology_of(cfg["topology"])
    return all(_holds(cfg, owner, rank, aid(p)) for p in topo.precursors(parse_aid(k)))


@pytest.mark.parametrize("name,cfg,sample,world", [
    ("C0", dict(C0), 0, 2),
    ("C1U", dict(C1U), 3, 2),
    ("C1U-w3", dict(C1U), 0, 3),
    ("T931-ee", dict(C1U, topology=TREE9, out_len=[[16, 64], 32, 32]), 1, 2),
])
def test_partitioned_engine_matches_single(name, cfg, sample, world):
    single = _single(cfg, sample)
    owner = capi.placement(cfg["topology"], world)
    assert len(set(owner.values())) == world
    for rank, o in enumerate(_partitioned(cfg, sample, world)):
        assert o["tokens"] == single["tokens"], (name, rank)
        assert [(m["completed"], m["evaluated"], m["q"], m["exited"], m["pruned"]) for m in o["metricq"]] == \
               [(m["completed"], m["evaluated"], m["q"], m["exited"], m["pruned"]) for m in single["metricq"]]
        for k, a in single["agents"].items():
            b = o["agents"][k]
            for f in ("complete", "decode_start", "pruned", "output_tokens", "prefill_only_calls",
                      "recomputed_tokens"):
                assert b[f] == a[f], (name, rank, k, f)
            if _holds_prompt(cfg, owner, rank, k):
                assert b["prompt"] == a["prompt"], (name, rank, k)
            if not _holds(cfg, owner, rank, k):
                continue
            n = len(a["output"])
            if a["pruned"] and owner[k] != rank:
                # a remote agent cut mid-chunk is known up to its last hand-off
                n = (n // cfg["chunk_size"]) * cfg["chunk_size"]
            assert b["output"][:n] == a["output"][:n], (name, rank, k)
            assert b["logprobs"][:n] == a["logprobs"][:n], (name, rank, k)


@pytest.mark.parametrize("name,cfg,sample,world", [
    ("C0", dict(C0), 0, 2),
    ("C1U", dict(C1U), 3, 2),
    ("C1U-w3", dict(C1U), 1, 3),
])
def test_partitioned_engine_tensor_core_path(name, cfg, sample, world):
    """The default (tensor-core) decode and prefill path under partitioning.
    Which rows share a forward differs between the ranks and the single
    engine, so bit-equality with the single run is not the contract; instead
    every rank must hold exactly the owners' tokens (the hand-off is lossless:
    the ranks agree bit for bit), every agent must pass the teacher-forced
    oracle check, and without early exit the schedule equals the single run's."""
    from oracle.model import CpuModel, make_spec
    from oracle.parity import check_agent
    outs = _partitioned(cfg, sample, world, gemv_only=False)
    single = _single(cfg, sample, gemv_only=False)
    owner = capi.placement(cfg["topology"], world)
    ref = outs[0]  # rank 0 receives every agent's chunks
    for rank, o in enumerate(outs):
        assert [(m["completed"], m["evaluated"], m["q"], m["exited"], m["pruned"]) for m in o["metricq"]] == \
               [(m["completed"], m["evaluated"], m["q"], m["exited"], m["pruned"]) for m in ref["metricq"]]
        for k, a in ref["agents"].items():
            b = o["agents"][k]
            if _holds_prompt(cfg, owner, rank, k):
                assert b["prompt"] == a["prompt"], (name, rank, k)
            if not _holds(cfg, owner, rank, k):
                continue
            n = len(a["output"])
            if a["pruned"] and owner[k] != rank:
                n = (n // cfg["chunk_size"]) * cfg["chunk_size"]
            assert b["output"][:n] == a["output"][:n], (name, rank, k)
    if not cfg["early_exit"]:
        for k, a in single["agents"].items():
            for f in ("complete", "decode_start", "output_tokens", "prefill_only_calls", "recomputed_tokens"):
                assert ref["agents"][k][f] == a[f], (name, k, f)
    models = {}
    for k, a in ref["agents"].items():
        if not a["output"] or a["pruned"]:
            continue
        layer, pos = (int(x) for x in k.split(":"))
        cyc = cfg["assign"][min(layer - 1, len(cfg["assign"]) - 1)]
        tag = cyc[pos % len(cyc)]
        mm = cfg["models"][tag]
        if tag not in models:
            models[tag] = CpuModel(make_spec(tag, mm["shape"], seed=mm["seed"]), 1024)
        chk = check_agent(models[tag], a["prompt"], a["output"], a["logprobs"])
        assert chk["mismatches"] == [] and chk["lp_ok"], (name, k, chk)
