"""Tick-engine contract on the CPU oracle: protocol errors (pdsim.cpp), replay
consistency, schedule-mode token invariance and the early-exit gate rules
(orchestrator.cpp:222-276)."""
import pytest

from oracle.configs import models_of, run_config
from oracle.engine import TickEngine
from oracle.model import CpuModel, make_spec
from oracle.orchestrator import run_query
from oracle.topology import RunError, ValidationError
from paper_2512_18126_b200.configs import C0, C1, C1U

_MODELS = {}


def tiny_models(cfg):
    key = tuple(sorted((t, m["seed"]) for t, m in cfg["models"].items()))
    if key not in _MODELS:
        _MODELS[key] = models_of(cfg, 512)
    return _MODELS[key]


def test_protocol_errors():
    eng = TickEngine({"m": CpuModel(make_spec("leaf", "tiny", seed=1), 64)})
    a = (1, 0)
    eng.add_agent(a, "m")
    with pytest.raises(ValidationError):
        eng.add_agent(a, "m")
    eng.submit_prefill_only(a, 0, [1, 2, 3])
    with pytest.raises(RunError):
        eng.submit_prefill_only(a, 5, [4])
    with pytest.raises(RunError):
        eng.submit_generate(a, [9, 2, 3, 4], 4, 2)
    with pytest.raises(ValidationError):
        eng.submit_generate(a, [1, 2, 3, 4], 4, 0)
    with pytest.raises(RunError):
        eng.reclaim(a, 7)
    eng.reclaim(a, 2)
    assert len(eng.reqs[a].prompt) == 2 and list(eng.reqs[a].queue) == [(0, 2, 1)]
    eng.submit_generate(a, [1, 2, 3, 4], 4, 2)
    with pytest.raises(RunError):
        eng.submit_generate(a, [1, 2, 3, 4], 4, 2)
    eng.run()
    with pytest.raises(RunError):
        eng.cancel(a)


def test_replay_reproduces_free_run():
    cfg = C1U
    o = run_query(run_config(cfg), tiny_models(cfg), 2)
    forced = {tuple(int(x) for x in k.split(":")): (a["output"], a["logprobs"], a["entropy"])
              for k, a in o["agents"].items()}
    r = run_query(run_config(cfg), {}, 2, forced=forced)
    for k in o["agents"]:
        for f in ("prompt", "output", "complete", "decode_start", "pruned", "prefill_only_calls"):
            assert r["agents"][k][f] == o["agents"][k][f], (k, f)
    assert [(m["completed"], m.get("q"), m["exited"]) for m in r["metricq"]] == \
           [(m["completed"], m.get("q"), m["exited"]) for m in o["metricq"]]


def test_schedule_modes_decode_identical_tokens():
    """acceptance_main.cpp:682-813: tokens are mode-invariant, zero recompute."""
    outs = {}
    for mode in ("sequential-pd", "dp-only", "dp-chunked-prefill", "incremental-overlap"):
        cfg = dict(C0, mode=mode, out_len=[16, 16, 16], query_tokens=32)
        o = run_query(run_config(cfg), tiny_models(cfg), 0)
        outs[mode] = {k: v["output"] for k, v in o["agents"].items()}
        assert all(v["recomputed_tokens"] == 0 for v in o["agents"].values())
        if mode == "incremental-overlap":
            inc = o
        if mode == "sequential-pd":
            seq = o
    assert all(v == outs["incremental-overlap"] for v in outs.values())
    # incremental overlap finishes no later than sequential (tick time)
    assert inc["e2e_ticks"] <= seq["e2e_ticks"]
    # aggregators issued prefill_only increments only in incremental mode
    assert inc["agents"]["2:0"]["prefill_only_calls"] > 0 and seq["agents"]["2:0"]["prefill_only_calls"] == 0


def test_force_q_gate_rules():
    """test_orchestrator.cpp:140-240: q=0 never exits (12 evals in 9-3-1 ->
    here every member evaluated); q=1 exits at the first completion of each
    group and prunes the still-decoding members."""
    base = dict(C1U, out_len=[[8, 24], 8, 8], query_tokens=16)
    o0 = run_query(run_config(dict(base, force_q=0.0)), tiny_models(base), 1)
    assert all(m["evaluated"] and not m["exited"] for m in o0["metricq"])
    assert len(o0["metricq"]) == 6
    o1 = run_query(run_config(dict(base, force_q=1.0)), tiny_models(base), 1)
    firsts = {}
    for m in o1["metricq"]:
        firsts.setdefault(m["group"], m)
    assert all(m["exited"] for m in firsts.values())
    pruned = [a for a, v in o1["agents"].items() if v["pruned"]]
    for a in pruned:
        assert o1["agents"][a]["output_tokens"] < o1["agents"][a]["decoded"] + 1
    # q = 0 is schedule-neutral (acceptance_main.cpp:923-976)
    n0 = run_query(run_config(dict(base, early_exit=False)), tiny_models(base), 1)
    assert {k: v["output"] for k, v in n0["agents"].items()} == {k: v["output"] for k, v in o0["agents"].items()}
    assert n0["e2e_ticks"] == o0["e2e_ticks"]


def test_oracle_hidden_state_provider():
    """The oracle's hidden-state provider (CpuModel.hidden_embed) feeds the
    MetricQ evaluator: rows are unit-RMS fp64, a C1H request evaluates."""
    import numpy as np
    from oracle.configs import models_of, run_config
    from oracle.orchestrator import run_query
    from paper_2512_18126_b200.configs import CONFIGS
    cfg = dict(CONFIGS["C1H"], out_len=[[8, 16], 8, 8], query_tokens=16, leaf_prefix_tokens=8,
               agg_prefix_tokens=8, suffix_tokens=4)
    rc = run_config(cfg)
    e = rc.embed_fn([5, 17, 99])
    assert e.shape == (3, 256) and e.dtype == np.float64
    assert np.allclose((e * e).mean(axis=1), 1.0, rtol=1e-4)
    r = run_query(rc, models_of(cfg, 256), 0)
    assert any(m["evaluated"] for m in r["metricq"])
