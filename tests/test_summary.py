"""RunSummary (a20): the C-ABI's moa_summarize / moa_percentile against the
reference's own run_repetitions + summarize (orchestrator.cpp:297-382) on the
reference's traces (tests/golden/summary.json, generated from oracle/_ref by
tests/golden/make_golden.py) -- bit-exact.  The GPU side (moa_run_repetitions)
is in tests/test_gpu_parity.py."""
import math

import pytest

from paper_2512_18126_b200 import capi


def _model_index(case):
    return {tag: i for i, tag in enumerate(sorted(case["spec"]["profiles"]))}


def test_summarize_matches_reference(golden):
    cases = golden("summary.json")
    assert len(cases) >= 6
    for c in cases:
        out = c["out"]
        ref = out["summary"]
        mine = capi.summarize(c["spec"]["topology"], out["traces"], _model_index(c))
        for k in ("samples", "mean_e2e", "p50_e2e", "p95_e2e", "mean_ee_latency_share", "mean_prefill_only_calls",
                  "mean_recomputed_tokens", "critical_path_prefill_share"):
            assert mine[k] == ref[k], (c["spec"], k, mine[k], ref[k])
        assert set(mine["activation"]) == set(ref["activation"])
        for tag, a in ref["activation"].items():
            for k in ("instances", "invoked", "pruned", "activation"):
                assert mine["activation"][tag][k] == a[k], (tag, k)


def test_critical_path_share_per_trace(golden):
    """Single-trace summaries reproduce the reference's per-trace
    critical_path_prefill_share (orchestrator.cpp:325-350)."""
    for c in golden("summary.json"):
        for t in c["out"]["traces"]:
            s = capi.summarize(c["spec"]["topology"], [t], _model_index(c))
            assert s["critical_path_prefill_share"] == t["prefill_share"]
            assert s["p50_e2e"] == t["e2e_latency"] == s["p95_e2e"]


def test_percentile_interpolation():
    # orchestrator.cpp:306-314: linear interpolation between closest ranks
    assert capi.percentile([], 0.5) == 0.0
    assert capi.percentile([3.0], 0.95) == 3.0
    assert capi.percentile([4.0, 1.0, 3.0, 2.0], 0.5) == 2.5
    v = [float(x) for x in range(1, 21)]
    assert math.isclose(capi.percentile(v, 0.95), 19.05, rel_tol=0, abs_tol=1e-12)
    assert capi.percentile([5.0, 1.0], 0.0) == 1.0 and capi.percentile([5.0, 1.0], 1.0) == 5.0


def test_summarize_errors():
    topo = dict(kind="tree", widths=[2, 1], branching=[2])
    # a trace without the root's record is a protocol error (the reference's map::at throws)
    t = dict(e2e_latency=1.0, ee_latency_total=0.0,
             agents=[dict(layer=1, position=0, model_tag="x", invoked=True, pruned=False, prefill_only_calls=0,
                          recomputed_tokens=0, complete_t=1.0, prefill=[])])
    with pytest.raises(capi.RunError):
        capi.summarize(topo, [t], {"x": 0})
    with pytest.raises(capi.ValidationError):
        capi.summarize(dict(kind="tree", widths=[3, 1], branching=[2]), [], {})
    s = capi.summarize(topo, [], {})
    assert s["samples"] == 0 and s["mean_e2e"] == 0.0 and s["activation"] == {}
