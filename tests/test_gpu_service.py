"""The engine service on the GPU: HTTP /prefill_only + /generate served by
the CUDA engine produce the oracle's greedy tokens, and a shell router gets
the same tokens whether it streams increments (split entrypoint) or degrades
to one generate (the reference's mode-invariance criterion,
acceptance_main.cpp:682-813, over its live-mode router,
engine_service.cpp:302-371)."""
import pytest

from oracle import rng as orng
from oracle.model import CpuModel, make_spec
from oracle.parity import check_agent
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.service import EngineService, HttpEngineBackend, HttpShellRouter, ServiceServer

pytestmark = pytest.mark.gpu


def _engine():
    return capi.Engine([capi.model_spec("leaf", "tiny", 1, max_agents=4), capi.model_spec("agg", "tiny", 2,
                                                                                            max_agents=4)],
                       max_ctx=1024, max_out=128)


def _model_for(a):
    return 0 if a[0] == 1 else 1


def test_service_generate_matches_oracle():
    eng = _engine()
    svc = EngineService(eng, _model_for)
    prompt = orng.synth_tokens(11, "svc", 48)
    with ServiceServer(svc) as srv:
        be = HttpEngineBackend(srv.url)
        assert be.prefill_only((1, 0), 0, prompt[:30])
        assert be.prefill_only((1, 0), 30, prompt[30:40])
        import json
        import urllib.request
        req = urllib.request.Request(srv.url + "/generate", method="POST",
                                     data=json.dumps({"agent": "1:0", "prompt": prompt, "output_tokens": 24,
                                                      "chunk_size": 8}).encode())
        with urllib.request.urlopen(req, timeout=120) as res:
            g = json.loads(res.read())
    assert (g["prompt_tokens"], g["remainder"], g["transfer_seconds"]) == (48, 8, 0.0)
    assert [(c["begin"], c["end"]) for c in g["chunks"]] == [(0, 8), (8, 16), (16, 24)]
    times = [g["prefill_end"]] + [c["t"] for c in g["chunks"]]
    assert all(b >= a for a, b in zip(times, times[1:])) and g["decode_end"] == g["chunks"][-1]["t"]
    toks = [t for c in g["chunks"] for t in c["tokens"]]
    _, lp, _ = eng.read_output((1, 0), 24)
    chk = check_agent(CpuModel(make_spec("leaf", "tiny", seed=1), 1024), prompt, toks, lp)
    assert chk["mismatches"] == [] and chk["lp_ok"], chk
    assert svc.prefill_only_calls == 2 and svc.generate_calls == 1
    eng.close()


def _route(split: bool, threshold: int):
    eng = _engine()
    svc = EngineService(eng, _model_for, default_output_tokens=32)
    a_out = orng.synth_tokens(21, "a", 40)
    b_out = orng.synth_tokens(22, "b", 40)
    with ServiceServer(svc, split=split) as srv:
        r = HttpShellRouter(HttpEngineBackend(srv.url), (2, 0), orng.synth_tokens(23, "pre", 24),
                            [((1, 0), [7, 8]), ((1, 1), [9])], orng.synth_tokens(24, "suf", 6), True, threshold)
        r.start()
        for k in range(0, 40, 16):
            r.on_chunk((1, 0), a_out[k:k + 16])
            r.on_chunk((1, 1), b_out[k:k + 16])
        r.on_precursor_done((1, 0))
        r.on_precursor_done((1, 1))
        g = r.generate_response()
    toks = [t for c in g["chunks"] for t in c["tokens"]]
    _, lp, _ = eng.read_output((2, 0), len(toks))
    calls = svc.prefill_only_calls
    eng.close()
    return toks, lp, r.final_prompt, r.degraded, calls


def test_router_split_and_degraded_decode_the_same_prompt():
    """Streamed, coalesced and degraded routing decode against the same prompt;
    each run's greedy tokens are the oracle's (teacher-forced; different
    prefill chunkings take different GEMM paths, so bit-identity across the
    three runs is not the contract -- DESIGN.md §8)."""
    runs = [_route(True, 0), _route(True, 12), _route(False, 0)]
    (t1, _, p1, d1, c1), (t2, _, p2, d2, c2), (t3, _, p3, d3, c3) = runs
    assert p1 == p2 == p3 and len(p1) == 24 + 2 + 40 + 1 + 40 + 6
    assert not d1 and not d2 and d3
    assert c1 > c2 > 0 and c3 == 0
    model = CpuModel(make_spec("agg", "tiny", seed=2), 1024)
    for toks, lp, prompt, _, _ in runs:
        assert len(toks) == 32
        chk = check_agent(model, prompt, toks, lp)
        assert chk["mismatches"] == [] and chk["lp_ok"], chk
