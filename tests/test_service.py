"""Engine service, HTTP backend and shell router (CPU): the reference's
test_engine_service.cpp cases that do not depend on its virtual-time rate
laws, over a deterministic stand-in engine (the GPU run is in
test_gpu_service.py).  The router cases are transcribed from
test_engine_service.cpp:436-590 (same template, same expected call
sequences)."""
import json
import urllib.request

import pytest

from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.capi import RunError, ValidationError
from paper_2512_18126_b200.service import (EngineBackend, EngineService, HttpEngineBackend, HttpShellRouter,
                                           ServiceServer, parse_agent)

SELF, A, B = (2, 0), (1, 0), (1, 1)


def two_slot():
    """{10,11} [sep {20} <- 1:0] [sep {21} <- 1:1] {30} (test_engine_service.cpp:41-46)."""
    return dict(prefix=[10, 11], slots=[(A, [20]), (B, [21])], suffix=[30])


class FakeBackend(EngineBackend):
    """Records every call and checks a real engine's invariants (test_engine_service.cpp:69-105)."""

    def __init__(self, accept_prefill=True):
        self.accept_prefill = accept_prefill
        self.calls, self.delivered = [], []
        self.generate_result = {"source": "fake"}

    def prefill_only(self, agent, start, tokens):
        assert tuple(agent) == SELF
        self.calls.append(("prefill", start, list(tokens)))
        if not self.accept_prefill:
            return False
        assert start == len(self.delivered) and tokens
        self.delivered += list(tokens)
        return True

    def generate(self, agent, prompt):
        self.calls.append(("generate", 0, list(prompt)))
        return self.generate_result

    def reclaim(self, agent, keep):
        self.calls.append(("reclaim", keep, []))
        assert 0 <= keep <= len(self.delivered)
        del self.delivered[keep:]


def router(backend, incremental=True, threshold=0):
    t = two_slot()
    return HttpShellRouter(backend, SELF, t["prefix"], t["slots"], t["suffix"], incremental, threshold)


def test_router_streams_incremental_fill():
    be = FakeBackend()
    r = router(be)
    with pytest.raises(RunError):
        r.generate_response()
    r.start()
    r.on_chunk(A, [100, 101])
    r.on_precursor_done(A)
    r.on_chunk(B, [200])
    assert not r.done
    r.on_precursor_done(B)
    assert r.done and not r.degraded
    assert r.generate_response() == be.generate_result
    prompt = [10, 11, 20, 100, 101, 21, 200, 30]
    assert [c[2] for c in be.calls[:5]] == [[10, 11, 20], [100, 101], [21], [200], [30]]
    assert be.calls[5] == ("generate", 0, prompt)
    assert be.delivered == prompt and r.final_prompt == prompt


def test_router_non_incremental_generates_once():
    be = FakeBackend()
    r = router(be, incremental=False)
    r.start()
    r.on_chunk(A, [100, 101])
    r.on_precursor_done(A)
    r.on_chunk(B, [200])
    r.on_precursor_done(B)
    assert r.done
    assert be.calls == [("generate", 0, [10, 11, 20, 100, 101, 21, 200, 30])]
    assert be.delivered == []


def test_router_degrades_on_missing_split_entrypoint():
    be = FakeBackend(accept_prefill=False)
    r = router(be)
    r.start()
    assert r.degraded and len(be.calls) == 1  # the one rejected attempt
    r.on_chunk(A, [100, 101])
    r.on_precursor_done(A)
    r.on_chunk(B, [200])
    assert len(be.calls) == 1
    r.on_precursor_done(B)
    assert r.done and len(be.calls) == 2
    assert be.calls[1] == ("generate", 0, [10, 11, 20, 100, 101, 21, 200, 30])
    assert be.delivered == []


def test_router_coalesces_below_threshold():
    be = FakeBackend()
    r = router(be, threshold=5)
    r.start()
    r.on_chunk(A, [100])
    assert be.calls == []
    r.on_chunk(A, [101, 102])
    assert be.calls == [("prefill", 0, [10, 11, 20, 100, 101, 102])]
    r.on_chunk(A, [103])
    r.on_precursor_done(A)
    assert len(be.calls) == 1
    r.on_chunk(B, [200, 201, 202])
    assert be.calls[1] == ("prefill", 6, [103, 21, 200, 201, 202])
    r.on_precursor_done(B)
    prompt = [10, 11, 20, 100, 101, 102, 103, 21, 200, 201, 202, 30]
    assert len(be.calls) == 3 and be.calls[2] == ("generate", 0, prompt)
    assert be.delivered == prompt[:-1]


def test_router_flushes_before_rollback():
    be = FakeBackend()
    r = router(be, threshold=100)
    r.start()
    r.on_chunk(A, [100, 101])
    assert be.calls == []
    r.on_precursor_cancelled(A)
    assert be.calls == [("prefill", 0, [10, 11, 20, 100, 101]), ("reclaim", 2, [])]
    assert be.delivered == [10, 11]
    r.on_chunk(B, [200])
    r.on_precursor_done(B)
    assert r.done and be.calls[2] == ("generate", 0, [10, 11, 21, 200, 30])


def test_router_rejects_negative_threshold():
    with pytest.raises(ValidationError):
        router(FakeBackend(), threshold=-1)


class StubEngine:
    """The capi.Engine protocol surface the service drives, with one token per
    tick per decoding agent (token = 1000 * layer + position + k) and chunk
    events every apc tokens -- enough to exercise the service and the HTTP
    layer without a GPU."""

    def __init__(self):
        self.reset()

    def reset(self):
        self.t, self.agents, self.times = 0, {}, []

    def trace(self, on):
        pass

    def mark_start(self):
        self.times = []

    def add_agent(self, a, model):
        self.agents[a] = dict(prompt=[], queued=0, gen=None, out=[], rec=dict(decode_start=-1, decode_end=-1))

    def prefill_only(self, a, start, tokens):
        g = self.agents[a]
        if start != len(g["prompt"]):
            raise RunError("sim: contiguity")
        g["prompt"] += list(tokens)
        g["queued"] += 1

    def generate(self, a, prompt, max_new, apc):
        g = self.agents[a]
        g["prompt"] = list(prompt)
        g["gen"] = dict(n=max_new, apc=apc, begin=0)

    def reclaim(self, a, keep):
        del self.agents[a]["prompt"][keep:]

    def busy(self):
        return any(g["queued"] or (g["gen"] and g["rec"]["decode_end"] < 0) for g in self.agents.values())

    def step(self):
        ev, tick = [], self.t
        for a, g in self.agents.items():
            if g["queued"]:
                g["queued"] = 0
            elif g["gen"] and g["rec"]["decode_end"] < 0:
                gen = g["gen"]
                if g["rec"]["decode_start"] < 0:
                    g["rec"]["decode_start"] = tick
                if len(g["out"]) < gen["n"]:
                    g["out"].append(1000 * a[0] + a[1] + len(g["out"]))
                n = len(g["out"])
                if n > gen["begin"] and (n - gen["begin"] >= gen["apc"] or n == gen["n"]):
                    ev.append(("chunk", tick, a, gen["begin"], n))
                    gen["begin"] = n
                if n == gen["n"]:
                    g["rec"]["decode_end"] = tick
                    ev.append(("decode_end", tick, a, n, 0))
        self.t += 1
        self.times.append(0.001 * self.t)
        return ev, self.busy()

    def tick(self):
        return self.t

    def tick_seconds(self, t):
        return self.times[t]

    def record(self, a):
        return dict(self.agents[a]["rec"])

    def read_output(self, a, n):
        return self.agents[a]["out"][:n], [0.0] * n, [0.0] * n


def post(url, route, body, raw=None):
    req = urllib.request.Request(url + route, data=raw if raw is not None else json.dumps(body).encode(),
                                 headers={"Content-Type": "application/json"}, method="POST")
    try:
        with urllib.request.urlopen(req, timeout=10) as res:
            return res.status, json.loads(res.read())
    except urllib.error.HTTPError as e:
        return e.code, json.loads(e.read())


def test_agent_id_parsing():
    assert parse_agent("2:0") == (2, 0) and parse_agent(" 3:+1x") == (3, 1)
    for bad in ("", ":1", "1:", "a:1", "12"):
        with pytest.raises(ValidationError):
            parse_agent(bad)


def test_service_prefill_contiguity_and_generate():
    svc = EngineService(StubEngine(), default_chunk_size=2)
    r = svc.prefill_only({"agent": "2:0", "start": 0, "tokens": [1, 2, 3]})
    assert (r["agent"], r["start"], r["end"]) == ("2:0", 0, 3) and r["t_end"] >= r["t_start"]
    with pytest.raises(ValidationError, match="contiguity violation"):
        svc.prefill_only({"agent": "2:0", "start": 2, "tokens": [4]})
    e = svc.prefill_only({"agent": "2:0", "start": 3, "tokens": []})  # empty increment: timestamped no-op
    assert e["end"] == 3 and e["t_start"] == e["t_end"]
    g = svc.generate({"agent": "2:0", "prompt": [1, 2, 3, 4], "output_tokens": 5})
    assert list(g) == ["agent", "prompt_tokens", "remainder", "prefill_end", "transfer_seconds", "decode_start",
                       "decode_end", "chunks"]
    assert (g["prompt_tokens"], g["remainder"], g["transfer_seconds"]) == (4, 1, 0.0)
    assert [(c["begin"], c["end"]) for c in g["chunks"]] == [(0, 2), (2, 4), (4, 5)]
    assert [t for c in g["chunks"] for t in c["tokens"]] == [2000, 2001, 2002, 2003, 2004]
    assert g["decode_end"] >= g["decode_start"] == g["prefill_end"]
    assert svc.prefill_only_calls == 3 and svc.generate_calls == 1


@pytest.mark.parametrize("body,match", [
    ({"agent": "2:0"}, "body.prompt: required"),
    ({"agent": "2:0", "prompt": [9]}, "does not extend"),
    ({"agent": "2:0", "prompt": [1, 2], "chunk_size": 0}, "chunk_size"),
    ({"agent": "2:0", "prompt": [1, 2], "output_tokens": -1}, "output_tokens"),
    ({"agent": "2:0", "prompt": [1, "x"]}, "array of token ids"),
    ({"agent": "bad", "prompt": [1]}, "agent id"),
    ({"prompt": [1]}, "body.agent"),
])
def test_service_generate_validation(body, match):
    """test_engine_service.cpp:234-282."""
    svc = EngineService(StubEngine())
    svc.prefill_only({"agent": "2:0", "start": 0, "tokens": [1, 2]})
    with pytest.raises(ValidationError, match=match):
        svc.generate(body)


def test_service_generate_seals_and_reclaim_bounds():
    svc = EngineService(StubEngine())
    svc.prefill_only({"agent": "2:0", "start": 0, "tokens": [1, 2, 3]})
    with pytest.raises(ValidationError, match="outside scheduled prompt"):
        svc.reclaim({"agent": "2:0", "keep": 4})
    assert svc.reclaim({"agent": "2:0", "keep": 1}) == {"agent": "2:0", "scheduled": 1}
    assert svc.prefill_only({"agent": "2:0", "start": 1, "tokens": [7]})["end"] == 2
    svc.generate({"agent": "2:0", "prompt": [1, 7], "output": [0, 0, 0]})
    with pytest.raises(ValidationError, match="twice"):
        svc.generate({"agent": "2:0", "prompt": [1, 7]})
    with pytest.raises(ValidationError, match="after generate"):
        svc.prefill_only({"agent": "2:0", "start": 2, "tokens": [1]})
    with pytest.raises(ValidationError, match="after generate"):
        svc.reclaim({"agent": "2:0", "keep": 0})


def test_http_routes_and_errors():
    """test_engine_service.cpp:305-384: 200 JSON, 400 on domain errors, 404 without the split entrypoint."""
    with ServiceServer(EngineService(StubEngine())) as srv:
        with urllib.request.urlopen(srv.url + "/healthz", timeout=10) as res:
            assert json.loads(res.read()) == {"ok": True}
        assert post(srv.url, "/prefill_only", {"agent": "2:0", "start": 0, "tokens": [5, 6]})[0] == 200
        st, body = post(srv.url, "/prefill_only", {"agent": "2:0", "start": 0, "tokens": [5]})
        assert st == 400 and "contiguity violation" in body["error"]
        st, body = post(srv.url, "/generate", None, raw=b"{not json")
        assert st == 400 and body["error"].startswith("invalid JSON body")
        st, body = post(srv.url, "/generate", {"agent": "2:0", "prompt": [5, 6, 7], "output_tokens": 2})
        assert st == 200 and body["remainder"] == 1 and len(body["chunks"]) == 1
    with ServiceServer(EngineService(StubEngine()), split=False) as srv:
        assert post(srv.url, "/prefill_only", {"agent": "2:0", "start": 0, "tokens": [1]})[0] == 404
        assert post(srv.url, "/reclaim", {"agent": "2:0", "keep": 0})[0] == 404
        assert post(srv.url, "/generate", {"agent": "2:0", "prompt": [1]})[0] == 200


def test_http_backend_round_trip_errors_and_sticky_downgrade():
    """test_engine_service.cpp:386-434."""
    with ServiceServer(EngineService(StubEngine())) as srv:
        be = HttpEngineBackend(srv.url)
        assert be.prefill_only(SELF, 0, [1, 2])
        with pytest.raises(RunError, match="status 400: contiguity violation"):
            be.prefill_only(SELF, 5, [3])
        be.reclaim(SELF, 1)
        g = be.generate(SELF, [1, 9])
        assert g["prompt_tokens"] == 2 and g["remainder"] == 1
    with ServiceServer(EngineService(StubEngine()), split=False) as srv:
        be = HttpEngineBackend(srv.url)
        assert not be.prefill_only(SELF, 0, [1]) and be.no_prefill_route
        assert not be.prefill_only(SELF, 0, [1])  # sticky: no further request
        assert be.generate(SELF, [1])["prompt_tokens"] == 1
    be = HttpEngineBackend("http://127.0.0.1:9", timeout_s=2)
    with pytest.raises(RunError, match="transport failure"):
        be.generate(SELF, [1])


def test_router_end_to_end_over_http_with_coalescing():
    """test_engine_service.cpp:560-586 (rates aside: prompt / remainder / call counts)."""
    svc = EngineService(StubEngine())
    with ServiceServer(svc) as srv:
        r = router(HttpEngineBackend(srv.url), threshold=4)
        r.start()
        r.on_chunk(A, [100, 101])
        r.on_precursor_done(A)
        r.on_chunk(B, [200, 201, 202])
        r.on_precursor_done(B)
        assert r.done and not r.degraded
        gen = r.generate_response()
        assert gen["prompt_tokens"] == 10 and gen["remainder"] == 1
        assert gen["transfer_seconds"] == 0.0 and gen["decode_end"] == gen["decode_start"]
        assert len(r.final_prompt) == 10
    assert svc.prefill_only_calls == 2 and svc.generate_calls == 1


def test_slotplan_wrapper_matches_router_actions():
    p = capi.SlotPlan(SELF, [10, 11], [(A, [20]), (B, [21])], [30], True)
    assert p.start() == [{"kind": "prefill_only", "start": 0, "tokens": [10, 11, 20]}]
    assert p.on_chunk(A, [100]) == [{"kind": "prefill_only", "start": 3, "tokens": [100]}]
    assert p.on_chunk((9, 9), [1]) == []  # not a slot of this plan: dropped (router.cpp:45-46)
    p.on_precursor_done(A)
    p.on_precursor_done(B)
    with pytest.raises(RunError, match="after generate"):  # router.cpp:47-49
        p.on_chunk(A, [1])
