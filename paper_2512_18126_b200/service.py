"""Engine service: the reference's two-entrypoint HTTP engine API
(`/prefill_only`, `/generate`, `/reclaim`, `/healthz`) served by the GPU
engine, the `EngineBackend` plugin interface with its HTTP client, and the
live-mode shell router that feeds one slot plan to a backend
(core/include/moaserve/engine_service.hpp:22-137, core/src/engine_service.cpp:36-371).

What changes against the reference: its `EngineService` computes a virtual
schedule from linear rate laws (engine_service.cpp:49-171); this one runs the
request on the GPU engine (`capi.Engine`: the SimWorld protocol over real
agents) and reports device time.  Request and response bodies keep the
reference's fields and error conditions:

  POST /prefill_only {"agent": "2:0", "start": 0, "tokens": [...]}
    -> {"agent", "start", "end", "t_start", "t_end"}
  POST /generate {"agent", "prompt": [...], "output_tokens": n | "output": [...],
                  "chunk_size": optional}
    -> {"agent", "prompt_tokens", "remainder", "prefill_end", "transfer_seconds",
        "decode_start", "decode_end", "chunks": [{"t", "begin", "end", "tokens"}]}
  POST /reclaim {"agent", "keep"} -> {"agent", "scheduled"}
  GET  /healthz -> {"ok": true}

Times are seconds of device time since the service started (tick-end
events).  "chunks[].tokens" are the tokens the agent decoded (greedy); an
explicit "output" only fixes how many ("t" submit times are accepted and
ignored: calls run when they arrive).  KV stays where it was prefilled, so
"transfer_seconds" is 0.  Domain errors answer HTTP 400 {"error": ...}; a
route the service does not expose answers 404, which `HttpEngineBackend`
turns into a sticky downgrade to accumulate-then-generate
(engine_service.cpp:266-277).

The transport is the Python standard library's threading HTTP server; every
call is serialised by one lock (engine_service.hpp:66) because the engine is
driven by one host thread.  This is host plumbing, not part of the device hot
path: a request's time is spent in `capi.Engine.step()`.
"""
from __future__ import annotations

import json
import re
import threading
import urllib.error
import urllib.request
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer

from . import capi
from .capi import RunError, ValidationError

_INT_PREFIX = re.compile(r"^\s*[+-]?\d+")


def parse_agent(s: str):
    """AgentId::parse (agent.hpp:26-36): '<layer>:<position>' with std::stoi semantics."""
    colon = s.find(":")
    if colon <= 0 or colon + 1 >= len(s):
        raise ValidationError(f"agent id '{s}': expected '<layer>:<position>'")
    a, b = _INT_PREFIX.match(s[:colon]), _INT_PREFIX.match(s[colon + 1:])
    if not a or not b:
        raise ValidationError(f"agent id '{s}': expected '<layer>:<position>'")
    return int(a.group()), int(b.group())


def agent_str(a) -> str:
    return f"{a[0]}:{a[1]}"


def _tokens(v, where):
    """tokens_from (engine_service.cpp:16-25)."""
    if not isinstance(v, list) or any(isinstance(e, bool) or not isinstance(e, int) for e in v):
        raise ValidationError(f"{where}: expected an array of token ids")
    return list(v)


def _agent_from(body):
    if not isinstance(body, dict) or not isinstance(body.get("agent"), str):
        raise ValidationError("body.agent: expected an agent id string")
    return body["agent"]


def _int_field(body, key, default):
    v = body.get(key, default)
    if isinstance(v, bool) or not isinstance(v, int):
        raise ValidationError(f"body.{key}: expected an integer")
    return v


class EngineService:
    """EngineService (engine_service.hpp:40-73) over a GPU engine.

    engine: a `capi.Engine` (or any object with its protocol methods);
    model_for(agent) -> model index, called once when an agent is first seen.
    """

    def __init__(self, engine, model_for=lambda agent: 0, default_chunk_size: int = 32,
                 default_output_tokens: int = 0):
        """default_output_tokens: decode length of a /generate that names neither
        "output" nor "output_tokens" (the reference's synthetic default is 0;
        HttpEngineBackend.generate sends neither, engine_service.cpp:283-289)."""
        if default_chunk_size <= 0:
            raise ValidationError("engine service: default_chunk_size must be > 0")
        if default_output_tokens < 0:
            raise ValidationError("engine service: default_output_tokens must be >= 0")
        self.default_output_tokens = default_output_tokens
        self.eng = engine
        self.model_for = model_for
        self.default_chunk_size = default_chunk_size
        self._lock = threading.Lock()
        self._req = {}
        self._prefill_calls = 0
        self._generate_calls = 0
        self._now = 0.0  # device time at the end of the last tick this service ran
        self.eng.trace(True)
        self.eng.mark_start()

    # -- bookkeeping ------------------------------------------------------
    def _state(self, agent: str):
        """Request state keyed by the parsed AgentId (so "01:0" and "1:0" are one
        agent, as AgentId::parse makes them); the engine slot is bound only
        once a request has passed validation (_bind)."""
        a = parse_agent(agent)  # rejects malformed ids
        r = self._req.get(a)
        if r is None:
            r = self._req[a] = {"id": a, "prompt": [], "generated": False, "bound": False}
        return r

    def _bind(self, r):
        if not r["bound"]:
            self.eng.add_agent(r["id"], self.model_for(r["id"]))
            r["bound"] = True

    def _drive(self):
        """Tick the engine until it is idle; returns its events."""
        events = []
        busy = self.eng.busy()
        while busy:
            ev, busy = self.eng.step()
            events += ev
        return events

    def _t(self, tick: int) -> float:
        return self.eng.tick_seconds(tick) if tick >= 0 else 0.0

    @property
    def prefill_only_calls(self) -> int:
        with self._lock:
            return self._prefill_calls

    @property
    def generate_calls(self) -> int:
        with self._lock:
            return self._generate_calls

    # -- the three entrypoints (engine_service.cpp:49-171) -------------------
    def prefill_only(self, body: dict) -> dict:
        with self._lock:
            self._prefill_calls += 1
            agent = _agent_from(body)
            r = self._state(agent)
            if r["generated"]:
                raise ValidationError(f"prefill_only after generate for agent {agent}")
            start = _int_field(body, "start", 0)
            tokens = _tokens(body["tokens"], "body.tokens") if "tokens" in body else []
            scheduled = len(r["prompt"])
            if start != scheduled:
                raise ValidationError(f"contiguity violation for agent {agent}: prefill starts at {start} but "
                                      f"{scheduled} tokens are scheduled")
            t_start = t_end = self._now
            if tokens:
                self._bind(r)
                self.eng.prefill_only(r["id"], start, tokens)
                r["prompt"] += tokens
                self._drive()
                t_end = self._now = self._last_tick_time()
            return {"agent": agent, "start": start, "end": len(r["prompt"]), "t_start": t_start, "t_end": t_end}

    def generate(self, body: dict) -> dict:
        with self._lock:
            self._generate_calls += 1
            agent = _agent_from(body)
            r = self._state(agent)
            if r["generated"]:
                raise ValidationError(f"generate submitted twice for agent {agent}")
            if "prompt" not in body:
                raise ValidationError("body.prompt: required")
            prompt = _tokens(body["prompt"], "body.prompt")
            have = r["prompt"]
            if len(prompt) < len(have) or prompt[:len(have)] != have:
                raise ValidationError(f"generate prompt for agent {agent} does not extend the prefilled prefix")
            if "output" in body:
                n = len(_tokens(body["output"], "body.output"))
            else:
                n = _int_field(body, "output_tokens", self.default_output_tokens)
                if n < 0:
                    raise ValidationError("body.output_tokens: must be >= 0")
            chunk = _int_field(body, "chunk_size", self.default_chunk_size)
            if chunk <= 0:
                raise ValidationError("body.chunk_size: must be > 0")
            remainder = len(prompt) - len(have)
            self._bind(r)
            self.eng.generate(r["id"], prompt, n, chunk)
            r["prompt"] = list(prompt)
            r["generated"] = True
            events = self._drive()
            rec = self.eng.record(r["id"])
            # the tick that prefilled the remainder also decoded token 0
            prefill_end = self._t(rec["decode_start"]) if rec["decode_start"] >= 0 else self._now
            decode_end = self._t(rec["decode_end"]) if n > 0 and rec["decode_end"] >= 0 else prefill_end
            out = self.eng.read_output(r["id"], n)[0] if n > 0 else []
            chunks = [{"t": self._t(tick), "begin": b, "end": e, "tokens": out[b:e]}
                      for kind, tick, a, b, e in events if kind == "chunk" and tuple(a) == r["id"]]
            self._now = max(self._now, decode_end, self._last_tick_time())
            return {"agent": agent, "prompt_tokens": len(prompt), "remainder": remainder, "prefill_end": prefill_end,
                    "transfer_seconds": 0.0, "decode_start": prefill_end, "decode_end": decode_end, "chunks": chunks}

    def reclaim(self, body: dict) -> dict:
        with self._lock:
            agent = _agent_from(body)
            r = self._state(agent)
            if r["generated"]:
                raise ValidationError(f"reclaim after generate for agent {agent}")
            keep = _int_field(body, "keep", 0)
            scheduled = len(r["prompt"])
            if keep < 0 or keep > scheduled:
                raise ValidationError(f"reclaim point {keep} outside scheduled prompt of {scheduled} tokens")
            if r["bound"]:
                self.eng.reclaim(r["id"], keep)
            del r["prompt"][keep:]
            return {"agent": agent, "scheduled": keep}

    def reset(self):
        """Drop every request (weights stay resident)."""
        with self._lock:
            self.eng.reset()
            self._req.clear()
            self.eng.mark_start()
            self._now = 0.0

    def _last_tick_time(self) -> float:
        t = self.eng.tick() - 1
        return self._t(t) if t >= 0 else self._now


# ---------------------------------------------------------------------------
# HTTP transport (engine_service.cpp:173-225)

class _Handler(BaseHTTPRequestHandler):
    protocol_version = "HTTP/1.1"

    def _reply(self, status, body):
        data = json.dumps(body).encode()
        self.send_response(status)
        self.send_header("Content-Type", "application/json")
        self.send_header("Content-Length", str(len(data)))
        self.end_headers()
        self.wfile.write(data)

    def do_POST(self):  # noqa: N802 (http.server API)
        n = int(self.headers.get("Content-Length") or 0)
        raw = self.rfile.read(n) if n else b""
        fn = self.server.routes.get(self.path)
        if fn is None:
            self._reply(404, {"error": f"no route {self.path}"})
            return
        try:
            body = json.loads(raw) if raw else {}
        except ValueError as e:
            self._reply(400, {"error": f"invalid JSON body: {e}"})
            return
        try:
            self._reply(200, fn(body))
        except (ValidationError, RunError, capi.UnsupportedError) as e:
            self._reply(400, {"error": str(e)})

    def do_GET(self):  # noqa: N802
        if self.path == "/healthz":
            self._reply(200, {"ok": True})
        else:
            self._reply(404, {"error": f"no route {self.path}"})

    def log_message(self, *args):
        pass


class ServiceServer:
    """An EngineService on a loopback port (attach / attach_without_prefill,
    engine_service.cpp:203-225).  split=False exposes only /generate and
    /healthz, emulating a backend without the split entrypoint."""

    def __init__(self, service: EngineService, host: str = "127.0.0.1", port: int = 0, split: bool = True):
        self.httpd = ThreadingHTTPServer((host, port), _Handler)
        self.httpd.daemon_threads = True
        routes = {"/generate": service.generate}
        if split:
            routes.update({"/prefill_only": service.prefill_only, "/reclaim": service.reclaim})
        self.httpd.routes = routes
        self.thread = threading.Thread(target=self.httpd.serve_forever, daemon=True)
        self.thread.start()

    @property
    def url(self) -> str:
        host, port = self.httpd.server_address[:2]
        return f"http://{host}:{port}"

    def close(self):
        self.httpd.shutdown()
        self.httpd.server_close()
        self.thread.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---------------------------------------------------------------------------
# EngineBackend plugin interface + HTTP client (engine_service.hpp:73-99,
# engine_service.cpp:229-298)

class EngineBackend:
    """How a shell router's actions reach an engine."""

    def prefill_only(self, agent, start: int, tokens) -> bool:
        """False: the backend has no split prefill entrypoint (the router degrades)."""
        raise NotImplementedError

    def generate(self, agent, prompt) -> dict:
        raise NotImplementedError

    def reclaim(self, agent, keep: int) -> None:
        raise NotImplementedError


class HttpEngineBackend(EngineBackend):
    def __init__(self, base_url: str, timeout_s: float = 30.0):
        self.base_url = base_url.rstrip("/")
        self.timeout_s = timeout_s
        self.no_prefill_route = False

    def _post(self, route, body):
        req = urllib.request.Request(self.base_url + route, data=json.dumps(body).encode(),
                                     headers={"Content-Type": "application/json"}, method="POST")
        try:
            with urllib.request.urlopen(req, timeout=self.timeout_s) as res:
                return res.status, res.read()
        except urllib.error.HTTPError as e:
            return e.code, e.read()
        except (urllib.error.URLError, OSError) as e:
            raise RunError(f"engine backend: transport failure on {route} ({e})") from e

    @staticmethod
    def _parse(status, raw, route):
        body = None
        if raw:
            try:
                body = json.loads(raw)
            except ValueError:
                raise RunError(f"engine backend: non-JSON response on {route}") from None
        if status != 200:
            detail = body.get("error", "") if isinstance(body, dict) else ""
            raise RunError(f"engine backend: {route} failed with status {status}" + (f": {detail}" if detail else ""))
        return body

    def prefill_only(self, agent, start, tokens):
        if self.no_prefill_route:
            return False
        status, raw = self._post("/prefill_only", {"agent": agent_str(agent), "start": start, "tokens": list(tokens)})
        if status == 404:
            self.no_prefill_route = True
            return False
        self._parse(status, raw, "/prefill_only")
        return True

    def generate(self, agent, prompt):
        status, raw = self._post("/generate", {"agent": agent_str(agent), "prompt": list(prompt)})
        return self._parse(status, raw, "/generate")

    def reclaim(self, agent, keep):
        status, raw = self._post("/reclaim", {"agent": agent_str(agent), "keep": keep})
        self._parse(status, raw, "/reclaim")


# ---------------------------------------------------------------------------
# Live-mode shell router (engine_service.hpp:101-135, engine_service.cpp:302-371)

class HttpShellRouter:
    """Feeds one consumer's slot plan to a backend as precursor chunks and
    completions arrive.  Degradation: when the backend rejects the split
    entrypoint every pending and later increment folds into the terminal
    generate.  Throttle: with min_tokens_per_call > 0 increments are coalesced
    until that many tokens are pending (slot rollback and the terminal
    generate flush first)."""

    def __init__(self, backend: EngineBackend, self_id, prefix, slots, suffix, incremental: bool,
                 min_tokens_per_call: int = 0):
        if min_tokens_per_call < 0:
            raise ValidationError("router: min_tokens_per_call must be >= 0")
        self.backend = backend
        self.self_id = tuple(self_id)
        self.plan = capi.SlotPlan(self_id, prefix, slots, suffix, incremental)
        self.min_tokens_per_call = min_tokens_per_call
        self.degraded = False
        self.done = False
        self.final_prompt = None
        self._buffer_start = -1
        self._buffer = []
        self._response = None

    def start(self):
        self._apply(self.plan.start())

    def on_chunk(self, producer, tokens):
        self._apply(self.plan.on_chunk(producer, tokens))

    def on_precursor_done(self, producer):
        self._apply(self.plan.on_precursor_done(producer))

    def on_precursor_cancelled(self, producer):
        self._apply(self.plan.on_precursor_cancelled(producer))

    def generate_response(self) -> dict:
        if not self.done:
            raise RunError("router: generate has not been issued yet")
        return self._response

    def _flush(self):
        if self._buffer and not self.degraded:
            if not self.backend.prefill_only(self.self_id, self._buffer_start, self._buffer):
                self.degraded = True
        self._buffer = []
        self._buffer_start = -1

    def _apply(self, actions):
        for a in actions:
            if a["kind"] == "prefill_only":
                if self.degraded:
                    continue  # increments fold into the terminal generate
                if self.min_tokens_per_call > 0:
                    if not self._buffer:
                        self._buffer_start = a["start"]
                    self._buffer += a["tokens"]
                    if len(self._buffer) >= self.min_tokens_per_call:
                        self._flush()
                elif not self.backend.prefill_only(self.self_id, a["start"], a["tokens"]):
                    self.degraded = True
            elif a["kind"] == "generate":
                self._buffer = []  # the full prompt carries any coalesced remainder
                self._buffer_start = -1
                self.final_prompt = list(a["tokens"])
                self._response = self.backend.generate(self.self_id, a["tokens"])
                self.done = True
            elif a["kind"] == "reclaim":
                self._flush()  # restore engine offsets before rolling back
                if not self.degraded:
                    self.backend.reclaim(self.self_id, a["start"])


def main(argv=None):
    """Serve the engine API on a loopback port: python -m paper_2512_18126_b200.service --config C1."""
    import argparse

    from .configs import CONFIGS

    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--config", default="C1", help="models of this config (configs.py); agents of layer 1 use the "
                                                   "leaf model, the others the aggregator model")
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--port", type=int, default=8080)
    ap.add_argument("--chunk-size", type=int, default=32)
    ap.add_argument("--output-tokens", type=int, default=0, help="decode length when a request names none")
    ap.add_argument("--no-prefill", action="store_true", help="expose only /generate (a backend without the split "
                                                             "entrypoint)")
    args = ap.parse_args(argv)
    cfg = CONFIGS[args.config]
    eng, _ = capi.engine_for(cfg)
    tags = list(cfg["models"])
    leaf = tags.index("leaf") if "leaf" in tags else 0
    agg = tags.index("agg") if "agg" in tags else leaf
    svc = EngineService(eng, lambda a: leaf if a[0] == 1 else agg, args.chunk_size, args.output_tokens)
    srv = ServiceServer(svc, args.host, args.port, split=not args.no_prefill)
    print(f"serving {args.config} on {srv.url}", flush=True)
    try:
        srv.thread.join()
    except KeyboardInterrupt:
        srv.close()


if __name__ == "__main__":
    main()
