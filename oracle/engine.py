"""Tick engine -- the engine protocol of SimWorld (pdsim.hpp:61-156) on
discrete engine ticks instead of a linear time law.  TEST INFRASTRUCTURE: the
CPU restatement that the CUDA engine (csrc/host/engine.cpp) must match
tick-for-tick (DESIGN.md §5 "tick contract").

Protocol checks are the reference's (pdsim.cpp:155-214, :374-418):
contiguity, generate-extends-prefix, apc_chunk > 0, cancel-after-completion,
reclaim bounds, late actions on cancelled requests dropped.

One tick:
  1. rows, in agent registration order (skip cancelled / finished):
     - decoding (n_out >= 1, n_out < max_new): one decode row at P+n_out-1;
     - else its queued prefill jobs, in order, while they fit the tick's row
       budget; the last row of the job that ends the sealed prompt yields out[0];
     - else a sealed, fully prefilled prompt that has not started decoding:
       one bootstrap row at P-1 (re-writes the identical KV) yielding out[0]
       (max_new == 0: no row, decode starts and ends this tick).
  2. one batched forward per model over its rows.
  3. state update (prefill commit, recompute accounting, n_out).
  4. phase A: chunk emission [begin, n_out) every apc_chunk tokens and at the
     end (pdsim.cpp:339-362) -> chunk callbacks, registration order;
     phase B: completions -> decode_end callbacks, registration order;
     phase C: deferred callbacks (FIFO, may enqueue more).
"""
from __future__ import annotations

from collections import deque

import numpy as np

from .model import logit_stats
from .topology import RunError, ValidationError, aid


class Request:
    def __init__(self, rid, model, kv, order):
        self.id, self.model, self.kv, self.order = rid, model, kv, order
        self.prompt = []
        self.prefilled = 0
        self.max_computed = 0
        self.gen = 0
        self.queue = deque()
        self.generate_pending = False
        self.decode_started = False
        self.finished = False
        self.cancelled = False
        self.max_new = 0
        self.apc_chunk = 0
        self.n_out = 0
        self.chunk_begin = 0
        self.out, self.lp, self.ent = [], [], []
        self.chunk_cbs, self.end_cbs = [], []
        self.rec = dict(invoked=False, pruned=False, empty_input=False, submit_tick=0,
                        precursor_ready_tick=0, prompt_tokens=0, output_tokens=0, prefill=[],
                        prefill_only_calls=0, recomputed_tokens=0, reclaimed_tokens=0,
                        wasted_prefill_tokens=0, decode_start=-1, decode_end=-1, complete=-1)


class TickEngine:
    def __init__(self, models: dict, max_rows_per_tick: int = 16384, keep_logits: bool = False,
                 forced: dict | None = None, owner: dict | None = None, rank: int = 0, exchange=None):
        """forced: agent -> (tokens, logprobs, entropy) replayed instead of the
        model's greedy outputs (record-and-replay parity: the schedule, routing
        and early-exit logic then run on exactly the GPU's completions).

        owner / rank / exchange: tree-partitioned mode (the C++ engine's
        replicated control plane): every rank runs this schedule for all
        agents but computes rows only for agents it owns; at each chunk,
        exchange(agent, owner, payload) returns the chunk's (tokens, logprobs,
        entropies) -- the owner passes its payload, the others receive it."""
        self.models = models  # tag -> CpuModel (unused when forced)
        self.forced = forced
        self.owner, self.rank, self.exchange = owner, rank, exchange
        self.reqs = {}
        self.order = []
        self.tick = 0
        self.max_rows = max_rows_per_tick
        self.deferred = deque()
        self.events = []
        self.keep_logits = keep_logits
        self.logits = {}  # (agent, k) -> logits row (when keep_logits)

    # ---- protocol (pdsim.hpp:61-156) ----
    def add_agent(self, rid, model_tag):
        if rid in self.reqs:
            raise ValidationError(f"sim: agent {aid(rid)} added twice")
        kv = None if self.forced is not None else self.models[model_tag].new_kv()
        r = Request(rid, model_tag, kv, len(self.order))
        r.rec["submit_tick"] = self.tick
        self.reqs[rid] = r
        self.order.append(rid)

    def req(self, rid):
        if rid not in self.reqs:
            raise RunError(f"sim: unknown agent {aid(rid)}")
        return self.reqs[rid]

    def submit_prefill_only(self, rid, expected_start, tokens):
        """pdsim.cpp:155-174."""
        r = self.req(rid)
        if r.cancelled:
            return
        if r.generate_pending or r.decode_started:
            raise RunError(f"sim: prefill_only after generate for agent {aid(rid)}")
        sched = len(r.prompt)
        if expected_start != sched:
            raise RunError(f"sim: contiguity violation for agent {aid(rid)}")
        if not tokens:
            return
        r.prompt += list(tokens)
        r.rec["prefill_only_calls"] += 1
        r.queue.append((sched, sched + len(tokens), r.gen))

    def submit_generate(self, rid, full_prompt, max_new, apc_chunk, prefill_chunk=0):
        """pdsim.cpp:176-214 (output length instead of planned output)."""
        r = self.req(rid)
        if r.cancelled:
            return
        if r.generate_pending or r.decode_started:
            raise RunError(f"sim: generate submitted twice for agent {aid(rid)}")
        sched = len(r.prompt)
        if len(full_prompt) < sched or list(full_prompt[:sched]) != r.prompt:
            raise RunError(f"sim: generate prompt for agent {aid(rid)} does not extend the prefilled prefix")
        if apc_chunk <= 0:
            raise ValidationError("sim: apc_chunk must be > 0")
        if max_new < 0:
            raise ValidationError("sim: max_new must be >= 0")
        r.prompt = list(full_prompt)
        r.max_new, r.apc_chunk = max_new, apc_chunk
        r.generate_pending = True
        r.rec["prompt_tokens"] = len(full_prompt)
        r.rec["invoked"] = True
        step = prefill_chunk if prefill_chunk > 0 else len(full_prompt) - sched
        b = sched
        while b < len(full_prompt):
            e = min(b + step, len(full_prompt))
            r.queue.append((b, e, r.gen))
            b = e

    def cancel(self, rid):
        """pdsim.cpp:374-398: output truncated to the tokens already decoded."""
        r = self.req(rid)
        if r.finished:
            raise RunError(f"sim: cancel after completion for agent {aid(rid)}")
        if r.cancelled:
            return
        r.cancelled = True
        r.rec["pruned"] = True
        r.gen += 1
        r.queue.clear()
        r.generate_pending = False
        r.rec["output_tokens"] = r.n_out if r.decode_started else 0
        self.events.append((self.tick, "cancel", rid, r.rec["output_tokens"]))

    def reclaim(self, rid, keep):
        """pdsim.cpp:400-418."""
        r = self.req(rid)
        if r.generate_pending or r.decode_started:
            raise RunError(f"sim: reclaim after generate for agent {aid(rid)}")
        if keep < 0 or keep > len(r.prompt):
            raise RunError("sim: reclaim point outside scheduled prompt")
        r.gen += 1
        # Jobs below the keep point survive (truncated at keep).  The
        # reference clears the whole queue (pdsim.cpp:411), which strands
        # [prefilled, keep) and later trips its own contiguity check
        # (pdsim.cpp:270-272); between ticks nothing is in flight, so the
        # correct rewind is expressible here.
        kept = deque()
        for b, e, _ in r.queue:
            if b < keep:
                kept.append((b, min(e, keep), r.gen))
        r.queue = kept
        del r.prompt[keep:]
        if r.prefilled > keep:
            r.rec["reclaimed_tokens"] += r.prefilled - keep
            r.prefilled = keep
        self.events.append((self.tick, "reclaim", rid, keep))

    def on_chunk(self, rid, cb):
        self.req(rid).chunk_cbs.append(cb)

    def on_decode_end(self, rid, cb):
        self.req(rid).end_cbs.append(cb)

    def defer(self, fn):
        self.deferred.append(fn)

    def note_precursor_ready(self, rid):
        r = self.req(rid)
        r.rec["precursor_ready_tick"] = max(r.rec["precursor_ready_tick"], self.tick)

    def mark_empty_input(self, rid):
        self.req(rid).rec["empty_input"] = True

    # ---- ticks ----
    def _computes(self, r):
        return self.owner is None or self.owner[r.id] == self.rank

    def busy(self):
        for r in self.reqs.values():
            if r.cancelled or r.finished:
                continue
            if r.queue or r.generate_pending or r.decode_started:
                return True
        return False

    def step(self):
        t = self.tick
        plan = []  # (req, kind, job)
        rows_by_model = {}
        budget = self.max_rows
        for rid in self.order:
            r = self.reqs[rid]
            if r.cancelled or r.finished:
                continue
            if r.decode_started:
                if r.n_out < r.max_new:
                    p = len(r.prompt) + r.n_out - 1
                    if self._computes(r):
                        rows_by_model.setdefault(r.model, []).append((r, p, r.out[r.n_out - 1], True))
                    plan.append((r, "decode", None))
                    budget -= 1
                continue
            if r.queue:
                took = False
                while r.queue and r.queue[0][1] - r.queue[0][0] <= budget:
                    b, e, _ = r.queue.popleft()
                    budget -= e - b
                    took = True
                    yields = r.generate_pending and e == len(r.prompt) and r.max_new > 0
                    if self._computes(r):
                        lst = rows_by_model.setdefault(r.model, [])
                        for p in range(b, e):
                            lst.append((r, p, r.prompt[p], yields and p == e - 1))
                    plan.append((r, "prefill", (b, e, yields)))
                if took or r.queue:
                    continue
            if r.generate_pending and r.prefilled == len(r.prompt):
                if r.max_new == 0:
                    plan.append((r, "empty", None))
                else:
                    P = len(r.prompt)
                    tok = r.prompt[P - 1] if P > 0 else 0
                    if self._computes(r):
                        rows_by_model.setdefault(r.model, []).append((r, max(P - 1, 0), tok, True))
                    plan.append((r, "bootstrap", None))
                    budget -= 1
        # 2. forward per model
        for tag, rows in rows_by_model.items():
            if self.forced is not None:
                for r, p, _, want in rows:
                    if want:
                        k = len(r.out)
                        tok, lp, ent = self.forced[r.id]
                        r.out.append(int(tok[k]))
                        r.lp.append(float(lp[k]))
                        r.ent.append(float(ent[k]))
                continue
            m = self.models[tag]
            logits = m.forward([(r.kv, p, tok) for r, p, tok, _ in rows], [w for *_, w in rows])
            if len(logits):
                tok, lp, ent = logit_stats(logits)
                k = 0
                for r, p, _, want in rows:
                    if want:
                        if self.keep_logits:
                            self.logits[(r.id, len(r.out))] = logits[k]
                        r.out.append(int(tok[k]))
                        r.lp.append(float(lp[k]))
                        r.ent.append(float(ent[k]))
                        k += 1
        # 3. state update
        for r, kind, job in plan:
            if kind == "decode":
                r.n_out += 1
            elif kind == "prefill":
                b, e, yields = job
                recomputed = max(0, min(e, r.max_computed) - b)
                r.max_computed = max(r.max_computed, e)
                r.rec["prefill"].append((t, b, e, False))
                r.rec["recomputed_tokens"] += recomputed
                if b != r.prefilled:
                    raise RunError(f"sim: internal contiguity breach for agent {aid(r.id)}")
                r.prefilled = e
                if yields:
                    self._start_decode(r, t, 1)
                elif r.generate_pending and r.prefilled == len(r.prompt) and r.max_new == 0:
                    self._start_decode(r, t, 0)
            elif kind == "bootstrap":
                self._start_decode(r, t, 1)
            elif kind == "empty":
                self._start_decode(r, t, 0)
        self.tick += 1
        # 4. phase A: chunks (partitioned mode: owner -> every rank first)
        if self.exchange is not None:
            for rid in self.order:
                r = self.reqs[rid]
                if r.cancelled or r.finished or not r.decode_started:
                    continue
                n = r.n_out
                if n > r.chunk_begin and (n - r.chunk_begin >= r.apc_chunk or n == r.max_new):
                    b = r.chunk_begin
                    mine = self._computes(r)
                    payload = (r.out[b:n], r.lp[b:n], r.ent[b:n]) if mine else None
                    toks, lps, ents = self.exchange(rid, self.owner[rid], n - b, payload)
                    if not mine:
                        r.out += [int(x) for x in toks]
                        r.lp += [float(x) for x in lps]
                        r.ent += [float(x) for x in ents]
        done = []
        for rid in self.order:
            r = self.reqs[rid]
            if r.cancelled or r.finished or not r.decode_started:
                continue
            n = r.n_out
            if n > r.chunk_begin and (n - r.chunk_begin >= r.apc_chunk or n == r.max_new):
                b = r.chunk_begin
                r.chunk_begin = n
                gen = r.gen
                toks = r.out[b:n]
                self.events.append((t, "chunk", rid, (b, n)))
                for cb in list(r.chunk_cbs):
                    cb(b, n, toks)
                    if r.gen != gen:
                        break
            if r.n_out == r.max_new and not r.cancelled:
                done.append(r)
        # phase B: completions
        for r in done:
            if r.cancelled or r.finished:
                continue
            r.finished = True
            r.rec["decode_end"] = t
            r.rec["complete"] = t
            r.rec["output_tokens"] = r.max_new
            self.events.append((t, "decode_end", r.id, r.max_new))
            for cb in list(r.end_cbs):
                cb(t)
        # phase C: deferred
        while self.deferred:
            self.deferred.popleft()()
        return True

    def _start_decode(self, r, t, n_out):
        r.generate_pending = False
        r.decode_started = True
        r.rec["decode_start"] = t
        r.n_out = n_out

    def run(self, max_ticks=1_000_000):
        while self.busy():
            self.step()
            if self.tick > max_ticks:
                raise RunError("engine: tick limit exceeded")
