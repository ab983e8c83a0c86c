"""run_query restated over the tick engine (orchestrator.cpp:130-295,
scenario.cpp:10-116).  TEST INFRASTRUCTURE: the checker for the CUDA path and
the CPU baseline timed by bench.py.

Differences from the reference are the contract of this tier:
agent outputs come from greedy decode of the agent's model instead of
make_output/make_logprobs (orchestrator.cpp:87-116); time is engine ticks;
ee_eval_latency is not modelled (evaluations complete between ticks).
Everything else -- prompt synthesis labels, slot filling, exit groups, RNG
streams, gate semantics, pruning rule -- is the reference's.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

from . import metricq as mq
from .engine import TickEngine
from .rng import RngStream, hash_combine, synth_tokens
from .router import PromptTemplate, SlotPlan
from .topology import Topology, ValidationError, aid

MODES = ("sequential-pd", "dp-only", "dp-chunked-prefill", "incremental-overlap")


@dataclass
class RunConfig:
    """orchestrator.hpp:23-53 (+ model assignment, which replaces rates)."""
    topology: Topology
    assign: dict  # agent -> model tag
    out_len: dict  # agent -> fixed output length, (lo, hi) uniform, or {"values": [...]} empirical
    mode: str = "incremental-overlap"
    early_exit: bool = False
    exit_scope: str = "cluster"
    tau: float = 0.7
    include_diagonal: bool = True
    force_q: Optional[float] = None
    chunk_size: int = 32
    seed: int = 0
    repetitions: int = 1
    query_tokens: int = 256
    leaf_prefix_tokens: int = 64
    agg_prefix_tokens: int = 96
    separator_tokens: int = 0
    suffix_tokens: int = 32
    hidden: int = 64
    provider_seed: int = 0
    # embedding provider: None = MockProvider(hidden, provider_seed); else a
    # callable tokens -> fp64 [n, h] (the hidden-state provider, CpuModel.hidden_embed)
    embed_fn: Optional[Callable] = None

    def validate(self):
        """orchestrator.cpp:21-62."""
        if len(self.topology.layers[-1]) != 1:
            raise ValidationError("run: last layer must hold a single aggregator")
        if not (0.0 < self.tau <= 1.0):
            raise ValidationError("run.tau: must be in (0, 1]")
        if self.chunk_size <= 0:
            raise ValidationError("run.chunk_size: must be > 0")
        if self.force_q is not None and not (0.0 <= self.force_q <= 1.0):
            raise ValidationError("run.force_q: must be in [0, 1]")
        if self.mode not in MODES:
            raise ValidationError(f"mode: unknown '{self.mode}'")
        for a, spec in self.out_len.items():
            if isinstance(spec, dict) and (not spec["values"] or min(spec["values"]) < 0):
                raise ValidationError(f"run: empirical output lengths need values >= 0 for agent {aid(a)}")
            if self.early_exit and out_len_min(spec) < 1:  # orchestrator.cpp:42-60
                raise ValidationError(f"run: early exit needs output_len >= 1 for agent {aid(a)}")


def sample_out_len(spec, ss, a):
    """OutputLenDist::sample with RngStream::derive(ss, "outlen:l:p") (agent.hpp:88-99):
    int = Fixed, (lo, hi) = Uniform, {"values": [...]} = Empirical (uniform over
    the support: values[next_int(0, size - 1)])."""
    if isinstance(spec, int):
        return spec
    if isinstance(spec, dict):
        v = spec["values"]
        return v[RngStream.derive_from(ss, "outlen:" + aid(a)).next_int(0, len(v) - 1)]
    lo, hi = spec
    return RngStream.derive_from(ss, "outlen:" + aid(a)).next_int(lo, hi)


def out_len_min(spec):
    if isinstance(spec, int):
        return spec
    if isinstance(spec, dict):
        return min(spec["values"])
    return spec[0]


class Driver:
    """SimDriver (scenario.cpp:10-116) over the tick engine."""

    def __init__(self, eng: TickEngine, mode: str, chunk: int):
        self.eng, self.mode, self.chunk = eng, mode, chunk
        self.order, self.plans, self.out_len, self.consumers, self.dependent = [], {}, {}, {}, {}
        self.gate = None

    def add_source(self, a, tag, prompt, out_len):
        self.eng.add_agent(a, tag)
        self.order.append(a)
        self.dependent[a] = False
        self.out_len[a] = out_len
        self.plans[a] = SlotPlan(a, PromptTemplate(prompt, [], []), False)

    def add_plan(self, a, tag, tmpl, out_len):
        self.eng.add_agent(a, tag)
        self.order.append(a)
        self.dependent[a] = bool(tmpl.slots)
        self.out_len[a] = out_len
        for p, _ in tmpl.slots:
            self.consumers.setdefault(p, []).append(a)
        self.plans[a] = SlotPlan(a, tmpl, self.mode == "incremental-overlap")

    def start(self):
        for dep in sorted(self.consumers):
            for c in self.consumers[dep]:
                self.eng.on_chunk(dep, lambda b, e, toks, c=c, d=dep: self.apply(c, self.plans[c].on_chunk(d, toks)))
        for a in self.order:
            self.eng.on_decode_end(a, lambda t, a=a: self.on_completion(a))
        for a in self.order:
            self.apply(a, self.plans[a].start())

    def apply(self, a, actions):
        for kind, start, toks in actions:
            if kind == "prefill_only":
                self.eng.submit_prefill_only(a, start, toks)
            elif kind == "generate":
                pc = self.chunk if (self.mode == "dp-chunked-prefill" and self.dependent[a]) else 0
                self.eng.submit_generate(a, toks, self.out_len[a], self.chunk, pc)
            else:
                self.eng.reclaim(a, start)

    def on_completion(self, a):
        if self.gate:
            self.gate(a)
        else:
            self.release(a)

    def release(self, p):
        for c in self.consumers.get(p, []):
            self.eng.note_precursor_ready(c)
            self.apply(c, self.plans[c].on_precursor_done(p))

    def prune(self, p):
        self.eng.cancel(p)
        for c in self.consumers.get(p, []):
            plan = self.plans[c]
            self.apply(c, plan.on_precursor_cancelled(p))
            if plan.all_inputs_pruned():
                self.eng.mark_empty_input(c)


@dataclass
class ExitGroup:
    label: str
    members: list
    evaluator: mq.MetricQEvaluator
    rng: RngStream
    exited: bool = False
    evals: int = 0


def build_query(cfg: RunConfig, sample: int, eng: TickEngine):
    """Prompt synthesis + registration (orchestrator.cpp:133-191)."""
    topo = cfg.topology
    ss = hash_combine(cfg.seed, sample)
    drv = Driver(eng, cfg.mode, cfg.chunk_size)
    query = synth_tokens(ss, "query", cfg.query_tokens)
    for layer in topo.layers:
        for a in layer:
            n = sample_out_len(cfg.out_len[a], ss, a)
            if not topo.precursors(a):
                prompt = synth_tokens(ss, "leaf_prefix:" + aid(a), cfg.leaf_prefix_tokens) + query
                drv.add_source(a, cfg.assign[a], prompt, n)
            else:
                slots = [(p, synth_tokens(ss, f"sep:{aid(a)}:{k}", cfg.separator_tokens))
                         for k, p in enumerate(topo.precursors(a))]
                tmpl = PromptTemplate(synth_tokens(ss, "agg_prefix:" + aid(a), cfg.agg_prefix_tokens),
                                      slots, synth_tokens(ss, "suffix:" + aid(a), cfg.suffix_tokens))
                drv.add_plan(a, cfg.assign[a], tmpl, n)
    return ss, drv


def exit_groups(cfg: RunConfig, ss: int):
    """orchestrator.cpp:204-219."""
    topo = cfg.topology
    if cfg.exit_scope == "layer" or topo.kind == "all_to_all":
        sets = [list(topo.layer(l)) for l in range(1, topo.depth)]
    else:
        sets = [c for l in range(2, topo.depth + 1) for c in topo.clusters_of_layer(l)]
    groups = []
    for g, members in enumerate(sets):
        label = f"ee:{g}"
        embed = cfg.embed_fn or (lambda t: mq.mock_embed(t, cfg.hidden, cfg.provider_seed))
        ev = mq.MetricQEvaluator(embed, cfg.tau, cfg.include_diagonal)
        groups.append(ExitGroup(label, members, ev, RngStream.derive_from(ss, label)))
    return groups


def tree_placement(topo: Topology, world: int) -> dict:
    """Owning rank per agent (mirrors csrc/host/orchestrator.cpp
    tree_placement): leaves in contiguous blocks over the ranks, every
    dependent agent on the rank of its first precursor."""
    leaves = topo.layers[0]
    at = {a: (i * world) // len(leaves) for i, a in enumerate(leaves)}
    for layer in topo.layers[1:]:
        for a in layer:
            at[a] = at[topo.precursors(a)[0]]
    return at


def run_query(cfg: RunConfig, models: dict, sample: int = 0, keep_logits: bool = False, forced=None,
              world: int = 1, rank: int = 0, exchange=None):
    """forced: agent -> (tokens, logprobs, entropy) -- replay mode (see TickEngine).
    world > 1: tree-partitioned mode -- this rank computes only the agents
    tree_placement gives it; `exchange` moves chunk payloads between ranks."""
    cfg.validate()
    owner = tree_placement(cfg.topology, world) if world > 1 else None
    eng = TickEngine(models, keep_logits=keep_logits, forced=forced, owner=owner, rank=rank, exchange=exchange)
    ss, drv = build_query(cfg, sample, eng)
    records = []
    if cfg.early_exit and cfg.topology.depth > 1:
        groups = exit_groups(cfg, ss)
        group_of = {m: g for g in groups for m in g.members}

        def gate(producer):
            g = group_of.get(producer)
            if g is None or g.exited:
                drv.release(producer)
                return

            def evaluate():
                rec = dict(tick=eng.tick, group=g.label, eval_index=g.evals, completed=aid(producer))
                if g.exited:
                    rec.update(evaluated=False, q=0.0, draw=1.0, exited=False, pruned=[])
                    records.append(rec)
                    drv.release(producer)
                    return
                g.evals += 1
                r = eng.reqs[producer]
                score = g.evaluator.add_completion(r.out[: r.max_new], [float(x) for x in r.lp[: r.max_new]])
                q = cfg.force_q if cfg.force_q is not None else score["q"]
                d = mq.decide_exit(q, g.rng)
                pruned = []
                if d["exited"]:
                    g.exited = True
                    for m in g.members:
                        if m == producer or eng.reqs[m].finished or eng.reqs[m].cancelled:
                            continue
                        pruned.append(m)
                rec.update(evaluated=True, q=d["q"], draw=d["draw"], exited=d["exited"],
                           pruned=[aid(m) for m in pruned], c=score["confidences"][-1],
                           score_q=score["q"], sim_row=[float(x) for x in score["sim"][-1]])
                for m in pruned:
                    drv.prune(m)
                records.append(rec)
                drv.release(producer)

            eng.defer(evaluate)

        drv.gate = gate
    drv.start()
    eng.run()
    return summarize_run(cfg, eng, drv, records)


def summarize_run(cfg, eng, drv, records):
    agents = {}
    for a in drv.order:
        r = eng.reqs[a]
        rec = dict(r.rec)
        agents[aid(a)] = dict(
            rec,
            model=r.model,
            prompt=list(r.prompt),
            output=list(r.out[: (r.rec["output_tokens"])]),
            logprobs=list(r.lp[: r.rec["output_tokens"]]),
            entropy=list(r.ent[: r.rec["output_tokens"]]),
            decoded=r.n_out,
        )
    ticks = max((v["complete"] for v in agents.values()), default=-1) + 1
    tokens = sum(v["output_tokens"] for v in agents.values() if v["invoked"] and not v["pruned"])
    return dict(agents=agents, metricq=records, e2e_ticks=ticks, tokens=tokens, events=eng.events)
