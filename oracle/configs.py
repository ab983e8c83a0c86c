"""Build oracle RunConfig/model objects from the plain config dicts shared with
the product (paper_2512_18126_b200/configs.py).  Test infrastructure only."""
from __future__ import annotations

from .model import CpuModel, make_spec
from .orchestrator import RunConfig
from .topology import Topology

_MODEL_CACHE = {}


def topology_of(t: dict) -> Topology:
    if t["kind"] == "all_to_all":
        return Topology.all_to_all(t["widths"])
    if "cluster_sizes" in t:
        return Topology.tree_custom(t["widths"], t["cluster_sizes"])
    return Topology.tree(t["widths"], t["branching"])


def run_config(cfg: dict) -> RunConfig:
    topo = topology_of(cfg["topology"])
    assign, out_len = {}, {}
    for layer in topo.layers:
        for a in layer:
            cyc = cfg["assign"][min(a[0] - 1, len(cfg["assign"]) - 1)]
            assign[a] = cyc[a[1] % len(cyc)]
            ol = cfg["out_len"][min(a[0] - 1, len(cfg["out_len"]) - 1)]
            out_len[a] = dict(ol) if isinstance(ol, dict) else tuple(ol) if isinstance(ol, (list, tuple)) else int(ol)
    keys = ("mode", "early_exit", "exit_scope", "tau", "include_diagonal", "chunk_size", "seed",
            "query_tokens", "leaf_prefix_tokens", "agg_prefix_tokens", "separator_tokens",
            "suffix_tokens", "hidden", "provider_seed")
    kw = {k: cfg[k] for k in keys if k in cfg}
    if cfg.get("force_q") is not None:
        kw["force_q"] = cfg["force_q"]
    if cfg.get("provider", "mock") == "hidden":  # hidden-state provider: the embedding model's final rows
        em = models_of(cfg, 1024)[cfg["embed_model"]]
        kw["embed_fn"] = em.hidden_embed
    return RunConfig(topology=topo, assign=assign, out_len=out_len, **kw)


def models_of(cfg: dict, max_ctx: int = 4096) -> dict:
    out = {}
    for tag, m in cfg["models"].items():
        over = {k: v for k, v in m.items() if k not in ("shape", "seed")}  # e.g. n_layers: the shape's first layers
        key = (tag, m["shape"], m.get("seed", 0), max_ctx, tuple(sorted(over.items())))
        if key not in _MODEL_CACHE:
            _MODEL_CACHE[key] = CpuModel(make_spec(tag, m["shape"], seed=m.get("seed", 0), **over), max_ctx)
        out[tag] = _MODEL_CACHE[key]
    return out
