"""Concrete instances of BASELINE.json `configs` (SURVEY.md §8 "Configs").

Plain data shared by the product host (passed to the C-ABI run config) and by
the tests (which feed the same dicts to the oracle).  Model shapes are the
builder's choice (SURVEY.md §8 "Illustrative model shapes"); the prompt shape
is the reference preset's (config.cpp:228-235).
"""
from __future__ import annotations

import copy

PRESET_PROMPT = dict(query_tokens=256, leaf_prefix_tokens=64, agg_prefix_tokens=96,
                     separator_tokens=0, suffix_tokens=32, chunk_size=32)

C0 = dict(
    name="C0",
    workload="tree 4-2-1, tiny random-init agents, greedy 64 tokens",
    topology=dict(kind="tree", widths=[4, 2, 1], branching=[2, 2]),
    models=dict(leaf=dict(shape="tiny", seed=1), agg=dict(shape="tiny", seed=2)),
    assign=[["leaf"], ["agg"], ["agg"]],
    out_len=[64, 64, 64],
    mode="incremental-overlap",
    early_exit=False,
    exit_scope="cluster",
    tau=0.7,
    include_diagonal=True,
    seed=0,
    hidden=64,
    provider_seed=0,
    **PRESET_PROMPT,
)

C1 = dict(copy.deepcopy(C0), name="C1", early_exit=True,
          workload="tree 4-2-1, tiny agents, greedy 64 tokens, adaptive early exit (cluster scope, tau 0.7)")

# OutputLenDist::Empirical (agent.hpp:40-103): leaf lengths drawn from a support
C1E = dict(copy.deepcopy(C0), name="C1E", early_exit=True, out_len=[{"values": [24, 40, 72, 96]}, 64, 64],
           workload="C1 with empirical leaf output lengths {24, 40, 72, 96}")

# EE parity variant: uneven leaf lengths (test_orchestrator.cpp:32-57 style) so
# exits actually prune still-decoding siblings.
C1U = dict(copy.deepcopy(C1), name="C1U", out_len=[[24, 96], 64, 64],
           workload="C1 with leaf outputs ~U(24,96) (exercises pruning)")

C2 = dict(
    copy.deepcopy(C0), name="C2",
    workload="tree 8-2-1, ~1B random-init agents, leaf prompt 320, greedy 512",
    topology=dict(kind="tree", widths=[8, 2, 1], branching=[4, 2]),
    models=dict(leaf=dict(shape="1b", seed=1), agg=dict(shape="1b", seed=2)),
    out_len=[512, 512, 512],
)

C3 = dict(
    copy.deepcopy(C0), name="C3",
    workload="tree 8-2-1, heterogeneous 1B/8B agents, leaf prompt 2048, greedy 512",
    topology=dict(kind="tree", widths=[8, 2, 1], branching=[4, 2]),
    models=dict(small=dict(shape="1b", seed=1), big=dict(shape="8b", seed=3), agg=dict(shape="1b", seed=2)),
    assign=[["small", "big"], ["agg"], ["big"]],
    out_len=[512, 512, 512],
    query_tokens=1984,
)

# The reference preset's scenario (config.cpp:182-240) at model scale: a 9-3-1
# tree whose leaves cycle three profiles (here 1B, 1B, 8B) with outputs
# ~U(192, 768) (the preset's U(256, 1024), scaled so the all-to-all
# aggregators' 9-output prompts fit the 8192-token context), aggregators with
# fixed 256-token outputs, adaptive early exit at cluster scope.  The
# ablation's paper-scale base (ablation.py --base C5).
C5 = dict(
    copy.deepcopy(C0), name="C5",
    workload="reference-preset analogue: tree 9-3-1, leaves 1B/1B/8B ~U(192,768), 1B aggregators 256, early exit",
    topology=dict(kind="tree", widths=[9, 3, 1], branching=[3, 3]),
    models=dict(fast=dict(shape="1b", seed=1), medium=dict(shape="1b", seed=4), slow=dict(shape="8b", seed=3),
                agg=dict(shape="1b", seed=2)),
    assign=[["fast", "medium", "slow"], ["agg"], ["agg"]],
    out_len=[[192, 768], 256, 256],
    early_exit=True,
)

C4_TREE = dict(copy.deepcopy(C0), name="C4-tree", workload="tree 9-3-1 (13 tiny agents)",
               topology=dict(kind="tree", widths=[9, 3, 1], branching=[3, 3]))
C4_DENSE = dict(copy.deepcopy(C0), name="C4-dense", workload="all-to-all 6-6-1 (13 tiny agents)",
                topology=dict(kind="all_to_all", widths=[6, 6, 1]))

# C1 with the hidden-state embedding provider: the
# semantic agreement is measured on the final hidden states of a separate
# random-init embedding model (the Qwen3-Embedding analogue)
# instead of the MockProvider hash embeddings.
C1H = dict(copy.deepcopy(C1U), name="C1H", provider="hidden", embed_model="embed",
           models=dict(leaf=dict(shape="tiny", seed=1), agg=dict(shape="tiny", seed=2), embed=dict(shape="tiny", seed=7)),
           workload="C1U with the hidden-state embedding provider (tiny embedding model, h = 256)")

# ... at a 1B-class embedding width (the first 2 layers of the `1b` shape,
# h = d_model = 2048 > completion length: the n x n cross-Gram FCS route)
C1H1B = dict(copy.deepcopy(C1H), name="C1H1B",
             models=dict(leaf=dict(shape="tiny", seed=1), agg=dict(shape="tiny", seed=2),
                         embed=dict(shape="1b", seed=7, n_layers=2)),
             workload="C1U with the hidden-state provider at 1B width (h = 2048, n x n FCS route)")

CONFIGS = {c["name"]: c for c in (C0, C1, C1E, C1U, C1H, C1H1B, C2, C3, C4_TREE, C4_DENSE, C5)}


def agent_tag(cfg: dict, layer: int, position: int) -> str:
    """Profile cycling per layer (config.cpp:252-265)."""
    cyc = cfg["assign"][min(layer - 1, len(cfg["assign"]) - 1)]
    return cyc[position % len(cyc)]


def agent_out_len(cfg: dict, layer: int):
    return cfg["out_len"][min(layer - 1, len(cfg["out_len"]) - 1)]
