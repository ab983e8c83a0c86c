"""Topology restated from topology.cpp (test infrastructure only).

Agents are ``(layer, position)`` tuples (agent.hpp:16-37); ``aid(a)`` gives the
reference's ``"l:p"`` string.
"""
from __future__ import annotations


class ValidationError(Exception):
    """errors.hpp:10-13 (CLI exit 2)."""


class RunError(Exception):
    """errors.hpp:17-20 (CLI exit 3)."""


def aid(a) -> str:
    return f"{a[0]}:{a[1]}"


def parse_aid(s: str):
    l, p = s.split(":")
    return (int(l), int(p))


class Topology:
    """Layered agent graph (topology.hpp:28-80)."""

    def __init__(self, kind, layers, cluster_sizes):
        self.kind = kind
        self.layers = layers
        self.cluster_sizes = cluster_sizes
        self.pre = {}
        self._index()

    @staticmethod
    def _check_widths(widths):
        if not widths:
            raise ValidationError("topology: widths must be non-empty")
        for i, w in enumerate(widths):
            if w <= 0:
                raise ValidationError(f"topology: layer {i + 1} has non-positive width {w}")

    @staticmethod
    def _make_layers(widths):
        return [[(l + 1, j) for j in range(w)] for l, w in enumerate(widths)]

    @classmethod
    def tree(cls, widths, branching):
        """topology.cpp:43-67."""
        cls._check_widths(widths)
        if len(branching) + 1 != len(widths):
            raise ValidationError("topology: branching count mismatch")
        sizes = []
        for l in range(len(widths) - 1):
            b = branching[l]
            if b <= 0:
                raise ValidationError(f"topology: branching factor for layer {l + 2} must be positive")
            if widths[l + 1] * b != widths[l]:
                raise ValidationError(f"topology: layer {l + 2} width does not cover layer {l + 1}")
            sizes.append([b] * widths[l + 1])
        return cls.tree_custom(widths, sizes)

    @classmethod
    def tree_custom(cls, widths, cluster_sizes):
        """topology.cpp:69-104."""
        cls._check_widths(widths)
        if len(cluster_sizes) + 1 != len(widths):
            raise ValidationError("topology: cluster size count mismatch")
        for l in range(len(widths) - 1):
            sizes = cluster_sizes[l]
            if len(sizes) != widths[l + 1]:
                raise ValidationError(f"topology: layer {l + 2} cluster count mismatch")
            if any(s <= 0 for s in sizes):
                raise ValidationError(f"topology: layer {l + 2} has a non-positive cluster size")
            if sum(sizes) != widths[l]:
                raise ValidationError(f"topology: layer {l + 2} cluster sizes do not sum")
        return cls("tree", cls._make_layers(widths), [list(s) for s in cluster_sizes])

    @classmethod
    def all_to_all(cls, widths):
        """topology.cpp:106-113."""
        cls._check_widths(widths)
        return cls("all_to_all", cls._make_layers(widths), [])

    def _index(self):
        """Contiguous cluster assignment (topology.cpp:115-142)."""
        for l, layer in enumerate(self.layers):
            if l == 0:
                for a in layer:
                    self.pre[a] = []
                continue
            if self.kind == "all_to_all":
                for a in layer:
                    self.pre[a] = list(self.layers[l - 1])
            else:
                cursor = 0
                for j, a in enumerate(layer):
                    n = self.cluster_sizes[l - 1][j]
                    self.pre[a] = list(self.layers[l - 1][cursor:cursor + n])
                    cursor += n

    @property
    def depth(self):
        return len(self.layers)

    def layer(self, l):
        if l < 1 or l > self.depth:
            raise ValidationError(f"topology: layer {l} out of range")
        return self.layers[l - 1]

    def agents(self):
        return [a for layer in self.layers for a in layer]

    def precursors(self, a):
        if a not in self.pre:
            raise ValidationError(f"topology: unknown agent {aid(a)}")
        return self.pre[a]

    def successors(self, a):
        """topology.cpp:167-175."""
        if a[0] >= self.depth:
            return []
        return [b for b in self.layers[a[0]] if a in self.pre[b]]

    def clusters_of_layer(self, l):
        """topology.cpp:177-187."""
        if l < 2 or l > self.depth:
            raise ValidationError("topology: clusters_of_layer range")
        return [list(self.pre[a]) for a in self.layers[l - 1]]

    def root(self):
        """topology.cpp:189-196."""
        if len(self.layers[-1]) != 1:
            raise ValidationError("topology: a single aggregator is required")
        return self.layers[-1][0]


def critical_path(topo: Topology, agent_time: dict) -> float:
    """topology.cpp:324-340."""
    finish, total = {}, 0.0
    for layer in topo.layers:
        for a in layer:
            ready = max([finish[p] for p in topo.precursors(a)], default=0.0)
            finish[a] = ready + agent_time[a]
            total = max(total, finish[a])
    return total
