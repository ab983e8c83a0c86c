"""MetricQ (Algorithm 1) and the deterministic mock embedder, restated.

Test infrastructure only.  fp64 numpy; summation orders follow the reference
where they matter for bit-exactness (sequential row mean in MockProvider,
embedding.cpp:104-109).  Gram products use BLAS (the reference's Eigen order
is unpinned; tests compare at 1e-12).
"""
from __future__ import annotations

import math

import numpy as np

from .rng import GOLDEN, RngStream, mix64_np
from .topology import ValidationError

DEFAULT_TAU = 0.7  # metricq.hpp:15


def validate_logprobs(values):
    """metricq.cpp:10-16."""
    if len(values) == 0:
        raise ValidationError("logprobs: need at least one token")
    for v in values:
        if not math.isfinite(v):
            raise ValidationError("logprobs: values must be finite")
        if v > 0.0:
            raise ValidationError("logprobs: values must be <= 0")


def geometric_mean_confidence(values) -> float:
    """metricq.cpp:18-23: exp(mean logprob), sequential sum."""
    validate_logprobs(values)
    s = 0.0
    for v in values:
        s += float(v)
    return math.exp(s / len(values))


def rms_aggregate(cs) -> float:
    """metricq.cpp:25-30."""
    if len(cs) == 0:
        raise ValidationError("rms_aggregate: empty confidence set")
    s = 0.0
    for c in cs:
        s += c * c
    return math.sqrt(s / len(cs))


def correlation_from_gram(g: np.ndarray, eps: float = 1e-12) -> np.ndarray:
    """metricq.cpp:32-53: cosine-normalised Gram, dead columns zeroed."""
    if g.shape[0] != g.shape[1]:
        raise ValidationError("correlation_from_gram: gram matrix must be square")
    d = np.diag(g).copy()
    live = d > eps
    inv = np.zeros_like(d)
    corr = np.zeros_like(g)
    idx = np.nonzero(live)[0]
    if len(idx):
        sub = g[np.ix_(idx, idx)] / np.sqrt(np.outer(d[idx], d[idx]))
        corr[np.ix_(idx, idx)] = sub
        corr[idx, idx] = 1.0
    del inv
    return corr


def frob_cos_sim_corr(cu: np.ndarray, cv: np.ndarray) -> float:
    """metricq.cpp:55-64."""
    if cu.shape != cv.shape:
        raise ValidationError("frob_cos_sim: correlation matrices must share dimensions")
    dot = float(np.sum(cu * cv))
    nu = float(np.sqrt(np.sum(cu * cu)))
    nv = float(np.sqrt(np.sum(cv * cv)))
    if nu == 0.0 or nv == 0.0:
        return 0.0
    return dot / (nu * nv)


def frob_cos_sim(gu, gv, eps=1e-12):
    return frob_cos_sim_corr(correlation_from_gram(gu, eps), correlation_from_gram(gv, eps))


def sim_matrix(embeddings, eps=1e-12):
    """metricq.cpp:72-90."""
    corrs = [correlation_from_gram(t.T @ t, eps) for t in embeddings]
    n = len(corrs)
    sim = np.zeros((n, n))
    for i in range(n):
        sim[i, i] = 1.0
        for j in range(i):
            v = frob_cos_sim_corr(corrs[i], corrs[j])
            sim[i, j] = sim[j, i] = v
    return sim


def weighted_similarity(cs, sim, include_diagonal=True):
    """metricq.cpp:92-111: W and P over the lower triangle."""
    n = len(cs)
    if sim.shape != (n, n):
        raise ValidationError("weighted_similarity: sim matrix does not match confidence count")
    wsum, acc = 0.0, 0.0
    for i in range(n):
        jmax = i if include_diagonal else i - 1
        for j in range(jmax + 1):
            w = cs[i] * cs[j]
            wsum += w
            acc += w * float(sim[i, j])
    return wsum, (acc / wsum if wsum > 0.0 else 0.0)


def calibrate(p, tau):
    """metricq.cpp:113-116."""
    if not tau > 0.0:
        raise ValidationError("calibrate: tau must be > 0")
    return min(max(1.0 - abs(p - tau) / tau, 0.0), 1.0)


def quality(c_bar, b):
    """metricq.cpp:118."""
    return math.sqrt(c_bar * b)


def decide_exit(q: float, rng: RngStream):
    """metricq.cpp:125-131: exit iff draw < q."""
    draw = rng.next_uniform()
    return {"q": q, "draw": draw, "exited": draw < q}


def mock_embed(tokens, hidden: int, seed: int) -> np.ndarray:
    """MockProvider::embed (embedding.cpp:91-113), bit-exact.

    row_seed = hash_combine(hash_combine(seed, token), row);
    x[r,c] = 2*unit_from_bits(mix64(hash_combine(row_seed, c))) - 1; then the
    sequential row mean is subtracted.
    """
    n = len(tokens)
    if n == 0:
        return np.zeros((0, hidden))
    g = np.uint64(GOLDEN)
    s = np.uint64(seed)

    def hc(a, b):
        return mix64_np(a ^ (b + g + (a << np.uint64(6)) + (a >> np.uint64(2))))

    with np.errstate(over="ignore"):
        tok = np.array([int(t) & ((1 << 64) - 1) for t in tokens], dtype=np.uint64)
        rows = np.arange(n, dtype=np.uint64)
        row_seed = hc(hc(np.full(n, s, dtype=np.uint64), tok), rows)
        cols = np.arange(hidden, dtype=np.uint64)
        bits = mix64_np(hc(row_seed[:, None], cols[None, :]))
    u = (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    x = 2.0 * u - 1.0
    mean = np.cumsum(x, axis=1)[:, -1] / float(hidden)  # sequential sum
    return x - mean[:, None]


class MetricQEvaluator:
    """Incremental evaluator (metricq.cpp:148-194)."""

    def __init__(self, embed_fn, tau=DEFAULT_TAU, include_diagonal=True, eps=1e-12):
        if not (0.0 < tau <= 1.0):
            raise ValidationError("metricq: tau must be in (0, 1]")
        self.embed_fn, self.tau, self.include_diagonal, self.eps = embed_fn, tau, include_diagonal, eps
        self.confidences, self.corrs = [], []
        self.sim = np.zeros((0, 0))

    def add_completion(self, output, logprobs):
        c = geometric_mean_confidence(logprobs)
        t = self.embed_fn(output)
        corr = correlation_from_gram(t.T @ t, self.eps)
        n = len(self.confidences) + 1
        grown = np.zeros((n, n))
        if n > 1:
            grown[: n - 1, : n - 1] = self.sim
        grown[n - 1, n - 1] = 1.0
        for j in range(n - 1):
            v = frob_cos_sim_corr(corr, self.corrs[j])
            grown[n - 1, j] = grown[j, n - 1] = v
        self.sim = grown
        self.corrs.append(corr)
        self.confidences.append(c)
        return self.current()

    def current(self):
        c_bar = rms_aggregate(self.confidences)
        w, p = weighted_similarity(self.confidences, self.sim, self.include_diagonal)
        b = calibrate(p, self.tau)
        return {
            "outputs": len(self.confidences),
            "confidences": list(self.confidences),
            "c_bar": c_bar,
            "sim": self.sim.copy(),
            "weight_sum": w,
            "weighted": p,
            "calibrated": b,
            "q": quality(c_bar, b),
            "tau": self.tau,
        }
