"""CPU transformer agent -- TEST INFRASTRUCTURE (the checker for the B200 path).

The reference has no model (it synthesises outputs, orchestrator.cpp:87-116),
so this is a restatement of OUR engine's numerics contract:
Llama-style decoder (RMSNorm, RoPE rotate-half, GQA, SwiGLU), bf16 weights,
fp32 math, with the activations rounded to bf16 at exactly the points the CUDA
kernels round them:

  rp1  h  = bf16(x)                         (GEMM A operand: the residual itself)
       y  = (h W^T) * inv_rms(x)             (RMSNorm applied to the fp32 product:
            inv_rms(x) = 1 / sqrt(mean(x^2) + eps); the norm gains are ones)
  rp2  q,k = bf16(rope(y)); v = bf16(y)      (KV cache is bf16)
  rp3  o  = bf16(softmax(q k^T / sqrt(hd)) v)
  rp4  a  = bf16(silu(g_acc) * u_acc)
  residual stream x stays fp32; logits fp32.

Weights: uniform hash init, bit-identical with the device init kernel:
bits_i = mix64(base_T + i), base_T = hash_combine(hash_combine(seed,
fnv1a(tag)), fnv1a(T)); w = bf16(fp32((bits>>40) * 2^-23 - 1) * scale_T).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .rng import fnv1a, hash_combine, mix64_np

VOCAB = 50000


@dataclass(frozen=True)
class ModelSpec:
    tag: str
    d: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int = VOCAB
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    lm_gain: float = 4.0
    seed: int = 0


# Shapes from SURVEY.md §8 (builder's choice; the reference has none).
SHAPES = {
    "tiny": dict(d=256, n_layers=4, n_heads=4, n_kv_heads=4, head_dim=64, ffn=1024),
    "1b": dict(d=2048, n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, ffn=8192),
    "8b": dict(d=4096, n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336),
}


def make_spec(tag: str, shape: str, seed: int = 0, **kw) -> ModelSpec:
    return ModelSpec(tag=tag, seed=seed, **{**SHAPES[shape], **kw})


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, like __float2bfloat16_rn."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    if nan.any():
        out = np.where(nan, x, out)
    return out


def tensor_scale(spec: ModelSpec, name: str) -> np.float32:
    """Per-tensor uniform half-width; fp64 formula then one cast to fp32."""
    if name == "emb":
        s = 1.0
    elif name == "lm":
        s = math.sqrt(3.0 / spec.d) * spec.lm_gain
    else:
        k = {"wq": spec.d, "wk": spec.d, "wv": spec.d, "wg": spec.d, "wu": spec.d,
             "wo": spec.n_heads * spec.head_dim, "wd": spec.ffn}[name.split(".")[-1]]
        s = math.sqrt(3.0 / k)
    return np.float32(s)


def _init_chunk(out, s0, s1, base, scale):
    with np.errstate(over="ignore"):
        idx = np.arange(s0, s1, dtype=np.uint64)
        bits = mix64_np(idx + np.uint64(base))
        u = (bits >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
        out[s0:s1] = bf16_round(u * scale)


def init_tensor(spec: ModelSpec, name: str, rows: int, cols: int) -> np.ndarray:
    """Hash-uniform bf16 weights (as fp32 values), logical [rows, cols].
    Chunks are independent (element i depends only on base + i), so they are
    generated on all host threads (numpy releases the GIL)."""
    base = hash_combine(hash_combine(spec.seed, fnv1a(spec.tag)), fnv1a(name))
    n = rows * cols
    out = np.empty(n, dtype=np.float32)
    scale = tensor_scale(spec, name)
    step = 1 << 22
    spans = [(s0, min(n, s0 + step)) for s0 in range(0, n, step)]
    if len(spans) == 1:
        _init_chunk(out, 0, n, base, scale)
    else:
        list(_pool().map(lambda sp: _init_chunk(out, sp[0], sp[1], base, scale), spans))
    return out.reshape(rows, cols)


_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)
    return _POOL


class Weights:
    def __init__(self, spec: ModelSpec):
        self.spec = spec
        d, hd, nh, nkv, f, V = spec.d, spec.head_dim, spec.n_heads, spec.n_kv_heads, spec.ffn, spec.vocab
        self.emb = init_tensor(spec, "emb", V, d)
        self.layers = []
        for l in range(spec.n_layers):
            p = f"L{l}."
            self.layers.append(dict(
                wq=init_tensor(spec, p + "wq", nh * hd, d),
                wk=init_tensor(spec, p + "wk", nkv * hd, d),
                wv=init_tensor(spec, p + "wv", nkv * hd, d),
                wo=init_tensor(spec, p + "wo", d, nh * hd),
                wg=init_tensor(spec, p + "wg", f, d),
                wu=init_tensor(spec, p + "wu", f, d),
                wd=init_tensor(spec, p + "wd", d, f),
            ))
        self.lm = init_tensor(spec, "lm", V, d)


def rope_table(spec: ModelSpec, max_pos: int):
    """cos/sin [max_pos, hd/2] in fp64 (libm) then cast to fp32 -- the device
    uses the identical table computed by the host library."""
    half = spec.head_dim // 2
    cos = np.empty((max_pos, half), dtype=np.float32)
    sin = np.empty((max_pos, half), dtype=np.float32)
    inv = [spec.rope_theta ** (-2.0 * i / spec.head_dim) for i in range(half)]
    for p in range(max_pos):
        for i in range(half):
            a = p * inv[i]
            cos[p, i] = math.cos(a)
            sin[p, i] = math.sin(a)
    return cos, sin


def inv_rms(x: np.ndarray, eps: float) -> np.ndarray:
    """1 / sqrt(mean(x^2) + eps) per row (fp32), shape [..., 1]."""
    ms = np.mean(x * x, axis=-1, keepdims=True, dtype=np.float32)
    return np.float32(1.0) / np.sqrt(ms + np.float32(eps))


def normed_linear(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    """RMSNorm (unit gains) fused with a linear map, as every GPU path computes
    it: the bf16 operand is the residual itself and the fp32 product is scaled
    by the row's inverse RMS -- mathematically rmsnorm(x) @ w.T, rounded at
    bf16(x) instead of bf16(rmsnorm(x))."""
    return (bf16_round(x) @ w.T) * inv_rms(x, eps)


def logit_stats(logits: np.ndarray):
    """argmax (lowest index on ties), logprob(argmax) = -log S, entropy
    H = log S - T/S with S = sum e^(l-m), T = sum (l-m) e^(l-m)."""
    tok = np.argmax(logits, axis=-1)
    m = logits.max(axis=-1, keepdims=True)
    z = logits - m
    e = np.exp(z)
    S = e.sum(axis=-1)
    T = (z * e).sum(axis=-1)
    lp = -np.log(S)
    ent = np.log(S) - T / S
    return tok.astype(np.int32), lp.astype(np.float32), ent.astype(np.float32)


def _runs(rows):
    """Maximal runs of rows of one agent at consecutive positions [i0, i1)."""
    out, i0 = [], 0
    for i in range(1, len(rows) + 1):
        if i == len(rows) or rows[i][0] is not rows[i - 1][0] or rows[i][1] != rows[i - 1][1] + 1:
            out.append((i0, i))
            i0 = i
    return out


class AgentKV:
    def __init__(self, spec: ModelSpec, max_ctx: int):
        self.k = np.zeros((spec.n_layers, spec.n_kv_heads, max_ctx, spec.head_dim), np.float32)
        self.v = np.zeros_like(self.k)


class CpuModel:
    """Batched ragged forward over rows (agent kv, position, token)."""

    def __init__(self, spec: ModelSpec, max_ctx: int = 4096):
        self.spec = spec
        self.w = Weights(spec)
        self.cos, self.sin = rope_table(spec, max_ctx)
        self.max_ctx = max_ctx

    def new_kv(self) -> AgentKV:
        return AgentKV(self.spec, self.max_ctx)

    def forward(self, rows, want_logits):
        """rows: list of (kv: AgentKV, pos, token); rows of one agent appear in
        ascending position order.  Returns (logits[n_out, V]) for rows whose
        want_logits flag is set."""
        sp, w = self.spec, self.w
        x = self.layers(rows)
        sel = np.nonzero(np.asarray(want_logits, bool))[0]
        if len(sel) == 0:
            return np.zeros((0, sp.vocab), np.float32)
        return normed_linear(x[sel], w.lm, sp.norm_eps)

    def hidden_embed(self, tokens) -> np.ndarray:
        """Hidden-state embedding provider (csrc ee_hidden_embed): the final
        residual rows of `tokens` at positions 0..n-1 on a fresh KV,
        RMS-normalised in fp64: e[r] = x[r] / sqrt(mean(x[r]^2) + eps)."""
        kv = self.new_kv()
        x = self.layers([(kv, i, int(t)) for i, t in enumerate(tokens)]).astype(np.float64)
        inv = 1.0 / np.sqrt((x * x).sum(axis=1) / x.shape[1] + self.spec.norm_eps)
        return x * inv[:, None]

    def layers(self, rows):
        """The transformer layers over a ragged batch of rows: final residual x [R, d] (fp32)."""
        sp, w = self.spec, self.w
        R = len(rows)
        hd, nh, nkv = sp.head_dim, sp.n_heads, sp.n_kv_heads
        half = hd // 2
        grp = nh // nkv
        pos = np.array([r[1] for r in rows])
        x = w.emb[np.array([r[2] for r in rows])].astype(np.float32)
        cos, sin = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        scale = np.float32(1.0 / math.sqrt(hd))
        for l, L in enumerate(w.layers):
            h, inv = bf16_round(x), inv_rms(x, sp.norm_eps)
            q = ((h @ L["wq"].T) * inv).reshape(R, nh, hd)
            k = ((h @ L["wk"].T) * inv).reshape(R, nkv, hd)
            v = bf16_round((h @ L["wv"].T) * inv).reshape(R, nkv, hd)

            def rope(t):
                a, b = t[..., :half], t[..., half:]
                return np.concatenate([a * cos - b * sin, b * cos + a * sin], axis=-1)

            q, k = bf16_round(rope(q)), bf16_round(rope(k))
            for i, (kv, p, _) in enumerate(rows):
                kv.k[l, :, p] = k[i]
                kv.v[l, :, p] = v[i]
            o = np.empty((R, nh, hd), np.float32)
            for i0, i1 in _runs(rows):
                kv, p1 = rows[i0][0], rows[i1 - 1][1] + 1
                K = kv.k[l, :, :p1]  # [nkv, p1, hd]
                V = kv.v[l, :, :p1]
                for c0 in range(i0, i1, 256):  # causal attention of a run of consecutive positions
                    c1 = min(i1, c0 + 256)
                    n = c1 - c0
                    qi = q[c0:c1].reshape(n, nkv, grp, hd).transpose(1, 0, 2, 3).reshape(nkv, n * grp, hd)
                    s = np.matmul(qi, K.transpose(0, 2, 1)) * scale  # [nkv, n*grp, p1]
                    s = s.reshape(nkv, n, grp, p1)
                    mask = np.arange(p1)[None, :] > pos[c0:c1][:, None]  # [n, p1]
                    s = np.where(mask[None, :, None, :], np.float32(-np.inf), s)
                    s = s - s.max(axis=-1, keepdims=True)
                    e = np.exp(s)
                    e = e / e.sum(axis=-1, keepdims=True)
                    oi = np.matmul(e.reshape(nkv, n * grp, p1), V)  # [nkv, n*grp, hd]
                    o[c0:c1] = oi.reshape(nkv, n, grp, hd).transpose(1, 0, 2, 3).reshape(n, nh, hd)
            o = bf16_round(o.reshape(R, nh * hd))
            x = x + o @ L["wo"].T
            h2, inv2 = bf16_round(x), inv_rms(x, sp.norm_eps)
            g = (h2 @ L["wg"].T) * inv2
            u = (h2 @ L["wu"].T) * inv2
            a = bf16_round(g / (np.float32(1.0) + np.exp(-g)) * u)
            x = x + a @ L["wd"].T
        return x
