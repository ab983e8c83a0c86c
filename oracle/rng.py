"""Deterministic RNG restated from rng.hpp (test infrastructure only).

Every function is bit-exact with the reference: Python ints masked to 64 bits,
doubles formed exactly as ``unit_from_bits`` does (rng.hpp:33-35).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    """splitmix64 finaliser (rng.hpp:14-19)."""
    z = (z + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def fnv1a(s: str) -> int:
    """fnv1a over the label bytes (rng.hpp:21-28)."""
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & M64
    return h


def unit_from_bits(x: int) -> float:
    """53-bit uniform in [0, 1) (rng.hpp:33-35)."""
    return float(x >> 11) * (2.0 ** -53)


def hash_combine(a: int, b: int) -> int:
    """rng.hpp:39-41."""
    return mix64(a ^ ((b + GOLDEN + ((a << 6) & M64) + (a >> 2)) & M64))


def hash_u64(seed: int, label: str, index: int) -> int:
    """rng.hpp:87-89."""
    return mix64(hash_combine(hash_combine(seed, fnv1a(label)), index))


def hash_unit(seed: int, label: str, index: int) -> float:
    return unit_from_bits(hash_u64(seed, label, index))


class RngStream:
    """splitmix64 stream (rng.hpp:46-83)."""

    def __init__(self, seed: int):
        self.state = seed & M64

    @staticmethod
    def derive_from(master: int, label: str) -> "RngStream":
        return RngStream(hash_combine(master, fnv1a(label)))

    def derive(self, label: str) -> "RngStream":
        return RngStream.derive_from(self.state, label)

    def next_u64(self) -> int:
        v = mix64(self.state)
        self.state = (self.state + 1) & M64
        return v

    def next_uniform(self) -> float:
        return unit_from_bits(self.next_u64())

    def next_int(self, lo: int, hi: int) -> int:
        if hi < lo:
            return lo
        span = (hi - lo) + 1
        return lo + (self.next_u64() % span)


def synth_tokens(seed: int, label: str, count: int) -> list[int]:
    """scenario.cpp:257-264: hash_u64(seed, label, i) % 50000."""
    base = hash_combine(seed, fnv1a(label))
    return [mix64(hash_combine(base, i)) % 50000 for i in range(max(count, 0))]


# ---- vectorised splitmix64 for weight init (numpy uint64 wraps mod 2^64) ----

def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))
