"""Synthetic KEEP workloads (the bench's inputs; not on the hot path).

Restates the reference's seeded instance generator so the GPU bench and the
CPU oracle see identical layouts: keep::Rng (prng.hpp:34-82) and
testutil::make_instance's draw order (tests/test_util.hpp:26-36).  Static
groups model the reference's static/dynamic memory layout
(memory_store.hpp:27-88): consecutive runs of segments share one joint KV
block (harness.hpp:520-531), the rest are dynamic per-segment owners.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def fnv1a64(name: str) -> int:
    h = 0xCBF29CE484222325
    for c in name.encode():
        h ^= c
        h = (h * 0x100000001B3) & MASK64
    return h


class Rng:
    """keep::Rng -- splitmix64 with two warm-up draws (prng.hpp:34-38)."""

    def __init__(self, seed: int):
        self.s = seed & MASK64
        self.next_u64()
        self.next_u64()

    @classmethod
    def stream(cls, seed: int, name: str) -> "Rng":
        return cls(seed ^ fnv1a64(name))

    def next_u64(self) -> int:
        self.s = (self.s + GAMMA) & MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def next_below(self, n: int) -> int:
        return self.next_u64() % n


def _stream_draws(seed: int, name: str, count: int) -> np.ndarray:
    """Vectorised: the first `count` outputs of Rng::stream(seed, name)."""
    s0 = (seed ^ fnv1a64(name)) & MASK64
    k = np.arange(3, count + 3, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(s0) + k * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


@dataclass
class Instance:
    seg_len: np.ndarray
    tokens: np.ndarray
    query: np.ndarray


def make_instance_layout(seed: int, S: int, V: int, lo: int = 8, hi: int = 12, qlen: int = 8) -> Instance:
    """Layout of testutil::make_instance (tests/test_util.hpp:26-36)."""
    # upper bound of draws: per segment 1 + hi, then qlen
    draws = _stream_draws(seed, "instance", S * (1 + hi) + qlen).tolist()
    pos = 0
    seg_len = np.empty(S, np.int32)
    toks = []
    for i in range(S):
        n = lo + int(draws[pos] % (hi - lo + 1))
        pos += 1
        seg_len[i] = n
        toks.extend(int(x % V) for x in draws[pos:pos + n])
        pos += n
    query = np.array([int(x % V) for x in draws[pos:pos + qlen]], np.int32)
    return Instance(seg_len, np.array(toks, np.int32), query)


def group_units(S: int, group_size: int, static_fraction: float, seed: int = 0):
    """Units (begin, end, owner_kind, owner_id): the first static_fraction of
    the segments in static groups of group_size, the rest dynamic."""
    from . import GROUP, SEGMENT
    units = []
    n_static = int(S * static_fraction) // group_size * group_size
    g = 0
    for b in range(0, n_static, group_size):
        units.append((b, b + group_size, GROUP, g))
        g += 1
    for i in range(n_static, S):
        units.append((i, i + 1, SEGMENT, i))
    return units
