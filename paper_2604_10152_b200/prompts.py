"""Deterministic synthetic prompts and the reference's seeded RNG primitives (host side).

``make_prompts`` restates the reference harness contract (harness.hpp:60-62, declared but
never defined in the reference): prompt b depends only on (seed, b), so it is identical at
every batch size.  Tokens are ``floor(uniform01 * V)`` drawn from
``mt19937_64(substream(seed, 0x70726f6d, b))`` -- the reference's RNG primitives
(common.hpp:23-42).
"""
from __future__ import annotations

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:  # common.hpp:27-32
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def substream(seed: int, tag0: int, tag1: int = 0) -> int:  # common.hpp:35-37
    return splitmix64(seed ^ splitmix64(tag0 ^ splitmix64(tag1)))


class MT19937_64:
    """std::mt19937_64 (sequence fixed by the C++ standard)."""

    def __init__(self, seed: int):
        s = [0] * 312
        s[0] = seed & MASK64
        for i in range(1, 312):
            s[i] = (6364136223846793005 * (s[i - 1] ^ (s[i - 1] >> 62)) + i) & MASK64
        self.s, self.i = s, 312

    def __call__(self) -> int:
        s = self.s
        if self.i >= 312:
            for k in range(312):
                y = (s[k] & 0xFFFFFFFF80000000) | (s[(k + 1) % 312] & 0x7FFFFFFF)
                v = s[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                s[k] = v
            self.i = 0
        x = s[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & MASK64

    def uniform01(self) -> float:  # common.hpp:40-42
        return float(self() >> 11) * (2.0 ** -53)


PROMPT_TAG = 0x70726F6D  # "prom"


def make_prompts(seed: int, batch: int, prompt_len: int, vocab: int) -> list[list[int]]:
    out = []
    for b in range(batch):
        rng = MT19937_64(substream(seed, PROMPT_TAG, b))
        out.append([min(vocab - 1, int(rng.uniform01() * vocab)) for _ in range(prompt_len)])
    return out
