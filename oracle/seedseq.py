"""Pure-Python restatement of numpy's SeedSequence -> PCG64 seeding and the
float32 draw stream that the reference renderer consumes.

TEST INFRASTRUCTURE ONLY.  This module is the checker for the C++ port in
``paper_2103_13744_b200/csrc/seedseq.cpp``; nothing in the product imports it.

Reference call site: ``render.py:375``
    rng = np.random.default_rng(np.random.SeedSequence([seed, block_start]))
and ``render.py:296`` ``rng.random((n, k), dtype=np.float32)``.
numpy (pinned here at 2.3.5, third-party, not under /root/reference) defines
the algorithm: SeedSequence pool mixing (pool size 4, 32-bit hashmix), PCG64
``set_seed`` from four generated 64-bit words, XSL-RR output, and float32
draws ``(next_uint32 >> 8) * 2**-24`` where ``next_uint32`` serves the low
half of a fresh 64-bit output first and buffers the high half.
"""

from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645

_INIT_A = 0x43B0D7E5
_MULT_A = 0x931E8875
_INIT_B = 0x8B51F9DD
_MULT_B = 0x58F38DED
_MIX_L = 0xCA01F9DD
_MIX_R = 0x4973F715
_POOL = 4


def _words(n: int) -> list[int]:
    if n < 0:
        raise ValueError("entropy must be non-negative")
    if n == 0:
        return [0]
    out = []
    while n:
        out.append(n & M32)
        n >>= 32
    return out


class _Hasher:
    def __init__(self, const: int, mult: int):
        self.const = const
        self.mult = mult

    def __call__(self, value: int) -> int:
        value = (value ^ self.const) & M32
        self.const = (self.const * self.mult) & M32
        value = (value * self.const) & M32
        return value ^ (value >> 16)


def _mix(x: int, y: int) -> int:
    r = (_MIX_L * x - _MIX_R * y) & M32
    return r ^ (r >> 16)


def seed_pool(entropy: list[int]) -> list[int]:
    """SeedSequence.mix_entropy over the flattened uint32 entropy words."""
    words: list[int] = []
    for e in entropy:
        words += _words(int(e))
    h = _Hasher(_INIT_A, _MULT_A)
    pool = [h(words[i]) if i < len(words) else h(0) for i in range(_POOL)]
    for s in range(_POOL):
        for d in range(_POOL):
            if s != d:
                pool[d] = _mix(pool[d], h(pool[s]))
    for s in range(_POOL, len(words)):
        for d in range(_POOL):
            pool[d] = _mix(pool[d], h(words[s]))
    return pool


def generate_u64(pool: list[int], n64: int) -> list[int]:
    h = _Hasher(_INIT_B, _MULT_B)
    w32 = [h(pool[i % _POOL]) for i in range(2 * n64)]
    return [w32[2 * i] | (w32[2 * i + 1] << 32) for i in range(n64)]


def pcg64_seed(entropy: list[int]) -> tuple[int, int]:
    """(state, inc) of ``PCG64(SeedSequence(entropy))`` as 128-bit ints."""
    v = generate_u64(seed_pool(entropy), 4)
    initstate = (v[0] << 64) | v[1]
    initseq = (v[2] << 64) | v[3]
    inc = ((initseq << 1) | 1) & M128
    state = (0 * PCG_MULT + inc) & M128
    state = (state + initstate) & M128
    state = (state * PCG_MULT + inc) & M128
    return state, inc


def pcg64_output(state: int) -> int:
    hi, lo = state >> 64, state & M64
    x = hi ^ lo
    rot = hi >> 58
    return ((x >> rot) | (x << ((64 - rot) & 63))) & M64


def float32_draws(state: int, inc: int, count: int) -> list[float]:
    """First ``count`` float32 draws of ``Generator.random(dtype=float32)``."""
    out = []
    for m in range((count + 1) // 2):
        state = (state * PCG_MULT + inc) & M128
        o = pcg64_output(state)
        for half in (o & M32, o >> 32):
            out.append((half >> 8) * (1.0 / 16777216.0))
    return out[:count]
