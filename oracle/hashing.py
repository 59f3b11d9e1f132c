"""Oracle hash family (implementation #1) — TEST INFRASTRUCTURE ONLY.

PAPER.md §4.1 only says "universal hash function" h1 : N -> {0..|M|-Z}
 and h2 : N^2 -> {0..|M|-Z1 Z2}, plus an independent sign hash
g : N^k -> {+-1}, each module with "independent hash functions"
(P:293).  The concrete family is the reading of SURVEY.md Appendix A /
DESIGN.md R1-R3, R8: a degree-3 polynomial over GF(2^61 - 1) whose
coefficients come from splitmix64, reduced to an A-aligned offset.

Everything here is plain Python integers (exact), written for reading, not
speed.  Pinned by tests/test_oracle_hash.py: range / alignment fuzz,
determinism, single-legal-offset, chi-square uniformity, birthday collision
rate, seed sensitivity, sign balance and 4-wise sign moments,
and the survey prototype's golden values (tests/golden/hash_c1.txt).  The
exact coefficient stream is a reading, not paper-fixed, so parity of the
*values* against the paper is unpinned; the properties the paper needs
(range, independence, balance) are pinned.
"""
from __future__ import annotations

import math

import numpy as np

P61 = (1 << 61) - 1
MASK64 = (1 << 64) - 1

ROLE_OFFSET = 0
ROLE_SIGN = 1


def splitmix64(z: int) -> int:
    """One splitmix64 output for state z (all arithmetic mod 2^64)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def coefficient(seed: int, module: int, role: int, r: int) -> int:
    """c_r of module `module`, role 0 (offset) or 1 (sign): App. A coef()."""
    inner = splitmix64(((module << 8) | (role << 4) | r) & MASK64)
    return splitmix64((seed ^ inner) & MASK64) % P61


def coefficients(seed: int, module: int, role: int) -> tuple[int, int, int, int]:
    return tuple(coefficient(seed, module, role, r) for r in range(4))


def poly61(c: tuple[int, int, int, int], key: int) -> int:
    """c3 k^3 + c2 k^2 + c1 k + c0 mod (2^61 - 1), key < 2^60."""
    assert 0 <= key < (1 << 60)
    c0, c1, c2, c3 = c
    return (((c3 * key + c2) * key + c1) * key + c0) % P61


def num_positions(mem_size: int, span: int, align: int) -> int:
    """R = floor((|M| - T) / A) + 1: the number of A-aligned legal offsets (R3)."""
    if span > mem_size:
        raise ValueError("geometry: tile/chunk larger than |M| (S:42, S:51)")
    return (mem_size - span) // align + 1


def tile_key(x: int, y: int) -> int:
    """Key of 2-D tile (x, y): x * 2^32 + y (R2)."""
    assert 0 <= x < (1 << 28) and 0 <= y < (1 << 32)
    return (x << 32) | y


def chunk_key(row: int, j: int, chunks_per_row: int) -> int:
    """Global chunk id c = row * ceil(d/Z) + j (R16)."""
    return row * chunks_per_row + j


def offset(seed: int, module: int, key: int, mem_size: int, span: int, align: int) -> int:
    """h(key) in A * {0..R-1}: offset of the tile/chunk inside M (R3)."""
    R = num_positions(mem_size, span, align)
    return align * (poly61(coefficients(seed, module, ROLE_OFFSET), key) % R)


def sign(seed: int, module: int, key: int) -> int:
    """g(key) in {+1, -1}: parity of the role-1 polynomial."""
    return -1 if poly61(coefficients(seed, module, ROLE_SIGN), key) & 1 else 1


def lam(C: float, fan_in: float) -> float:
    """lambda = C / sqrt(n), computed in fp64 then rounded once to fp32 (R7)."""
    return float(np.float32(C / math.sqrt(fan_in)))


def lms_segments(sizes, mem_size: int, align: int) -> list[tuple[int, int]]:
    """Local memory sharing: piece i of n_i parameters gets its own
    memory M_i of |M_i| = f_i |M|, f_i = n_i / n, sum |M_i| = |M|.  Reading R14/R23:
    |M_i| = floor(f_i |M|) rounded down to a multiple of A (so every segment base
    stays A-aligned), the remainder goes to the last piece.  Returns (base, size)."""
    n = sum(sizes)
    out, base = [], 0
    for i, ni in enumerate(sizes):
        if i == len(sizes) - 1:
            size = mem_size - base
        else:
            size = (ni * mem_size // n) // align * align
        out.append((base, size))
        base += size
    return out


class ModuleHash:
    """The hash functions of one registered module (offset + sign), cached coefficients.

    GMS: the module hashes into all of M (base 0, mem_size = |M|).  LMS
    (P:320): into its own segment M_i = M[base, base + mem_size)."""

    def __init__(self, seed: int, module: int, mem_size: int, span: int, align: int,
                 use_sign: bool = True, base: int = 0):
        self.c_off = coefficients(seed, module, ROLE_OFFSET)
        self.c_sgn = coefficients(seed, module, ROLE_SIGN)
        self.R = num_positions(mem_size, span, align)
        self.align = align
        self.use_sign = use_sign
        self.base = base

    def offset(self, key: int) -> int:
        return self.base + self.align * (poly61(self.c_off, key) % self.R)

    def sign(self, key: int) -> int:
        if not self.use_sign:
            return 1
        return -1 if poly61(self.c_sgn, key) & 1 else 1
