"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of ROAST's arithmetic (no hashing, no mapping, no
matmul, no scatter).  It only turns a seed into arrays of the shapes and
distributions the paper's workloads use (SURVEY.md §8(d) "Inputs"):

  * counter-based stream  u_i = (splitmix64(seed * 2^32 + i) >> 11) * 2^-53
  * uniform(a, b)         a + (b - a) * u
  * normal                Box-Muller on consecutive pairs of the stream
  * bf16 operands         fp32 draw rounded to bf16 (round-to-nearest-even)
  * embedding indices     uniform on [0, rows) or Zipf(s) by inverse-CDF

Seeds: M = 1, X = 2, dY = 3, idx = 4; hash master seed
0x5EED.  Both the oracle tests and the GPU parity tests / bench draw their
inputs from here, so the two sides see identical bytes.
"""
from __future__ import annotations

import numpy as np

SEED_M = 1
SEED_X = 2
SEED_DY = 3
SEED_IDX = 4
HASH_SEED = 0x5EED

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def _stream_u64(seed: int, n: int, start: int = 0) -> np.ndarray:
    """n raw 64-bit words of the counter stream (vectorised, wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) << np.uint64(32)) + np.arange(start, start + n, dtype=np.uint64)
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, n: int) -> np.ndarray:
    """u_i in [0, 1), fp64, 53-bit resolution."""
    return (_stream_u64(seed, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(seed: int, shape, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    n = int(np.prod(shape))
    return (lo + (hi - lo) * uniform01(seed, n)).reshape(shape)


def normal(seed: int, shape) -> np.ndarray:
    n = int(np.prod(shape))
    u = uniform01(seed, 2 * n)
    u1 = 1.0 - u[0::2]                 # (0, 1]: log is finite
    u2 = u[1::2]
    return (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).reshape(shape)


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (RNE), returned as fp32 values (exactly representable in bf16)."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).reshape(f.shape)


def bf16_bits(a_bf16_valued_f32: np.ndarray) -> np.ndarray:
    """The uint16 bit patterns of fp32 arrays that hold bf16-representable values."""
    f = np.ascontiguousarray(a_bf16_valued_f32, dtype=np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def uniform_indices(seed: int, n: int, rows: int) -> np.ndarray:
    """int64 indices uniform on [0, rows)."""
    return np.minimum((uniform01(seed, n) * rows).astype(np.int64), rows - 1)


def zipf_indices(seed: int, n: int, rows: int, s: float = 1.05) -> np.ndarray:
    """int64 indices on [0, rows) with P(r) proportional to (r+1)^-s.

    Inverse-CDF of the continuous power law on [1, rows+1), floored; then a
    fixed multiplicative scramble (odd constant mod rows is NOT a bijection in
    general, so we use a seeded permutation of hot ranks instead: hot rank r maps
    to row (r * 2654435761) % rows when gcd == 1, else identity).  Only the
    skew matters for the workload; the paper has no DLRM data.
    """
    u = uniform01(seed, n)
    a = 1.0 - s
    hi = float(rows + 1)
    r = np.floor((1.0 + u * (hi ** a - 1.0)) ** (1.0 / a)).astype(np.int64) - 1
    r = np.clip(r, 0, rows - 1)
    mult = 2654435761
    if np.gcd(mult, rows) == 1:
        r = (r * mult) % rows
    return r.astype(np.int64)


def compressed_size(n_virtual: int, ratio: float, align: int = 8) -> int:
    """|M| = ceil(n / ratio) rounded up to a multiple of `align`."""
    m = int(np.ceil(n_virtual / ratio))
    return ((m + align - 1) // align) * align


def mlp_block(ratio: float, tokens: int = 8192, d_model: int = 768, d_ff: int = 3072):
    """C2 shapes: L1 d_model->d_ff, L2 d_ff->d_model and the |M| for `ratio`."""
    n = 2 * d_model * d_ff
    return dict(tokens=tokens, layers=[(d_model, d_ff), (d_ff, d_model)],
                mem_size=compressed_size(n, ratio), n_virtual=n)
