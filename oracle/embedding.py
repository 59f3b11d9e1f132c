"""Oracle ROAST / ROBE block embedding (the L operation) — TEST INFRASTRUCTURE ONLY.

    w[i] = lambda * M[h1(C(i)) + O(i)]                         (§4.1 "Lookup")

with chunks of Z elements; the global chunk id of element k of logical row r
is c = r * ceil(d / Z) + k // Z (rows padded to a multiple of Z, reading R16),
O(i) = k mod Z, and the optional sign g(c).  Backward:

    dM[h1(c) + o] += lambda * g(c) * dOut[b, jZ + o]           (duplicates add, R15)

lambda = fp32(C / sqrt(fan_in)), fan_in = d by default (R7).

Pinned by tests/test_oracle_embedding.py: the single-row store m = Z = d
(S:180), zero store, linearity + adjoint, central finite
differences over every slot, duplicate accumulation and the collision
example, and the bit-exact fp32 value definition.
"""
from __future__ import annotations

import numpy as np

from . import hashing


class EmbeddingSpec:
    def __init__(self, num_rows, dim, chunk, mem_size, seed, module, align=8, C=1.0,
                 fan_in=None, use_sign=True, segment=None):
        self.num_rows, self.dim, self.chunk = num_rows, dim, chunk
        self.mem_size = mem_size
        self.chunks_per_row = -(-dim // chunk)
        # segment = (base, size): LMS memory M_i of this table; None = GMS
        seg_base, seg_size = segment if segment is not None else (0, mem_size)
        assert 0 <= seg_base and seg_base + seg_size <= mem_size
        self.mh = hashing.ModuleHash(seed, module, seg_size, chunk, align, use_sign, base=seg_base)
        self.lam = hashing.lam(C, dim if fan_in is None else fan_in)

    def chunk_map(self, rows) -> tuple[np.ndarray, np.ndarray]:
        """(offset, sign) of every chunk of every requested row: shape (n, ceil(d/Z))."""
        rows = np.asarray(rows, dtype=np.int64)
        n, q = len(rows), self.chunks_per_row
        off = np.empty((n, q), dtype=np.int64)
        sgn = np.empty((n, q), dtype=np.int64)
        for b, r in enumerate(rows.tolist()):
            if not 0 <= r < self.num_rows:
                raise IndexError("bounds: row index out of range (S:178)")
            for j in range(q):
                k = hashing.chunk_key(r, j, q)
                off[b, j] = self.mh.offset(k)
                sgn[b, j] = self.mh.sign(k)
        return off, sgn

    def _slots(self, off):
        """slot[b, k] = h1(C(k)) + O(k) for k < d."""
        k = np.arange(self.dim, dtype=np.int64)
        return off[:, k // self.chunk] + (k % self.chunk)

    def forward(self, rows, M, kind: str = "fp32") -> np.ndarray:
        """out[b, k]; kind="fp32" is the bit-exact fp32 value g * fp32(lambda32 * M32)."""
        off, sgn = self.chunk_map(rows)
        k = np.arange(self.dim)
        g = sgn[:, k // self.chunk].astype(np.float64)
        prod = np.float64(self.lam) * np.asarray(M, dtype=np.float64)[self._slots(off)]
        if kind == "fp32":
            return g * prod.astype(np.float32).astype(np.float64)
        if kind == "exact":
            return g * prod
        raise ValueError(kind)

    def backward(self, rows, dOut, dM=None) -> np.ndarray:
        """dM += scatter of lambda * g * dOut, in (b, k) order; duplicates accumulate."""
        if dM is None:
            dM = np.zeros(self.mem_size, dtype=np.float64)
        off, sgn = self.chunk_map(rows)
        k = np.arange(self.dim)
        g = sgn[:, k // self.chunk].astype(np.float64)
        contrib = np.float64(self.lam) * g * np.asarray(dOut, dtype=np.float64)
        np.add.at(dM, self._slots(off).ravel(), contrib.ravel())
        return dM
