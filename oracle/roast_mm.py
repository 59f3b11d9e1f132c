"""Oracle ROAST-MM (linear layer) — TEST INFRASTRUCTURE ONLY.

The plain definition (SURVEY.md §8(c) "Nature of the result"): ROAST-MM is a
dense layer whose weights are tied through the hash, so

    W[i, j] = g(C1, C2) * lambda * M[h2(C1, C2) + pi(O1, O2)]
    Y  = X W            (Algorithm 1; lambda once per output tile)
    dX = dY W^T         (backward through the same mapping)
    dM[s] = sum_{(i,j): slot(i,j) = s} lambda * g * (X^T dY)[i, j]
                        (P:340 gradient rule, with g by the chain rule, R12)

implemented literally: materialise W in fp64, use numpy's fp64 matmul as the
library primitive, and scatter with np.add.at in fixed (i, j) order.
pi(O1, O2) = Z2*O1 + O2 ("row-major") or the SW128 bijection of
reading R4.  Edge tiles (H % Z1 != 0 or O % Z2 != 0) are zero-padded (R9).

Pinned by tests/test_oracle_mm.py: identity mapping == dense reshape (R22,
north star), X = I gives W, zero store, single tile,
adjoint identities, central finite differences over every slot
of a tiny two-layer GMS model, sum-of-partials across layers,
the collision example, padding invariance, and the bit-exact
fp32 recovered-weight definition.
"""
from __future__ import annotations

import numpy as np
import torch

from . import hashing

ROW_MAJOR = 0
SW128 = 1

HASH = 0
IDENTITY = 1


def pi(o1: int, o2: int, z2: int, layout: int) -> int:
    """Position of tile element (o1, o2) inside its Z1 x Z2 block of M."""
    if layout == ROW_MAJOR:
        return z2 * o1 + o2
    if layout == SW128:
        assert z2 * 2 == 128, "SW128 layout needs Z2 * 2 B = 128 B (R4)"
        return z2 * o1 + 8 * ((o2 >> 3) ^ (o1 & 7)) + (o2 & 7)       # R4
    raise ValueError(layout)


def bf16_round(a) -> np.ndarray:
    """fp32 -> bf16 round-to-nearest-even, as fp64 values (plain PyTorch CPU cast)."""
    t = torch.as_tensor(np.asarray(a, dtype=np.float32))
    return t.to(torch.bfloat16).to(torch.float64).numpy()


class LinearSpec:
    """One registered ROAST linear: its tile map (offsets, signs) and lambda.

    seed/module select the module's independent hash functions (R8);
    fan_in is H (R7); lambda = fp32(C / sqrt(H)).
    """

    def __init__(self, H, O, z1, z2, mem_size, seed, module, align=8, C=1.0,
                 mapping=HASH, use_sign=True, layout=ROW_MAJOR, base=0, lam=None, segment=None):
        self.H, self.O, self.z1, self.z2 = H, O, z1, z2
        self.mem_size = mem_size
        self.layout = layout
        self.nx = -(-H // z1)
        self.ny = -(-O // z2)
        T = z1 * z2
        self.off = np.zeros((self.nx, self.ny), dtype=np.int64)
        self.sgn = np.ones((self.nx, self.ny), dtype=np.int64)
        if mapping == HASH:
            # segment = (base, size): LMS memory M_i of this module; None = GMS
            seg_base, seg_size = segment if segment is not None else (0, mem_size)
            assert 0 <= seg_base and seg_base + seg_size <= mem_size
            mh = hashing.ModuleHash(seed, module, seg_size, T, align, use_sign, base=seg_base)
            for x in range(self.nx):
                for y in range(self.ny):
                    k = hashing.tile_key(x, y)
                    self.off[x, y] = mh.offset(k)
                    self.sgn[x, y] = mh.sign(k)
            self.lam = hashing.lam(C, H) if lam is None else lam
        elif mapping == IDENTITY:                                    # R22
            for x in range(self.nx):
                for y in range(self.ny):
                    self.off[x, y] = base + T * (x * self.ny + y)
            assert base + T * self.nx * self.ny <= mem_size, "identity needs |M| >= n"
            self.lam = 1.0 if lam is None else lam
        else:
            raise ValueError(mapping)

    # -- the mapping, element by element ------------------------------------
    def slot_index(self) -> np.ndarray:
        """slot[i, j] = h2(C1, C2) + pi(O1, O2) for every weight (i, j)."""
        i = np.arange(self.H, dtype=np.int64)[:, None]
        j = np.arange(self.O, dtype=np.int64)[None, :]
        x, o1 = i // self.z1, i % self.z1          # C1(i,j), O1(i,j)
        y, o2 = j // self.z2, j % self.z2          # C2(i,j), O2(i,j)
        return self.off[x, y] + pi(o1, o2, self.z2, self.layout)

    def sign_matrix(self) -> np.ndarray:
        """g(C1(i,j), C2(i,j)) for every weight."""
        return np.repeat(np.repeat(self.sgn, self.z1, 0), self.z2, 1)[:self.H, :self.O]

    def materialize(self, M, kind: str = "exact") -> np.ndarray:
        """Recovered W (H x O), fp64.

        kind="exact":   g * lambda * M, exact real value (lambda32 * M32 fits fp64 exactly)
        kind="fp32":    g * fp32_RNE(lambda32 * M32)   -- bit-exact fp32 definition (§8(c) step 4)
        kind="operand": g * bf16_RNE(M32)               -- bf16 tensor-core operand, lambda deferred
        """
        M = np.asarray(M)
        slot = self.slot_index()
        g = self.sign_matrix().astype(np.float64)
        m = M.astype(np.float64)[slot]
        if kind == "exact":
            return g * (np.float64(self.lam) * m)
        if kind == "fp32":
            return g * (np.float64(self.lam) * m).astype(np.float32).astype(np.float64)
        if kind == "operand":
            return g * bf16_round(M.astype(np.float32))[slot]
        raise ValueError(kind)

    # -- the passes -----------------------------------------------------------
    def _weights(self, M, bf16_operand: bool) -> np.ndarray:
        if bf16_operand:      # bf16 path (R18): operand g * bf16(M), lambda once per output
            return np.float64(self.lam) * self.materialize(M, "operand")
        return self.materialize(M)

    def forward(self, X, M, bf16_operand: bool = False) -> np.ndarray:
        """Y = X W  (Algorithm 1)."""
        return np.asarray(X, dtype=np.float64) @ self._weights(M, bf16_operand)

    def backward_dx(self, dY, M, bf16_operand: bool = False) -> np.ndarray:
        """dX = dY W^T."""
        return np.asarray(dY, dtype=np.float64) @ self._weights(M, bf16_operand).T

    def grad_weights(self, X, dY) -> np.ndarray:
        """G = X^T dY, the gradient w.r.t. the virtual weights theta (H x O)."""
        return np.asarray(X, dtype=np.float64).T @ np.asarray(dY, dtype=np.float64)

    def scatter(self, G, dM: np.ndarray) -> np.ndarray:
        """dM[slot(i,j)] += lambda * g * G[i, j] in (i, j) order (R12)."""
        contrib = np.float64(self.lam) * self.sign_matrix() * G
        np.add.at(dM, self.slot_index().ravel(), contrib.ravel())
        return dM

    def backward_dm(self, X, dY, dM=None) -> np.ndarray:
        if dM is None:
            dM = np.zeros(self.mem_size, dtype=np.float64)
        return self.scatter(self.grad_weights(X, dY), dM)

    # -- per-slot form for sampled parity at full size --------------------------
    def grad_slot(self, X, dY, s: int) -> float:
        """dM[s] for this module alone, computed one slot at a time.

        Enumerates every tile whose block [off, off + Z1 Z2) covers s, recovers
        the (i, j) it maps to, and sums lambda * g * <X[:, i], dY[:, j]>.
        """
        X = np.asarray(X, dtype=np.float64)
        dY = np.asarray(dY, dtype=np.float64)
        T = self.z1 * self.z2
        inv = {}
        for o1 in range(self.z1):
            for o2 in range(self.z2):
                inv[pi(o1, o2, self.z2, self.layout)] = (o1, o2)
        total = 0.0
        for x in range(self.nx):
            for y in range(self.ny):
                e = s - int(self.off[x, y])
                if 0 <= e < T:
                    o1, o2 = inv[e]
                    i, j = x * self.z1 + o1, y * self.z2 + o2
                    if i < self.H and j < self.O:
                        total += self.lam * self.sgn[x, y] * float(X[:, i] @ dY[:, j])
        return total
