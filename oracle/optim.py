"""Oracle optimizer updates on the compressed array — TEST INFRASTRUCTURE ONLY.

The paper trains ROAST models with PyTorch's SGD / Adagrad / Adam on the compressed
parameters and notes the optimizer cost scales with |M| (`tab:total-opt`
P:749-813); it gives no formulas of its own, so the oracle writes out the standard
(PyTorch) definitions in fp64, element by element:

    g = dM + wd * M
    SGD      M <- M - lr g
    Adagrad  G <- G + g^2;            M <- M - lr g / (sqrt(G) + eps)
    Adam     m <- b1 m + (1 - b1) g;  v <- b2 v + (1 - b2) g^2
             M <- M - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)

Pinned by tests/test_oracle_optim.py: one SGD step on a quadratic reduces to the
closed form; Adam's first step moves every coordinate by lr * sign(g) (bias-corrected
m / sqrt(v) = g / |g|, up to eps); Adagrad's first step likewise by lr * g / (|g| + eps).
The recurrences with carried state (t >= 2) are pinned by hand-derived exact values for
the scalar gradient sequence (1, -2, 3) (Adam with b1 = 1/2, b2 = 3/4; Adagrad), the
Adagrad constant-gradient closed form sum 1/sqrt(s), three SGD steps on a quadratic, and
torch.optim (a second, independent implementation) over five steps with weight decay.
Dropping Adam's b1 m / b2 v decay, not carrying Adagrad's G, or a t >= 2 bias-correction
slip each fails a pin.
"""
from __future__ import annotations

import numpy as np


def step(kind, M, dM, state, lr, t=1, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
    """Return (M_new, state_new).  kind in {"sgd", "adagrad", "adam"}; state is a dict of arrays."""
    M = np.asarray(M, dtype=np.float64)
    g = np.asarray(dM, dtype=np.float64) + wd * M
    st = {k: np.asarray(v, dtype=np.float64).copy() for k, v in state.items()}
    if kind == "sgd":
        return M - lr * g, st
    if kind == "adagrad":
        G = st.get("G", np.zeros_like(M)) + g * g
        st["G"] = G
        return M - lr * g / (np.sqrt(G) + eps), st
    if kind == "adam":
        m = b1 * st.get("m", np.zeros_like(M)) + (1 - b1) * g
        v = b2 * st.get("v", np.zeros_like(M)) + (1 - b2) * g * g
        st["m"], st["v"] = m, v
        mh = m / (1 - b1 ** t)
        vh = v / (1 - b2 ** t)
        return M - lr * mh / (np.sqrt(vh) + eps), st
    raise ValueError(kind)
