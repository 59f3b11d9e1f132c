"""Shared helpers for the -m gpu parity tests: build inputs with synth, move them to the GPU."""
import numpy as np

import synth


def rel_frob(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def to_dev(a, dtype):
    import torch
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def bf16_input(seed, shape, dist="normal"):
    """bf16-valued fp32 numpy array (R18: rounded once, both sides consume it)."""
    x = synth.normal(seed, shape) if dist == "normal" else synth.uniform(seed, shape)
    return synth.round_to_bf16(x.astype(np.float32))


def store(mem_size, seed=synth.SEED_M):
    """M ~ U(-1, 1) (C = 1) as fp32."""
    return synth.uniform(seed, (mem_size,)).astype(np.float32)
