"""dM launch time, atomic (TMA reduce-add) vs deterministic (workspace + fixed-order reduce), at
C5 (4096 x 4096, 16384 tokens; |M| 8 MB and 2 GB) and C2 L1 (768 x 3072, 8192 tokens, 100x)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_10702_b200 import roast as R  # noqa: E402


def time_dm(mem, H, O, T, det):
    M = torch.tensor(synth.uniform(synth.SEED_M, (mem,)).astype(np.float32), device="cuda")
    ctx = R.Roast(M, 64, 64, seed=synth.HASH_SEED, deterministic=det)
    mid = ctx.linear(H, O)
    X = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    dY = torch.randn(T, O, device="cuda", dtype=torch.bfloat16)
    ctx.touched_size()
    for _ in range(3):
        ctx.bwd_dm(mid, X, dY)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.bwd_dm(mid, X, dY)
    times = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ctx.close()
    return float(np.median(times))


for name, mem, H, O, T in [("C5 8MB", 2 << 20, 4096, 4096, 16384), ("C5 2GB", 512 << 20, 4096, 4096, 16384),
                           ("C2 L1 100x", synth.mlp_block(100)["mem_size"], 768, 3072, 8192)]:
    print(json.dumps(dict(config=name, atomic_ms=time_dm(mem, H, O, T, False),
                          deterministic_ms=time_dm(mem, H, O, T, True))), flush=True)
