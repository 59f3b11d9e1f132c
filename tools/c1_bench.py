"""C1 (BASELINE.json configs[0]): one ROAST linear 256 x 256, batch 64, tile
32 x 32, |M| = 8192 fp32 (8x), fwd + bwd on the fp32 SIMT path — a correctness config
(latency-bound, 25.2 MFLOP per fwd+bwd; no roofline claim).  Reports the GPU time per
fwd + bwd (atomic and deterministic dM; CUDA-graph replays) next to the oracle (fp64 numpy)
on 1 host thread and on all of them, plus the parity of this very run.

    python tools/c1_bench.py > profiles/round1/c1.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import roast_mm as OM  # noqa: E402
from paper_2207_10702_b200 import roast as R  # noqa: E402

H = O = 256
T, Z, MEM = 64, 32, 8192


def gpu_us(deterministic):
    M_np = synth.uniform(synth.SEED_M, (MEM,)).astype(np.float32)
    ctx = R.Roast(torch.tensor(M_np, device="cuda"), Z, Z, seed=synth.HASH_SEED, deterministic=deterministic,
                  simt_bf16=True)   # C1 (32 x 32 tiles) is the SIMT path by construction
    mid = ctx.linear(H, O)
    X_np = synth.uniform(synth.SEED_X, (T, H)).astype(np.float32)
    dY_np = synth.uniform(synth.SEED_DY, (T, O)).astype(np.float32)
    X, dY = torch.tensor(X_np, device="cuda"), torch.tensor(dY_np, device="cuda")
    Y = torch.empty(T, O, device="cuda")
    dX = torch.empty(T, H, device="cuda")

    def step():
        ctx.zero_grad()
        ctx.fwd(mid, X, Y)
        ctx.bwd(mid, X, dY, dX)
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(10):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    spec = OM.LinearSpec(H, O, Z, Z, MEM, synth.HASH_SEED, mid)
    err = dict(Y=float(np.linalg.norm(Y.cpu().numpy() - spec.forward(X_np, M_np)) / np.linalg.norm(spec.forward(X_np, M_np))),
               dX=float(np.linalg.norm(dX.cpu().numpy() - spec.backward_dx(dY_np, M_np)) /
                        np.linalg.norm(spec.backward_dx(dY_np, M_np))),
               dM=float(np.linalg.norm(ctx.dM.cpu().numpy() - spec.backward_dm(X_np, dY_np)) /
                        np.linalg.norm(spec.backward_dm(X_np, dY_np))))
    launches = ctx.launch_count()
    ctx.close()
    return us, err, launches


def oracle_us(threads):
    from threadpoolctl import threadpool_limits
    M_np = synth.uniform(synth.SEED_M, (MEM,)).astype(np.float32)
    spec = OM.LinearSpec(H, O, Z, Z, MEM, synth.HASH_SEED, 0)
    X_np = synth.uniform(synth.SEED_X, (T, H))
    dY_np = synth.uniform(synth.SEED_DY, (T, O))
    with threadpool_limits(limits=threads):
        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 3.0:
            spec.forward(X_np, M_np)
            spec.backward_dx(dY_np, M_np)
            spec.backward_dm(X_np, dY_np)
            n += 1
        return (time.perf_counter() - t0) / n * 1e6


def main():
    flop = 6.0 * T * H * O
    res = dict(config="C1 256x256 ROAST linear, batch 64, tile 32x32, |M| = 8192 fp32 (8x), fp32 SIMT path",
               flop_per_fwd_bwd=flop)
    for det in (False, True):
        us, err, launches = gpu_us(det)
        res["gpu_deterministic" if det else "gpu_atomic"] = dict(us_per_fwd_bwd=round(us, 2),
                                                                 gflops=round(flop / us / 1e3, 2),
                                                                 rel_err_vs_oracle=err, tol=1e-5)
    res["oracle_1_thread_us"] = round(oracle_us(1), 1)
    res["oracle_all_threads_us"] = round(oracle_us(os.cpu_count()), 1)
    res["host_threads"] = os.cpu_count()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
