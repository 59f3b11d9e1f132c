"""B200 analogue of the paper's `tab:fwd` / `tab:total-*`: square D x D
weights, batch 512, |M| = 4 MB fp32 (1 048 576 elements): ROAST-MM (tcgen05, 64x64 tiles),
HashedNet (per-element hashing = 1x1 tiles, A = 1, SIMT gather path) and dense
cuBLAS, forward and forward+backward times.  bf16 on B200 vs the paper's TF32 on A100:
context only, not the same hardware or precision.

    python tools/tabfwd_bench.py [--dims 512,1024,2048,4096,8192] [--hashednet-max 4096]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="512,1024,2048,4096,8192,10240,20480")
    ap.add_argument("--hashednet-max", type=int, default=4096)
    ap.add_argument("--mem", type=int, default=1 << 20)
    ap.add_argument("--batch", type=int, default=512)
    args = ap.parse_args()
    rows = []
    bf = torch.bfloat16
    for D in [int(x) for x in args.dims.split(",")]:
        T = args.batch
        X = torch.randn(T, D, device="cuda").to(bf)
        dY = torch.randn(T, D, device="cuda").to(bf)
        res = dict(dim=D, batch=T, mem_fp32_MB=args.mem * 4 / 2 ** 20)
        M = torch.rand(args.mem, device="cuda") * 2 - 1
        ro = R.Roast(M, 64, 64)
        l = ro.linear(D, D)
        Y = torch.empty(T, D, device="cuda", dtype=bf)
        dX = torch.empty_like(X)
        res["roast_fwd_ms"] = timeit(lambda: ro.fwd(l, X, Y))
        res["roast_fwdbwd_ms"] = timeit(lambda: (ro.fwd(l, X, Y), ro.bwd(l, X, dY, dX)))
        W = ro.materialize(l, bf)
        res["dense_fwd_ms"] = timeit(lambda: X @ W)
        res["dense_fwdbwd_ms"] = timeit(lambda: (X @ W, dY @ W.t(), X.t() @ dY))
        ro.close()
        if D <= args.hashednet_max:
            hn = R.Roast(M, 1, 1, align=1, simt_bf16=True)
            lh = hn.linear(D, D)
            res["hashednet_fwd_ms"] = timeit(lambda: hn.fwd(lh, X, Y), iters=3)
            res["hashednet_fwdbwd_ms"] = timeit(lambda: (hn.fwd(lh, X, Y), hn.bwd(lh, X, dY, dX)), iters=3)
            res["roast_vs_hashednet_fwd"] = res["hashednet_fwd_ms"] / res["roast_fwd_ms"]
            hn.close()
        res["roast_vs_dense_fwd"] = res["dense_fwd_ms"] / res["roast_fwd_ms"]
        res["roast_vs_dense_fwdbwd"] = res["dense_fwdbwd_ms"] / res["roast_fwdbwd_ms"]
        print(json.dumps(res), flush=True)
        rows.append(res)


if __name__ == "__main__":
    main()
