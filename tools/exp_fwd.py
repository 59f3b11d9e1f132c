"""Micro-experiments on the tcgen05 forward kernel (timing only, ROAST_EXP knobs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def main():
    T = 8192
    M = torch.rand(47192, device="cuda") * 2 - 1
    ctx = R.Roast(M, 64, 64)
    l1 = ctx.linear(768, 3072)
    l2 = ctx.linear(3072, 768)
    X = torch.randn(T, 768, device="cuda").bfloat16()
    H = torch.randn(T, 3072, device="cuda").bfloat16()
    Y1 = torch.empty(T, 3072, device="cuda", dtype=torch.bfloat16)
    Y2 = torch.empty(T, 768, device="cuda", dtype=torch.bfloat16)
    dense = torch.randn(768, 3072, device="cuda").bfloat16()
    for exp in [0]:
        os.environ["ROAST_EXP"] = str(exp)
        res = []
        for name, fn in [("L1", lambda: ctx.fwd(l1, X, Y1)), ("L2", lambda: ctx.fwd(l2, H, Y2))]:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                fn()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / 20 * 1e3
            res.append(f"{name} {us:7.1f} us {2*T*768*3072/us/1e6:7.1f} TF")
        print(f"exp={exp}: " + " | ".join(res), flush=True)
    os.environ.pop("ROAST_EXP")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        X @ dense
    a.record()
    for _ in range(20):
        X @ dense
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    print(f"cuBLAS X@W (8192x768x3072): {us:.1f} us {2*T*768*3072/us/1e6:.1f} TF")


if __name__ == "__main__":
    main()
