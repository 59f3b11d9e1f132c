"""One C2 step with ROAST_PROF=1: per-kernel cycle breakdown printed by libroast (debug)."""
import os
import sys

os.environ["ROAST_PROF"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def main():
    T = 8192
    M = torch.rand(47192, device="cuda") * 2 - 1
    ctx = R.Roast(M, 64, 64)
    l1 = ctx.linear(768, 3072)
    l2 = ctx.linear(3072, 768)
    bf = torch.bfloat16
    X = torch.randn(T, 768, device="cuda").to(bf)
    dY2 = torch.randn(T, 768, device="cuda").to(bf)
    Y1 = torch.empty(T, 3072, device="cuda", dtype=bf)
    Y2 = torch.empty(T, 768, device="cuda", dtype=bf)
    dY1 = torch.empty(T, 3072, device="cuda", dtype=bf)
    dX = torch.empty(T, 768, device="cuda", dtype=bf)
    for it in range(2):
        print(f"--- iteration {it}", file=sys.stderr, flush=True)
        ctx.fwd(l1, X, Y1)
        ctx.fwd(l2, Y1, Y2)
        ctx.bwd_dx(l2, dY2, dY1)
        ctx.bwd_dm(l2, Y1, dY2)
        ctx.bwd_dx(l1, dY1, dX)
        ctx.bwd_dm(l1, X, dY1)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
