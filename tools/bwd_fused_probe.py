"""Time roast_linear_bwd_chain (one fused launch for the MLP block's backward) against the
separate launches (two streams, as bench.py's step), graph-replayed with L2 flushed."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
MEM = int(sys.argv[2]) if len(sys.argv) > 2 else 47192   # |M|: 471864 / 47192 / 4720 = 10x / 100x / 1000x
M = torch.rand(MEM, device="cuda") * 2 - 1
ctx = R.Roast(M, 64, 64)
ctx.set_autotune(2)
a, b = ctx.linear(768, 3072), ctx.linear(3072, 768)
bf = torch.bfloat16
X = torch.randn(T, 768, device="cuda").to(bf)
Ya = torch.randn(T, 3072, device="cuda").to(bf)
dYb = torch.randn(T, 768, device="cuda").to(bf)
dYa = torch.empty(T, 3072, device="cuda", dtype=bf)
dXa = torch.empty(T, 768, device="cuda", dtype=bf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()


def sep():
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    ctx.bwd_dx(b, dYb, dYa)
    e = torch.cuda.Event()
    e.record(cur)
    with torch.cuda.stream(side):
        ctx.bwd_dm(b, Ya, dYb)
    ctx.bwd_dx(a, dYa, dXa)
    side.wait_event(e)
    with torch.cuda.stream(side):
        ctx.bwd_dm(a, X, dYa)
    cur.wait_stream(side)


def fused():
    ctx.bwd_chain(a, b, X, Ya, dYb, dYa, dXa)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


# tune the single kernels first (eager), then plan the fused one
sep()
torch.cuda.synchronize()
ctx.zero_grad()
fused()
torch.cuda.synchronize()
ref_dYa, ref_dXa = dYa.clone(), dXa.clone()
ctx.zero_grad(); sep(); torch.cuda.synchronize(); dM_sep = ctx.dM.clone()
ctx.zero_grad(); fused(); torch.cuda.synchronize(); dM_f = ctx.dM.clone()
err = float((dM_f - dM_sep).norm() / dM_sep.norm())
ctx.check()
flop = 4 * 2.0 * T * 768 * 3072
t_sep, t_f = timeit(sep), timeit(fused)
print(json.dumps(dict(T=T, sep_us=t_sep, fused_us=t_f, sep_tflops=flop / t_sep / 1e6, fused_tflops=flop / t_f / 1e6,
                      dM_rel_diff=err)))
