"""C3's LayerNorm (65 536 x 768 bf16 activations): fwd + bwd time with bf16 vs fp32 parameters
(N-op of the BERT workload, outside the ROAST path)."""
import torch

N, D = 65536, 768
x = torch.randn(N, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
dy = torch.randn(N, D, device="cuda", dtype=torch.bfloat16)


def run(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for pdt in (torch.bfloat16, torch.float32):
    ln = torch.nn.LayerNorm(D, device="cuda", dtype=pdt)
    try:
        def f():
            y = ln(x)
            y.backward(dy)
        print("params", pdt, round(run(f), 3), "ms fwd+bwd", ln(x).dtype)
    except Exception as e:  # noqa: BLE001
        print("params", pdt, "error", repr(e)[:100])
ln = torch.nn.LayerNorm(D, device="cuda", dtype=torch.bfloat16, elementwise_affine=False)
def g():
    y = ln(x)
    y.backward(dy)
print("no affine", round(run(g), 3))

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import nn as RN  # noqa: E402
mine = RN.LayerNorm(D, device="cuda", dtype=torch.bfloat16)
r = torch.randn(N, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
def h():
    y = mine(x)
    y.backward(dy)
def h2():
    y = mine(x, r)
    y.backward(dy)
print("libroast LayerNorm", round(run(h), 3), "ms fwd+bwd; with the residual fused", round(run(h2), 3))
