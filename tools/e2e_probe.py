"""Why does bench.py's e2e H2D run below the link rate?  H2D of the step's two 12.6 MB inputs,
(a) back to back, (b) each followed by a ~0.2 ms GEMM on the same stream (serial pattern),
(c) on a copy stream while GEMMs run (pipelined pattern)."""
import json
import torch

n = 8192 * 768
Xh = torch.randn(n, dtype=torch.bfloat16).pin_memory()
Yh = torch.randn(n, dtype=torch.bfloat16).pin_memory()
X = torch.empty(n, dtype=torch.bfloat16, device="cuda")
Y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
A = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
cs = torch.cuda.Stream()
res = {}


def timed(fn, it=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def copies():
    X.copy_(Xh, non_blocking=True)
    Y.copy_(Yh, non_blocking=True)


def serial():
    copies()
    A @ A


def pipelined():
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        copies()
    A @ A
    torch.cuda.current_stream().wait_stream(cs)


Xd = torch.randn(8192, 768, dtype=torch.bfloat16, device="cuda")
Xh2 = Xd.cpu().pin_memory()             # bench.py's way of staging its inputs
Xh3 = torch.empty(Xd.shape, dtype=Xd.dtype, pin_memory=True)
Xh3.copy_(Xd)
Xd2 = torch.empty_like(Xd)
for name, src in [("cpu_then_pin_memory", Xh2), ("empty_pinned_then_copy", Xh3)]:
    ms = timed(lambda: Xd2.copy_(src, non_blocking=True))
    res[name + "_GBps"] = n * 2 / (ms * 1e-3) / 1e9
for rep in range(2):
    ms = timed(copies)
    res[f"copies_GBps_{rep}"] = 2 * n * 2 / (ms * 1e-3) / 1e9
    res[f"gemm_ms_{rep}"] = timed(lambda: A @ A)
    res[f"serial_ms_{rep}"] = timed(serial)
    res[f"pipelined_ms_{rep}"] = timed(pipelined)
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
