"""LayerNorm kernels (K11, N-op of the C3 workload) timed alone through the C ABI: forward with the
residual fused and backward (+ its parameter reduce), at C3's 65 536 x 768 and the 8192-token shard.
Prints one JSON line per (rows, direction): us per call and the algorithmic HBM GB/s (fwd reads x, r
and writes s, y; bwd reads dy, s and writes ds; bf16), with the HBM fraction of MEASURED_PEAKS."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402

D = 768
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    pass


def timed(fn, reps=50):
    """device time per call (CUDA events around `reps` back-to-back calls) and the host time per
    call (if the two agree, the loop was launch-bound, not kernel-bound)"""
    import time
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3, (t1 - t0) / reps * 1e6


for rows in (65536, 8192):
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(rows, D, device="cuda", generator=g).to(torch.bfloat16)
    r = torch.randn(rows, D, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(rows, D, device="cuda", generator=g).to(torch.bfloat16)
    gam = (1 + 0.1 * torch.randn(D, device="cuda", generator=g)).to(torch.bfloat16)
    bet = (0.1 * torch.randn(D, device="cuda", generator=g)).to(torch.bfloat16)
    y, s, ds = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    dg = torch.empty(D, device="cuda")
    db = torch.empty(D, device="cuda")
    strm = torch.cuda.current_stream().cuda_stream

    def fwd():
        R.roast_layernorm_fwd(x.data_ptr(), r.data_ptr(), gam.data_ptr(), bet.data_ptr(), y.data_ptr(), s.data_ptr(),
                              mean.data_ptr(), rstd.data_ptr(), rows, D, 1e-12, R.BF16, R.BF16, strm)

    def bwd():
        R.roast_layernorm_bwd(dy.data_ptr(), s.data_ptr(), gam.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                              ds.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, D, R.BF16, R.BF16, strm)

    # correctness against torch on this input (fp32 math)
    fwd()
    bwd()
    sr = (x.float() + r.float()).to(torch.bfloat16).float().requires_grad_(True)
    gr = gam.float().requires_grad_(True)
    br = bet.float().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(sr, (D,), gr, br, 1e-12)
    yr.backward(dy.float())
    err = {"y": float((y.float() - yr).abs().max()), "ds": float((ds.float() - sr.grad).abs().max()),
           "dg": float((dg - gr.grad).abs().max() / gr.grad.abs().max()),
           "db": float((db - br.grad).abs().max() / br.grad.abs().max())}
    for name, fn, nbytes in (("fwd", fwd, 4 * rows * D * 2), ("bwd", bwd, 3 * rows * D * 2)):
        us, host_us = timed(fn)
        gbs = nbytes / us / 1e3
        print(json.dumps({"rows": rows, "dir": name, "us": round(us, 2), "host_us": round(host_us, 1),
                          "GB/s": round(gbs, 1),
                          "hbm_frac": round(gbs / peak, 3) if peak else None, "err": err}), flush=True)

# per-kernel device durations (torch.profiler: CUPTI activity records, not the wall clock), to
# separate the kernels from launch / allocation effects in the loop above
if os.environ.get("LN_PROFILE"):
    from torch.profiler import ProfilerActivity, profile
    for rows in (65536, 8192):
        x = torch.randn(rows, D, device="cuda").to(torch.bfloat16)
        r, dy = torch.randn_like(x), torch.randn_like(x)
        gam, bet = torch.ones(D, device="cuda", dtype=torch.bfloat16), torch.zeros(D, device="cuda", dtype=torch.bfloat16)
        y, s, ds = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
        dg, db = torch.empty(D, device="cuda"), torch.empty(D, device="cuda")
        strm = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            R.roast_layernorm_fwd(x.data_ptr(), r.data_ptr(), gam.data_ptr(), bet.data_ptr(), y.data_ptr(),
                                  s.data_ptr(), mean.data_ptr(), rstd.data_ptr(), rows, D, 1e-12, R.BF16, R.BF16, strm)
            R.roast_layernorm_bwd(dy.data_ptr(), s.data_ptr(), gam.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                  ds.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, D, R.BF16, R.BF16, strm)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(20):
                R.roast_layernorm_fwd(x.data_ptr(), r.data_ptr(), gam.data_ptr(), bet.data_ptr(), y.data_ptr(),
                                      s.data_ptr(), mean.data_ptr(), rstd.data_ptr(), rows, D, 1e-12, R.BF16, R.BF16,
                                      strm)
                R.roast_layernorm_bwd(dy.data_ptr(), s.data_ptr(), gam.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                      ds.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, D, R.BF16, R.BF16, strm)
            torch.cuda.synchronize()
        agg = {}
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA and "ln_" in ev.name:
                k = ev.name.split("<")[0].split("::")[-1].split("(")[0]
                agg.setdefault(k, []).append(ev.device_time)
        print(json.dumps({"rows": rows, "kernel_us": {k: [round(sum(v) / len(v), 2), round(min(v), 2), round(max(v), 2)]
                                                      for k, v in agg.items()}}), flush=True)
