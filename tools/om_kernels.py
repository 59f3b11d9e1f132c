"""The O(|M|) kernels of the large-|M| regime (C5, |M| = 512 M fp32 = 2 GB) for an ncu capture:
bf16 shadow refresh (sync_shadow_kernel), fused Adam step over M (opt_kernel<2,4>) and over the
touched set, and the touched-set pack / unpack (pack_kernel) of one 4096 x 4096 linear.
Prints the CUDA-event time and the algorithmic HBM bytes of each (HBM roofline).

    python tools/om_kernels.py
    ncu --set full -k regex:"opt_kernel|pack_kernel|sync_shadow" -c 5 -o gpurun_out/prof_om python tools/om_kernels.py --once
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mem", type=int, default=512, help="|M| in mega-elements")
    ap.add_argument("--once", action="store_true", help="one launch each (under ncu)")
    args = ap.parse_args()
    mem = args.mem << 20
    gen = torch.Generator(device="cuda").manual_seed(1)
    M = torch.rand(mem, device="cuda", generator=gen) * 2 - 1
    ctx = R.Roast(M, 64, 64)
    ctx.linear(4096, 4096)
    n_touched, _ = ctx.touched_size()
    ctx.optimizer_step(R.OPT_ADAM, 1e-3, step=1)   # allocate the state
    s = torch.cuda.current_stream().cuda_stream
    calls = [("sync_shadow", ctx.sync_shadow, 4 * mem + 2 * 2 * mem),
             ("adam_dense", lambda: ctx.optimizer_step(R.OPT_ADAM, 1e-3, step=1), 36 * mem),
             ("adam_touched", lambda: ctx.optimizer_step(R.OPT_ADAM, 1e-3, step=1, touched_only=True), 36 * n_touched),
             ("pack_unpack", lambda: R.roast_debug_exchange(ctx.h, 1.0, s), 2 * 8 * n_touched)]
    out = {}
    for name, f, nbytes in calls:
        f()
        torch.cuda.synchronize()
        if args.once:
            continue
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            f()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 10 * 1e3
        out[name] = dict(us=round(us, 1), algorithmic_bytes=nbytes, gbs=round(nbytes / us / 1e3, 1))
    if not args.once:
        print(json.dumps(dict(config=f"|M| = {args.mem} M fp32, one 4096x4096 linear (touched {n_touched})", **out)))


if __name__ == "__main__":
    main()
