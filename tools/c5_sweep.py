"""C5 (BASELINE.json configs[4]): the |M| sweep of a 4096 x 4096 ROAST-MM at
batch 16384 per GPU, |M| from L2-resident (8 MB fp32) to HBM-resident (2 GB), on one B200.

Per |M| it reports, all CUDA-event timed (each call captured in a CUDA graph, median of
replays; the 134 MB activations exceed the 126 MB L2, so no flush is needed):
  * ROAST fwd, dX, dM and the fwd + bwd sequence (effective TFLOP/s = 6 T H O / t);
  * dense cuBLAS fwd + bwd on the same virtual shape (materialised bf16 W);
  * the O(|M|) passes the paper's optimizer tables time: bf16 shadow refresh,
    fused Adam step (+ shadow + dM zero; 36 B per slot of HBM traffic) over all of M and over
    the touched set only, dM zeroing;
  * the exchange (a6 at W ranks): dense all-reduce bytes 4 |M| vs the touched-set exchange
    (4 n_touched) and the pack + unpack time it adds.

    python tools/c5_sweep.py [--mems 2,8,32,128,512] [--T 16384] > profiles/round1/c5_sweep.jsonl
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def graph_time_us(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mems", default="2,8,32,128,512", help="|M| in mega-elements (fp32: x4 MB)")
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--D", type=int, default=4096)
    args = ap.parse_args()
    T, D = args.T, args.D
    bf = torch.bfloat16
    gen = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(T, D, device="cuda", generator=gen).to(bf)
    dY = torch.randn(T, D, device="cuda", generator=gen).to(bf)
    Y = torch.empty(T, D, device="cuda", dtype=bf)
    dX = torch.empty(T, D, device="cuda", dtype=bf)
    flop = 6.0 * T * D * D
    side = torch.cuda.Stream()
    dense_us = None
    for mm in [int(v) for v in args.mems.split(",")]:
        mem = mm << 20
        M = torch.rand(mem, device="cuda", generator=gen) * 2 - 1
        ctx = R.Roast(M, 64, 64)
        ctx.set_autotune(2)
        lid = ctx.linear(D, D)
        ctx.fwd(lid, X, Y)                                   # tune outside capture
        ctx.bwd_dx(lid, dY, dX)
        ctx.bwd_dm(lid, X, dY)
        torch.cuda.synchronize()

        def step():
            ctx.fwd(lid, X, Y)
            side.wait_stream(torch.cuda.current_stream())
            ctx.bwd_dx(lid, dY, dX)
            with torch.cuda.stream(side):
                ctx.bwd_dm(lid, X, dY, stream=side)
            torch.cuda.current_stream().wait_stream(side)

        t_fwd = graph_time_us(lambda: ctx.fwd(lid, X, Y))
        t_dx = graph_time_us(lambda: ctx.bwd_dx(lid, dY, dX))
        t_dm = graph_time_us(lambda: ctx.bwd_dm(lid, X, dY))
        t_step = graph_time_us(step)
        if dense_us is None:
            W = ctx.materialize(lid, bf)

            def dense():
                torch.matmul(X, W, out=Y)
                torch.matmul(dY, W.t(), out=dX)
                torch.matmul(X.t(), dY)
            dense_us = graph_time_us(dense)
            del W
        t_shadow = graph_time_us(ctx.sync_shadow)
        ctx.optimizer_step(R.OPT_ADAM, 1e-3, step=1)
        t_adam = graph_time_us(lambda: ctx.optimizer_step(R.OPT_ADAM, 1e-3, step=1))
        t_zero = graph_time_us(ctx.zero_grad)
        n_touched, n_iv = ctx.touched_size()
        t_adam_t = graph_time_us(lambda: ctx.optimizer_step(R.OPT_ADAM, 1e-3, step=1, touched_only=True))
        t_pack = graph_time_us(lambda: R.roast_debug_exchange(ctx.h, 1.0, torch.cuda.current_stream().cuda_stream))
        line = dict(config="C5 4096x4096 ROAST-MM, batch 16384, 1 B200", mem_elems=mem, mem_mb_fp32=mem * 4 / 2 ** 20,
                    compression=round(D * D / mem, 3), us=dict(fwd=round(t_fwd, 1), dx=round(t_dx, 1),
                                                               dm=round(t_dm, 1), fwd_bwd=round(t_step, 1)),
                    tflops=round(flop / t_step / 1e6, 1), dense_fwd_bwd_us=round(dense_us, 1),
                    dense_tflops=round(flop / dense_us / 1e6, 1), roast_over_dense=round(dense_us / t_step, 3),
                    tuned={k: ctx.tuned(lid, j, T) for j, k in enumerate(("fwd", "dx", "dm"))},
                    o_m_passes_us=dict(sync_shadow=round(t_shadow, 1), adam_step=round(t_adam, 1),
                                       adam_step_touched_only=round(t_adam_t, 1), zero_grad=round(t_zero, 1),
                                       adam_hbm_gbs=round(36.0 * mem / t_adam / 1e3, 1)),
                    exchange=dict(dense_bytes=mem * 4, touched_elems=n_touched, touched_intervals=n_iv,
                                  touched_bytes=n_touched * 4, reduction=round(mem / max(n_touched, 1), 2),
                                  pack_unpack_us=round(t_pack, 1),
                                  ring_bytes_per_rank_w8=dict(dense=int(2 * 7 / 8 * 4 * mem),
                                                              touched=int(2 * 7 / 8 * 4 * n_touched))))
        print(json.dumps(line), flush=True)
        ctx.close()
        del M, ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
