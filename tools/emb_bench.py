"""C4 (BASELINE.json configs[3]): DLRM-shaped ROAST block embeddings on one B200.

26 tables x 10^7 virtual rows x dim 128, chunk Z = 32, 1000x compression
(|M| = 33 280 000 fp32 = 133 MB, HBM-resident), 65 536 samples x 26 tables,
single-hot.  Reports achieved GB/s against the HBM roofline with the
algorithmic bytes per lookup: fwd 8 + 512 + 512 = 1032 B,
bwd 8 + 512 + 1024 (read-modify-write of M's gradient) = 1544 B.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_10702_b200 import roast as R  # noqa: E402



def _hbm_gbs():
    """HBM roofline: MEASURED_PEAKS.json when present (driver-written), else the measured copy
    bandwidth of this pool recorded in SURVEY.md §8(d) (6558.1 GB/s)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import bench
        _, _, hbm, src = bench.load_peaks()
        return hbm if src == "measured" else 6558.1
    except Exception:
        return 6558.1


HBM_GBS = _hbm_gbs()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--dist", default="uniform", choices=["uniform", "zipf"])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--align", type=int, default=32, help="offset alignment A in elements (32 = 128-B lines)")
    ap.add_argument("--deterministic", action="store_true", help="fixed-order dM (sort-based backward)")
    ap.add_argument("--nvtx", action="store_true", help="one eager fused fwd + bwd in NVTX range 'emb_step' (ncu)")
    args = ap.parse_args()
    tables, rows, dim, Z = 26, 10 ** 7, 128, 32
    batch = 8192 if args.quick else 65536
    mem = synth.compressed_size(tables * rows * dim, 1000, align=args.align)
    M = torch.tensor(synth.uniform(synth.SEED_M, (mem,)).astype(np.float32), device="cuda")
    ctx = R.Roast(M, 64, 64, seed=synth.HASH_SEED, align=args.align, deterministic=args.deterministic)
    ids = [ctx.embedding(rows, dim, Z) for _ in range(tables)]
    gen = synth.uniform_indices if args.dist == "uniform" else synth.zipf_indices
    idx = [torch.tensor(gen(synth.SEED_IDX + t, batch, rows), device="cuda") for t in range(tables)]
    out = [torch.empty(batch, dim, device="cuda") for _ in range(tables)]
    dout = torch.randn(batch, dim, device="cuda")

    def fwd():
        for t in range(tables):
            ctx.emb_fwd(ids[t], idx[t], out[t])

    def bwd():
        for t in range(tables):
            ctx.emb_bwd(ids[t], idx[t], dout)

    idx_all = torch.cat(idx)                       # table-major 26 x batch
    out_all = torch.empty(tables * batch, dim, device="cuda")
    dout_all = dout.repeat(tables, 1)

    def fwd_multi():                               # all 26 tables in one launch
        ctx.emb_fwd_multi(ids, idx_all, out_all)

    def bwd_multi():
        ctx.emb_bwd_multi(ids, idx_all, dout_all)

    res = {}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    if args.nvtx:
        fwd_multi()
        bwd_multi()
        flush.zero_()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("emb_step")
        fwd_multi()
        bwd_multi()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    for name, fn, bpl in [("fwd", fwd, 1032), ("bwd", bwd, 1544), ("fwd_multi", fwd_multi, 1032),
                          ("bwd_multi", bwd_multi, 1544)]:
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        times = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = float(np.median(times))
        gbs = tables * batch * bpl / (ms * 1e-3) / 1e9
        res[name] = dict(ms=ms, GBps=gbs, hbm_frac=gbs / HBM_GBS, lookups=tables * batch)
    ctx.check()
    # library baseline: torch gather / index_add_ of the same 128-B chunks at the same offsets
    # (precomputed, no hashing) -> what the raw access pattern costs on this GPU
    if args.align * 4 == 128:
        offs = torch.cat([ctx.chunk_map(ids[t], idx[t])[0].reshape(-1) for t in range(tables)]) // 32
        Mv = M.view(-1, 32)
        dflat = dout.reshape(-1, 32).repeat(tables, 1)
        g = torch.empty(offs.numel(), 32, device="cuda")
        for name, fn in [("torch_gather", lambda: torch.index_select(Mv, 0, offs, out=g)),
                         ("torch_index_add", lambda: Mv.index_add_(0, offs, dflat))]:
            for _ in range(3):
                fn()
            times = []
            for _ in range(args.steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            ms = float(np.median(times))
            bpl = 1032 if name == "torch_gather" else 1544
            res[name] = dict(ms=ms, GBps=tables * batch * bpl / (ms * 1e-3) / 1e9)
    print(json.dumps(dict(config="C4 26x1e7x128 chunk 32 1000x", dist=args.dist, batch=batch, align=args.align,
                          deterministic=args.deterministic,
                          **res)))


if __name__ == "__main__":
    main()
