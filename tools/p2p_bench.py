"""Exchange + update on one B200: NCCL path (roast_grad_exchange_step: pack, all-reduce, update)
against the one-shot P2P path (roast_grad_exchange_p2p: pack + signal, sum-of-peers + update) and
the two-shot one (roast_grad_exchange_p2p2: pack + signal, slice reduce + update, gather).

On one GPU the NCCL all-reduce is a 1-rank no-op, so this measures what each path costs around
the communication itself; the P2P path at W virtual ranks (W handles in one process attached by
device pointer) reads W packed buffers from local HBM, the HBM-bound stand-in for reading them
from the peers over NVSwitch.  Configs: C2 at 100x (|M| = 47 192, every slot touched) and C5
at 2 GB (4096 x 4096 layer, 16.8 M touched slots of 512 M).
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


def make(mem, layers, M0):
    ctx = R.Roast(M0.clone(), 64, 64, seed=synth.HASH_SEED)
    for H, O in layers:
        ctx.linear(H, O)
    return ctx


def timed(fn, iters=20):
    """Per-call device time of fn, captured once in a CUDA graph and replayed (the host-side
    launch cost of the Python wrapper would otherwise dominate the small configs)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,8")
    args = ap.parse_args()
    configs = [("C2 100x", synth.mlp_block(100)["mem_size"], [(768, 3072), (3072, 768)]),
               ("C5 2GB", 512 * 1024 * 1024, [(4096, 4096)])]
    for name, mem, layers in configs:
        M0 = torch.tensor(synth.uniform(synth.SEED_M, (mem,)).astype(np.float32), device="cuda")
        for kind, kname in [(0, "sgd"), (2, "adam")]:
            res = dict(config=name, mem=mem, opt=kname)
            ctx = make(mem, layers, M0)
            R.roast_comm_init(ctx.h, 0, 1, R.roast_comm_unique_id())
            n, _ = ctx.touched_size()
            res["touched"] = n
            ctx.dM.normal_()
            res["nccl_exchange_step_us"] = timed(lambda: ctx.exchange_step(kind, 1e-4, step=1, zero_grad=False))
            ctx.close()
            for W in [int(w) for w in args.worlds.split(",")]:
                ranks = [make(mem, layers, M0) for _ in range(W)]
                wins = [c.p2p_window()[0] for c in ranks]
                for r, c in enumerate(ranks):
                    c.p2p_attach(r, wins)
                    c.dM.normal_()

                def post():
                    for c in ranks:
                        c.p2p_post()

                def finish():
                    for c in ranks:
                        c.p2p_finish(kind, 1e-4, step=1, zero_grad=False)

                def both():
                    post()
                    finish()
                t_both = timed(both) / W                     # per rank (W ranks share the GPU)
                # one rank's finish alone: capture post(all) + finish(rank 0), minus post(all)
                t_post = timed(post)

                def post_finish0():
                    post()
                    ranks[0].p2p_finish(kind, 1e-4, step=1, zero_grad=False)
                t_fin = timed(post_finish0) - t_post
                state = {0: 0, 1: 1, 2: 2}[kind]
                # algorithmic bytes of one rank's finish: W packed reads + M, state r/w + shadow write
                byts = n * (4 * W + 8 + 8 * state + 4)
                def two_shot():
                    post()
                    for c in ranks:
                        c.p2p_reduce(kind, 1e-4, step=1)
                    for c in ranks:
                        c.p2p_gather()
                res[f"p2p2_W{W}_us_per_rank"] = timed(two_shot) / W
                res[f"p2p_W{W}_us_per_rank"] = t_both
                res[f"p2p_W{W}_post_us_per_rank"] = t_post / W
                res[f"p2p_W{W}_finish_us"] = t_fin
                res[f"p2p_W{W}_finish_GBps"] = byts / (t_fin * 1e-6) / 1e9
                for c in ranks:
                    c.close()
            print(json.dumps(res), flush=True)
        del M0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
