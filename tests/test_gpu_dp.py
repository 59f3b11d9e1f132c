"""The data-parallel C2 step through libroast in two processes (split the tokens,
replicate M, sum dM over the ranks, identical update everywhere; P:194 + P:440).

One GPU stands in for two: each process runs the MLP block (768 -> 3072 -> 768, 100x) on its
half of the tokens with the product path — the chained forward and the fused backward
(roast_linear_fwd_chain / roast_linear_bwd_chain) — then the fused exchange + SGD step
(Roast.exchange_init: NVLS where the driver allows it, else the CUDA-IPC two-shot), twice.
Checked against the fp64 oracle on the WHOLE batch: after each step both ranks hold the same M
bit for bit, and the update M_new - M_old equals -lr * dM_full (dM of the full batch, the
oracle's own dY_a chain) at the bf16 tolerance."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import synth
from oracle import roast_mm as OM
from tests.gpu_helpers import bf16_input, rel_frob, store

pytestmark = pytest.mark.gpu
HS = synth.HASH_SEED
T, LR, RATIO = 1024, 1e-2, 100

_WORKER = textwrap.dedent("""
    import os, sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.getcwd())
    import synth
    from paper_2207_10702_b200 import roast as R
    rank, world, out, port = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + port, rank=rank, world_size=world)
    d = np.load(out + "_in.npz")
    T = d["X"].shape[0]
    lo, hi = rank * T // world, (rank + 1) * T // world          # this rank's shard of the tokens
    ctx = R.Roast(torch.tensor(d["M"], device="cuda"), 64, 64, seed=synth.HASH_SEED)
    a, b = ctx.linear(768, 3072), ctx.linear(3072, 768)
    path = ctx.exchange_init()
    bf = torch.bfloat16
    for t in (1, 2):
        X = torch.tensor(d["X%d" % t][lo:hi], device="cuda").to(bf)
        dY = torch.tensor(d["dY%d" % t][lo:hi], device="cuda").to(bf)
        Y1 = torch.empty(hi - lo, 3072, device="cuda", dtype=bf)
        Y2 = torch.empty(hi - lo, 768, device="cuda", dtype=bf)
        ctx.zero_grad()
        ctx.fwd_chain(a, b, X, Y1, Y2)
        ctx.bwd_chain(a, b, X, Y1, dY)
        np.save(out + "_Y1_%d_%d.npy" % (t, rank), Y1.float().cpu().numpy())
        ctx.exchange_fused(R.OPT_SGD, float(sys.argv[5]), step=t)
        torch.cuda.synchronize()
        np.save(out + "_M%d_%d.npy" % (t, rank), ctx.M.cpu().numpy())
    with open(out + "_path_%d.txt" % rank, "w") as f:
        f.write(path)
    ctx.check()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
""")


def test_data_parallel_step_two_processes_equals_full_batch(tmp_path):
    cfg = synth.mlp_block(RATIO, tokens=T)
    mem = cfg["mem_size"]
    M0 = store(mem)
    ins = {"M": M0}
    for t in (1, 2):
        ins["X%d" % t] = bf16_input(synth.SEED_X + 100 * t, (T, 768))
        ins["dY%d" % t] = bf16_input(synth.SEED_DY + 100 * t, (T, 768))
    ins["X"] = ins["X1"]
    out = str(tmp_path / "dp")
    np.savez(out + "_in.npz", **ins)
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    port = str(27500 + os.getpid() % 1000)
    env = dict(os.environ, PYTHONPATH=os.getcwd())
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2", out, port, str(LR)], cwd=os.getcwd(),
                              env=env) for r in range(2)]
    assert [p.wait(timeout=600) for p in procs] == [0, 0]
    paths = [open(out + "_path_%d.txt" % r).read() for r in range(2)]
    assert paths[0] == paths[1] and paths[0] in ("nvls", "p2p")
    sa = OM.LinearSpec(768, 3072, 64, 64, mem, HS, 0)
    sb = OM.LinearSpec(3072, 768, 64, 64, mem, HS, 1)
    M_prev = M0.astype(np.float64)
    for t in (1, 2):
        Ms = [np.load(out + "_M%d_%d.npy" % (t, r)) for r in range(2)]
        assert np.array_equal(Ms[0], Ms[1])                 # replicated bit for bit
        # the full batch's gradient: Y1 as the ranks computed it (bf16, checked against the
        # oracle forward below), dY_a from the oracle's own fp64 chain
        Y1 = np.concatenate([np.load(out + "_Y1_%d_%d.npy" % (t, r)) for r in range(2)])
        Mp32 = M_prev.astype(np.float32)
        X, dY = ins["X%d" % t], ins["dY%d" % t]
        assert rel_frob(Y1, sa.forward(X, Mp32, True)) <= 1e-2
        dYa = sb.backward_dx(dY, Mp32, True)
        dM = sb.backward_dm(Y1, dY) + sa.backward_dm(X, dYa)
        step = Ms[0].astype(np.float64) - M_prev
        assert rel_frob(step, -LR * dM) <= 1e-2, rel_frob(step, -LR * dM)
        M_prev = Ms[0].astype(np.float64)
