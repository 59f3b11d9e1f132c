"""One-shot P2P exchange fused with the update (include/roast.h roast_p2p_*, p2p.cu;
SURVEY.md §8(f) NEXT #1 = a6 P:194 + a7 P:440 / P:749-813).

One GPU stands in for the node: W "ranks" are W handles in one process whose windows are
attached to each other by device pointer (the kernels cannot tell a peer's HBM from their own),
plus a two-process test that maps the windows through CUDA IPC.  Every rank must end with the
same M, bit for bit, equal to roast_optimizer_step (touched_only) on the fp32 sum of the W
gradients in rank order, and its update within 1e-5 of the fp64 oracle's (tests.gpu_helpers.check_update)."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import synth
from oracle import embedding as OE
from oracle import optim as OO
from oracle import roast_mm as OM
from tests.gpu_helpers import check_update, grad_condition, rel_frob, store, to_dev

pytestmark = pytest.mark.gpu
HS = synth.HASH_SEED
# optimizer hyper-parameters exactly as the library receives them (fp32 in roast_opt_config_t)
HP32 = {k: float(np.float32(v)) for k, v in dict(lr=1e-2, wd=0.01, b1=0.9, b2=0.999, eps=1e-8).items()}
MEM = 1 << 22
NAMES = {0: "sgd", 1: "adagrad", 2: "adam"}


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def R():
    from paper_2207_10702_b200 import roast
    return roast


def _model(R, torch, M0):
    ctx = R.Roast(to_dev(M0, torch.float32), 64, 64, seed=HS)
    ids = [ctx.linear(512, 1024), ctx.linear(1024, 512), ctx.embedding(3000, 64, 32)]
    return ctx, ids


def _touched(ids):
    m = np.zeros(MEM, dtype=bool)
    for sp in [OM.LinearSpec(512, 1024, 64, 64, MEM, HS, ids[0]), OM.LinearSpec(1024, 512, 64, 64, MEM, HS, ids[1])]:
        m[sp.slot_index().ravel()] = True
    emb = OE.EmbeddingSpec(3000, 64, 32, MEM, HS, ids[2])
    for off in emb.chunk_map(np.arange(3000))[0].ravel():
        m[int(off):int(off) + 32] = True
    return m


def _grads(torch, inside, W, t):
    out = []
    for r in range(W):
        g = torch.zeros(MEM, device="cuda")
        g[inside] = to_dev(synth.normal(1000 * t + r, (int(inside.sum()),)).astype(np.float32), torch.float32)
        out.append(g)
    return out


@pytest.mark.parametrize("W", [1, 2, 4])
@pytest.mark.parametrize("kind,zero", [(0, True), (2, True), (2, False), (1, True)])
def test_p2p_virtual_ranks(R, torch, W, kind, zero):
    M0 = store(MEM)
    ranks = [_model(R, torch, M0) for _ in range(W)]
    ids = ranks[0][1]
    inside_np = _touched(ids)
    n, _ = ranks[0][0].touched_size()
    assert n == int(inside_np.sum())
    inside = torch.tensor(inside_np, device="cuda")
    wins = [c.p2p_window()[0] for c, _ in ranks]
    for r, (c, _) in enumerate(ranks):
        c.p2p_attach(r, wins)
    ref, _ = _model(R, torch, M0)                      # one handle, summed gradient, plain update
    ref_M, st = M0.astype(np.float64), {}
    for t in (1, 2, 3):                                # both buffer parities, then reuse of the first
        gs = _grads(torch, inside, W, t)
        for (c, _), g in zip(ranks, gs):
            c.dM.copy_(g)
        for c, _ in ranks:
            c.p2p_post()
        for c, _ in ranks:
            c.p2p_finish(kind, 1e-2, step=t, weight_decay=0.01, zero_grad=zero)
        gsum = gs[0].clone()
        for g in gs[1:]:
            gsum += g
        ref.dM.copy_(gsum)
        ref.optimizer_step(kind, 1e-2, step=t, weight_decay=0.01, zero_grad=zero, touched_only=True)
        torch.cuda.synchronize()
        for c, _ in ranks:
            assert torch.equal(c.M, ref.M)
            assert torch.equal(c.dM, ref.dM)
            assert torch.equal(c.materialize(ids[0], torch.bfloat16), ref.materialize(ids[0], torch.bfloat16))
        # the fp64 oracle on the touched slots (the other slots are dead and stay as they were),
        # started from the device's M and state; the UPDATE and the new state are compared
        gsum64 = sum(g.double().cpu().numpy() for g in gs)
        new, st_ref = OO.step(NAMES[kind], ref_M, gsum64, st, **HP32, t=t)   # fp32 hyper-parameters, as received
        got = ranks[0][0].M.cpu().numpy()
        gabs = sum(g.double().abs().cpu().numpy() for g in gs)
        cond = grad_condition(gsum64[inside_np], ref_M[inside_np], 0.01, dM_abs=gabs[inside_np])
        check_update(ref_M[inside_np], got[inside_np], new[inside_np], cond=cond)
        assert np.array_equal(got[~inside_np], M0[~inside_np])
        keys = {0: [], 1: ["G"], 2: ["m", "v"]}[kind]
        for i, k in enumerate(keys):
            assert rel_frob(ranks[0][0].opt_state(i)[inside_np], st_ref[k][inside_np]) <= 1e-6, (k, t)
        st = {k: ranks[0][0].opt_state(i).astype(np.float64) for i, k in enumerate(keys)}
        ref_M = got.astype(np.float64)
    for c, _ in ranks:
        c.close()
    ref.close()


@pytest.mark.parametrize("W", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", [0, 2])
def test_p2p_two_shot_virtual_ranks(R, torch, W, kind):
    """Two-shot (reduce-scatter of the packed gradient + update of each rank's slice, then a
    gather of the slices): every rank's M, shadow and dM equal one handle's update of the
    summed gradient, bit for bit, over three steps (Adam's state lives on the slice owner)."""
    M0 = store(MEM)
    ranks = [_model(R, torch, M0) for _ in range(W)]
    ids = ranks[0][1]
    inside = torch.tensor(_touched(ids), device="cuda")
    wins = [c.p2p_window()[0] for c, _ in ranks]
    for r, (c, _) in enumerate(ranks):
        c.p2p_attach(r, wins)
    ref, _ = _model(R, torch, M0)
    for t in (1, 2, 3):
        gs = _grads(torch, inside, W, t)
        for (c, _), g in zip(ranks, gs):
            c.dM.copy_(g)
        for c, _ in ranks:
            c.p2p_post()
        for c, _ in ranks:
            c.p2p_reduce(kind, 1e-2, step=t, weight_decay=0.01)
        for c, _ in ranks:
            c.p2p_gather()
        gsum = gs[0].clone()
        for g in gs[1:]:
            gsum += g
        ref.dM.copy_(gsum)
        ref.optimizer_step(kind, 1e-2, step=t, weight_decay=0.01, touched_only=True)
        torch.cuda.synchronize()
        for c, _ in ranks:
            assert torch.equal(c.M, ref.M)
            assert torch.count_nonzero(c.dM).item() == 0
            for mid in ids[:2]:
                assert torch.equal(c.materialize(mid, torch.bfloat16), ref.materialize(mid, torch.bfloat16))
    for c, _ in ranks:
        c.close()
    ref.close()


def test_p2p_graph_capture_replays_advance_the_epoch(R, torch):
    """post + finish of two ranks captured once and replayed: the epoch and the buffer parity
    live in device memory, so every replay is a new step (same result as eager calls)."""
    M0 = store(MEM)
    res = []
    for graph in (False, True):
        ranks = [_model(R, torch, M0) for _ in range(2)]
        inside = torch.tensor(_touched(ranks[0][1]), device="cuda")
        wins = [c.p2p_window()[0] for c, _ in ranks]
        for r, (c, _) in enumerate(ranks):
            c.p2p_attach(r, wins)
        s = torch.cuda.Stream()
        gbuf = [torch.zeros(MEM, device="cuda") for _ in range(2)]

        def step():
            for (c, _), g in zip(ranks, gbuf):
                c.dM.copy_(g)
            for c, _ in ranks:
                c.p2p_post(stream=s)
            for c, _ in ranks:
                c.p2p_finish(0, 1e-2, step=1, stream=s)
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                step()
        for t in (1, 2, 3):
            for r in range(2):
                gbuf[r].copy_(_grads(torch, inside, 2, t)[r])
            torch.cuda.synchronize()
            if graph:
                g.replay()
            else:
                with torch.cuda.stream(s):
                    step()
            torch.cuda.synchronize()
        res.append([c.M.clone() for c, _ in ranks])
        for c, _ in ranks:
            c.close()
    assert torch.equal(res[0][0], res[0][1])
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[1][0], res[1][1])


_WORKER = textwrap.dedent("""
    import os, sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.getcwd())
    import synth
    from paper_2207_10702_b200 import roast as R
    rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[4], rank=rank, world_size=world)
    mem = 1 << 22
    M0 = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    ctx = R.Roast(torch.tensor(M0, device="cuda"), 64, 64, seed=synth.HASH_SEED)
    ctx.linear(512, 1024); ctx.linear(1024, 512); ctx.embedding(3000, 64, 32)
    ctx.p2p_init()
    for t in (1, 2):
        ctx.dM.copy_(torch.tensor(np.load(out + f"_g{t}_{rank}.npy"), device="cuda"))
        if sys.argv[5] == "2":
            ctx.exchange_p2p2(2, 1e-2, step=t, weight_decay=0.01)
        else:
            ctx.exchange_p2p(2, 1e-2, step=t, weight_decay=0.01)
    torch.cuda.synchronize()
    np.save(out + f"_M_{rank}.npy", ctx.M.cpu().numpy())
    ctx.check()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
""")


@pytest.mark.parametrize("shots", ["1", "2"])
def test_p2p_two_processes_through_cuda_ipc(R, torch, tmp_path, shots):
    """Two processes on one GPU, windows mapped with cudaIpcOpenMemHandle after a gloo
    all_gather of the handles (what p2p_init does on a node): both end with the single-handle
    update of the summed gradient, bit for bit."""
    M0 = store(MEM)
    ref, ids = _model(R, torch, M0)
    inside = torch.tensor(_touched(ids), device="cuda")
    out = str(tmp_path / "p2p")
    for t in (1, 2):
        gs = _grads(torch, inside, 2, t)
        for r in range(2):
            np.save(out + f"_g{t}_{r}.npy", gs[r].cpu().numpy())
        ref.dM.copy_(gs[0] + gs[1])
        ref.optimizer_step(2, 1e-2, step=t, weight_decay=0.01, touched_only=True)
    torch.cuda.synchronize()
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    port = str(29500 + os.getpid() % 1000 + int(shots))
    env = dict(os.environ, PYTHONPATH=os.getcwd())
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2", out, port, shots], cwd=os.getcwd(), env=env)
             for r in range(2)]
    codes = [p.wait(timeout=300) for p in procs]
    assert codes == [0, 0]
    M_ref = ref.M.cpu().numpy()
    for r in range(2):
        assert np.array_equal(np.load(out + f"_M_{r}.npy"), M_ref)
    ref.close()


def test_p2p_missing_peer_times_out_instead_of_hanging(tmp_path):
    """Rank 0 finishes while rank 1 never posts: the wait gives up after 20 s, sets the sticky
    error and traps (in a child process: the trap ends that CUDA context)."""
    code = textwrap.dedent("""
        import os, sys
        import numpy as np, torch
        sys.path.insert(0, os.getcwd())
        import synth
        from paper_2207_10702_b200 import roast as R
        M0 = synth.uniform(synth.SEED_M, (1 << 20,)).astype(np.float32)
        cs = [R.Roast(torch.tensor(M0, device="cuda"), 64, 64, seed=synth.HASH_SEED) for _ in range(2)]
        for c in cs:
            c.linear(512, 512)
        w = [c.p2p_window()[0] for c in cs]
        for r, c in enumerate(cs):
            c.p2p_attach(r, w)
        cs[0].p2p_post()
        cs[0].p2p_finish(0, 1e-2)
        try:
            torch.cuda.synchronize()
        except Exception as e:
            print("SYNC_ERROR", type(e).__name__)
            sys.exit(3)
        sys.exit(0)
    """)
    script = tmp_path / "timeout.py"
    script.write_text(code)
    p = subprocess.run([sys.executable, str(script)], cwd=os.getcwd(), capture_output=True, text=True, timeout=180,
                       env=dict(os.environ, PYTHONPATH=os.getcwd()))
    assert p.returncode == 3, p.stdout + p.stderr
    assert "SYNC_ERROR" in p.stdout
