"""NVLS (NVSwitch multicast) exchange fused with the update, and its fallback to the CUDA-IPC
P2P path (include/roast.h roast_nvls_*, nvls.cu; SURVEY.md §8(e) / §8(f) NEXT #1 = a6 P:194 +
a7 P:440 / P:749-813).

The gpurun boxes have one GPU and no NVSwitch fabric, so what runs here depends on the driver:
- where it accepts a one-device multicast object, the multimem kernels run for real at W = 1
  (ld_reduce over one copy is that copy) and must match the plain update bit for bit;
- otherwise the set-up must fail cleanly on every rank together and fall back to the P2P
  two-shot path, which must then match the plain update bit for bit.
Either way each test asserts which branch it took and checks the result of that branch."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import synth
from tests.gpu_helpers import store, to_dev
from tests.test_gpu_p2p import MEM, _grads, _model, _touched

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def R():
    from paper_2207_10702_b200 import roast
    return roast


def _run_steps(torch, ctx, ref, ids, fused, kind=2):
    inside = torch.tensor(_touched(ids), device="cuda")
    for t in (1, 2, 3):
        g = _grads(torch, inside, 1, t)[0]
        ctx.dM.copy_(g)
        fused(t)
        ref.dM.copy_(g)
        ref.optimizer_step(kind, 1e-2, step=t, weight_decay=0.01, touched_only=True)
        torch.cuda.synchronize()
        ctx.check()
        assert torch.equal(ctx.M, ref.M)
        assert torch.count_nonzero(ctx.dM).item() == 0
        for mid in ids[:2]:
            assert torch.equal(ctx.materialize(mid, torch.bfloat16), ref.materialize(mid, torch.bfloat16))


def test_nvls_probe_reports_a_bool(R, torch):
    assert R.roast_nvls_supported(torch.cuda.current_device()) in (True, False)


@pytest.mark.parametrize("prefer", ["auto", "p2p"])
def test_exchange_init_selects_a_path_and_matches_the_update(R, torch, prefer):
    """exchange_init picks NVLS or falls back to P2P (recording why); the fused two-shot
    exchange + Adam of the chosen path equals one handle's touched-only update, bit for bit,
    over three steps."""
    M0 = store(MEM)
    ctx, ids = _model(R, torch, M0)
    ref, _ = _model(R, torch, M0)
    path = ctx.exchange_init(prefer=prefer)
    assert path in ("nvls", "p2p")
    if prefer == "p2p":
        assert path == "p2p" and ctx.exchange_fallback is None
    if path == "p2p" and prefer == "auto":
        assert ctx.exchange_fallback and not R.roast_nvls_bound(ctx.h)
    if path == "nvls":
        assert R.roast_nvls_bound(ctx.h)
    print(f"exchange path: {path}; fallback: {getattr(ctx, 'exchange_fallback', None)}")
    _run_steps(torch, ctx, ref, ids, lambda t: ctx.exchange_fused(2, 1e-2, step=t, weight_decay=0.01))
    ctx.close()
    ref.close()


@pytest.mark.parametrize("shots", [1, 2])
def test_prefer_nvls_runs_multimem_or_fails_cleanly(R, torch, shots):
    """prefer="nvls" either binds (then the multimem one-shot / two-shot kernels run at W = 1
    and must equal the plain update bit for bit) or raises a RoastError; after the error the
    handle's P2P path still works (the failed set-up was fully undone)."""
    M0 = store(MEM)
    ctx, ids = _model(R, torch, M0)
    ref, _ = _model(R, torch, M0)
    try:
        ctx.exchange_init(prefer="nvls")
        bound = True
    except R.RoastError as e:
        bound = False
        print("NVLS refused on this box:", e)
        assert not R.roast_nvls_bound(ctx.h)
        R.roast_nvls_reset(ctx.h)
        ctx.p2p_init()
    if shots == 1:
        step = lambda t: ctx.exchange_p2p(2, 1e-2, step=t, weight_decay=0.01)   # noqa: E731
    else:
        step = lambda t: ctx.exchange_p2p2(2, 1e-2, step=t, weight_decay=0.01)  # noqa: E731
    _run_steps(torch, ctx, ref, ids, step)
    assert R.roast_nvls_bound(ctx.h) == bound
    ctx.close()
    ref.close()


def test_nvls_calls_validate_their_state(R, torch):
    M0 = store(MEM)
    ctx, _ = _model(R, torch, M0)
    with pytest.raises(R.RoastError):
        R.roast_nvls_add_device(ctx.h)     # no multicast object yet
    with pytest.raises(R.RoastError):
        R.roast_nvls_bind(ctx.h, 0)        # nothing added
    with pytest.raises(R.RoastError):
        R.roast_nvls_create(ctx.h, 9)      # world > 8
    R.roast_nvls_reset(ctx.h)              # no-op in the initial state
    ctx.close()


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
    path = ctx.exchange_init()
    for t in (1, 2):
        ctx.dM.copy_(torch.tensor(np.load(out + f"_g{t}_{rank}.npy"), device="cuda"))
        ctx.exchange_fused(2, 1e-2, step=t, weight_decay=0.01)
    torch.cuda.synchronize()
    np.save(out + f"_M_{rank}.npy", ctx.M.cpu().numpy())
    with open(out + f"_path_{rank}.txt", "w") as f:
        f.write(path + "\\n" + str(ctx.exchange_fallback))
    ctx.check()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
""")


def test_exchange_init_two_processes_agree_on_the_path(R, torch, tmp_path):
    """Two processes on one GPU run the whole negotiation (probe, create on rank 0, descriptor
    over a unix socket, import, add device, bind — or a fallback decided together): both
    report the same path and end with the single-handle update of the summed gradient."""
    M0 = store(MEM)
    ref, ids = _model(R, torch, M0)
    inside = torch.tensor(_touched(ids), device="cuda")
    out = str(tmp_path / "nvls")
    for t in (1, 2):
        gs = _grads(torch, inside, 2, t)
        for r in range(2):
            np.save(out + f"_g{t}_{r}.npy", gs[r].cpu().numpy())
        ref.dM.copy_(gs[0] + gs[1])
        ref.optimizer_step(2, 1e-2, step=t, weight_decay=0.01, touched_only=True)
    torch.cuda.synchronize()
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    port = str(28500 + os.getpid() % 1000)
    env = dict(os.environ, PYTHONPATH=os.getcwd())
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2", out, port], cwd=os.getcwd(), env=env)
             for r in range(2)]
    codes = [p.wait(timeout=300) for p in procs]
    assert codes == [0, 0]
    paths = [open(out + f"_path_{r}.txt").read().split("\n")[0] for r in range(2)]
    print("two-process paths:", paths, open(out + "_path_0.txt").read())
    assert paths[0] == paths[1] and paths[0] in ("nvls", "p2p")
    M_ref = ref.M.cpu().numpy()
    for r in range(2):
        assert np.array_equal(np.load(out + f"_M_{r}.npy"), M_ref)
    ref.close()
