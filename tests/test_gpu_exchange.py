"""Touched-set dM exchange on the GPU: the library's interval tables equal
the oracle's slot set, pack / unpack move exactly the touched slots, and the NCCL exchange in
TOUCHED mode gives the same sum as the dense one (1-rank communicator on one B200)."""
import numpy as np
import pytest

import synth
from oracle import embedding as OE
from oracle import roast_mm as OM
from tests.gpu_helpers import store, to_dev

pytestmark = pytest.mark.gpu
HS = synth.HASH_SEED


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def R():
    from paper_2207_10702_b200 import roast
    return roast


def _oracle_slots(specs, mem, extra=()):
    m = np.zeros(mem, dtype=bool)
    for sp in specs:
        m[sp.slot_index().ravel()] = True
    for s, n in extra:
        m[s:s + n] = True
    return m


@pytest.mark.parametrize("mem", [1 << 21, 47192])
def test_touched_size_equals_oracle_slot_set(R, torch, mem):
    M = to_dev(store(mem), torch.float32)
    ctx = R.Roast(M, 64, 64, seed=HS)
    l1, l2 = ctx.linear(768, 3072), ctx.linear(3072, 768)
    bias = ctx.embedding(1, 3072, 64, fan_in=768.0)             # a bias via L: its exact 48 chunks
    n, k = ctx.touched_size()
    specs = [OM.LinearSpec(768, 3072, 64, 64, mem, HS, l1), OM.LinearSpec(3072, 768, 64, 64, mem, HS, l2)]
    be = OE.EmbeddingSpec(1, 3072, 64, mem, HS, bias)
    boff = [int(o) for o in be.chunk_map(np.zeros(1, dtype=np.int64))[0].ravel()]
    slots = _oracle_slots(specs, mem, [(o, 64) for o in boff])
    assert n == int(slots.sum())
    runs = np.diff(np.concatenate([[0], slots.astype(np.int8), [0]]))
    assert k == int((runs == 1).sum())
    ctx.close()


def test_large_table_touches_its_whole_memory(R, torch):
    mem = 1 << 20
    M = to_dev(store(mem), torch.float32)
    ctx = R.Roast(M, 64, 64, seed=HS)
    ctx.embedding(10 ** 7, 128, 32)
    assert ctx.touched_size() == (mem, 1)                      # every legal chunk position: all of M
    ctx.close()


def test_pack_unpack_moves_exactly_the_touched_slots(R, torch):
    mem = 1 << 21
    M = to_dev(store(mem), torch.float32)
    ctx = R.Roast(M, 64, 64, seed=HS)
    l1 = ctx.linear(1024, 2048)
    g = to_dev(synth.normal(9, (mem,)).astype(np.float32), torch.float32)   # every slot nonzero
    ctx.dM.copy_(g)
    R.roast_debug_exchange(ctx.h, 3.0, 0)
    torch.cuda.synchronize()
    spec = OM.LinearSpec(1024, 2048, 64, 64, mem, HS, l1)
    inside = torch.tensor(_oracle_slots([spec], mem), device="cuda")
    assert torch.equal(ctx.dM[inside], 3.0 * g[inside])
    assert torch.equal(ctx.dM[~inside], g[~inside])
    ctx.close()


def test_touched_exchange_nccl_matches_dense(R, torch):
    """C5 geometry (4096 x 4096, |M| = 32M elements = 128 MB fp32, 2x the virtual layer):
    backward, then the exchange in TOUCHED and DENSE mode on a 1-rank communicator — both the
    identity sum; TOUCHED launches the pack / unpack pair and captures into a CUDA graph."""
    from tests.gpu_helpers import bf16_input
    mem = 32 << 20
    M = to_dev(store(mem), torch.float32)
    ctx = R.Roast(M, 64, 64, seed=HS)
    lid = ctx.linear(4096, 4096)
    R.roast_comm_init(ctx.h, 0, 1, R.roast_comm_unique_id())
    X = to_dev(bf16_input(2, (256, 4096)), torch.bfloat16)
    dY = to_dev(bf16_input(3, (256, 4096)), torch.bfloat16)
    ctx.zero_grad()
    ctx.bwd(lid, X, dY, need_dx=False)
    torch.cuda.synchronize()
    ref = ctx.dM.clone()
    n, _ = ctx.touched_size()
    assert 2 * n <= mem                                         # AUTO picks the touched exchange
    for mode, launches in [(R.EXCHANGE_TOUCHED, 2), (R.EXCHANGE_AUTO, 2), (R.EXCHANGE_DENSE, 0)]:
        ctx.set_exchange(mode)
        c0 = ctx.launch_count()
        ctx.allreduce()
        torch.cuda.synchronize()
        assert ctx.launch_count() - c0 == launches
        assert torch.equal(ctx.dM, ref)
    ctx.set_exchange(R.EXCHANGE_TOUCHED)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ctx.allreduce()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(ctx.dM, ref)
    ctx.close()


@pytest.mark.parametrize("kind", [0, 2])
def test_optimizer_touched_only_equals_dense_on_the_touched_set(R, torch, kind):
    """Update restricted to the touched set: touched slots of M, state, shadow
    and dM bit-identical to the dense pass; every other slot left as it was; the recovered
    weights (what any module reads) identical."""
    mem = 1 << 20
    M0 = store(mem)
    g = to_dev(synth.normal(11, (mem,)).astype(np.float32), torch.float32)
    ctxs = []
    for touched in (False, True):
        ctx = R.Roast(to_dev(M0, torch.float32), 64, 64, seed=HS)
        lid = ctx.linear(256, 512)
        ctx.touched_size()
        for t in (1, 2):
            ctx.dM.copy_(g)
            ctx.optimizer_step(kind, 1e-2, step=t, weight_decay=0.01, touched_only=touched)
        torch.cuda.synchronize()
        ctxs.append((ctx, lid))
    (dense, l0), (tch, l1) = ctxs
    spec = OM.LinearSpec(256, 512, 64, 64, mem, HS, l0)
    inside = torch.tensor(_oracle_slots([spec], mem), device="cuda")
    M0d = to_dev(M0, torch.float32)
    assert torch.equal(tch.M[inside], dense.M[inside])
    assert torch.equal(tch.M[~inside], M0d[~inside])
    assert torch.count_nonzero(tch.dM[inside]).item() == 0 and torch.equal(tch.dM[~inside], g[~inside])
    assert torch.equal(tch.materialize(l1, torch.bfloat16), dense.materialize(l0, torch.bfloat16))
    assert torch.equal(tch.materialize(l1, torch.float32), dense.materialize(l0, torch.float32))
    for c, _ in ctxs:
        c.close()


@pytest.mark.parametrize("kind", [0, 2])
@pytest.mark.parametrize("mode,comm,zero", [(0, True, True), (2, False, True), (1, True, True), (0, True, False)])
def test_exchange_step_equals_allreduce_then_update(R, torch, kind, mode, comm, zero):
    """roast_grad_exchange_step (exchange fused with the update; the touched path reads the summed
    gradient from the packed buffer) == roast_grad_allreduce + roast_optimizer_step, bit for bit,
    over two steps: M, the bf16 shadow (recovered operand tiles) and dM."""
    mem = 1 << 22
    M0 = store(mem)
    g = to_dev(synth.normal(13, (mem,)).astype(np.float32), torch.float32)
    res = []
    for fused in (False, True):
        ctx = R.Roast(to_dev(M0, torch.float32), 64, 64, seed=HS)
        lid = ctx.linear(512, 1024)
        if comm:
            R.roast_comm_init(ctx.h, 0, 1, R.roast_comm_unique_id())
        ctx.set_exchange(mode)
        n, _ = ctx.touched_size()
        touched = mode == 2 or (mode == 0 and 2 * n <= mem)
        spec = OM.LinearSpec(512, 1024, 64, 64, mem, HS, lid)
        inside = torch.tensor(_oracle_slots([spec], mem), device="cuda")
        for t in (1, 2):
            ctx.dM.zero_()
            ctx.dM[inside] = g[inside]          # a backward writes only the touched slots
            if fused:
                ctx.exchange_step(kind, 1e-2, step=t, weight_decay=0.01, zero_grad=zero)
            else:
                ctx.allreduce()
                ctx.optimizer_step(kind, 1e-2, step=t, weight_decay=0.01, zero_grad=zero, touched_only=touched)
        torch.cuda.synchronize()
        res.append((ctx.M.clone(), ctx.dM.clone(), ctx.materialize(lid, torch.bfloat16)))
        ctx.close()
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)
