"""Multi-process (gloo, world size 2, CPU) coverage of the data-parallel host logic.

The north star's partitioning: split the batch, replicate M, all-reduce dM.  Under
GMS the gradient is linear in the batch, so the sum over ranks of the
per-shard dM must equal the full-batch dM of the oracle; the NCCL unique id must
reach every rank intact.  (The NCCL exchange itself runs on the GPU box.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import embedding as OE
from oracle import roast_mm as OM
from paper_2207_10702_b200 import dp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. the 128-byte id broadcast used to bootstrap NCCL
        uid = bytes(range(128)) if rank == 0 else None
        got = dp.broadcast_bytes(uid, rank, 128)
        assert got == bytes(range(128))
        # 2. linear layers: sharded dM, summed over ranks == full-batch oracle dM
        mem = 4720
        M = synth.uniform(synth.SEED_M, (mem,))
        T = 203                                           # ragged: shards of 102 / 101 tokens
        layers = [OM.LinearSpec(128, 192, 64, 64, mem, synth.HASH_SEED, 0),
                  OM.LinearSpec(192, 128, 64, 64, mem, synth.HASH_SEED, 1)]
        X1 = synth.normal(synth.SEED_X, (T, 128))
        dY1 = synth.normal(synth.SEED_DY, (T, 192))
        X2 = synth.normal(synth.SEED_X + 10, (T, 192))
        dY2 = synth.normal(synth.SEED_DY + 10, (T, 128))
        a, b = dp.shard(T, rank, world)
        local = np.zeros(mem)
        layers[0].backward_dm(X1[a:b], dY1[a:b], local)
        layers[1].backward_dm(X2[a:b], dY2[a:b], local)
        t = torch.tensor(local)
        dist.all_reduce(t)
        full = np.zeros(mem)
        layers[0].backward_dm(X1, dY1, full)
        layers[1].backward_dm(X2, dY2, full)
        err_mm = float(np.max(np.abs(t.numpy() - full)) / np.max(np.abs(full)))
        # 3. embeddings: sharded samples
        emb = OE.EmbeddingSpec(10 ** 6, 64, 32, mem, synth.HASH_SEED, 2)
        idx = synth.zipf_indices(synth.SEED_IDX, 301, 10 ** 6)
        dout = synth.normal(synth.SEED_DY + 20, (301, 64))
        a, b = dp.shard(301, rank, world)
        te = torch.tensor(emb.backward(idx[a:b], dout[a:b]))
        dist.all_reduce(te)
        full_e = emb.backward(idx, dout)
        err_emb = float(np.max(np.abs(te.numpy() - full_e)) / np.max(np.abs(full_e)))
        q.put((rank, err_mm, err_emb))
    finally:
        dist.destroy_process_group()


def test_shard_partitions_exactly():
    for n in [0, 1, 7, 8192, 65537]:
        for world in [1, 2, 3, 8]:
            parts = [dp.shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2, 8])     # "at world = 2 and 8"
def test_world_allreduce_equals_full_batch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = [q.get(timeout=5) for _ in range(world)]
    assert all(p.exitcode == 0 for p in procs)
    for rank, err_mm, err_emb in results:
        assert err_mm <= 1e-12 and err_emb <= 1e-12, (rank, err_mm, err_emb)


def _touched_worker(rank, world, port, q):
    """The touched-set exchange at world 2: pack the library's intervals,
    all-reduce only the packed vector, unpack — equals the dense full-batch dM."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2207_10702_b200 import roast as R
        mem = 1 << 18                                      # |M| >> n: most of dM is never written
        layers = [OM.LinearSpec(128, 192, 64, 64, mem, synth.HASH_SEED, 0),
                  OM.LinearSpec(192, 128, 64, 64, mem, synth.HASH_SEED, 1)]
        T = 77
        X1, dY1 = synth.normal(2, (T, 128)), synth.normal(3, (T, 192))
        X2, dY2 = synth.normal(4, (T, 192)), synth.normal(5, (T, 128))
        a, b = dp.shard(T, rank, world)
        local = np.zeros(mem)
        layers[0].backward_dm(X1[a:b], dY1[a:b], local)
        layers[1].backward_dm(X2[a:b], dY2[a:b], local)
        starts, lens = R.roast_touched_intervals(np.concatenate([sp.off.ravel() for sp in layers]), 64 * 64)
        packed = torch.tensor(np.concatenate([local[s:s + n] for s, n in zip(starts, lens)]))
        dist.all_reduce(packed)
        out = np.zeros(mem)
        p = 0
        for s, n in zip(starts, lens):
            out[s:s + n] = packed.numpy()[p:p + n]
            p += n
        full = np.zeros(mem)
        layers[0].backward_dm(X1, dY1, full)
        layers[1].backward_dm(X2, dY2, full)
        err = float(np.max(np.abs(out - full)) / np.max(np.abs(full)))
        q.put((rank, err, int(lens.sum()), mem))
    finally:
        dist.destroy_process_group()


def test_world2_touched_set_exchange_equals_dense():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_touched_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = [q.get(timeout=5) for _ in range(2)]
    assert all(p.exitcode == 0 for p in procs)
    for rank, err, moved, mem in results:
        assert err <= 1e-12, (rank, err)
        assert moved <= 2 * 6 * 4096 < mem       # 2 x 6 tiles of 4096 slots at most, << |M|
