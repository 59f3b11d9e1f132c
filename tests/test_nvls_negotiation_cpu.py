"""The multi-rank NVLS negotiation of Roast.exchange_init (roast.py; include/roast.h roast_nvls_*)
at world size 2 on CPU (gloo): the driver steps are replaced by recording fakes, so what runs is
the host protocol itself — the capability probe, rank 0's multicast object exported as a file
descriptor and passed to the other rank over an abstract unix socket (SCM_RIGHTS), the status
all-gather after every step, and the joint fallback to the P2P window when any rank fails any
step (every rank must take the same path, or the exchange kernels would wait on each other)."""
import os
import socket
import tempfile
import types

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

PAYLOAD = b"roast-nvls-multicast-object"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scenario, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_10702_b200 import roast as R
    log = []
    fail = lambda step: scenario == f"{step}_fails_rank{rank}"   # noqa: E731

    def boom(step):
        raise R.RoastError(7, step)   # what a refused driver call raises

    def supported(dev):
        log.append("probe")
        return not fail("probe")

    def create(h, w):
        log.append(("create", w))
        if fail("create"):
            boom("create")
        f = tempfile.TemporaryFile()
        f.write(PAYLOAD)
        f.flush()
        return os.dup(f.fileno())   # the object's descriptor, owned by the caller

    def imp(h, w, fd):
        os.lseek(fd, 0, 0)
        log.append(("import", w, os.read(fd, 64) == PAYLOAD))
        if fail("import"):
            boom("import")

    def add(h):
        log.append("add")
        if fail("add"):
            boom("add_device")

    def bind(h, r):
        log.append(("bind", r))
        if fail("bind"):
            boom("bind")

    R.roast_nvls_supported, R.roast_nvls_create, R.roast_nvls_import = supported, create, imp
    R.roast_nvls_add_device, R.roast_nvls_bind = add, bind
    R.roast_nvls_reset = lambda h: log.append("reset")
    fake = types.SimpleNamespace(h=None, torch=None, M=types.SimpleNamespace(device=types.SimpleNamespace(index=0)))
    fake.p2p_init = lambda group=None: log.append("p2p_init")
    fake._nvls_init = types.MethodType(R.Roast._nvls_init, fake)
    try:
        path = R.Roast.exchange_init(fake)
        q.put((rank, path, fake.exchange_fallback, log))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), log))
    finally:
        dist.destroy_process_group()


def _run(scenario):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, scenario, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, path, why, log = q.get(timeout=180)
        res[r] = (path, why, log)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_all_steps_succeed_every_rank_binds_nvls():
    res = _run("ok")
    for r in range(2):
        path, why, log = res[r]
        assert path == "nvls" and why is None
        assert log[-2:] == ["add", ("bind", r)] and "p2p_init" not in log
    assert ("create", 2) in res[0][2]
    assert ("import", 2, True) in res[1][2]          # the descriptor reached rank 1 intact


@pytest.mark.parametrize("scenario", ["probe_fails_rank1", "create_fails_rank0", "import_fails_rank1",
                                      "add_fails_rank0", "bind_fails_rank1"])
def test_any_failure_makes_every_rank_fall_back_together(scenario):
    res = _run(scenario)
    for r in range(2):
        path, why, log = res[r]
        assert path == "p2p", (r, path, why)
        assert why and "nvls" in why
        assert log[-2:] == ["reset", "p2p_init"]     # partial set-up undone, then the IPC window
    step = scenario.split("_")[0]
    if step in ("add", "bind"):       # every rank reached the failing step: all-gathered after it
        assert all(("bind", r) in res[r][2] or "add" in res[r][2] for r in range(2))
