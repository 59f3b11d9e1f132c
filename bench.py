#!/usr/bin/env python
"""bench.py — ROAST-MM fwd+bwd effective TFLOP/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the metric's config):
BERT-base MLP block, L1 768->3072 and L2 3072->768 in ONE global M (GMS) at
100x compression (|M| = 47 192 fp32), hash tile 64x64, 8192 tokens per GPU,
bf16 operands / fp32 accumulate.  One step = the whole hot path over one batch:

    Y1 = L1(X); Y2 = L2(Y1)                      (a1, the N-op between them is identity)
    dY1 = L2.dX(dY2); dM += L2.dM(Y1, dY2)       (a2, a3)
    dX  = L1.dX(dY1); dM += L1.dM(X, dY1)        (a2, a3)
    dM  = allreduce(dM)                          (a6; no-op at N = 1)

Effective FLOPs per step per GPU = sum over layers of 6 T H O (ROAST does
not reduce compute).  Multi-GPU: one process per GPU, tokens per GPU fixed
(weak scaling), dM all-reduced with NCCL through the C ABI.

`--impl reference` times the oracle (oracle/, CPU fp64) as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RATIO = 100   # the metric's configuration (BASELINE.json configs[1] at 100x); --ratio 10 / 1000 for the others


def _num(x):
    return int(x) if float(x).is_integer() else x


def workload(ratio, mem):
    """config.workload of both arms (the same string: same metric, same configuration)."""
    r = int(ratio) if float(ratio).is_integer() else ratio
    return "C2 BERT-base MLP block 768->3072->768 fwd+bwd, %sx (|M|=%d), tile 64x64" % (r, mem)


def synth_mem(ratio):
    import synth
    return synth.mlp_block(ratio)["mem_size"]


def args_ratio():
    """--ratio of the current command line (the reference arm's sample uses the same |M|)."""
    for i, a in enumerate(sys.argv):
        if a == "--ratio" and i + 1 < len(sys.argv):
            return float(sys.argv[i + 1])
        if a.startswith("--ratio="):
            return float(a.split("=", 1)[1])
    return RATIO
TOKENS = 8192
LAYERS = [(768, 3072), (3072, 768)]
TILE = 64
METRIC = "ROAST-MM fwd+bwd effective TFLOP/s vs dense cuBLAS & bf16 peak, 1/2/4/8 B200"
UNIT = "TFLOP/s"


def flops_per_step(tokens):
    return sum(6.0 * tokens * H * O for H, O in LAYERS)


def load_peaks():
    """(bf16 burst TFLOP/s, sustained, HBM GB/s, source) from the driver-written
    MEASURED_PEAKS.json, else the B200_PROFILING.md fallback (1590 / ~1400 / 6650).
    Tolerates a missing file, missing keys or a nested layout (never fails the bench)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))

        def find(key):
            if isinstance(d, dict) and key in d:
                return float(d[key])
            for v in (d.values() if isinstance(d, dict) else []):
                if isinstance(v, dict) and key in v:
                    return float(v[key])
            return None
        burst, sus, hbm = find("bf16_tflops"), find("bf16_tflops_sustained"), find("hbm_gbs")
        if burst and hbm:
            return burst, sus, hbm, "measured"
    except Exception:
        pass
    return 1590.0, 1400.0, 6650.0, "fallback"


def ncu_traffic(kind):
    """DRAM bytes (read + write) per launch of `kind` from the newest committed ncu --set full
    capture summary (profiles/round*/traffic.json, written by tools/traffic_from_ncu.py), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "round*", "traffic.json")))
    if not files:
        return None
    try:
        return json.load(open(files[-1])).get(kind)
    except Exception:
        return None


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------------ reference arm
def cpu_sample(seconds_target=10.0, tokens=256):
    """Time the oracle on a bounded sample of the workload: `tokens` of the 8192."""
    import numpy as np

    import synth
    from oracle import roast_mm as OM
    mem = synth.mlp_block(args_ratio())["mem_size"]
    M = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    specs = [OM.LinearSpec(H, O, TILE, TILE, mem, synth.HASH_SEED, i) for i, (H, O) in enumerate(LAYERS)]
    X = synth.round_to_bf16(synth.normal(synth.SEED_X, (tokens, 768)).astype(np.float32))
    dY2 = synth.round_to_bf16(synth.normal(synth.SEED_DY, (tokens, 768)).astype(np.float32))
    t0 = time.perf_counter()
    steps = 0
    while True:
        Y1 = specs[0].forward(X, M, True)
        specs[1].forward(Y1, M, True)
        dM = np.zeros(mem)
        dY1 = specs[1].backward_dx(dY2, M, True)
        specs[1].backward_dm(Y1, dY2, dM)
        specs[0].backward_dx(dY1, M, True)
        specs[0].backward_dm(X, dY1, dM)
        steps += 1
        el = time.perf_counter() - t0
        if el >= seconds_target:
            break
    per_step = el / steps
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return dict(value=flops_per_step(tokens) / per_step / 1e12, unit=UNIT, cores=cores, kind="oracle",
                sample=f"MLP block fwd+bwd at T={tokens} of {TOKENS} tokens (oracle cost is linear in T), "
                       f"{steps} steps in {el:.1f}s, fp64 numpy", seconds_per_sample_step=per_step)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    for _ in range(args.warmup):
        pass
    cb = cpu_sample(seconds_target=max(3.0, 2.0 * args.steps))
    line = dict(metric=METRIC, value=cb["value"], unit=UNIT, n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=cb["seconds_per_sample_step"] * 1e3, higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=workload(args_ratio(), synth_mem(args_ratio())),
                            tokens_per_gpu=TOKENS, ratio=_num(args_ratio())),
                impl="reference",
                cpu_baseline=dict(value=cb["value"], unit=UNIT, cores=cb["cores"], kind="oracle",
                                  sample=cb["sample"]),
                e2e=dict(value=cb["value"], unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
class ClockSampler:
    """SM clock + clock-event reasons sampled every ~2 ms by an NVML thread during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None

    def _run(self):
        import pynvml as N
        names = {N.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 N.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 N.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        while not self.stop:
            self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in names.items():
                if r & bit:
                    self.reasons.add(name)
            time.sleep(0.002)

    def __enter__(self):
        import threading
        self.stop = False
        self.thread = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *a):
        self.stop = True
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        import statistics
        if not self.samples:
            return dict(sm_mhz=None, sm_max_mhz=self.max_mhz, reasons=["unsampled"])
        return dict(sm_mhz=statistics.median(self.samples), sm_max_mhz=self.max_mhz,
                    reasons=sorted(self.reasons), samples=len(self.samples))


def run_gpu(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2207_10702_b200 import roast as R
    import synth

    T = TOKENS
    mem = synth.mlp_block(args.ratio)["mem_size"]
    stream = torch.cuda.current_stream()
    M = torch.tensor(synth.uniform(synth.SEED_M, (mem,)).astype(np.float32), device=dev)
    ctx = R.Roast(M, TILE, TILE, seed=synth.HASH_SEED, deterministic=args.deterministic)
    ctx.set_autotune(args.autotune)   # tuned in the eager warm-up, before graph capture
    from paper_2207_10702_b200 import dp
    dp.init_comm(ctx, rank, world, device=dev)   # NCCL communicator inside libroast (no-op at N = 1)
    l1 = ctx.linear(*LAYERS[0])
    l2 = ctx.linear(*LAYERS[1])
    bf = torch.bfloat16
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    X = torch.randn(T, 768, device=dev, generator=g).to(bf)
    dY2 = torch.randn(T, 768, device=dev, generator=g).to(bf)
    Y1 = torch.empty(T, 3072, device=dev, dtype=bf)
    Y2 = torch.empty(T, 768, device=dev, dtype=bf)
    dY1 = torch.empty(T, 3072, device=dev, dtype=bf)
    dX = torch.empty(T, 768, device=dev, dtype=bf)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    side = torch.cuda.Stream(device=dev)

    def step_body(Xin, dY2in):
        """One step of the hot path: Y1 = X W1, Y2 = Y1 W2, dY1 = dY2 W2^T, dX = dY1 W1^T,
        dM += scatter(X^T dY1) + scatter(Y1^T dY2), then the dM exchange.  With --chain the
        forward pair (and with --chain 2 the dX pair) runs as ONE persistent launch.  dX and dM
        of each layer are independent, so with --streams 2 every dM GEMM runs on a second
        stream and fills the SMs the dX GEMMs leave idle (roast_linear_bwd_dx / _dm)."""
        cur = torch.cuda.current_stream()
        ctx.zero_grad()
        if args.chain:
            ctx.fwd_chain(l1, l2, Xin, Y1, Y2)
        else:
            ctx.fwd(l1, Xin, Y1)
            ctx.fwd(l2, Y1, Y2)
        if args.streams == 2 and args.chain == 2:
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                ctx.bwd_dm(l2, Y1, dY2in)
            ctx.bwd_dx_chain(l1, l2, dY2in, dY1, dX)   # dY1 and dX in one launch
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                ctx.bwd_dm(l1, Xin, dY1)
            cur.wait_stream(side)
        elif args.streams == 2:
            side.wait_stream(cur)
            ctx.bwd_dx(l2, dY2in, dY1)
            e_dy1 = torch.cuda.Event()
            e_dy1.record(cur)
            with torch.cuda.stream(side):
                ctx.bwd_dm(l2, Y1, dY2in)
            ctx.bwd_dx(l1, dY1, dX)
            side.wait_event(e_dy1)
            with torch.cuda.stream(side):
                ctx.bwd_dm(l1, Xin, dY1)
            cur.wait_stream(side)
        else:
            if args.chain == 2:
                ctx.bwd_dx_chain(l1, l2, dY2in, dY1, dX)
            else:
                ctx.bwd_dx(l2, dY2in, dY1)
                ctx.bwd_dx(l1, dY1, dX)
            ctx.bwd_dm(l2, Y1, dY2in)
            ctx.bwd_dm(l1, Xin, dY1)
        ctx.allreduce()

    if args.tuned_file:   # reuse a tuning (e.g. the plain bench run's) instead of timing under a profiler
        saved = json.load(open(args.tuned_file))
        saved = saved.get("config", {}).get("tuned", saved)
        for i, mid in enumerate((l1, l2)):
            for j, k in enumerate(("fwd", "dx", "dm")):
                v = saved.get(f"L{i + 1}.{k}")
                if v:
                    ctx.set_tuned(mid, j, T, int(v[0]), int(v[1]))
    if args.autotune:   # tune every kernel once, sequentially on one stream (no concurrent work skews it)
        ctx.zero_grad()
        ctx.fwd(l1, X, Y1)
        ctx.fwd(l2, Y1, Y2)
        if args.chain:
            ctx.fwd_chain(l1, l2, X, Y1, Y2)            # plans the chained schedules eagerly
            ctx.bwd_dx_chain(l1, l2, dY2, dY1, dX)
        ctx.bwd_dx(l2, dY2, dY1)
        ctx.bwd_dm(l2, Y1, dY2)
        ctx.bwd_dx(l1, dY1, dX)
        ctx.bwd_dm(l1, X, dY1)
        torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    if world > 1:
        # every rank must run the same configuration: the step-level choice below replays steps
        # with the NCCL exchange inside, so a rank-dependent branch would mismatch collectives
        import torch.distributed as dist
        cfgs = torch.tensor([v for mid in (l1, l2) for j in range(3) for v in (ctx.tuned(mid, j, T) or (0, 0))],
                            dtype=torch.int32, device=dev)
        dist.broadcast(cfgs, 0)
        vals = cfgs.tolist()
        for i, mid in enumerate((l1, l2)):
            for j in range(3):
                wm, sp = vals[6 * i + 2 * j], vals[6 * i + 2 * j + 1]
                if wm:
                    ctx.set_tuned(mid, j, T, wm, sp)

    # training-optimal at the step level (P:428-429 tunes forward and backward together): a dX
    # GEMM tuned alone may pick 192-column units, which fill more CTA pairs but leave fewer
    # SMs to the dM GEMM running beside it on the second stream; keep whichever whole step
    # (graph-replayed, L2 flushed) is faster
    if args.autotune == 2 and not args.tuned_file:
        def step_ms(reps=15):
            for _ in range(3):
                step_body(X, dY2)
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_):
                step_body(X, dY2)
            ts = []
            for _ in range(reps):
                flush.zero_()
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                g_.replay()
                b_.record(stream)
                torch.cuda.synchronize()
                ts.append(a_.elapsed_time(b_))
            return sorted(ts)[len(ts) // 2]
        for mid in (l1, l2):
            wm, nu = ctx.tuned(mid, 1, T)
            if nu == 3:
                t192 = step_ms()
                ctx.set_tuned(mid, 1, T, wm, 4)
                t256 = step_ms()
                keep = t192 < t256
                if world > 1:   # rank 0 decides for everyone (same configuration on every rank)
                    import torch.distributed as dist
                    flag = torch.tensor([int(keep)], dtype=torch.int32, device=dev)
                    dist.broadcast(flag, 0)
                    keep = bool(flag.item())
                if keep:
                    ctx.set_tuned(mid, 1, T, wm, 3)

    # warm-up (eager), launches per step, then capture the step in a CUDA graph
    for _ in range(args.warmup):
        step_body(X, dY2)
    barrier()
    l0 = ctx.launch_count()
    step_body(X, dY2)
    launches_per_step = ctx.launch_count() - l0
    barrier()
    graph = None
    if args.graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_body(X, dY2)
        for _ in range(args.warmup):
            graph.replay()
        barrier()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step_body(X, dY2)

    # timed region: per-step CUDA events; L2 flushed between steps (outside the events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            run_step()
            ends[i].record(stream)
        barrier()
    launches = launches_per_step * args.steps
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = world * flops_per_step(T) / (ms_per_step * 1e-3) / 1e12

    # per-kernel-kind launch durations: each call captured alone in a CUDA graph and replayed
    # between CUDA events (device time of exactly that launch, no host launch latency)
    gemm_flop = 2.0 * T * 768 * 3072                       # every GEMM is one 2*T*H*O contraction
    if args.chain:
        calls = [("fwd_chain", lambda: ctx.fwd_chain(l1, l2, X, Y1, Y2), 2 * gemm_flop)]
    else:
        calls = [("fwd", lambda: ctx.fwd(l1, X, Y1), gemm_flop), ("fwd", lambda: ctx.fwd(l2, Y1, Y2), gemm_flop)]
    if args.chain == 2:
        calls += [("dx_chain", lambda: ctx.bwd_dx_chain(l1, l2, dY2, dY1, dX), 2 * gemm_flop)]
    else:
        calls += [("dx", lambda: ctx.bwd_dx(l2, dY2, dY1), gemm_flop), ("dx", lambda: ctx.bwd_dx(l1, dY1, dX), gemm_flop)]
    calls += [("dm", lambda: ctx.bwd_dm(l2, Y1, dY2), gemm_flop), ("dm", lambda: ctx.bwd_dm(l1, X, dY1), gemm_flop)]
    kinds = list(dict.fromkeys(k for k, _, _ in calls))
    ev = {k: [] for k in kinds}
    kind_flop = {k: f for k, _, f in calls}
    kind_count = {k: sum(1 for c in calls if c[0] == k) for k in kinds}
    call_graphs = []
    for kind, fn, _ in calls:
        cg_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg_):
            fn()
        call_graphs.append((kind, cg_))
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        for kind, cg_ in call_graphs:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cg_.replay()
            b.record(stream)
            ev[kind].append((a, b))
    torch.cuda.synchronize()
    kind_ms = {k: float(np.mean([a.elapsed_time(b) for a, b in ev[k]])) for k in kinds}
    # dominant kernel = the kind with the largest share of the step's launch time
    dom = max(kinds, key=lambda k: kind_ms[k] * kind_count[k])
    burst, sustained, hbm, src = load_peaks()
    achieved = kind_flop[dom] / (kind_ms[dom] * 1e-3) / 1e12

    # end-to-end through the C ABI with host buffers: every step's inputs (X, dY2) are copied
    # host -> device from pinned memory and its result (dM) read back, all inside the timed
    # region.  As in a training input pipeline, step k + 1's inputs are copied on a second
    # stream into the other of two device buffers while step k computes (double-buffered
    # prefetch), so PCIe and the kernels overlap; each step still waits for its own copy.
    # pinned staging buffers from the pinned allocator (torch.empty(pin_memory=True)): on these
    # boxes `X.cpu().pin_memory()` gave host memory that copies at 13 GB/s instead of 54 GB/s
    # (tools/e2e_probe.py), which had made e2e swing between 150 and 480 TFLOP/s
    Xh = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
    Xh.copy_(X)
    dY2h = torch.empty(dY2.shape, dtype=dY2.dtype, pin_memory=True)
    dY2h.copy_(dY2)
    dMh = torch.empty(mem, dtype=torch.float32, pin_memory=True)
    bufs = [(torch.empty_like(X), torch.empty_like(dY2)) for _ in range(2)]
    copy_s = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def e2e_compute(i):
        step_body(*bufs[i])
        dMh.copy_(ctx.dM, non_blocking=True)

    def issue_copy(i):
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(free[i])            # the step that last read buffer i is done
            bufs[i][0].copy_(Xh, non_blocking=True)
            bufs[i][1].copy_(dY2h, non_blocking=True)
            ready[i].record(copy_s)

    for i in range(2):
        bufs[i][0].copy_(X)
        bufs[i][1].copy_(dY2)
        e2e_compute(i)
    barrier()
    e2e_graphs = [None, None]
    if args.graph:
        for i in range(2):
            e2e_graphs[i] = torch.cuda.CUDAGraph()
            with torch.cuda.graph(e2e_graphs[i]):
                e2e_compute(i)
            e2e_graphs[i].replay()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(2):
        free[i].record(stream)
    if args.e2e_mode == "pipelined":
        issue_copy(0)
    for k in range(args.steps):
        i = k % 2
        if args.e2e_mode == "serial":     # copy, compute, read back, one after the other
            bufs[i][0].copy_(Xh, non_blocking=True)
            bufs[i][1].copy_(dY2h, non_blocking=True)
        elif k + 1 < args.steps:
            issue_copy((k + 1) % 2)
        if args.e2e_mode == "pipelined":
            stream.wait_event(ready[i])
        if e2e_graphs[i] is not None:
            e2e_graphs[i].replay()
        else:
            e2e_compute(i)
        free[i].record(stream)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = world * flops_per_step(T) / (e2e_ms * 1e-3) / 1e12

    # dense cuBLAS layer of the same virtual shapes, same run (context for the metric)
    W1 = ctx.materialize(l1, bf)
    W2 = ctx.materialize(l2, bf)

    def dense_step():
        y1 = X @ W1
        y2 = y1 @ W2
        d1 = dY2 @ W2.t()
        g2 = y1.t() @ dY2
        dx = d1 @ W1.t()
        g1 = X.t() @ d1
        return y2, dx, g1, g2
    for _ in range(3):
        dense_step()
    torch.cuda.synchronize()
    dense_graph = None
    if args.graph:   # same launch discipline as the ROAST step
        dense_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(dense_graph):
            dense_step()
        dense_graph.replay()
        torch.cuda.synchronize()
    d0, d1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dn = []
    for _ in range(max(5, args.steps)):
        flush.zero_()
        d0.record(stream)
        if dense_graph is not None:
            dense_graph.replay()
        else:
            dense_step()
        d1e.record(stream)
        torch.cuda.synchronize()
        dn.append(d0.elapsed_time(d1e))
    dense_ms = float(np.mean(dn))
    dense_tflops = flops_per_step(T) / (dense_ms * 1e-3) / 1e12

    if args.nvtx_step:   # one more eager step inside an NVTX range, for `ncu --nvtx-include roast_step/`
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("roast_step")
        step_body(X, dY2)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    # the oracle baseline on the host cores: rank 0 at N = 1 only (the contract's cpu_baseline)
    cb = cpu_sample(seconds_target=args.cpu_seconds) if not args.no_cpu and world == 1 else None
    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=ms_per_step, higher_is_better=True, scaling="weak", vs_baseline=None, dtype="bf16",
        data="synthetic (M ~ U(-1,1) from synth seed 1; X, dY ~ N(0,1) bf16)",
        config=dict(workload=workload(args.ratio, mem),
                    tokens_per_gpu=T, global_tokens=T * world, ratio=_num(args.ratio), mem_size=mem,
                    l2="flushed between timed steps (256 MB write outside the events)",
                    dm_mode="deterministic" if args.deterministic else "atomic",
                    streams=args.streams, cuda_graph=bool(args.graph),
                    chain=["off", "forward pair", "forward + dX pairs"][args.chain],
                    autotune=["makespan model", "inference-optimal", "training-optimal"][args.autotune],
                    tuned={f"L{i + 1}.{k}": ctx.tuned(mid, j, T) for i, mid in enumerate((l1, l2))
                           for j, k in enumerate(("fwd", "dx", "dm"))},
                    parallelism=f"dp{world}"),
        roofline=dict(bound="tensor", kernel=dom, achieved=achieved, peak=burst, unit="TFLOP/s",
                      frac=achieved / burst, traffic=ncu_traffic(dom),
                      note=f"peak = {src} bf16 burst ({'of measured, MEASURED_PEAKS.json' if src == 'measured' else 'of fallback, B200_PROFILING.md: MEASURED_PEAKS.json absent'}); algorithmic 2*T*H*O = "
                           f"{kind_flop[dom]/1e9:.2f} GFLOP per launch / mean CUDA-event duration",
                      per_kind_ms=kind_ms, sustained_peak=sustained),
        dense_cublas=dict(tflops=dense_tflops, ms_per_step=dense_ms, roast_over_dense=value / world / dense_tflops),
        e2e=dict(value=e2e_value, unit=UNIT, pipeline="H2D of step k+1 on a copy stream overlaps step k "
                 "(double-buffered device inputs); every step's copies inside the timed region",
                 h2d_bytes_per_step=int(Xh.numel() * 2 + dY2h.numel() * 2),
                 d2h_bytes_per_step=int(mem * 4)),
        gpu_launches=int(launches),
        clocks=clk.summary(),
        cpu_baseline=None if cb is None else {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
    )
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="roast", choices=["roast", "reference"])
    ap.add_argument("--deterministic", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--streams", type=int, default=2, choices=[1, 2])
    ap.add_argument("--ratio", type=float, default=RATIO, help="compression (C2 at 10x / 100x / 1000x)")
    ap.add_argument("--e2e-mode", default="pipelined", choices=["pipelined", "serial"],
                    help="e2e: H2D of the next step overlapped with this step's kernels, or in sequence")
    ap.add_argument("--graph", type=int, default=1, choices=[0, 1])
    ap.add_argument("--tuned-file", default=None,
                    help="bench JSON (or its config.tuned dict) whose kernel choices seed the tuner")
    ap.add_argument("--nvtx-step", action="store_true",
                    help="run one extra eager step in NVTX range 'roast_step' (profiling)")
    ap.add_argument("--chain", type=int, default=1, choices=[0, 1, 2],
                    help="1: forward GEMM pair in one launch (roast_linear_fwd_chain); 2: also the dX pair")
    ap.add_argument("--autotune", type=int, default=2, choices=[0, 1, 2],
                    help="kernel-config autotuner: 0 makespan model, 1 inference-optimal, 2 training-optimal")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
