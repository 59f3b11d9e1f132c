#!/usr/bin/env python
"""bench.py — ROAST-MM fwd+bwd effective TFLOP/s on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[1], the metric's config):
BERT-base MLP block, L1 768->3072 and L2 3072->768 in ONE global M (GMS) at 100x
compression (|M| = 47 192 fp32), hash tile 64x64, 8192 tokens per GPU, bf16 operands /
fp32 accumulate.  One step = the whole hot path over one batch:

    Y1 = L1(X); Y2 = L2(Y1)                      (a1, the N-op between them is identity)
    dY1 = L2.dX(dY2); dM += L2.dM(Y1, dY2)       (a2, a3)
    dX  = L1.dX(dY1); dM += L1.dM(X, dY1)        (a2, a3)
    dM  = allreduce(dM)                          (a6; no-op at N = 1)

Effective FLOPs per step per GPU = sum over layers of 6 T H O (ROAST does not
reduce compute).  Multi-GPU: one process per GPU, tokens per GPU fixed (weak scaling), dM
all-reduced with NCCL through the C ABI.  `--gpus N` without torchrun re-launches itself
under torch.distributed.run with N ranks.

`--workload c3` (the strong-scaling headline): the 12-layer BERT-base
encoder (72 ROAST linears in one GMS M at 100x), global 65 536 tokens split over the N ranks,
one training step = forward + backward + (all-reduce + SGD + shadow refresh + dM zeroing in
one roast_grad_exchange_step); reports t_step split into linears / N-ops / exchange /
update and the all-reduce's algbw / busbw.

At N = 1 the default run adds `extra` (about a minute in all): C2 at 10x and 1000x, the
deterministic C2 step, C1's fp32 case, C4 embeddings (GB/s, HBM fraction), C5's |M| endpoints (8 MB and 2 GB)
against cuBLAS, C3 at 8192 tokens (encoder and whole BERT, ROAST vs dense), per-GEMM ROAST /
cuBLAS ratios, the oracle at 1 thread and all cores with the CPU model, and the paper's own
numbers (A100 TF32, context only).

`--impl reference` times the oracle (oracle/, CPU fp64) as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
# C3: BERT-base encoder, 12 layers x {Q, K, V, O: 768x768; FFN1 768x3072; FFN2 3072x768}
C3_D, C3_FF, C3_HEADS, C3_LAYERS, C3_SEQ = 768, 3072, 12, 12, 128
C3_N_LIN = C3_LAYERS * (4 * C3_D * C3_D + 2 * C3_D * C3_FF)   # 84 934 656 ("~85M MM params")

# The paper's own numbers for this path (PAPER.md lines): NVIDIA A100, TF32,
# batch 512, square D x D, Triton ROAST-MM.  Different hardware and precision: context only.
PAPER_CONTEXT = {
    "hardware": "NVIDIA A100 (paper prints 'A100 (48GB)'), TF32, batch 512, square D x D; context only",
    "fwd_ms_D8096": {"pytorch_dense": 0.69, "roast_4MB": 0.99, "hashednet_4MB": 6.20, "cite": "P:408, P:415, P:409"},
    "fwd_ms_D20480": {"pytorch_dense": 3.91, "roast_4MB": 4.83, "roast_512MB": 4.95, "hashednet_512MB": 272.23,
                      "cite": "P:408, P:415, P:420, P:414"},
    "fwd_bwd_ms_D20480": {"dense": 10.68, "roast_4MB": 21.53, "roast_512MB": 27.69, "roast_over_dense_4MB": 0.50,
                          "cite": "P:708/P:732, P:715/P:739, P:720/P:744"},
    "fwd_bwd_eff_tflops_D20480": {"dense": 120.6, "roast_4MB": 59.8, "note": "6*512*D^2/t (BASELINE.md §1.2)"},
    "adam_step_ms_512MB": {"value": 7.89, "cite": "P:792"},
    "claims": "ROAST fwd 1.34x slower than dense on average (P:435); training up to 2x slower at large |M| (P:440)",
}


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


def cpu_model():
    """(model name, logical CPUs usable by this process) of the host."""
    name = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                name = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count()
    return name, n


# ------------------------------------------------------------------------------ reference arm
def cpu_sample(seconds_target=10.0, tokens=256, threads=None):
    """Time the oracle on a bounded sample of the workload: `tokens` of the 8192.  threads:
    limit the BLAS pool (None = all cores)."""
    import numpy as np

    import synth
    from oracle import roast_mm as OM
    mem = synth.mlp_block(args_ratio())["mem_size"]
    M = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    specs = [OM.LinearSpec(H, O, TILE, TILE, mem, synth.HASH_SEED, i) for i, (H, O) in enumerate(LAYERS)]
    X = synth.round_to_bf16(synth.normal(synth.SEED_X, (tokens, 768)).astype(np.float32))
    dY2 = synth.round_to_bf16(synth.normal(synth.SEED_DY, (tokens, 768)).astype(np.float32))
    import contextlib
    limiter = contextlib.nullcontext()
    if threads is not None:
        try:
            from threadpoolctl import threadpool_limits
            limiter = threadpool_limits(limits=threads)
        except Exception:
            pass
    with limiter:
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
        try:
            from threadpoolctl import threadpool_info
            cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
        except Exception:
            cores = os.cpu_count()
    per_step = el / steps
    return dict(value=flops_per_step(tokens) / per_step / 1e12, unit=UNIT, cores=cores, kind="oracle",
                sample=f"MLP block fwd+bwd at T={tokens} of {TOKENS} tokens (oracle cost is linear in T), "
                       f"{steps} steps in {el:.1f}s, fp64 numpy", seconds_per_sample_step=per_step)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cb = cpu_sample(seconds_target=args.cpu_seconds if args.cpu_seconds else max(3.0, 2.0 * args.steps))
    line = dict(metric=METRIC, value=cb["value"], unit=UNIT, n_gpus=world, steps=args.steps,
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


def _events(torch, n):
    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


def graph_of(torch, fn):
    """fn captured in a CUDA graph (one warm-up call first)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    return g


def mean_replay_ms(torch, g, reps, flush, stream):
    """Mean device time of one replay of graph g, L2 flushed (outside the events) before each."""
    import numpy as np
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = _events(torch, 2)
        a.record(stream)
        g.replay()
        b.record(stream)
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in ts]))


class C2Step:
    """The C2 MLP-block step (fwd pair, 2x dX, 2x dM, exchange) on one rank, with its tensors,
    tuned and planned eagerly (kernel- and step-level training-optimal tuning)."""

    def __init__(self, torch, dev, ratio, deterministic=False, autotune=2, chain=1, streams=2, rank=0, world=1,
                 tuned_file=None, flush=None, bwd="fused"):
        import numpy as np

        from paper_2207_10702_b200 import dp
        from paper_2207_10702_b200 import roast as R
        import synth
        self.torch, self.dev, self.chain, self.streams, self.world = torch, dev, chain, streams, world
        # fused: the whole backward as ONE persistent launch (roast_linear_bwd_chain: dY1, dM of
        # L2, dX, dM of L1 co-scheduled; deterministic mode adds the fixed-order reduces)
        self.bwd = bwd
        T = self.T = TOKENS
        self.mem = synth.mlp_block(ratio)["mem_size"]
        M = torch.tensor(synth.uniform(synth.SEED_M, (self.mem,)).astype(np.float32), device=dev)
        self.ctx = ctx = R.Roast(M, TILE, TILE, seed=synth.HASH_SEED, deterministic=deterministic)
        ctx.set_autotune(autotune)   # tuned in the eager warm-up, before graph capture
        dp.init_comm(ctx, rank, world, device=dev)   # NCCL communicator inside libroast (no-op at N = 1)
        self.l1 = ctx.linear(*LAYERS[0])
        self.l2 = ctx.linear(*LAYERS[1])
        bf = torch.bfloat16
        g = torch.Generator(device=dev)
        g.manual_seed(1234 + rank)
        self.X = torch.randn(T, 768, device=dev, generator=g).to(bf)
        self.dY2 = torch.randn(T, 768, device=dev, generator=g).to(bf)
        self.Y1 = torch.empty(T, 3072, device=dev, dtype=bf)
        self.Y2 = torch.empty(T, 768, device=dev, dtype=bf)
        self.dY1 = torch.empty(T, 3072, device=dev, dtype=bf)
        self.dX = torch.empty(T, 768, device=dev, dtype=bf)
        self.flush = flush if flush is not None else torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        self.side = torch.cuda.Stream(device=dev)
        l1, l2, X, dY2, Y1, Y2, dY1, dX = self.l1, self.l2, self.X, self.dY2, self.Y1, self.Y2, self.dY1, self.dX
        if tuned_file:   # reuse a tuning (e.g. the plain bench run's) instead of timing under a profiler
            saved = json.load(open(tuned_file))
            saved = saved.get("config", {}).get("tuned", saved)
            for i, mid in enumerate((l1, l2)):
                for j, k in enumerate(("fwd", "dx", "dm")):
                    v = saved.get(f"L{i + 1}.{k}")
                    if v:
                        ctx.set_tuned(mid, j, T, int(v[0]), int(v[1]))
        if autotune:   # tune every kernel once, sequentially on one stream (no concurrent work skews it)
            ctx.zero_grad()
            ctx.fwd(l1, X, Y1)
            ctx.fwd(l2, Y1, Y2)
            if chain:
                ctx.fwd_chain(l1, l2, X, Y1, Y2)            # plans the chained schedules eagerly
                ctx.bwd_dx_chain(l1, l2, dY2, dY1, dX)
            ctx.bwd_dx(l2, dY2, dY1)
            ctx.bwd_dm(l2, Y1, dY2)
            ctx.bwd_dx(l1, dY1, dX)
            ctx.bwd_dm(l1, X, dY1)
            if self.bwd == "fused":
                ctx.bwd_chain(l1, l2, X, Y1, dY2, dY1, dX)   # plans the fused backward eagerly
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
        # the backward's schedule, training-optimal at the step level: the fused launch unless the
        # separate dX / dM launches on two streams make the whole step faster (e.g. at 1000x the
        # tiny dM's reduce-add hot spot favours spreading the dM GEMMs out)
        if autotune == 2 and not tuned_file and self.bwd == "fused" and not os.environ.get("ROAST_BENCH_KEEP_BWD"):
            t_fused = self.step_ms()
            self.bwd = "streams"
            t_streams = self.step_ms()
            keep_fused = t_fused <= t_streams
            if world > 1:
                import torch.distributed as dist
                flag = torch.tensor([int(keep_fused)], dtype=torch.int32, device=dev)
                dist.broadcast(flag, 0)
                keep_fused = bool(flag.item())
            self.bwd = "fused" if keep_fused else "streams"
        if autotune == 2 and not tuned_file and self.bwd != "fused":
            for mid in (l1, l2):
                wm, nu = ctx.tuned(mid, 1, T)
                if nu == 3:
                    t192 = self.step_ms()
                    ctx.set_tuned(mid, 1, T, wm, 4)
                    t256 = self.step_ms()
                    keep = t192 < t256
                    if world > 1:   # rank 0 decides for everyone (same configuration on every rank)
                        import torch.distributed as dist
                        flag = torch.tensor([int(keep)], dtype=torch.int32, device=dev)
                        dist.broadcast(flag, 0)
                        keep = bool(flag.item())
                    if keep:
                        ctx.set_tuned(mid, 1, T, wm, 3)

    def step_body(self, Xin=None, dY2in=None):
        """One step of the hot path: Y1 = X W1, Y2 = Y1 W2, dY1 = dY2 W2^T, dX = dY1 W1^T,
        dM += scatter(X^T dY1) + scatter(Y1^T dY2), then the dM exchange.  With chain the
        forward pair (and with chain 2 the dX pair) runs as ONE persistent launch.  dX and dM
        of each layer are independent, so with streams 2 every dM GEMM runs on a second
        stream and fills the SMs the dX GEMMs leave idle (roast_linear_bwd_dx / _dm)."""
        torch, ctx, side = self.torch, self.ctx, self.side
        Xin = self.X if Xin is None else Xin
        dY2in = self.dY2 if dY2in is None else dY2in
        l1, l2, Y1, Y2, dY1, dX = self.l1, self.l2, self.Y1, self.Y2, self.dY1, self.dX
        cur = torch.cuda.current_stream()
        ctx.zero_grad()
        if self.chain:
            ctx.fwd_chain(l1, l2, Xin, Y1, Y2)
        else:
            ctx.fwd(l1, Xin, Y1)
            ctx.fwd(l2, Y1, Y2)
        if self.bwd == "fused":
            ctx.bwd_chain(l1, l2, Xin, Y1, dY2in, dY1, dX)   # a2 + a3 of both layers, one launch
        elif self.streams == 2 and self.chain == 2:
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                ctx.bwd_dm(l2, Y1, dY2in)
            ctx.bwd_dx_chain(l1, l2, dY2in, dY1, dX)   # dY1 and dX in one launch
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                ctx.bwd_dm(l1, Xin, dY1)
            cur.wait_stream(side)
        elif self.streams == 2:
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
            if self.chain == 2:
                ctx.bwd_dx_chain(l1, l2, dY2in, dY1, dX)
            else:
                ctx.bwd_dx(l2, dY2in, dY1)
                ctx.bwd_dx(l1, dY1, dX)
            ctx.bwd_dm(l2, Y1, dY2in)
            ctx.bwd_dm(l1, Xin, dY1)
        ctx.allreduce()

    def step_ms(self, reps=15):
        """Median graph-replayed step time (L2 flushed between replays)."""
        torch = self.torch
        for _ in range(3):
            self.step_body()
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_):
            self.step_body()
        ts = []
        stream = torch.cuda.current_stream()
        for _ in range(reps):
            self.flush.zero_()
            a_, b_ = _events(torch, 2)
            a_.record(stream)
            g_.replay()
            b_.record(stream)
            torch.cuda.synchronize()
            ts.append(a_.elapsed_time(b_))
        return sorted(ts)[len(ts) // 2]

    def tuned(self):
        return {f"L{i + 1}.{k}": self.ctx.tuned(mid, j, self.T) for i, mid in enumerate((self.l1, self.l2))
                for j, k in enumerate(("fwd", "dx", "dm"))}


def allreduce_stats(torch, ctx, mem, world, stream, reps=20):
    """Median device time of roast_grad_allreduce alone: algbw = |M| 4 B / t,
    busbw = algbw 2 (W - 1) / W (nccl-tests convention)."""
    import numpy as np
    for _ in range(3):
        ctx.allreduce()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = _events(torch, 2)
        a.record(stream)
        ctx.allreduce()
        b.record(stream)
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ts]))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=stream.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    algbw = mem * 4 / (ms * 1e-3) / 1e9 if ms > 0 else None
    return dict(ms=ms, bytes=mem * 4, algbw_gbs=algbw,
                busbw_gbs=None if algbw is None else algbw * 2 * (world - 1) / world,
                note="median of %d roast_grad_allreduce calls (dense dM, ncclAllReduce fp32 sum)" % reps)


def run_gpu(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    S = C2Step(torch, dev, args.ratio, deterministic=args.deterministic, autotune=args.autotune, chain=args.chain,
               streams=args.streams, rank=rank, world=world, tuned_file=args.tuned_file, flush=flush, bwd=args.bwd)
    ctx, T, mem = S.ctx, S.T, S.mem
    l1, l2, X, dY2, Y1, Y2, dY1, dX = S.l1, S.l2, S.X, S.dY2, S.Y1, S.Y2, S.dY1, S.dX
    step_body = S.step_body

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

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
    starts, ends = _events(torch, args.steps), _events(torch, args.steps)
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
    if S.bwd == "fused":
        calls += [("bwd_fused", lambda: ctx.bwd_chain(l1, l2, X, Y1, dY2, dY1, dX), 4 * gemm_flop)]
    elif args.chain == 2:
        calls += [("dx_chain", lambda: ctx.bwd_dx_chain(l1, l2, dY2, dY1, dX), 2 * gemm_flop)]
    else:
        calls += [("dx", lambda: ctx.bwd_dx(l2, dY2, dY1), gemm_flop), ("dx", lambda: ctx.bwd_dx(l1, dY1, dX), gemm_flop)]
    if S.bwd != "fused":
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
            a, b = _events(torch, 2)
            a.record(stream)
            cg_.replay()
            b.record(stream)
            ev[kind].append((a, b))
    torch.cuda.synchronize()
    kind_ms = {k: float(np.mean([a.elapsed_time(b) for a, b in ev[k]])) for k in kinds}
    # dominant kernel = the kind with the largest share of the step's launch time
    dom = max(kinds, key=lambda k: kind_ms[k] * kind_count[k])
    burst, sustained_peak, hbm, src = load_peaks()
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
    e0, e1 = _events(torch, 2)
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

    # dense cuBLAS layer of the same virtual shapes, same run (context for the metric): one
    # stream, and with the same two-stream overlap of the weight-gradient GEMMs as ROAST
    W1 = ctx.materialize(l1, torch.bfloat16)
    W2 = ctx.materialize(l2, torch.bfloat16)
    side_d = torch.cuda.Stream(device=dev)

    def dense_step():
        y1 = X @ W1
        y2 = y1 @ W2
        d1 = dY2 @ W2.t()
        g2 = y1.t() @ dY2
        dx = d1 @ W1.t()
        g1 = X.t() @ d1
        return y2, dx, g1, g2

    def dense_step_2s():
        cur = torch.cuda.current_stream()
        y1 = X @ W1
        y2 = y1 @ W2
        side_d.wait_stream(cur)
        with torch.cuda.stream(side_d):
            g2 = y1.t() @ dY2
        d1 = dY2 @ W2.t()
        e = torch.cuda.Event()
        e.record(cur)
        dx = d1 @ W1.t()
        side_d.wait_event(e)
        with torch.cuda.stream(side_d):
            g1 = X.t() @ d1
        cur.wait_stream(side_d)
        return y2, dx, g1, g2
    dense = {}
    for name, fn in (("one_stream", dense_step), ("two_streams", dense_step_2s)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g_ = graph_of(torch, fn) if args.graph else None
        dn = []
        for _ in range(max(5, args.steps)):
            flush.zero_()
            a, b = _events(torch, 2)
            a.record(stream)
            if g_ is not None:
                g_.replay()
            else:
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            dn.append(a.elapsed_time(b))
        dense[name] = float(np.mean(dn))
    dense_ms = min(dense.values())
    dense_tflops = flops_per_step(T) / (dense_ms * 1e-3) / 1e12

    if args.nvtx_step:   # one more eager step inside an NVTX range, for `ncu --nvtx-include roast_step/`
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("roast_step")
        step_body(X, dY2)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()

    ar = allreduce_stats(torch, ctx, mem, world, stream) if world > 1 else None
    extra = None
    if world == 1 and args.extras and not args.nvtx_step:
        extra = c2_extras(torch, dev, args, S, flush, stream, W1, W2)

    # sustained (last: it heats the GPU): the same graph back to back for ~args.sustained_seconds
    # (no flush, clocks sampled): the number a long training run sees once power / clocks settle
    sustained = None
    if graph is not None and args.sustained_seconds > 0:
        n_sus = max(50, int(args.sustained_seconds / max(ms_per_step * 1e-3, 1e-6)))
        a, b = _events(torch, 2)
        with ClockSampler(local) as clk_s:
            barrier()
            a.record(stream)
            for _ in range(n_sus):
                graph.replay()
            b.record(stream)
            barrier()
        sus_ms = a.elapsed_time(b) / n_sus
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([sus_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sus_ms = float(tt.item())
        sustained = dict(value=world * flops_per_step(T) / (sus_ms * 1e-3) / 1e12, unit=UNIT, ms_per_step=sus_ms,
                         steps=n_sus, seconds=sus_ms * n_sus / 1e3, l2="not flushed (back-to-back replays)",
                         clocks=clk_s.summary())


    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    # the oracle baseline on the host cores: rank 0 at N = 1 only (the contract's cpu_baseline)
    cb = cpu_sample(seconds_target=args.cpu_seconds) if not args.no_cpu and world == 1 else None
    if extra is not None and cb is not None and not args.no_cpu:
        extra["oracle_cpu"] = oracle_cpu_extra(cb)
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
                    backward="one fused launch (roast_linear_bwd_chain)" if S.bwd == "fused" else
                             "separate dX / dM launches on %d stream(s)" % args.streams,
                    autotune=["makespan model", "inference-optimal", "training-optimal"][args.autotune],
                    tuned=S.tuned(), parallelism=f"dp{world}"),
        roofline=dict(bound="tensor", kernel=dom, achieved=achieved, peak=burst, unit="TFLOP/s",
                      frac=achieved / burst, traffic=ncu_traffic(dom),
                      note=f"peak = {src} bf16 burst ({'of measured, MEASURED_PEAKS.json' if src == 'measured' else 'of fallback, B200_PROFILING.md: MEASURED_PEAKS.json absent'}); algorithmic 2*T*H*O = "
                           f"{kind_flop[dom]/1e9:.2f} GFLOP per launch / mean CUDA-event duration",
                      per_kind_ms=kind_ms, sustained_peak=sustained_peak,
                      frac_of_sustained=achieved / sustained_peak if sustained_peak else None),
        dense_cublas=dict(tflops=dense_tflops, ms_per_step=dense_ms, roast_over_dense=value / world / dense_tflops,
                          ms_per_step_by_schedule=dense, note="the faster of one-stream and two-stream cuBLAS "
                          "(the two-stream one overlaps the weight-gradient GEMMs like ROAST's step)"),
        e2e=dict(value=e2e_value, unit=UNIT, pipeline="H2D of step k+1 on a copy stream overlaps step k "
                 "(double-buffered device inputs); every step's copies inside the timed region",
                 h2d_bytes_per_step=int(Xh.numel() * 2 + dY2h.numel() * 2),
                 d2h_bytes_per_step=int(mem * 4)),
        gpu_launches=int(launches),
        clocks=clk.summary(),
        sustained=sustained,
        allreduce=ar,
        cpu_baseline=None if cb is None else {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        extra=extra,
    )
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def oracle_cpu_extra(cb_all):
    """the oracle at 1 thread and at all cores, with the CPU model."""
    name, ncpu = cpu_model()
    one = cpu_sample(seconds_target=5.0, threads=1)
    return dict(cpu_model=name, logical_cpus=ncpu,
                one_thread=dict(value=one["value"], unit=UNIT, sample=one["sample"]),
                all_cores=dict(value=cb_all["value"], unit=UNIT, threads=cb_all["cores"], sample=cb_all["sample"]),
                note="fp64 numpy oracle (BLAS matmul for the dense passes), reported baseline only")


def c2_extras(torch, dev, args, S, flush, stream, W1, W2):
    """Breadth in the same run (N = 1): per-GEMM ROAST vs cuBLAS, C2 at 10x / 1000x and
    deterministic, C4 embeddings, and the paper's own numbers as context.  Each part is bounded
    (a few seconds); a failure is reported in place instead of failing the bench."""
    import numpy as np
    out = {}
    t0 = time.perf_counter()
    ctx, T = S.ctx, S.T
    l1, l2, X, dY2, Y1, Y2, dY1, dX = S.l1, S.l2, S.X, S.dY2, S.Y1, S.Y2, S.dY1, S.dX
    gemm_flop = 2.0 * T * 768 * 3072
    try:   # per-GEMM: each ROAST call and its cuBLAS counterpart alone, graph-replayed, L2 flushed
        rows = [("fwd L1 768->3072", lambda: ctx.fwd(l1, X, Y1), lambda: torch.matmul(X, W1, out=Y1)),
                ("fwd L2 3072->768", lambda: ctx.fwd(l2, Y1, Y2), lambda: torch.matmul(Y1, W2, out=Y2)),
                ("dX L2 768->3072", lambda: ctx.bwd_dx(l2, dY2, dY1), lambda: torch.matmul(dY2, W2.t(), out=dY1)),
                ("dX L1 3072->768", lambda: ctx.bwd_dx(l1, dY1, dX), lambda: torch.matmul(dY1, W1.t(), out=dX)),
                ("dM L2 3072x768", lambda: ctx.bwd_dm(l2, Y1, dY2), lambda: torch.matmul(Y1.t(), dY2)),
                ("dM L1 768x3072", lambda: ctx.bwd_dm(l1, X, dY1), lambda: torch.matmul(X.t(), dY1))]
        per = {}
        for name, fr, fd in rows:
            r_ms = mean_replay_ms(torch, graph_of(torch, fr), 10, flush, stream)
            d_ms = mean_replay_ms(torch, graph_of(torch, fd), 10, flush, stream)
            per[name] = dict(roast_us=r_ms * 1e3, cublas_us=d_ms * 1e3, roast_tflops=gemm_flop / (r_ms * 1e-3) / 1e12,
                             cublas_tflops=gemm_flop / (d_ms * 1e-3) / 1e12, roast_over_cublas=d_ms / r_ms)
        tot_r = sum(v["roast_us"] for v in per.values())
        tot_d = sum(v["cublas_us"] for v in per.values())
        out["per_gemm"] = dict(gemms=per, sum_roast_us=tot_r, sum_cublas_us=tot_d, roast_over_cublas=tot_d / tot_r,
                               note="each GEMM alone (graph replay, L2 flushed); the step ratio also includes "
                                    "ROAST's chained forward and two-stream backward")
    except Exception as e:  # noqa: BLE001
        out["per_gemm"] = dict(error=repr(e))
    ctx.zero_grad()
    # C2 at the other compressions and in deterministic mode: the same step, a fresh handle each
    variants = {}
    for key, ratio, det in (("10x", 10, False), ("1000x", 1000, False), ("100x_deterministic", 100, True)):
        try:
            V = C2Step(torch, dev, ratio, deterministic=det, autotune=args.autotune, chain=args.chain,
                       streams=args.streams, flush=flush, bwd=args.bwd)
            g = graph_of(torch, V.step_body)
            ms = mean_replay_ms(torch, g, 10, flush, stream)
            variants[key] = dict(value=flops_per_step(T) / (ms * 1e-3) / 1e12, unit=UNIT, ms_per_step=ms,
                                 mem_size=V.mem, dm_mode="deterministic" if det else "atomic", bwd=V.bwd,
                                 tuned=V.tuned())
            V.ctx.close()
            del V, g
        except Exception as e:  # noqa: BLE001
            variants[key] = dict(error=repr(e))
    out["c2_variants"] = variants
    try:
        out["c4_embeddings"] = c4_extra(torch, dev, flush, stream)
    except Exception as e:  # noqa: BLE001
        out["c4_embeddings"] = dict(error=repr(e))
    try:
        out["c5_sweep_endpoints"] = c5_extra(torch)
    except Exception as e:  # noqa: BLE001
        out["c5_sweep_endpoints"] = dict(error=repr(e))
    out["c3_bert_step"] = c3_extra()
    try:
        out["c1_fp32"] = c1_extra(torch)
    except Exception as e:  # noqa: BLE001
        out["c1_fp32"] = dict(error=repr(e))
    out["paper_context"] = PAPER_CONTEXT
    out["seconds"] = time.perf_counter() - t0
    return out


def c5_extra(torch, mems=(2 << 20, 512 << 20), T=16384, D=4096):
    """C5 (BASELINE.json configs[4]) at its two endpoints, |M| = 8 MB (L2-resident) and 2 GB
    (HBM-resident) fp32: one 4096 x 4096 ROAST linear at batch 16384, fwd + bwd (dX and dM on
    two streams, as tools/c5_sweep.py), graph-replayed (the 134 MB activations exceed L2: no
    flush), against dense cuBLAS on the materialised W; plus the touched-only Adam step."""
    bf = torch.bfloat16
    gen = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn(T, D, device="cuda", generator=gen).to(bf)
    dY = torch.randn(T, D, device="cuda", generator=gen).to(bf)
    Y = torch.empty(T, D, device="cuda", dtype=bf)
    dX = torch.empty(T, D, device="cuda", dtype=bf)
    flop = 6.0 * T * D * D
    side = torch.cuda.Stream()
    stream = torch.cuda.current_stream()
    res = {}
    dense_ms = None
    for mem in mems:
        M = torch.rand(mem, device="cuda", generator=gen) * 2 - 1
        ctx = R_mod().Roast(M, 64, 64)
        ctx.set_autotune(2)
        lid = ctx.linear(D, D)
        ctx.fwd(lid, X, Y)
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
        nothing = torch.empty(0, dtype=torch.uint8, device="cuda")
        ms = mean_replay_ms(torch, graph_of(torch, step), 10, nothing, stream)
        if dense_ms is None:
            W = ctx.materialize(lid, bf)

            def dense():
                torch.matmul(X, W, out=Y)
                torch.matmul(dY, W.t(), out=dX)
                torch.matmul(X.t(), dY)
            dense_ms = mean_replay_ms(torch, graph_of(torch, dense), 10, nothing, stream)
            del W
        ctx.optimizer_step(2, 1e-3, step=1, touched_only=True)
        adam_ms = mean_replay_ms(torch, graph_of(torch, lambda: ctx.optimizer_step(2, 1e-3, step=1, touched_only=True)),
                                 5, nothing, stream)
        res["%d_MB" % (mem * 4 >> 20)] = dict(mem_elems=mem, fwd_bwd_ms=ms, tflops=flop / (ms * 1e-3) / 1e12,
                                            dense_tflops=flop / (dense_ms * 1e-3) / 1e12,
                                            roast_over_dense=dense_ms / ms, adam_touched_only_ms=adam_ms)
        ctx.close()
        del M, ctx
        torch.cuda.empty_cache()
    res["config"] = "C5: 4096 x 4096 ROAST-MM, batch 16384, |M| endpoints of the 8 MB - 2 GB sweep (1 GPU)"
    return res


def c1_extra(torch):
    """C1 (BASELINE.json configs[0]): one ROAST linear 256 x 256, batch 64, tile 32 x 32, |M| =
    8192 fp32 (8x), fwd + bwd on the fp32 SIMT path (the oracle-comparison case; its parity is
    tests/test_gpu_parity.py::test_c1_fp32_path).  Latency-bound: no roofline claim."""
    import numpy as np
    import synth
    R = R_mod()
    res = {}
    for det in (False, True):
        M = torch.tensor(synth.uniform(synth.SEED_M, (8192,)).astype(np.float32), device="cuda")
        ctx = R.Roast(M, 32, 32, seed=synth.HASH_SEED, deterministic=det, simt_bf16=True)
        mid = ctx.linear(256, 256)
        X = torch.tensor(synth.uniform(synth.SEED_X, (64, 256)).astype(np.float32), device="cuda")
        dY = torch.tensor(synth.uniform(synth.SEED_DY, (64, 256)).astype(np.float32), device="cuda")
        Y, dX = torch.empty(64, 256, device="cuda"), torch.empty(64, 256, device="cuda")

        def step():
            ctx.zero_grad()
            ctx.fwd(mid, X, Y)
            ctx.bwd(mid, X, dY, dX)
        g = graph_of(torch, step)
        for _ in range(10):
            g.replay()
        a, b = _events(torch, 2)
        a.record()
        for _ in range(200):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 200 * 1e3
        res["deterministic" if det else "atomic"] = dict(us_per_fwd_bwd=us, gflops=6 * 64 * 256 * 256 / us / 1e3)
        ctx.close()
    res["config"] = "C1: 256 x 256 linear, batch 64, tile 32 x 32, |M| = 8192 fp32, fp32 SIMT path (graph replays)"
    return res


def R_mod():
    from paper_2207_10702_b200 import roast as R
    return R


def c3_extra(timeout=180):
    """C3 (BASELINE.json configs[2]) at one GPU, 8192 tokens: the BERT-base encoder step (72
    ROAST linears in one GMS M) and the whole BERT (embeddings and biases via L), each against the
    same model with dense bf16 weights (tools/bert_step.py, separate processes, CUDA graphs)."""
    out = {}
    for key, extra in (("encoder", []), ("encoder_dense", ["--dense"]), ("full_bert", ["--full"]),
                       ("full_bert_dense", ["--full", "--dense"])):
        try:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bert_step.py"), "--steps", "10"] + extra,
                               capture_output=True, text=True, timeout=timeout, cwd=ROOT)
            line = json.loads(r.stdout.strip().splitlines()[-1])
            out[key] = dict(ms_per_step=line["ms_per_step"], tokens_per_s=line["tokens_per_s"],
                            linear_eff_tflops=line["linear_eff_tflops"])
        except Exception as e:  # noqa: BLE001
            out[key] = dict(error=repr(e)[:200])
    try:   # the strong-scaling line's 1-GPU point: 65 536 tokens (bench.py --workload c3)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c3", "--steps", "5",
                            "--warmup", "2", "--no-breakdown"], capture_output=True, text=True, timeout=timeout,
                           cwd=ROOT, env=dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
        line = json.loads(r.stdout.strip().splitlines()[-1])
        out["strong_scaling_1gpu_65536_tokens"] = dict(ms_per_step=line["ms_per_step"], value=line["value"],
                                                       unit=line["unit"], tokens_per_s=line["tokens_per_s"])
    except Exception as e:  # noqa: BLE001
        out["strong_scaling_1gpu_65536_tokens"] = dict(error=repr(e)[:200])
    try:
        out["roast_over_dense_encoder"] = out["encoder_dense"]["ms_per_step"] / out["encoder"]["ms_per_step"]
        out["roast_over_dense_full_bert"] = out["full_bert_dense"]["ms_per_step"] / out["full_bert"]["ms_per_step"]
    except Exception:  # noqa: BLE001
        pass
    return out


def c4_extra(torch, dev, flush, stream, reps=10):
    """C4 (BASELINE.json configs[3]): 26 tables x 10^7 virtual rows x dim 128, chunk 32, 1000x
    (|M| = 133 MB fp32, A = 32), 65 536 uniform single-hot lookups per table, all tables in one
    launch each way.  Algorithmic bytes per lookup: fwd 8 + 512 + 512 = 1032,
    bwd 8 + 512 + 1024 (read-modify-write of dM) = 1544; fraction of the measured HBM peak."""
    import numpy as np

    from paper_2207_10702_b200 import roast as R
    import synth
    tables, rows, dim, Z, batch, align = 26, 10 ** 7, 128, 32, 65536, 32
    mem = synth.compressed_size(tables * rows * dim, 1000, align=align)
    M = torch.tensor(synth.uniform(synth.SEED_M, (mem,)).astype(np.float32), device=dev)
    ctx = R.Roast(M, 64, 64, seed=synth.HASH_SEED, align=align)
    ids = [ctx.embedding(rows, dim, Z) for _ in range(tables)]
    idx = torch.tensor(np.concatenate([synth.uniform_indices(synth.SEED_IDX + t, batch, rows) for t in range(tables)]),
                       device=dev)
    out = torch.empty(tables * batch, dim, device=dev)
    dout = torch.randn(tables * batch, dim, device=dev)
    n = tables * batch
    _, _, hbm, src = load_peaks()
    res = dict(config="26 x 10^7 x 128, chunk 32, 1000x (|M| = %d fp32), %d lookups, uniform" % (mem, n),
               hbm_peak_gbs=hbm, hbm_peak_source=src)
    for name, fn, per in (("fwd", lambda: ctx.emb_fwd_multi(ids, idx, out), 1032),
                          ("bwd", lambda: ctx.emb_bwd_multi(ids, idx, dout), 1544)):
        ms = mean_replay_ms(torch, graph_of(torch, fn), reps, flush, stream)
        gbs = n * per / (ms * 1e-3) / 1e9
        res[name] = dict(us=ms * 1e3, algorithmic_bytes=n * per, gbs=gbs, hbm_frac=gbs / hbm)
    ctx.close()
    return res


# ------------------------------------------------------------------------------ C3 (strong scaling)
def run_gpu_c3(args):
    """BERT-base encoder training step, global tokens split over the ranks."""
    import numpy as np
    import torch

    from paper_2207_10702_b200 import dp, nn as RN, roast as R
    import synth
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    gtok = args.c3_tokens
    if gtok % (world * C3_SEQ):
        raise SystemExit(f"--c3-tokens {gtok} must split into whole sequences of {C3_SEQ} over {world} ranks")
    T = gtok // world
    B, Sq, D = T // C3_SEQ, C3_SEQ, C3_D
    mem = synth.compressed_size(C3_N_LIN, args.ratio)
    M = torch.tensor(synth.uniform(synth.SEED_M, (mem,)).astype(np.float32), device=dev)
    store = R.Roast(M, 64, 64, seed=synth.HASH_SEED)
    store.set_autotune(args.autotune)
    dp.init_comm(store, rank, world, device=dev)
    model = torch.nn.Sequential(*[RN.EncoderLayer(store, D, C3_FF, C3_HEADS) for _ in range(C3_LAYERS)]).to(dev)
    for m in model.modules():
        if isinstance(m, torch.nn.LayerNorm):
            m.to(torch.bfloat16)
    g = torch.Generator(device=dev)
    g.manual_seed(4321 + rank)
    x = torch.randn(B, Sq, D, device=dev, generator=g).to(torch.bfloat16)
    proj = torch.randn(B, Sq, D, device=dev, generator=g).to(torch.bfloat16)   # L = <proj, y> / T_global

    def step(xin=None):
        y = model(x if xin is None else xin)
        loss = (y * proj).float().sum() / gtok
        loss.backward()
        # a6 + a7 in one call: all-reduce of dM, M -= lr dM, bf16 shadow refresh, dM <- 0
        store.exchange_step(R.OPT_SGD, 1e-4, zero_grad=True)
        return loss

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):            # eager warm-up: tuning, lazy state, chain plans
        for _ in range(max(args.warmup, 2)):
            step()
    stream.wait_stream(side)
    barrier()
    l0 = store.launch_count()
    step()
    launches_per_step = store.launch_count() - l0
    barrier()
    # t_step split of one eager step by kernel category (rank 0; torch.profiler, kernel time)
    breakdown = None
    if rank == 0 and not args.no_breakdown:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        cats = {"linears": 0.0, "n_ops": 0.0, "exchange": 0.0, "update": 0.0}
        gemm_ms = 0.0
        for ev in prof.key_averages():
            t = getattr(ev, "device_time_total", getattr(ev, "cuda_time_total", 0.0)) / 1e3
            n = ev.key
            if "roast_mm_sm100" in n or "roast_mix_sm100" in n or "det_reduce" in n:
                cats["linears"] += t
                gemm_ms += t
            elif "nccl" in n.lower() or "pack_kernel" in n:
                cats["exchange"] += t
            elif "opt_kernel" in n or "sync_shadow" in n:
                cats["update"] += t
            elif "memset" not in n.lower() and "memcpy" not in n.lower():
                cats["n_ops"] += t
        top = sorted(((getattr(ev, "device_time_total", getattr(ev, "cuda_time_total", 0.0)) / 1e3, ev.key)
                      for ev in prof.key_averages()), reverse=True)[:20]
        breakdown = dict(ms={k: round(v, 4) for k, v in cats.items()},
                         top_kernels_ms=[[round(t, 4), k[:80]] for t, k in top],
                         note="one eager step under torch.profiler: kernel time by category (launch gaps "
                              "excluded); linears = the tcgen05 GEMMs incl. the fused backward")
        barrier()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        static_loss = step()
    graph.replay()
    barrier()
    starts, ends = _events(torch, args.steps), _events(torch, args.steps)
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            starts[i].record(stream)
            graph.replay()
            ends[i].record(stream)
        barrier()
    total = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    ms = total / args.steps
    flop = 6.0 * gtok * C3_N_LIN
    value = flop / (ms * 1e-3) / 1e12

    # e2e: every step copies its inputs host -> device (pinned) and reads the loss back
    xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    xh.copy_(x)
    ph = torch.empty(proj.shape, dtype=proj.dtype, pin_memory=True)
    ph.copy_(proj)
    lh = torch.empty((), dtype=torch.float32, pin_memory=True)
    barrier()
    a, b = _events(torch, 2)
    a.record(stream)
    for _ in range(args.steps):
        x.copy_(xh, non_blocking=True)
        proj.copy_(ph, non_blocking=True)
        graph.replay()
        lh.copy_(static_loss.detach(), non_blocking=True)
    b.record(stream)
    barrier()
    e2e_ms = a.elapsed_time(b) / args.steps
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    ar = allreduce_stats(torch, store, mem, world, stream)
    roofline = None
    burst, sustained_peak, hbm, src = load_peaks()
    if breakdown is not None and gemm_ms > 0:
        ach = 6.0 * T * C3_N_LIN / (gemm_ms * 1e-3) / 1e12
        roofline = dict(bound="tensor", kernel="roast_mm_sm100 (all GEMM launches of one step)", achieved=ach,
                        peak=burst, unit="TFLOP/s", frac=ach / burst, traffic=None,
                        note=f"6 T n_linear FLOP per rank-step / summed GEMM kernel time of one eager step; "
                             f"peak = {src} bf16 burst")
    if rank == 0:
        line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
                    ms_per_step=ms, higher_is_better=True, scaling="strong", vs_baseline=None, dtype="bf16",
                    data="synthetic (x, proj ~ N(0,1) bf16; M ~ U(-1,1))",
                    config=dict(workload=f"C3 BERT-base encoder training step (12 layers, 72 ROAST linears in one "
                                         f"GMS M), {_num(args.ratio)}x (|M|={mem}), global {gtok} tokens",
                                global_tokens=gtok, tokens_per_gpu=T, ratio=_num(args.ratio), mem_size=mem,
                                virtual_linear_params=C3_N_LIN, l2="inputs and activations > L2 (not flushed)",
                                cuda_graph=True, update="roast_grad_exchange_step: all-reduce + SGD + shadow + zero",
                                parallelism=f"dp{world}"),
                    tokens_per_s=gtok / (ms * 1e-3),
                    breakdown=breakdown, allreduce=ar, roofline=roofline,
                    e2e=dict(value=flop / (e2e_ms * 1e-3) / 1e12, unit=UNIT,
                             h2d_bytes_per_step=int(world * (xh.numel() + ph.numel()) * 2),
                             d2h_bytes_per_step=4 * world),
                    gpu_launches=int(launches_per_step * args.steps), clocks=clk.summary(),
                    note="value = 6 x global tokens x 84.9M linear params / t_step (N-ops timed, not counted)")
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ launcher
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(args_gpus):
    """`--gpus N` (N > 1) outside torchrun: re-run this script under torch.distributed.run with N
    ranks (one process per GPU, 127.0.0.1 rendezvous) and return its exit code.  Only rank 0
    prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args_gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stderr.write("[bench] launching %d ranks: %s\n" % (args_gpus, " ".join(cmd)))
    return subprocess.call(cmd, cwd=ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="N ranks (one per GPU); without torchrun, N > 1 re-launches under torch.distributed.run")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="roast", choices=["roast", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c3"],
                    help="c2: BASELINE configs[1] MLP block (weak scaling); c3: BERT-base encoder (strong scaling)")
    ap.add_argument("--deterministic", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extras", type=int, default=1, choices=[0, 1],
                    help="N = 1: per-GEMM ratios, C2 10x / 1000x / deterministic, C4, oracle timings, paper context")
    ap.add_argument("--sustained-seconds", type=float, default=2.0,
                    help="also replay the step back to back for this long and report it as `sustained`")
    ap.add_argument("--streams", type=int, default=2, choices=[1, 2])
    ap.add_argument("--bwd", default="fused", choices=["fused", "streams"],
                    help="backward: one fused launch (roast_linear_bwd_chain) or separate dX / dM launches")
    ap.add_argument("--ratio", type=float, default=RATIO, help="compression (C2 at 10x / 100x / 1000x)")
    ap.add_argument("--c3-tokens", type=int, default=65536, help="C3 global tokens (512 x 128), split over ranks")
    ap.add_argument("--no-breakdown", action="store_true", help="C3: skip the profiler breakdown step")
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
    if "WORLD_SIZE" not in os.environ:
        if args.gpus is not None and args.gpus > 1:
            sys.exit(spawn(args.gpus))
    else:
        world = int(os.environ["WORLD_SIZE"])
        if args.gpus is not None and args.gpus != world:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}\n")
            sys.exit(2)
        sys.stderr.write("[bench] rank %s of %d\n" % (os.environ.get("RANK", "0"), world))
    if args.gpus is None:
        args.gpus = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c3":
        run_gpu_c3(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
