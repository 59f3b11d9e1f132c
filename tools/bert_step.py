"""C3 (BASELINE.json configs[2]): full BERT-base-shaped encoder training step, all 72 linears
(12 layers x Q, K, V, O, FFN1, FFN2) ROAST-hashed into ONE global M at 100x
(|M| = 849 352 fp32), data parallel: per-GPU batch 64 x 128 tokens, dM all-reduced with
NCCL inside libroast, SGD on M + bf16 shadow refresh + dM zeroing fused in one kernel
(roast_grad_exchange_step).

    python tools/bert_step.py [--steps 10] [--dense]          (1 GPU)
    torchrun --nproc-per-node N tools/bert_step.py             (N GPUs, weak scaling)

Reports tokens/s, ms per step and the linears' effective TFLOP/s (6 T n_linear_params per
step); --dense runs the same model with dense bf16 nn.Linear weights for comparison.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_10702_b200 import dp, nn as RN, roast as R  # noqa: E402

D, FF, HEADS, LAYERS = 768, 3072, 12, 12
N_LIN = LAYERS * (4 * D * D + 2 * D * FF)   # 84 934 656 ("~85M MM params")


class DenseLayer(torch.nn.Module):
    """The same layer with dense bf16 weights; Q, K, V fused into one 768 x 2304 Linear exactly
    as the ROAST layer fuses them (one GEMM each way), so the comparison is like for like."""

    def __init__(self, bias=False):
        super().__init__()
        L = lambda i, o: torch.nn.Linear(i, o, bias=bias, dtype=torch.bfloat16)  # noqa: E731
        self.qkv_dense, self.o, self.ff1, self.ff2 = L(D, 3 * D), L(D, D), L(D, FF), L(FF, D)
        self.ln1 = RN.LayerNorm(D, dtype=torch.bfloat16)   # the same LayerNorm kernels as the ROAST layer
        self.ln2 = RN.LayerNorm(D, dtype=torch.bfloat16)

    forward = RN.EncoderLayer.forward
    _qkv = RN.EncoderLayer._qkv
    _qkv_packed = RN.EncoderLayer._qkv_packed
    heads = HEADS


class DenseBert(torch.nn.Module):
    """The --full model with dense torch weights: nn.Embedding word / position / type,
    LayerNorm, 12 layers with biased bf16 nn.Linear."""

    def __init__(self, vocab=30522, max_pos=512):
        super().__init__()
        self.word = torch.nn.Embedding(vocab, D)
        self.pos = torch.nn.Embedding(max_pos, D)
        self.tok_type = torch.nn.Embedding(2, D)
        self.ln = RN.LayerNorm(D)
        self.layers = torch.nn.ModuleList([DenseLayer(bias=True) for _ in range(LAYERS)])

    def forward(self, ids, types):
        B, S = ids.shape
        pos = torch.arange(S, device=ids.device).expand(B, S)
        x = self.ln(self.word(ids) + self.pos(pos) + self.tok_type(types)).to(torch.bfloat16)
        for layer in self.layers:
            x = layer(x)
        return x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--ratio", type=float, default=100)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--graph", type=int, default=1, choices=[0, 1],
                    help="capture the whole training step (fwd + bwd + all-reduce + update) in a CUDA graph")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--autotune", type=int, default=2, choices=[0, 1, 2],
                    help="kernel-configuration tuning: 0 makespan model, 1 inference-, 2 training-optimal")
    ap.add_argument("--breakdown", action="store_true",
                    help="SURVEY §8(d): split one step's GPU time into linears / N-ops / exchange / update")
    ap.add_argument("--full", action="store_true",
                    help="whole BERT-base: word/pos/type embeddings and biases via L too (NEXT #3)")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(1234 + rank)
    B, S = args.batch, args.seq
    T = B * S
    x = torch.randn(B, S, D, device=dev, dtype=torch.bfloat16)
    proj = torch.randn(B, S, D, device=dev, dtype=torch.bfloat16)   # L = <proj, y> / T
    ids = torch.randint(0, 30522, (B, S), device=dev)
    types = torch.randint(0, 2, (B, S), device=dev)
    n_virtual = RN.bert_param_count() if args.full else N_LIN
    if args.dense:
        if args.full:
            model = DenseBert().to(dev)
        else:
            model = torch.nn.Sequential(*[DenseLayer() for _ in range(LAYERS)]).to(dev)
        opt = torch.optim.SGD(model.parameters(), lr=1e-4)
        store = None
    else:
        mem = synth.compressed_size(n_virtual, args.ratio)
        M = (torch.rand(mem, device=dev) * 2 - 1).contiguous()
        store = R.Roast(M, 64, 64, seed=synth.HASH_SEED)
        store.set_autotune(args.autotune)   # tuned during the eager warm-up, before capture
        store.batch_biases = True           # 72 biases via L: one lookup / one scatter per step
        dp.init_comm(store, rank, world, device=dev)
        if args.full:
            model = RN.RoastBert(store).to(dev)
        else:
            model = torch.nn.Sequential(*[RN.EncoderLayer(store, D, FF, HEADS) for _ in range(LAYERS)]).to(dev)
            for m in model.modules():
                if isinstance(m, torch.nn.LayerNorm):
                    m.to(torch.bfloat16)

    def step():
        y = model(ids, types) if args.full else model(x)
        loss = (y * proj).float().sum() / T
        if store is None:
            opt.zero_grad(set_to_none=False)
            loss.backward()
            if world > 1:
                import torch.distributed as dist
                for p in model.parameters():
                    dist.all_reduce(p.grad)
            opt.step()
        else:
            loss.backward()                # dM starts zeroed: the exchange step below zeroes it
            # a6 + a7 in one call: ncclAllReduce of dM (or of its packed touched set), then
            # M -= lr dM, bf16 shadow refresh and dM <- 0 in the same pass
            store.exchange_step(R.OPT_SGD, 1e-4, zero_grad=True)
        return loss

    side = torch.cuda.Stream(device=dev) if args.graph else torch.cuda.current_stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):          # eager warm-up (also allocates grads / lazy state)
        for _ in range(args.warmup):
            step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    if args.breakdown and rank == 0:       # GPU time of one eager step by kernel category
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        cats = {"linears (ROAST-MM / dense GEMM)": 0.0, "embeddings + biases via L": 0.0, "exchange": 0.0,
                "update + shadow": 0.0, "N-ops (attention, LayerNorm, GELU, elementwise)": 0.0}
        for ev in prof.key_averages():
            t = getattr(ev, "device_time_total", getattr(ev, "cuda_time_total", 0.0)) / 1e3   # ms
            n = ev.key
            if "roast_mm_sm100" in n or "gemm" in n.lower() or "sm90_xmma" in n or "cutlass" in n.lower() or "nvjet" in n:
                cats["linears (ROAST-MM / dense GEMM)"] += t
            elif "embed" in n or "colsum" in n or "bias" in n:
                cats["embeddings + biases via L"] += t
            elif "nccl" in n.lower() or "pack_kernel" in n:
                cats["exchange"] += t
            elif "opt_kernel" in n or "sync_shadow" in n or "Sgd" in n or "sgd" in n or "foreach" in n:
                cats["update + shadow"] += t
            elif "memset" not in n.lower() and "memcpy" not in n.lower():
                cats["N-ops (attention, LayerNorm, GELU, elementwise)"] += t
        print(json.dumps(dict(breakdown_ms={k: round(v, 3) for k, v in cats.items()},
                              impl="dense-torch" if args.dense else "roast", full=bool(args.full),
                              note="one eager step under torch.profiler (kernel time; launch gaps excluded)")))
    if args.profile and rank == 0:         # top GPU kernels of one eager step
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25), file=sys.stderr)
    run = step
    if args.graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            static_loss = step()
        run = lambda: (g.replay(), static_loss)[1]   # noqa: E731
        run()
        torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        loss = run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        print(json.dumps(dict(config="C3 BERT-base encoder step, 72 linears in one GMS M" +
                              (" + word/pos/type embeddings and biases via L" if args.full else ""),
                              virtual_params=n_virtual, cuda_graph=bool(args.graph),
                              impl="dense-torch" if args.dense else "roast", ratio=args.ratio,
                              mem_size=None if store is None else store.mem_size, n_gpus=world,
                              tokens_per_gpu=T, ms_per_step=ms, tokens_per_s=world * T / (ms * 1e-3),
                              linear_eff_tflops=world * 6.0 * T * N_LIN / (ms * 1e-3) / 1e12,
                              loss=float(loss.detach()))))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
