"""Long randomized parity campaign on the GPU (a tool, not a test: minutes of cases).

Every case draws a random geometry and mode, runs it through libroast's C ABI, and compares with
the fp64 oracle (oracle/, P:294-313 / P:338-346 / P:268-276) at the bars of the parity suite
(bf16 1e-2, fp32 1e-5, embeddings forward bit-exact, backward 1e-5):
  linear    fwd / dX / dM of one module, forced kernel configuration, fast or deterministic mode
  chain     roast_linear_fwd_chain + roast_linear_bwd_chain (the bench's launches) on random MLP shapes
  act       fused GELU forward / GELU' dX and the residual dX epilogue
  emb       multi-table embedding forward / backward, uniform or Zipf rows, fast or deterministic
|M| is drawn from tiny (shadow / dM replicas) to large.  Prints one JSON line per failing case and
a summary line; exit code 1 if any case failed.

    python tools/fuzz_long.py [seconds] [seed]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import embedding as OE  # noqa: E402
from oracle import roast_mm as OM  # noqa: E402
from paper_2207_10702_b200 import roast as R  # noqa: E402

HS = synth.HASH_SEED
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
rng = np.random.default_rng(seed)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))


def bf16(sd, shape):
    return synth.round_to_bf16(synth.normal(sd, shape).astype(np.float32))


def dev(a, dt):
    return torch.tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def pick_mem(n_virtual):
    kind = rng.integers(0, 3)
    if kind == 0:      # tiny: shadow and dM replicas
        return int(max(4096 + 8, rng.integers(4100, 16000)) // 8 * 8)
    if kind == 1:
        return int(rng.integers(20_000, 300_000) // 8 * 8)
    return int(max(8192, n_virtual // int(rng.choice([2, 10]))) // 8 * 8)


def case_linear(i):
    H, O = 64 * int(rng.integers(1, 33)), 64 * int(rng.integers(1, 33))
    T = int(rng.integers(1, 3000))
    det = bool(rng.random() < 0.3)
    mem = pick_mem(H * O)
    M_np = synth.uniform(synth.SEED_M + i, (mem,)).astype(np.float32)
    ctx = R.Roast(dev(M_np, torch.float32), 64, 64, seed=HS, deterministic=det)
    mid = ctx.linear(H, O)
    wm = int(rng.integers(1, 3))
    ctx.set_tuned(mid, 0, T, wm, 3 if (wm == 2 and O % 192 == 0 and rng.random() < 0.5) else 4)
    ctx.set_tuned(mid, 1, T, wm, 3 if (wm == 2 and H % 192 == 0 and rng.random() < 0.5) else 4)
    ctx.set_tuned(mid, 2, T, int(rng.integers(1, 3)), int(rng.integers(1, 5)))
    X_np, dY_np = bf16(synth.SEED_X + i, (T, H)), bf16(synth.SEED_DY + i, (T, O))
    X, dY = dev(X_np, torch.bfloat16), dev(dY_np, torch.bfloat16)
    ctx.zero_grad()
    Y = ctx.fwd(mid, X)
    dX = ctx.bwd(mid, X, dY)
    torch.cuda.synchronize()
    ctx.check()
    sp = OM.LinearSpec(H, O, 64, 64, mem, HS, mid)
    errs = dict(Y=rel(f64(Y), sp.forward(X_np, M_np, True)), dX=rel(f64(dX), sp.backward_dx(dY_np, M_np, True)),
                dM=rel(ctx.dM.cpu().numpy(), sp.backward_dm(X_np, dY_np)))
    ctx.close()
    return dict(kind="linear", H=H, O=O, T=T, mem=mem, det=det, wm=wm), errs, 1e-2


def case_chain(i):
    H = 256 * int(rng.integers(1, 5))
    F = 256 * int(rng.integers(1, 17))
    T = int(rng.integers(1, 4097))
    det = bool(rng.random() < 0.3)
    mem = pick_mem(2 * H * F)
    M_np = synth.uniform(synth.SEED_M + i, (mem,)).astype(np.float32)
    ctx = R.Roast(dev(M_np, torch.float32), 64, 64, seed=HS, deterministic=det)
    ctx.set_autotune(0)
    a, b = ctx.linear(H, F), ctx.linear(F, H)
    X_np, dY_np = bf16(synth.SEED_X + i, (T, H)), bf16(synth.SEED_DY + i, (T, H))
    X, dY = dev(X_np, torch.bfloat16), dev(dY_np, torch.bfloat16)
    ctx.zero_grad()
    Ya, Yb = ctx.fwd_chain(a, b, X)
    dYa, dXa = ctx.bwd_chain(a, b, X, Ya, dY)
    torch.cuda.synchronize()
    ctx.check()
    sa, sb = OM.LinearSpec(H, F, 64, 64, mem, HS, a), OM.LinearSpec(F, H, 64, 64, mem, HS, b)
    Ya_np = f64(Ya)
    dYa_o = sb.backward_dx(dY_np, M_np, True)
    errs = dict(Ya=rel(Ya_np, sa.forward(X_np, M_np, True)), Yb=rel(f64(Yb), sb.forward(Ya_np, M_np, True)),
                dYa=rel(f64(dYa), dYa_o), dXa=rel(f64(dXa), sa.backward_dx(f64(dYa), M_np, True)),
                dM=rel(ctx.dM.cpu().numpy(), sb.backward_dm(Ya_np, dY_np) + sa.backward_dm(X_np, f64(dYa))))
    ctx.close()
    return dict(kind="chain", H=H, F=F, T=T, mem=mem, det=det), errs, 1e-2


def gelu(x):
    return 0.5 * x * (1 + np.tanh(np.sqrt(2 / np.pi) * (x + 0.044715 * x ** 3)))


def gelu_grad(x):
    t = np.tanh(np.sqrt(2 / np.pi) * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * np.sqrt(2 / np.pi) * (1 + 3 * 0.044715 * x * x)


def case_act(i):
    H = 64 * int(rng.integers(1, 25))
    O = 192 * int(rng.integers(1, 9)) if rng.random() < 0.5 else 64 * int(rng.integers(1, 33))
    T = int(rng.integers(1, 3000))
    mem = pick_mem(H * O)
    M_np = synth.uniform(synth.SEED_M + i, (mem,)).astype(np.float32)
    ctx = R.Roast(dev(M_np, torch.float32), 64, 64, seed=HS)
    mid = ctx.linear(H, O)
    sp = OM.LinearSpec(H, O, 64, 64, mem, HS, mid)
    X_np, dY_np, U_np = bf16(synth.SEED_X + i, (T, H)), bf16(synth.SEED_DY + i, (T, O)), bf16(synth.SEED_X + 99 + i, (T, H))
    X, dY, U = dev(X_np, torch.bfloat16), dev(dY_np, torch.bfloat16), dev(U_np, torch.bfloat16)
    for _ in range(2):   # the first call tunes the unit width
        Y, A = ctx.fwd_act(mid, X)
        dXg = ctx.bwd_dx_act(mid, dY, U)
        dXr = ctx.bwd_dx_act(mid, dY, U, act=R.ACT_RESIDUAL)
    plain = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    ctx.bwd_dx(mid, dY, plain)
    torch.cuda.synchronize()
    ctx.check()
    Y_np = f64(Y)
    dx_o = sp.backward_dx(dY_np, M_np, True)
    errs = dict(Y=rel(Y_np, sp.forward(X_np, M_np, True)), A=rel(f64(A), gelu(Y_np)),
                dX_gelu=rel(f64(dXg), dx_o * gelu_grad(U_np.astype(np.float64))),
                dX_res=rel(f64(dXr), dx_o + U_np), res_bits=float(not torch.equal(dXr, plain + U)))
    ctx.close()
    return dict(kind="act", H=H, O=O, T=T, mem=mem), errs, 1e-2


def case_emb(i):
    nt = int(rng.integers(1, 6))
    d = int(rng.choice([32, 64, 128, 256]))
    Z = int(rng.choice([z for z in (8, 16, 32, 64) if d % z == 0]))
    rows = int(rng.choice([50, 10 ** 4, 10 ** 7]))
    n = int(rng.integers(0, 5000))
    det = bool(rng.random() < 0.5)
    mem = pick_mem(10 ** 6)
    M_np = synth.uniform(synth.SEED_M + i, (mem,)).astype(np.float32)
    ctx = R.Roast(dev(M_np, torch.float32), 64, 64, seed=HS, deterministic=det)
    mids = [ctx.embedding(rows, d, Z) for _ in range(nt)]
    if rng.random() < 0.5:
        idx_np = rng.integers(0, rows, (nt, n))
    else:   # Zipf-hot rows
        idx_np = np.minimum(rng.zipf(1.05, (nt, n)) - 1, rows - 1)
    dout_np = synth.normal(synth.SEED_DY + i, (nt, n, d)).astype(np.float32)
    idx = torch.tensor(idx_np, dtype=torch.int64, device="cuda")
    dout = torch.tensor(dout_np, device="cuda")
    ctx.zero_grad()
    out = ctx.emb_fwd_multi(mids, idx)
    ctx.emb_bwd_multi(mids, idx, dout)
    torch.cuda.synchronize()
    ctx.check()
    out_np = out.cpu().numpy().reshape(nt, n, d)
    ref_dM = np.zeros(mem)
    fwd_bits = 0.0
    for t, m in enumerate(mids):
        sp = OE.EmbeddingSpec(rows, d, Z, mem, HS, m)
        if n:
            fwd_bits += float(not np.array_equal(out_np[t], sp.forward(idx_np[t], M_np)))
            sp.backward(idx_np[t], dout_np[t], ref_dM)
    errs = dict(fwd_bits=fwd_bits, dM=rel(ctx.dM.cpu().numpy(), ref_dM) if n else 0.0)
    ctx.close()
    return dict(kind="emb", nt=nt, d=d, Z=Z, rows=rows, n=n, mem=mem, det=det), errs, 1e-5


cases = [case_linear, case_chain, case_act, case_emb]
t0 = time.time()
counts, fails = {}, 0
i = 0
while time.time() - t0 < budget:
    fn = cases[i % len(cases)]
    try:
        where, errs, tol = fn(i)
        bad = {k: v for k, v in errs.items() if v > (0 if k.endswith("bits") else tol)}
    except Exception as e:  # noqa: BLE001  (a raised error is a failure of the case, reported)
        where, bad = dict(kind=fn.__name__, case=i), {"exception": repr(e)[:300]}
    counts[where["kind"]] = counts.get(where["kind"], 0) + 1
    if bad:
        fails += 1
        print(json.dumps(dict(fail=True, case=i, where=where, bad=bad)), flush=True)
    i += 1
print(json.dumps(dict(summary=True, seed=seed, seconds=round(time.time() - t0, 1), cases=i, by_kind=counts,
                      failures=fails)), flush=True)
sys.exit(1 if fails else 0)
