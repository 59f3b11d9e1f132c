"""Debug: per-linear dM of the autograd composition vs the oracle on the SAME captured (X, dY)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import roast_mm as OM  # noqa: E402
from paper_2207_10702_b200 import nn as RN, roast as R  # noqa: E402

d, ff, heads, B, S = 256, 512, 4, 2, 128
n = 4 * d * d + 2 * d * ff
mem = synth.compressed_size(n, 8)
M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
store = R.Roast(torch.tensor(M_np, device="cuda"), 64, 64, seed=synth.HASH_SEED)
layer = RN.EncoderLayer(store, d, ff, heads).cuda()
for m in layer.modules():
    if isinstance(m, torch.nn.LayerNorm):
        m.to(torch.bfloat16)
captured = []
orig = store.bwd_dm


def spy(mid, X, dY, stream=None):
    captured.append((mid, X.float().cpu().numpy().astype(np.float64), dY.float().cpu().numpy().astype(np.float64)))
    return orig(mid, X, dY, stream)


store.bwd_dm = spy
x = torch.randn(B, S, d, device="cuda").to(torch.bfloat16)
store.zero_grad()
y = layer(x)
(0.5 * (y.float() ** 2).sum()).backward()
torch.cuda.synchronize()
dM = store.dM.cpu().numpy().astype(np.float64)
ref = np.zeros(mem)
for mid, X, dY in captured:
    _, H, O = store.dims[mid]
    spec = OM.LinearSpec(H, O, 64, 64, mem, synth.HASH_SEED, mid)
    part = spec.backward_dm(X, dY)
    ref += part
    print(mid, H, O, X.shape, dY.shape, "norm part", np.linalg.norm(part))
print("rel err library vs oracle on captured inputs:", np.linalg.norm(dM - ref) / np.linalg.norm(ref))
# single module check via a fresh store
for mid, X, dY in captured[:2]:
    store.zero_grad()
    orig(mid, torch.tensor(X, device="cuda").to(torch.bfloat16), torch.tensor(dY, device="cuda").to(torch.bfloat16))
    torch.cuda.synchronize()
    _, H, O = store.dims[mid]
    spec = OM.LinearSpec(H, O, 64, 64, mem, synth.HASH_SEED, mid)
    r1 = spec.backward_dm(X, dY)
    g1 = store.dM.cpu().numpy()
    print("single", mid, np.linalg.norm(g1 - r1) / np.linalg.norm(r1))

# dense fp32 reference exactly as tests/test_gpu_model.py
lins = [layer.q, layer.k, layer.v, layer.o, layer.ff1, layer.ff2]
lam = lambda l: OM.LinearSpec(store.dims[l.mid][1], store.dims[l.mid][2], 64, 64, mem, synth.HASH_SEED, l.mid).lam  # noqa
W = [torch.nn.Parameter(store.materialize(l.mid, torch.bfloat16).float() * lam(l)) for l in lins]
xr = x.float()
def split(t):
    return t.reshape(B, S, heads, d // heads).transpose(1, 2)
a = torch.nn.functional.scaled_dot_product_attention(split(xr @ W[0]), split(xr @ W[1]), split(xr @ W[2]))
a = a.transpose(1, 2).reshape(B, S, d)
h1 = torch.nn.functional.layer_norm(xr + a @ W[3], (d,))
yr = torch.nn.functional.layer_norm(h1 + torch.nn.functional.gelu(h1 @ W[4]) @ W[5], (d,))
(0.5 * (yr ** 2).sum()).backward()
print("n captured", len(captured), "y rel err", float((y.float() - yr).norm() / yr.norm()))
for l, w in zip(lins, W):
    _, H, O = store.dims[l.mid]
    spec = OM.LinearSpec(H, O, 64, 64, mem, synth.HASH_SEED, l.mid)
    r = spec.scatter(w.grad.double().cpu().numpy(), np.zeros(mem))
    cap = [c for c in captured if c[0] == l.mid]
    o = spec.backward_dm(cap[0][1], cap[0][2]) if cap else np.zeros(mem)
    print(l.mid, "dense-ref norm", np.linalg.norm(r), "captured-oracle norm", np.linalg.norm(o),
          "rel", np.linalg.norm(o - r) / max(np.linalg.norm(r), 1e-30))
