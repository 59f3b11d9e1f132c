"""End-to-end composition check (GPU): a BERT encoder layer whose six linears are ROAST
linears in one GMS store, trained through torch autograd + the C ABI, against the same
model in fp32 torch autograd with the recovered weights materialised densely.

The dense reference weights, biases and embedding tables are built by the oracle's own
materialisation (oracle/), never read back from the library.  The reference dM is the paper's gradient rule applied to the dense model's weight
gradients: dM[slot] = sum over (i, j) mapped to slot of lambda * g * dL/dW[i, j]
(R12), scattered by the oracle (oracle/roast_mm.py).  Activations are bf16 on
the ROAST side (fp32 in the reference), so the tolerance is a composition bound (3e-2),
not the per-operation 1e-2 of the parity tests.
"""
import numpy as np
import pytest

import synth
from oracle import roast_mm as OM

pytestmark = pytest.mark.gpu


def test_encoder_layer_gradients_match_dense_autograd():
    import torch
    from paper_2207_10702_b200 import nn as RN, roast as R
    torch.manual_seed(0)
    d, ff, heads, B, S = 256, 512, 4, 2, 128
    n = 4 * d * d + 2 * d * ff
    mem = synth.compressed_size(n, 8)
    M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    M = torch.tensor(M_np, device="cuda")
    store = R.Roast(M, 64, 64, seed=synth.HASH_SEED)
    layer = RN.EncoderLayer(store, d, ff, heads).cuda()
    for m in layer.modules():
        if isinstance(m, torch.nn.LayerNorm):
            m.to(torch.bfloat16)
    x = torch.randn(B, S, d, device="cuda").to(torch.bfloat16)
    Rw = torch.randn(B, S, d, device="cuda")       # L = <R, y>: not invariant under the final LayerNorm
    store.zero_grad()
    y = layer(x)
    loss = (y.float() * Rw).sum()
    loss.backward()
    store.flush_bias_grads()
    torch.cuda.synchronize()
    dM = store.dM.cpu().numpy().astype(np.float64)

    # dense fp32 reference with W = lambda * g * bf16(M) (the tensor-core operand, R18)
    lins = [layer.q, layer.k, layer.v, layer.o, layer.ff1, layer.ff2]
    W = [torch.nn.Parameter(oracle_weight(store, l, M_np)) for l in lins]
    xr = x.float()

    def lin(t, i):
        return t @ W[i]

    def split(t):
        return t.reshape(B, S, heads, d // heads).transpose(1, 2)
    a = torch.nn.functional.scaled_dot_product_attention(split(lin(xr, 0)), split(lin(xr, 1)), split(lin(xr, 2)))
    a = a.transpose(1, 2).reshape(B, S, d)
    h1 = torch.nn.functional.layer_norm(xr + lin(a, 3), (d,))
    yr = torch.nn.functional.layer_norm(h1 + lin(torch.nn.functional.gelu(lin(h1, 4), approximate="tanh"), 5), (d,))
    lr = (yr * Rw).sum()
    lr.backward()
    assert abs(float(loss) - float(lr)) <= 2e-2 * float((yr.abs() * Rw.abs()).sum())
    dM_ref = np.zeros(mem)
    for l, w in zip(lins, W):
        _, H, O = store.dims[l.mid]
        spec = OM.LinearSpec(H, O, 64, 64, mem, synth.HASH_SEED, l.mid)
        spec.scatter(w.grad.double().cpu().numpy(), dM_ref)
    err = np.linalg.norm(dM - dM_ref) / np.linalg.norm(dM_ref)
    assert err < 3e-2, err


def oracle_weight(store, lin, M_np):
    """W = lambda * g * bf16(M) (the tensor-core operand, R18) built by the ORACLE's
    materialisation (oracle/roast_mm.py), fp32 on the GPU."""
    import torch
    _, H, O = store.dims[lin.mid]
    spec = OM.LinearSpec(H, O, 64, 64, len(M_np), synth.HASH_SEED, lin.mid)
    return torch.tensor(np.float64(spec.lam) * spec.materialize(M_np, "operand"), dtype=torch.float32, device="cuda")


def oracle_bias(store, lin, M_np):
    """A bias via L (R24): row 0 of its own 1 x O embedding, lambda from the linear's fan-in,
    recovered by the oracle (oracle/embedding.py)."""
    import torch
    from oracle import embedding as OE
    _, H, O = store.dims[lin.mid]
    v = OE.EmbeddingSpec(1, O, 64, len(M_np), synth.HASH_SEED, lin.bias.mid, fan_in=H).forward(
        np.zeros(1, np.int64), M_np.astype(np.float64))[0]
    return torch.tensor(v, dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("batch_biases", [False, True])
def test_roast_bert_embeddings_and_biases_match_dense_autograd(batch_biases):
    """NEXT #3: word / position / type embeddings and every linear's bias via L, plus the
    linears via ROAST-MM, all in ONE GMS store; dM of the whole model vs the
    dense fp32 model built from the recovered weights, its gradients scattered by the oracle
    (linears: the MM rule; embeddings and biases: the L rule)."""
    import torch
    from oracle import embedding as OE
    from paper_2207_10702_b200 import nn as RN, roast as R
    torch.manual_seed(1)
    vocab, max_pos, d, ff, heads, B, S, Z = 1000, 128, 256, 512, 4, 2, 64, 32
    n = RN.bert_param_count(vocab, d, ff, 1, max_pos, 2, True)
    mem = synth.compressed_size(n, 8)
    M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    M = torch.tensor(M_np, device="cuda")
    store = R.Roast(M, 64, 64, seed=synth.HASH_SEED)
    store.batch_biases = batch_biases   # True: one multi-table lookup / scatter for all biases
    model = RN.RoastBert(store, vocab, d, ff, heads, 1, max_pos, 2, Z, bias=True).cuda()
    ids = torch.randint(0, vocab, (B, S), device="cuda")
    types = torch.randint(0, 2, (B, S), device="cuda")
    Rw = torch.randn(B, S, d, device="cuda")
    store.zero_grad()
    y = model(ids, types)
    loss = (y.float() * Rw).sum()
    loss.backward()
    store.flush_bias_grads()
    torch.cuda.synchronize()
    dM = store.dM.cpu().numpy().astype(np.float64)

    # dense fp32 reference from the recovered weights
    emb = model.emb
    tables = [torch.nn.Parameter(torch.tensor(
        OE.EmbeddingSpec(r, d, Z, mem, synth.HASH_SEED, m.mid).forward(np.arange(r), M_np.astype(np.float64)),
        dtype=torch.float32, device="cuda")) for m, r in [(emb.word, vocab), (emb.pos, max_pos), (emb.tok_type, 2)]]
    layer = model.layers[0]
    lins = [layer.q, layer.k, layer.v, layer.o, layer.ff1, layer.ff2]
    W = [torch.nn.Parameter(oracle_weight(store, l, M_np)) for l in lins]
    bs = [torch.nn.Parameter(oracle_bias(store, l, M_np)) for l in lins]
    pos = torch.arange(S, device="cuda").expand(B, S)
    e = tables[0][ids] + tables[1][pos] + tables[2][types]
    xr = torch.nn.functional.layer_norm(e, (d,))

    def lin(t, i):
        return t @ W[i] + bs[i]

    def split(t):
        return t.reshape(B, S, heads, d // heads).transpose(1, 2)
    a = torch.nn.functional.scaled_dot_product_attention(split(lin(xr, 0)), split(lin(xr, 1)), split(lin(xr, 2)))
    a = a.transpose(1, 2).reshape(B, S, d)
    h1 = torch.nn.functional.layer_norm(xr + lin(a, 3), (d,))
    yr = torch.nn.functional.layer_norm(h1 + lin(torch.nn.functional.gelu(lin(h1, 4), approximate="tanh"), 5), (d,))
    (yr * Rw).sum().backward()
    parts = {k: np.zeros(mem) for k in ("linears", "biases", "embeddings")}
    for l, w, b in zip(lins, W, bs):
        _, H, O = store.dims[l.mid]
        OM.LinearSpec(H, O, 64, 64, mem, synth.HASH_SEED, l.mid).scatter(w.grad.double().cpu().numpy(),
                                                                         parts["linears"])
        OE.EmbeddingSpec(1, O, 64, mem, synth.HASH_SEED, l.bias.mid, fan_in=H).backward(
            np.zeros(1, np.int64), b.grad.double().cpu().numpy()[None], parts["biases"])
    for m, r, t in [(emb.word, vocab, tables[0]), (emb.pos, max_pos, tables[1]), (emb.tok_type, 2, tables[2])]:
        OE.EmbeddingSpec(r, d, Z, mem, synth.HASH_SEED, m.mid).backward(
            np.arange(r, dtype=np.int64), t.grad.double().cpu().numpy(), parts["embeddings"])
    dM_ref = sum(parts.values())
    for k, v in parts.items():   # every family contributes a visible share of the whole
        assert np.linalg.norm(v) > 1e-3 * np.linalg.norm(dM_ref), k
    err = np.linalg.norm(dM - dM_ref) / np.linalg.norm(dM_ref)
    assert err < 3e-2, err


def test_batched_bias_grads_accumulate_over_two_backwards_and_zero_grad_discards():
    """with batch_biases the bias backward only collects column sums until
    flush_bias_grads.  Two backwards before the flush (micro-batch accumulation, a layer applied
    twice) must keep both contributions; zero_grad must discard collected-but-unflushed ones.
    Reference: the same steps with per-call L backwards (batch_biases = False)."""
    import torch
    from paper_2207_10702_b200 import nn as RN, roast as R
    d, T, mem = 256, 192, 40_000
    M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    xs = [torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3)]
    rs = [torch.randn(T, d, device="cuda", generator=g) for _ in range(3)]

    def run(batched, discard_first):
        store = R.Roast(torch.tensor(M_np, device="cuda"), 64, 64, seed=synth.HASH_SEED)
        store.batch_biases = batched
        lin = RN.RoastLinear(store, d, d, bias=True)
        store.zero_grad()
        if discard_first:                       # a step whose gradients are thrown away
            (lin(xs[2]).float() * rs[2]).sum().backward()
            store.zero_grad()
        for x, r in zip(xs[:2], rs[:2]):        # two micro-batches, one flush
            (lin(x).float() * r).sum().backward()
        store.flush_bias_grads()
        torch.cuda.synchronize()
        out = store.dM.cpu().numpy().astype(np.float64)
        store.close()
        return out

    ref = run(False, False)
    assert np.linalg.norm(ref) > 0
    for discard in (False, True):
        got = run(True, discard)
        assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref), discard
