"""torch.autograd glue over the C ABI: a ROAST linear / embedding usable inside a model.

Forward calls roast_linear_fwd; backward calls roast_linear_bwd_dx for the input gradient
and roast_linear_bwd_dm, which accumulates the compressed-array gradient dM inside
libroast (the paper's custom backward that never materialises W, P:26 / P:592).  The
shared array M is not a torch Parameter: its gradient lives in the handle's dM and the
update is roast_sgd_step (after roast_grad_allreduce in data parallel).  Argument
marshalling only — all compute runs in libroast's kernels.
"""
from __future__ import annotations

import torch

from . import roast as R


def _anchor(store):
    """A 0-d tensor requiring grad, passed to every Function of this store so autograd records
    the op even when its tensor input does not require grad (the weights live in M, not in a
    torch Parameter).  Its gradient is always None."""
    a = getattr(store, "_autograd_anchor", None)
    if a is None:
        a = torch.zeros((), device=store.M.device, requires_grad=True)
        store._autograd_anchor = a
    return a


class _LinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, anchor, store, mid):
        H = store.dims[mid][1]
        x2 = x.reshape(-1, H).contiguous()
        y = store.fwd(mid, x2)
        ctx.save_for_backward(x2)
        ctx.store, ctx.mid, ctx.shape = store, mid, x.shape
        return y.reshape(*x.shape[:-1], y.shape[-1])

    @staticmethod
    def backward(ctx, dy):
        (x2,) = ctx.saved_tensors
        store, mid = ctx.store, ctx.mid
        dy2 = dy.reshape(x2.shape[0], -1).contiguous().to(x2.dtype)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = torch.empty_like(x2)
            store.bwd_dx(mid, dy2, dx)
        store.bwd_dm(mid, x2, dy2)          # dM += lambda g X^T dY scattered into M's slots
        return (dx.reshape(ctx.shape) if dx is not None else None), None, None, None


class RoastLinear(torch.nn.Module):
    """y = x W~ with W~ (in x out) read from the shared store through the ROAST-MM mapping."""

    def __init__(self, store: "R.Roast", in_features: int, out_features: int):
        super().__init__()
        self.store = store
        self.mid = store.linear(in_features, out_features)

    def forward(self, x):
        return _LinearFn.apply(x, _anchor(self.store), self.store, self.mid)


class _EmbeddingFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, idx, anchor, store, mid):
        out = store.emb_fwd(mid, idx.reshape(-1).contiguous())
        ctx.save_for_backward(idx)
        ctx.store, ctx.mid = store, mid
        return out.reshape(*idx.shape, out.shape[-1])

    @staticmethod
    def backward(ctx, dout):
        (idx,) = ctx.saved_tensors
        ctx.store.emb_bwd(ctx.mid, idx.reshape(-1).contiguous(), dout.reshape(idx.numel(), -1).float().contiguous())
        return None, None, None, None


class RoastEmbedding(torch.nn.Module):
    """ROAST/ROBE block embedding (rows x dim, chunks of `chunk`) over the shared store."""

    def __init__(self, store: "R.Roast", num_rows: int, dim: int, chunk: int):
        super().__init__()
        self.store = store
        self.mid = store.embedding(num_rows, dim, chunk)

    def forward(self, idx):
        return _EmbeddingFn.apply(idx, _anchor(self.store), self.store, self.mid)


class EncoderLayer(torch.nn.Module):
    """Post-LN BERT encoder layer whose six linears are ROAST linears in one GMS store.
    N-operations (attention math, GELU, LayerNorm) are plain torch."""

    def __init__(self, store, d_model=768, d_ff=3072, heads=12):
        super().__init__()
        self.heads = heads
        self.q = RoastLinear(store, d_model, d_model)
        self.k = RoastLinear(store, d_model, d_model)
        self.v = RoastLinear(store, d_model, d_model)
        self.o = RoastLinear(store, d_model, d_model)
        self.ff1 = RoastLinear(store, d_model, d_ff)
        self.ff2 = RoastLinear(store, d_ff, d_model)
        self.ln1 = torch.nn.LayerNorm(d_model)
        self.ln2 = torch.nn.LayerNorm(d_model)

    def forward(self, x):                   # x: [B, S, d]
        B, S, d = x.shape
        h = self.heads

        def split(t):
            return t.reshape(B, S, h, d // h).transpose(1, 2)
        a = torch.nn.functional.scaled_dot_product_attention(split(self.q(x)), split(self.k(x)), split(self.v(x)))
        a = a.transpose(1, 2).reshape(B, S, d)
        x = self.ln1(x + self.o(a))
        return self.ln2(x + self.ff2(torch.nn.functional.gelu(self.ff1(x))))
