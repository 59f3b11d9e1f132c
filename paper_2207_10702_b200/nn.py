"""torch.autograd glue over the C ABI: a ROAST linear / embedding usable inside a model.

Forward calls roast_linear_fwd; backward calls roast_linear_bwd_dx for the input gradient
and roast_linear_bwd_dm, which accumulates the compressed-array gradient dM inside
libroast (the paper's custom backward that never materialises W, P:26 / P:592).  The
shared array M is not a torch Parameter: its gradient lives in the handle's dM and the
update is roast_sgd_step (after roast_grad_allreduce in data parallel).  Argument
marshalling only — all compute runs in libroast's kernels.
"""
from __future__ import annotations

import os

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


class ResidualGrad:
    """Hand-off of a residual connection's gradient to the GEMM that produces the same input's
    other gradient.  In y = LayerNorm(f(x) + x) the input x receives ds (through the residual) and
    f's input gradient; instead of autograd adding the two (a separate bf16 add over the whole
    activation), the LayerNorm backward leaves ds here and f's first linear writes
    dX = bf16(dX_gemm) + ds in its dX GEMM's epilogue (roast_linear_bwd_dx_act, ROAST_ACT_RESIDUAL:
    the same bits).  The LayerNorm backward always runs first: f's backward needs its output."""

    __slots__ = ("ds",)

    def __init__(self):
        self.ds = None

    def take(self):
        ds, self.ds = self.ds, None
        return ds


# the fused residual add pays for itself once the dX launch has several units per CTA pair (its
# epilogue then overlaps the next unit's MMAs): tools/act_probe.py, 768-wide dX GEMMs, vs the plain
# dX GEMM + a bf16 add: T = 65 536 234 vs 270 us (ff1), 177 vs 215 us (QKV); T = 8192 51 vs 48 us
RESIDUAL_FUSE_MIN_TOKENS = 32768


def _linear_backward(store, mid, x2, dy2, box, need_dx):
    """dM += module `mid`'s gradient for (x2, dy2) and, if need_dx, its dX plus the residual
    gradient left in `box`.  Large token counts: the residual added in the dX epilogue, dM
    separately; otherwise dX and dM from roast_linear_bwd_fused (one co-scheduled launch where
    that pays: a 768-wide dX alone fills 48 of 74 CTA pairs at 8192 tokens) and the residual
    added after."""
    r = box.take() if box is not None else None
    if not need_dx:
        store.bwd_dm(mid, x2, dy2)
        return None
    if r is not None and x2.shape[0] >= RESIDUAL_FUSE_MIN_TOKENS:
        r2 = r.reshape(x2.shape).contiguous()
        try:
            dx = store.bwd_dx_act(mid, dy2, r2, act=R.ACT_RESIDUAL)
        except R.RoastError as e:
            if e.status != R.ERR_UNSUPPORTED:
                raise
            dx = torch.empty_like(x2)
            store.bwd_dx(mid, dy2, dx)
            dx = dx + r2
        store.bwd_dm(mid, x2, dy2)
        return dx
    dx = store.bwd_fused(mid, x2, dy2)
    if r is not None:
        dx.add_(r.reshape(x2.shape))
    return dx


class _LinearFn(torch.autograd.Function):
    """y = x W~ (+ b).  With a bias via L the bias is recovered by roast_bias_fwd and
    added inside the forward GEMM's epilogue; its gradient (column sums of dy, scattered by
    the L rule) is roast_bias_bwd."""

    @staticmethod
    def forward(ctx, x, anchor, store, mid, bias_mid):
        H = store.dims[mid][1]
        x2 = x.reshape(-1, H).contiguous()
        b = store.bias_vector(bias_mid) if bias_mid is not None else None
        y = store.fwd(mid, x2, bias=b)
        ctx.save_for_backward(x2)
        ctx.store, ctx.mid, ctx.bias_mid, ctx.shape = store, mid, bias_mid, x.shape
        return y.reshape(*x.shape[:-1], y.shape[-1])

    @staticmethod
    def backward(ctx, dy):
        (x2,) = ctx.saved_tensors
        store, mid = ctx.store, ctx.mid
        dy2 = dy.reshape(x2.shape[0], -1).contiguous().to(x2.dtype)
        # dM += lambda g X^T dY scattered into M's slots, and dX
        dx = _linear_backward(store, mid, x2, dy2, None, ctx.needs_input_grad[0])
        if ctx.bias_mid is not None:
            store.bias_grad(ctx.bias_mid, dy2)
        return (dx.reshape(ctx.shape) if dx is not None else None), None, None, None, None


class _LinearGroupFn(torch.autograd.Function):
    """y = x [W_1 | ... | W_n] (+ [b_1 | ... | b_n]) for a roast_register_linear_concat group:
    one forward GEMM, one dX GEMM (dX = sum_i dY_i W_i^T over the concatenated K), one dM GEMM;
    each member bias's backward reads its column slice of dY in place."""

    @staticmethod
    def forward(ctx, x, anchor, store, gid, bias_mids, box=None):
        H = store.dims[gid][1]
        x2 = x.reshape(-1, H).contiguous()
        b = torch.cat([store.bias_vector(m) for m in bias_mids]) if bias_mids else None
        y = store.fwd(gid, x2, bias=b)
        ctx.save_for_backward(x2)
        ctx.store, ctx.gid, ctx.bias_mids, ctx.shape, ctx.box = store, gid, bias_mids, x.shape, box
        return y.reshape(*x.shape[:-1], y.shape[-1])

    @staticmethod
    def backward(ctx, dy):
        (x2,) = ctx.saved_tensors
        store, gid = ctx.store, ctx.gid
        dy2 = dy.reshape(x2.shape[0], -1).contiguous().to(x2.dtype)
        # dM, and dX + the residual gradient if handed off
        dx = _linear_backward(store, gid, x2, dy2, ctx.box, ctx.needs_input_grad[0])
        if ctx.bias_mids:
            c0 = 0
            for m in ctx.bias_mids:
                n = store.dims[m][2]
                store.bias_grad(m, dy2[:, c0:c0 + n])
                c0 += n
        return (dx.reshape(ctx.shape) if dx is not None else None), None, None, None, None, None


def gelu(x):
    """The BERT MLP's activation: GELU in its tanh form (the original BERT's; torch's
    gelu(approximate="tanh")), the one roast_linear_fwd_act fuses into the GEMM epilogue."""
    return torch.nn.functional.gelu(x, approximate="tanh")


def _gelu_grad(u):
    k0, k1 = 0.7978845608028654, 0.044715
    uf = u.float()
    t = torch.tanh(k0 * (uf + k1 * uf * uf * uf))
    return 0.5 * (1 + t) + 0.5 * uf * (1 - t * t) * k0 * (1 + 3 * k1 * uf * uf)


class _MLPFn(torch.autograd.Function):
    """y = ff2(gelu(ff1(x))) with the GELU inside the GEMM epilogues: the forward of ff1 writes
    u = x W1 (+ b1) and h = gelu(u); the backward's dX GEMM of ff2 writes du = (dy W2^T) * gelu'(u)
    directly.  Off the fused path (roast_linear_*_act UNSUPPORTED) the same math runs unfused.
    The forward keeps separate launches (one chained launch, roast_linear_fwd_chain_act, was not
    faster in the BERT step); the backward is one fused launch below RESIDUAL_FUSE_MIN_TOKENS
    (_mlp_fused_bwd), separate launches above."""

    @staticmethod
    def forward(ctx, x, anchor, store, m1, b1, m2, b2, box=None):
        H = store.dims[m1][1]
        x2 = x.reshape(-1, H).contiguous()
        bv1 = store.bias_vector(b1) if b1 is not None else None
        bv2 = store.bias_vector(b2) if b2 is not None else None
        try:
            u, h = store.fwd_act(m1, x2, bias=bv1)
            ctx.fused = True
        except R.RoastError as e:
            if e.status != R.ERR_UNSUPPORTED:
                raise
            u = store.fwd(m1, x2, bias=bv1)
            h = gelu(u)
            ctx.fused = False
        y = store.fwd(m2, h, bias=bv2)
        ctx.save_for_backward(x2, u, h)
        ctx.store, ctx.m1, ctx.b1, ctx.m2, ctx.b2, ctx.shape = store, m1, b1, m2, b2, x.shape
        ctx.box = box
        return y.reshape(*x.shape[:-1], y.shape[-1])

    @staticmethod
    def backward(ctx, dy):
        x2, u, h = ctx.saved_tensors
        store = ctx.store
        dy2 = dy.reshape(x2.shape[0], -1).contiguous().to(x2.dtype)
        if ctx.fused and _mlp_fused_bwd(x2.shape[0]):   # the four GEMMs in one launch (bwd_chain_act)
            du, dx = store.bwd_chain_act(ctx.m1, ctx.m2, x2, h, u, dy2)
            if ctx.b2 is not None:
                store.bias_grad(ctx.b2, dy2)
            if ctx.b1 is not None:
                store.bias_grad(ctx.b1, du)
            r = ctx.box.take() if ctx.box is not None else None
            if r is not None:
                dx.add_(r.reshape(dx.shape))
            return dx.reshape(ctx.shape), None, None, None, None, None, None, None
        store.bwd_dm(ctx.m2, h, dy2)
        if ctx.b2 is not None:
            store.bias_grad(ctx.b2, dy2)
        if ctx.fused:
            du = store.bwd_dx_act(ctx.m2, dy2, u)
        else:
            dh = torch.empty_like(h)
            store.bwd_dx(ctx.m2, dy2, dh)
            du = (dh.float() * _gelu_grad(u)).to(h.dtype)
        if ctx.b1 is not None:
            store.bias_grad(ctx.b1, du)
        # dM of ff1, and dX + the residual gradient if handed off
        dx = _linear_backward(store, ctx.m1, x2, du, ctx.box, ctx.needs_input_grad[0])
        return (dx.reshape(ctx.shape) if dx is not None else None), None, None, None, None, None, None, None


def _mlp_fused_bwd(tokens):
    """The MLP's backward as ONE launch (roast_linear_bwd_chain_act: dY_a with GELU', dM_b, dX_a,
    dM_a co-scheduled) below RESIDUAL_FUSE_MIN_TOKENS, where its four GEMMs alone quantise badly:
    C3 at 8192 tokens 6.08 -> 5.93 ms; at 65 536 the separate launches with the residual fused into
    ff1's dX epilogue are faster (40.1 vs 41.6 ms).  ROAST_MLP_FUSED_BWD=0 / 1 forces it (A/B)."""
    force = os.environ.get("ROAST_MLP_FUSED_BWD")
    if force in ("0", "1"):
        return force == "1"
    return tokens < RESIDUAL_FUSE_MIN_TOKENS


def _mlp_fusable(ff1, ff2, x):
    return isinstance(ff1, RoastLinear) and isinstance(ff2, RoastLinear) and ff1.store is ff2.store and x.is_cuda \
        and x.dtype == torch.bfloat16


def mlp(ff1, ff2, x, box=None):
    """ff2(gelu(ff1(x))): one fused autograd op for two ROAST linears, plain modules otherwise.
    `box` (fused op only): a ResidualGrad whose gradient is added into x's gradient."""
    if _mlp_fusable(ff1, ff2, x):
        return _MLPFn.apply(x, _anchor(ff1.store), ff1.store, ff1.mid, ff1.bias.mid if ff1.bias is not None else None,
                            ff2.mid, ff2.bias.mid if ff2.bias is not None else None, box)
    assert box is None
    return ff2(gelu(ff1(x)))


class RoastBias(torch.nn.Module):
    """A bias vector of n elements recovered with L in chunks of `chunk` (reading R24:
    registered as a 1 x n embedding, lambda = fp32(C / sqrt(fan_in)) with fan_in the
    owning linear's in_features, the nn.Linear bias scale).  Used by RoastLinear."""

    def __init__(self, store: "R.Roast", n: int, fan_in: float, chunk: int = 64):
        super().__init__()
        self.store = store
        self.mid = store.bias(n, fan_in, chunk)

    def vector(self):
        """The recovered bias (fp32), e.g. for a dense reference."""
        return self.store.bias_fwd(self.mid)


class RoastLinear(torch.nn.Module):
    """y = x W~ (+ b) with W~ (in x out) read from the shared store through the ROAST-MM
    mapping and the optional bias b through L, both in the same GMS store."""

    def __init__(self, store: "R.Roast", in_features: int, out_features: int, bias: bool = False):
        super().__init__()
        self.store = store
        self.mid = store.linear(in_features, out_features)
        self.bias = RoastBias(store, out_features, in_features) if bias else None

    def forward(self, x):
        return _LinearFn.apply(x, _anchor(self.store), self.store, self.mid,
                               self.bias.mid if self.bias is not None else None)


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


try:   # attention is an N-op of the BERT workload: library kernels, as cuBLAS would be
    from flash_attn import flash_attn_func as _flash_attn
    from flash_attn import flash_attn_qkvpacked_func as _flash_attn_packed
except Exception:  # noqa: BLE001
    _flash_attn = _flash_attn_packed = None


def _cdt(t):
    return R.BF16 if t.dtype == torch.bfloat16 else R.FP32


class _LayerNormFn(torch.autograd.Function):
    """y = LayerNorm(x (+ r)) * weight + bias through roast_layernorm_fwd / _bwd (one pass each
    way, the residual add fused).  The gradient of x and of r is the same ds."""

    @staticmethod
    def forward(ctx, x, r, weight, bias, eps, box=None):
        n = x.shape[-1]
        x = x.contiguous()
        rows = x.numel() // n
        y = torch.empty_like(x)
        s = torch.empty_like(x) if r is not None else x
        mean = torch.empty(rows, device=x.device, dtype=torch.float32)
        rstd = torch.empty(rows, device=x.device, dtype=torch.float32)
        rr = r.contiguous() if r is not None else None
        strm = torch.cuda.current_stream().cuda_stream
        R.roast_layernorm_fwd(x.data_ptr(), rr.data_ptr() if rr is not None else None, weight.data_ptr(),
                              bias.data_ptr(), y.data_ptr(), s.data_ptr() if r is not None else None,
                              mean.data_ptr(), rstd.data_ptr(), rows, n, float(eps), _cdt(x), _cdt(weight), strm)
        ctx.save_for_backward(s, weight, mean, rstd)
        ctx.has_r = r is not None
        ctx.box = box
        return y

    @staticmethod
    def backward(ctx, dy):
        s, weight, mean, rstd = ctx.saved_tensors
        n = s.shape[-1]
        rows = s.numel() // n
        dy = dy.contiguous()
        ds = torch.empty_like(s)
        dg = torch.empty(n, device=s.device, dtype=torch.float32)
        db = torch.empty(n, device=s.device, dtype=torch.float32)
        R.roast_layernorm_bwd(dy.data_ptr(), s.data_ptr(), weight.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                              ds.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, n, _cdt(s), _cdt(weight),
                              torch.cuda.current_stream().cuda_stream)
        if ctx.box is not None:   # the residual's gradient goes to the GEMM that adds it (ResidualGrad)
            ctx.box.ds = ds
            return ds, None, dg.to(weight.dtype), db.to(weight.dtype), None, None
        return ds, (ds if ctx.has_r else None), dg.to(weight.dtype), db.to(weight.dtype), None, None


class LayerNorm(torch.nn.LayerNorm):
    """torch.nn.LayerNorm (same parameters, same function) computed by libroast's fused kernels;
    forward(x, residual=None) normalises x + residual in the same pass.  Falls back to torch's
    kernel off the GPU or without an affine part."""

    def fused(self, x):
        return x.is_cuda and self.elementwise_affine and self.bias is not None and x.shape[-1] % 8 == 0 \
            and x.shape[-1] <= 2048 and x.dtype in (torch.bfloat16, torch.float32)

    def forward(self, x, residual=None, residual_grad=None):
        """residual_grad (fused kernel only): a ResidualGrad that receives the residual's gradient
        instead of autograd (the residual must then reach the loss through that hand-off)."""
        if self.fused(x):
            if residual_grad is not None:
                return _LayerNormFn.apply(x, residual.detach(), self.weight, self.bias, self.eps, residual_grad)
            return _LayerNormFn.apply(x, residual, self.weight, self.bias, self.eps)
        assert residual_grad is None
        return super().forward(x if residual is None else x + residual)


_RESIDUAL_HANDOFF = os.environ.get("ROAST_RESIDUAL_HANDOFF", "1") != "0"   # A/B switch (ResidualGrad)


class EncoderLayer(torch.nn.Module):
    """Post-LN BERT encoder layer whose six linears (and, with bias=True, their biases via L)
    are ROAST modules in one GMS store.  N-operations (attention math, GELU, LayerNorm;
    P:263-265) are plain torch."""

    def __init__(self, store, d_model=768, d_ff=3072, heads=12, bias=False, fuse_qkv=True):
        super().__init__()
        self.heads = heads
        self.q = RoastLinear(store, d_model, d_model, bias)
        self.k = RoastLinear(store, d_model, d_model, bias)
        self.v = RoastLinear(store, d_model, d_model, bias)
        self.o = RoastLinear(store, d_model, d_model, bias)
        self.ff1 = RoastLinear(store, d_model, d_ff, bias)
        self.ff2 = RoastLinear(store, d_ff, d_model, bias)
        self.ln1 = LayerNorm(d_model)
        self.ln2 = LayerNorm(d_model)
        # Q, K, V read the same input: one 768 x 2304 GEMM over the three modules' own tiles
        # (registration order and hashes unchanged; the group id lives outside the module ids)
        self.qkv_gid = store.linear_concat([self.q.mid, self.k.mid, self.v.mid]) if fuse_qkv else None

    def _qkv_packed(self, x, box=None):
        """[q | k | v] as one [.., 3 d] tensor (the fused ROAST group or dense Linear), else None.
        `box` (ROAST group only): a ResidualGrad added into x's gradient by the dX GEMM."""
        dense = getattr(self, "qkv_dense", None)
        if dense is not None:
            assert box is None
            return dense(x)
        if getattr(self, "qkv_gid", None) is not None:
            bias = tuple(lin.bias.mid for lin in (self.q, self.k, self.v)) if self.q.bias is not None else ()
            return _LinearGroupFn.apply(x, _anchor(self.q.store), self.q.store, self.qkv_gid, bias, box)
        assert box is None
        return None

    def _qkv(self, x):
        """(q, k, v) projections: fused ROAST group, a fused dense Linear, or three calls."""
        packed = self._qkv_packed(x)
        if packed is not None:
            return packed.split(x.shape[-1], dim=-1)
        return self.q(x), self.k(x), self.v(x)

    def forward(self, x):                   # x: [B, S, d]
        B, S, d = x.shape
        h = self.heads

        # residual gradients handed to the GEMMs that add them (ResidualGrad): the QKV group's and
        # the MLP's dX epilogues write dX + ds instead of autograd adding the two afterwards
        hand_off = getattr(self, "fuse_residual_grad", _RESIDUAL_HANDOFF) and self.ln1.fused(x) and \
            x.dtype == torch.bfloat16
        box1 = ResidualGrad() if hand_off and getattr(self, "qkv_dense", None) is None and \
            getattr(self, "qkv_gid", None) is not None else None
        packed = self._qkv_packed(x, box1) if _flash_attn_packed is not None and x.is_cuda and \
            x.dtype == torch.bfloat16 else None
        if packed is not None:
            # the packed QKV GEMM output viewed as [B, S, 3, heads, d_head]: flash-attn's packed form
            # returns d(qkv) packed too (no concatenation of dq, dk, dv in the backward)
            a = _flash_attn_packed(packed.view(B, S, 3, h, d // h)).reshape(B, S, d)
            x = self.ln1(self.o(a), x, residual_grad=box1)
            box2 = ResidualGrad() if hand_off and self.ln2.fused(x) and _mlp_fusable(self.ff1, self.ff2, x) else None
            return self.ln2(mlp(self.ff1, self.ff2, x, box2), x, residual_grad=box2)
        q, k, v = self._qkv(x)
        if _flash_attn is not None and x.is_cuda and x.dtype == torch.bfloat16:
            # flash-attn (library kernel) reads [B, S, heads, d_head] strided views of the QKV
            # output directly: no transposes either way (0.77 vs 0.88 ms per C3 layer for SDPA)
            def heads(t):
                return t.view(B, S, h, d // h) if t.stride(-1) == 1 else t.reshape(B, S, h, d // h)
            a = _flash_attn(heads(q), heads(k), heads(v)).reshape(B, S, d)
        else:
            def split(t):
                return t.reshape(B, S, h, d // h).transpose(1, 2)
            a = torch.nn.functional.scaled_dot_product_attention(split(q), split(k), split(v))
            a = a.transpose(1, 2).reshape(B, S, d)
        x = self.ln1(self.o(a), x)            # LayerNorm(x + attention), the residual add fused
        return self.ln2(mlp(self.ff1, self.ff2, x), x)


class BertEmbeddings(torch.nn.Module):
    """Word + position + token-type embeddings, each a ROAST block embedding via L in the
    same GMS store (NEXT #3), summed in fp32 and LayerNorm-ed, output bf16."""

    def __init__(self, store, vocab=30522, d_model=768, max_pos=512, type_vocab=2, chunk=32):
        super().__init__()
        self.word = RoastEmbedding(store, vocab, d_model, chunk)
        self.pos = RoastEmbedding(store, max_pos, d_model, chunk)
        self.tok_type = RoastEmbedding(store, type_vocab, d_model, chunk)
        self.ln = LayerNorm(d_model)

    def forward(self, ids, types=None):                 # ids: [B, S] int64
        B, S = ids.shape
        pos = torch.arange(S, device=ids.device).expand(B, S)
        types = torch.zeros_like(ids) if types is None else types
        e = self.word(ids) + self.pos(pos.contiguous()) + self.tok_type(types)
        return self.ln(e).to(torch.bfloat16)


class RoastBert(torch.nn.Module):
    """ROASTed BERT-base encoder (NEXT #3): embeddings via L, 12 post-LN layers of
    ROAST linears with biases via L — every weight of the model except the LayerNorm
    affines lives in ONE global array M (GMS).  Returns the last hidden states."""

    def __init__(self, store, vocab=30522, d_model=768, d_ff=3072, heads=12, layers=12, max_pos=512,
                 type_vocab=2, chunk=32, bias=True):
        super().__init__()
        self.emb = BertEmbeddings(store, vocab, d_model, max_pos, type_vocab, chunk)
        self.layers = torch.nn.ModuleList([EncoderLayer(store, d_model, d_ff, heads, bias) for _ in range(layers)])
        for m in self.layers.modules():
            if isinstance(m, torch.nn.LayerNorm):
                m.to(torch.bfloat16)

    def forward(self, ids, types=None):
        x = self.emb(ids, types)
        for layer in self.layers:
            x = layer(x)
        return x


def bert_param_count(vocab=30522, d_model=768, d_ff=3072, layers=12, max_pos=512, type_vocab=2, bias=True):
    """Virtual parameters RoastBert maps into M (for sizing |M| = n / ratio)."""
    lin = layers * (4 * d_model * d_model + 2 * d_model * d_ff)
    b = layers * (5 * d_model + d_ff) if bias else 0
    return lin + b + (vocab + max_pos + type_vocab) * d_model
