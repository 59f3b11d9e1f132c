"""C3's attention (B = 512 sequences, 12 heads, S = 128, d = 64, bf16): fwd + bwd time per
SDPA backend and flash_attn, to pick the one the BERT layer uses (N-op, not the ROAST path)."""
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

B, H, S, D = 512, 12, 128, 64
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
dy = torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16)


def run(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, be in [("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)]:
    try:
        def f():
            with sdpa_kernel(be):
                o = torch.nn.functional.scaled_dot_product_attention(q, k, v)
            o.backward(dy)
        print(name, round(run(f), 3), "ms fwd+bwd")
    except Exception as e:  # noqa: BLE001
        print(name, "unavailable:", repr(e)[:120])
try:
    from flash_attn import flash_attn_func
    qt, kt, vt = (t.detach().transpose(1, 2).contiguous().requires_grad_(True) for t in (q, k, v))
    dyt = dy.transpose(1, 2).contiguous()

    def g():
        o = flash_attn_func(qt, kt, vt)
        o.backward(dyt)
    print("flash_attn", round(run(g), 3), "ms fwd+bwd")
except Exception as e:  # noqa: BLE001
    print("flash_attn unavailable:", repr(e)[:120])
