"""H2D bandwidth probe for bench.py's e2e leg: 2 x 12.6 MB pinned -> device per step, on one copy
stream vs split over two copy streams."""
import json
import torch

n = 8192 * 768
h = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
s = [torch.cuda.Stream() for _ in range(2)]
res = {}
for mode in ("one", "two", "one", "two"):
    for rep in range(2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for st in s:
            st.wait_event(a)
        for _ in range(50):
            for i in range(2):
                st = s[0] if mode == "one" else s[i]
                with torch.cuda.stream(st):
                    d[i].copy_(h[i], non_blocking=True)
        for st in s:
            torch.cuda.current_stream().wait_stream(st)
        b.record()
        torch.cuda.synchronize()
    res[mode] = 50 * 2 * n * 2 / (a.elapsed_time(b) * 1e-3) / 1e9
print(json.dumps({"h2d_GBps": res}))
