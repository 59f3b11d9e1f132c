for e in 0; do
ROAST_PROF=1 timeout 300 python - <<'PY' 2>&1 | grep "prof\] mix" | tail -1
import sys, torch
sys.path.insert(0,'.')
from paper_2207_10702_b200 import roast as R
c=R.Roast(torch.rand(47192,device='cuda'),64,64); c.set_autotune(0)
a,b=c.linear(768,3072),c.linear(3072,768)
T=8192; bf=torch.bfloat16
X=torch.randn(T,768,device='cuda').to(bf); Ya=torch.randn(T,3072,device='cuda').to(bf); dY=torch.randn(T,768,device='cuda').to(bf)
for _ in range(3): c.bwd_chain(a,b,X,Ya,dY)
torch.cuda.synchronize()
PY
done
timeout 300 python tools/bwd_fused_probe.py 8192 2>&1 | tail -1
