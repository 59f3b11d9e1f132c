ROAST_VERBOSE=1 python - <<'PY'
import torch, sys
sys.path.insert(0,'.')
from paper_2207_10702_b200 import roast as R
M=torch.rand(47192,device='cuda')
c=R.Roast(M,64,64)
l1=c.linear(768,3072); l2=c.linear(3072,768)
X=torch.randn(8192,768,device='cuda').bfloat16()
c.fwd_chain(l1,l2,X)
torch.cuda.synchronize()
print(torch.cuda.get_device_properties(0))
PY
