"""float32 (x,+) at 4096^3 on the device (the DFMA-in-float64 route), for ncu (tools probe)."""
import sys; sys.path.insert(0,'.')
import torch, paper_0907_0792_b200 as moa
from paper_0907_0792_b200.kernel import launch, plan_inner
n=4096
a=torch.rand(n*n,device='cuda'); b=torch.rand(n*n,device='cuda'); c=torch.empty(n*n,device='cuda')
p=plan_inner((n,n),(n,n))
for _ in range(2): launch(p,c,a,b,moa.MUL_ADD)
torch.cuda.synchronize()
