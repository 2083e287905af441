import sys, torch
sys.path.insert(0, '.')
import paper_2509_06220_b200 as nrmf
for lg in (12, 16, 20):
    x = torch.randn(1 << lg, dtype=torch.float64, device='cuda')
    out = torch.empty((), dtype=torch.float64, device='cuda')
    for _ in range(5):
        nrmf.norm(x, out=out)
torch.cuda.synchronize()
print("ok")
