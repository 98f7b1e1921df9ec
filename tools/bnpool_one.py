import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import maml
DEV = "cuda:0"
T, C, B, H, W = 32, 64, 25, 28, 28
g = torch.Generator(device=DEV).manual_seed(0)
x = torch.randn(T, C, B, H, W, device=DEV, generator=g).requires_grad_(True)
ga = (torch.rand(T, C, device=DEV, generator=g) + 0.5).requires_grad_(True)
be = torch.randn(T, C, device=DEV, generator=g).requires_grad_(True)
out = maml._BnPool.apply(x, ga, be)
dp = torch.randn(out.shape, device=DEV, generator=g)
for _ in range(3):
    torch.autograd.grad(out, (x, ga, be), dp, retain_graph=True)
torch.cuda.synchronize()
