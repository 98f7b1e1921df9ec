import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import _net as N
DEV = "cuda:0"
T, nsp = 32, 14700
W = torch.randn(T, 64, 576, device=DEV)
cols = torch.randn(T, 576, nsp, device=DEV)
Y = torch.empty(T, 64, nsp, device=DEV)
A = cols.transpose(1, 2)
for _ in range(3):
    N.net_tc_gemm(T, nsp, 64, 576, A, A.stride(1), A.stride(2), A.stride(0), W, W.stride(1), W.stride(2), W.stride(0), Y, nsp, 64 * nsp, None, 1, None)
torch.cuda.synchronize()
