import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, torch
sys.path.insert(0, %r)
from paper_2211_06934_b200 import _net as N
DEV = "cuda:0"
T, nsp = 32, 14700
W = torch.randn(T, 64, 576, device=DEV); cols = torch.randn(T, 576, nsp, device=DEV)
Y = torch.empty(T, 64, nsp, device=DEV); A = cols.transpose(1, 2)
f = lambda: N.net_tc_gemm(T, nsp, 64, 576, A, A.stride(1), A.stride(2), A.stride(0), W, W.stride(1), W.stride(2), W.stride(0), Y, nsp, 64 * nsp, None, 1, None)
for _ in range(3): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): f()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(os.environ.get("NET_TC_DBG", "0"), round(ms * 1e3, 1), "us", round(2 * T * 64 * 576 * nsp / ms / 1e9, 1), "TF/s")
''' % ROOT
for d in ("0", "1", "2", "4", "3", "5", "6", "7"):
    env = dict(os.environ, NET_TC_DBG=d)
    print(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip(), flush=True)
