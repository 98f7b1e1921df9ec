"""Accuracy of the 3xTF32 tcgen05 GEMM (net_tc_gemm) vs fp32 SIMT SGEMM
(cuBLAS, TF32 off) vs single-pass TF32 (cuBLAS), all against float64, on
the MAML convolution shapes. Prints max and rms error relative to the
rms of the result."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import _net as N
DEV = "cuda:0"

def tc(A, B):
    T, M, K = A.shape
    Nn = B.shape[1]
    D = torch.empty(T, Nn, M, device=DEV)
    N.net_tc_gemm(T, M, Nn, K, A, A.stride(1), A.stride(2), A.stride(0), B, B.stride(1),
                  B.stride(2), B.stride(0), D, M, M * Nn, None, 1, None)
    return D

for (T, M, Nn, K) in [(4, 4900, 64, 576), (4, 576, 64, 4900), (4, 4900, 576, 64)]:
    g = torch.Generator(device=DEV).manual_seed(0)
    A = torch.randn(T, M, K, device=DEV, generator=g)
    B = torch.randn(T, Nn, K, device=DEV, generator=g)
    ref = torch.bmm(B.double(), A.double().transpose(1, 2))
    rms = float(ref.pow(2).mean().sqrt())
    out = {"shape": [T, M, Nn, K]}
    torch.backends.cuda.matmul.allow_tf32 = False
    for name, D in (("tc3xtf32", tc(A, B)), ("sgemm", torch.bmm(B, A.transpose(1, 2)))):
        e = (D.double() - ref)
        out[name] = {"max_rel": float(e.abs().max()) / rms, "rms_rel": float(e.pow(2).mean().sqrt()) / rms}
    torch.backends.cuda.matmul.allow_tf32 = True
    D = torch.bmm(B, A.transpose(1, 2))
    e = (D.double() - ref)
    out["tf32"] = {"max_rel": float(e.abs().max()) / rms, "rms_rel": float(e.pow(2).mean().sqrt()) / rms}
    torch.backends.cuda.matmul.allow_tf32 = False
    print(json.dumps(out), flush=True)
