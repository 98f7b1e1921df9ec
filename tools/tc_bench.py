"""Throughput of net_tc_gemm (tcgen05 3xTF32) vs cuBLAS SIMT SGEMM on the
three MAML convolution contractions: fwd Y = W cols, dcols = W^T dY,
wgrad = dY cols^T (effective fp32 TFLOP/s = 2 M N K / time)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import _net as N
DEV = "cuda:0"
torch.backends.cuda.matmul.allow_tf32 = False

def timed(fn, reps=10):
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

def tc(A, B, D, splits=1, ws=None):
    T, M, K = A.shape
    Nn = B.shape[1]
    N.net_tc_gemm(T, M, Nn, K, A, A.stride(1), A.stride(2), A.stride(0), B, B.stride(1),
                  B.stride(2), B.stride(0), D, M, M * Nn, None, splits, ws)

for T in (4, 32):
    for nsp in (14700, 4900, 1225):
        W = torch.randn(T, 64, 576, device=DEV)
        cols = torch.randn(T, 576, nsp, device=DEV)
        dY = torch.randn(T, 64, nsp, device=DEV)
        res = {"T": T, "n": nsp}
        fl = 2.0 * T * 64 * 576 * nsp
        # fwd: D(m=n_sp, n=co) = sum_k cols[k][m] W[co][k]
        Y = torch.empty(T, 64, nsp, device=DEV)
        res["fwd_tc_tf"] = round(fl / timed(lambda: tc(cols.transpose(1, 2), W, Y)) / 1e9, 1)
        res["fwd_sgemm_tf"] = round(fl / timed(lambda: torch.bmm(W, cols)) / 1e9, 1)
        # dcols: D(m=n_sp, n=p) = sum_co dY[co][m] W[co][p]
        C = torch.empty(T, 576, nsp, device=DEV)
        res["dcols_tc_tf"] = round(fl / timed(lambda: tc(dY.transpose(1, 2), W.transpose(1, 2), C)) / 1e9, 1)
        res["dcols_sgemm_tf"] = round(fl / timed(lambda: torch.bmm(W.transpose(1, 2), dY)) / 1e9, 1)
        # wgrad: D(m=p, n=co) = sum_n cols[p][n] dY[co][n]
        G = torch.empty(T, 64, 576, device=DEV)
        best = None
        for sp in (1, 2, 4, 8, 16):
            wb = N.net_tc_gemm_workspace_bytes(T, 576, 64, nsp, sp)
            ws = torch.empty((wb + 3) // 4, device=DEV) if wb else None
            tf = fl / timed(lambda: tc(cols, dY, G, sp, ws)) / 1e9
            if best is None or tf > best[1]:
                best = (sp, tf)
        res["wgrad_tc_tf"] = round(best[1], 1)
        res["wgrad_tc_splits"] = best[0]
        res["wgrad_sgemm_tf"] = round(fl / timed(lambda: torch.bmm(dY, cols.transpose(1, 2))) / 1e9, 1)
        print(json.dumps(res), flush=True)
