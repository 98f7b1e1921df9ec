"""Throughput of net_gemm_nt (split-K fp32) vs torch.bmm (cuBLAS SGEMM) on
the MAML weight-gradient shapes: C[t] = A[t] B[t]^T, A [T, 64, n],
B [T, P, n]. Prints one JSON line per shape."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import maml  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
DEV = "cuda:0"


def timed(fn, reps=20):
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


for T in (4, 32):
    for P, n in ((576, 4900), (576, 14700), (576, 1225), (576, 225), (9, 19600), (9, 58800)):
        A = torch.randn(T, 64, n, device=DEV)
        B = torch.randn(T, P, n, device=DEV)
        flops = 2.0 * T * 64 * P * n
        ms_k = timed(lambda: maml._gemm_nt(A, B))
        ms_c = timed(lambda: torch.bmm(A, B.transpose(1, 2)))
        print(json.dumps({"T": T, "M": 64, "P": P, "n": n, "gemm_nt_us": round(ms_k * 1e3, 1),
                          "gemm_nt_tflops": round(flops / ms_k / 1e9, 2),
                          "cublas_us": round(ms_c * 1e3, 1),
                          "cublas_tflops": round(flops / ms_c / 1e9, 2)}), flush=True)
