"""Per-kernel timing of libmamlnet.so's memory-bound kernels (norm/pool
fwd/bwd/bwd2, im2col, col2im) at the C4 network's layer shapes: CUDA events
over back-to-back launches (same buffers: layer inputs are as L2-warm as in
the step, where the producer just wrote them), algorithmic bytes per launch
(each array read or written once) / time.

    python tools/netk_bench.py [--tasks 32 4] [--batch 25 75]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_06934_b200 import _net as N  # noqa: E402

DEV = "cuda:0"
LAYERS = [(28, 28), (14, 14), (7, 7), (3, 3)]


def ev(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", type=int, nargs="+", default=[32, 4])
    ap.add_argument("--batch", type=int, nargs="+", default=[25])
    args = ap.parse_args()
    g = torch.Generator(device=DEV).manual_seed(0)
    for T in args.tasks:
        for B in args.batch:
            for H, W in LAYERS:
                G = T * 64
                n, np_ = B * H * W, B * (H // 2) * (W // 2)
                x = torch.randn(G * n, device=DEV, generator=g)
                ga = torch.rand(G, device=DEV, generator=g) + 0.5
                be = torch.randn(G, device=DEV, generator=g)
                out = torch.empty(G * np_, device=DEV)
                code = torch.empty(G * np_, dtype=torch.uint8, device=DEV)
                mean, rstd = torch.empty(G, device=DEV), torch.empty(G, device=DEV)
                dp = torch.randn(G * np_, device=DEV, generator=g)
                dx, dg, db = torch.empty_like(x), torch.empty(G, device=DEV), torch.empty(G, device=DEV)
                gdx = torch.randn_like(x)
                gdg, gdb = torch.randn(G, device=DEV, generator=g), torch.randn(G, device=DEV, generator=g)
                g_dp, g_x, g_g = torch.empty_like(dp), torch.empty_like(x), torch.empty(G, device=DEV)
                cols = torch.empty(G * 9 * n, device=DEV)
                N.net_bnpool_fwd(G, B, H, W, x, ga, be, 1e-5, out, code, mean, rstd, 0)
                N.net_bnpool_bwd(G, B, H, W, dp, code, x, ga, mean, rstd, dx, dg, db, 0)
                res = {"T": T, "B": B, "HW": f"{H}x{W}"}
                tot = G * n
                jobs = {
                    "fwd": (lambda: N.net_bnpool_fwd(G, B, H, W, x, ga, be, 1e-5, out, code, mean,
                                                     rstd, 0), 4 * tot + 5 * G * np_),
                    "bwd": (lambda: N.net_bnpool_bwd(G, B, H, W, dp, code, x, ga, mean, rstd, dx, dg,
                                                     db, 0), 8 * tot + 5 * G * np_),
                    "bwd2": (lambda: N.net_bnpool_bwd2(G, B, H, W, gdx, gdg, gdb, dp, code, x, ga, mean,
                                                       rstd, dg, db, g_dp, g_x, g_g, 0),
                             12 * tot + 9 * G * np_),
                    "im2col": (lambda: N.net_im2col3x3(G, B, H, W, x, cols, 0), 40 * tot),
                    "col2im": (lambda: N.net_col2im3x3(G, B, H, W, cols, dx, 0), 40 * tot),
                }
                for k, (fn, by) in jobs.items():
                    us = ev(fn)
                    res[k] = [round(us, 2), round(by / us / 1e3, 0)]  # us, GB/s
                print(json.dumps(res), flush=True)
                del x, cols, gdx, g_x, dx


if __name__ == "__main__":
    main()
