"""Bandwidth of the centred momentum RMSProp kernels (NEXT-1): forward and
backward at 2^24 and 2^26 elements, fp32 state, GB/s on algorithmic bytes
(fwd: g, v, a, b in; u, v', a', b' out = 32 B/elem; bwd: g, v, a, b, du,
dv1, da1, db1 in; dg, dv, da, db out = 48 B/elem), back-to-back launches
timed with CUDA events, 2 rotating buffer sets (> 4 x L2 at 2^26).

    python tools/rms_cm_bench.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import _lib as L  # noqa: E402


def timed(fns, reps=30):
    for f in fns:
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        fns[i % len(fns)]()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    dev = torch.device("cuda", 0)
    g0 = torch.Generator(device=dev).manual_seed(0)
    for lg in (24, 26):
        n = 1 << lg
        tree = L.Tree(numel=n, device=dev)
        ext = L._ext()
        ws = tree.workspace(dev)
        hp = (1e-2, 0.95, 1e-6, 0.9, True)
        sets = []
        for _ in range(2):
            r = lambda: torch.randn(n, device=dev, generator=g0)
            a = 0.5 * r()
            x = dict(g=r(), a=a, v=a * a + r() ** 2 + 0.01, b=r(), du=r(), dv1=r(), da1=r(),
                     db1=r())
            x.update({k: torch.empty(n, device=dev) for k in
                      ("u", "v1", "a1", "b1", "dg", "dv", "da", "db")})
            x["dhp"] = torch.empty(5, dtype=torch.float64, device=dev)
            sets.append(x)
        fwd = [lambda x=x: L.opt_rmsprop_cm_fwd(tree, hp, ext, 0, 0, x["g"], x["v"], x["a"],
                                                x["b"], None, x["u"], x["v1"], x["a1"], x["b1"])
               for x in sets]
        bwd = [lambda x=x: L.opt_rmsprop_cm_bwd(tree, hp, ext, 0, 0, x["g"], x["v"], x["a"],
                                                x["b"], None, x["du"], x["dv1"], x["da1"],
                                                x["db1"], x["dg"], x["dv"], x["da"], x["db"],
                                                None, x["dhp"], None, ws)
               for x in sets]
        tf, tb = timed(fwd), timed(bwd)
        print(json.dumps({"op": "rmsprop centred+momentum", "n": f"2^{lg}",
                          "fwd_us": round(tf, 2), "fwd_gbs": round(32 * n / tf / 1e3, 1),
                          "bwd_us": round(tb, 2), "bwd_gbs": round(48 * n / tb / 1e3, 1)}),
              flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
