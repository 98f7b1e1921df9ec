"""Where does the C2 Adam backward lose time? Back-to-back launch averages
(CUDA events around K launches, rotating buffer sets) for: sizes C2/4 .. 4xC2
(fixed overhead = intercept of time vs bytes), with and without the
hyper-gradient reduction (d_hp NULL skips block partials and the last-block
sum), and a 4-element launch (pure launch + PDL overhead)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2211_06934_b200 import _lib as L  # noqa: E402

dev = "cuda:0"
HP = (1e-3, 0.9, 0.999, 1e-8, 0.0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 200


def sets_for(n, nsets):
    gen = torch.Generator(device=dev).manual_seed(n)
    out = []
    for _ in range(nsets):
        s = {k: torch.randn(n, device=dev, generator=gen) * 1e-2 for k in ("g", "m", "du", "dm1", "dv1")}
        s["v"] = torch.rand(n, device=dev, generator=gen) * 1e-4
        for k in ("dg", "dm", "dv"):
            s[k] = torch.empty(n, device=dev)
        s["dhp"] = torch.empty(4, dtype=torch.float64, device=dev)
        out.append(s)
    return out


def loop(fn, nsets):
    st = torch.cuda.current_stream()
    for i in range(20):
        fn(i % nsets)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(K):
        fn(i % nsets)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3  # us


rows = []
c2 = 11689512
for n in (c2 // 4, c2 // 2, c2, 2 * c2, 4 * c2, 4):
    nsets = max(1, min(6, int(np.ceil(4 * 126e6 / (n * 36))) + 1)) if n > 4 else 1
    S = sets_for(n, nsets)
    tree = L.Tree(numel=n, device=dev)
    ws = tree.workspace(dev)
    for hp in (True, False):
        def f(i, hp=hp):
            s = S[i]
            L.opt_adam_bwd(tree, 10, HP, 0, 0, s["g"], s["m"], s["v"], s["du"], s["dm1"], s["dv1"],
                           s["dg"], s["dm"], s["dv"], s["dhp"] if hp else None, None,
                           ws if hp else None)
        us = loop(f, nsets)
        rows.append({"n": n, "hp": hp, "us": round(us, 3), "gbs": round(n * 36 / us / 1e3, 1)})
        print(json.dumps(rows[-1]), flush=True)
    del S
    torch.cuda.empty_cache()
# fit t = a + bytes / BW over the four largest sizes, per hp mode
for hp in (True, False):
    pts = [(r["n"] * 36, r["us"]) for r in rows if r["hp"] == hp and r["n"] >= c2 // 2]
    x, y = np.array([p[0] for p in pts], float), np.array([p[1] for p in pts], float)
    slope, icpt = np.polyfit(x, y, 1)
    print(json.dumps({"fit": "hp" if hp else "no-hp", "fixed_us": round(icpt, 3),
                      "stream_gbs": round(1e-3 / slope, 1)}))
