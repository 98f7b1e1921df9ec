"""Leaf-count sweep: the same 11,689,512-element Adam step split into 1, 62
(ResNet-18), 558 (9 x ResNet-18 shape, rescaled), 4096 and 4096-ragged
leaves; forward and backward timed in the uniform path (leaf count is free:
flat buffers) and in per-leaf mode (d_hp_leaf: leaf-aligned tiles over the
shared-memory offset table), GB/s on algorithmic bytes.

    python tools/leaf_sweep.py [--out gpurun_out/leaf_sweep.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2211_06934_b200 import _lib as L  # noqa: E402

N = int(sum(synth.RESNET18_LEAVES))
HP = (1e-3, 0.9, 0.999, 1e-8, 0.0)


def trees():
    rng = np.random.default_rng(0)
    r18 = list(synth.RESNET18_LEAVES)
    out = {"1 leaf": [N], "62 (resnet18)": r18}
    big = np.array(r18 * 9, dtype=np.float64)
    big = np.floor(big / big.sum() * N).astype(np.int64)
    big[-1] += N - big.sum()
    out["558 (9x resnet18 shape)"] = big.tolist()
    even = [N // 4096] * 4096
    even[-1] += N - sum(even)
    out["4096 equal"] = even
    w = rng.lognormal(0, 2, 4096)
    rag = np.floor(w / w.sum() * N).astype(np.int64)
    rag[-1] += N - rag.sum()
    out["4096 lognormal"] = rag.tolist()
    return out


def timed(fn, reps=50):
    for _ in range(5):
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
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "leaf_sweep.json"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(0)
    t = lambda: torch.randn(N, device=dev, generator=gen)
    g, m, du, dm1, dv1 = t(), t(), t(), t(), t()
    v = t().abs()
    u, m1, v1, dg, dmo, dvo = (torch.empty(N, device=dev) for _ in range(6))
    rows = []
    for name, leaves in trees().items():
        tree = L.Tree(offsets=synth.offsets_of(leaves), device=dev)
        dhp = torch.empty(5, dtype=torch.float64, device=dev)
        dhl = torch.empty(len(leaves) * 4, dtype=torch.float64, device=dev)
        ws = tree.workspace(dev, per_leaf=True)
        fwd = lambda: L.opt_adam_fwd(tree, 10, HP, 0, 0, g, m, v, u, m1, v1)
        bwd = lambda: L.opt_adam_bwd(tree, 10, HP, 0, 0, g, m, v, du, dm1, dv1, dg, dmo, dvo,
                                     dhp, None, ws)
        bwd_leaf = lambda: L.opt_adam_bwd(tree, 10, HP, 0, 0, g, m, v, du, dm1, dv1, dg, dmo,
                                          dvo, dhp, dhl, ws)
        r = {"tree": name, "n_leaves": len(leaves), "min_leaf": int(min(leaves)),
             "max_leaf": int(max(leaves))}
        for key, fn, by in (("fwd", fwd, 24), ("bwd", bwd, 36), ("bwd_per_leaf", bwd_leaf, 36)):
            us = timed(fn)
            r[key] = {"us": round(us, 2), "gbs": round(by * N / (us * 1e-6) / 1e9, 1)}
        rows.append(r)
        print(json.dumps(r), flush=True)
    json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
