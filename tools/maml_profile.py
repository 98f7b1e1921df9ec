"""Kernel-time breakdown of one MAML outer step (C4) with torch.profiler
(CUPTI): which kernels the task-batched graph replay spends its time in.

    python tools/maml_profile.py [--tasks 32] [--impl batched|streams] [--tf32]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_06934_b200 import maml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", type=int, default=32)
    ap.add_argument("--impl", default="batched")
    ap.add_argument("--tf32", action="store_true")
    ap.add_argument("--net", default="cudnn")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = args.tf32
    torch.backends.cuda.matmul.allow_tf32 = args.tf32
    cfg = maml.MamlConfig(tasks=args.tasks, net=args.net)
    phi = maml.init_params(0, dev)
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), dev, cfg)
    outer = maml.FusedAdamOuter(phi.numel(), dev, cfg.outer_lr)
    shard = maml.GraphedShard(range(cfg.tasks), cfg, inner, dev, batched=args.impl == "batched",
                              streams=1 if args.impl == "batched" else 8)
    for i in range(3):
        phi, _, _ = maml.outer_step(phi, i, cfg, inner, outer, shard=shard)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        phi, _, _ = maml.outer_step(phi, 5, cfg, inner, outer, shard=shard)
        torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name[:110]
            c, t = tot.get(k, (0, 0.0))
            tot[k] = (c + 1, t + e.device_time_total if hasattr(e, "device_time_total") else t + e.cuda_time_total)
    s = sum(t for _, t in tot.values())
    print(f"total kernel time {s/1e3:.2f} ms over {sum(c for c, _ in tot.values())} kernels")
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{t/1e3:9.3f} ms {100*t/s:5.1f}% x{c:5d}  {k}")


if __name__ == "__main__":
    main()
