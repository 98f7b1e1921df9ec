"""Kernel timeline of one replay of the explicit MAML shard (C4) with
torch.profiler (CUPTI): span, busy time, idle gaps between kernels, the
kernel-time breakdown by name, and (--timeline FILE) every kernel in order.

    python tools/maml_explicit_profile.py [--tasks 4] [--timeline out.txt]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_06934_b200 import maml, maml_explicit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", type=int, default=4)
    ap.add_argument("--timeline", default=None)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--groups", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = maml.MamlConfig(tasks=args.tasks)
    phi = maml.init_params(0, dev)
    shard = maml_explicit.ExplicitShard(range(cfg.tasks), cfg, dev, groups=args.groups)
    for i in range(3):
        shard(phi, range(cfg.tasks), i, cfg)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        shard.graph.replay()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    gaps = sum(max(0, b.time_range.start - a.time_range.end) for a, b in zip(ev, ev[1:]))
    print(f"T={cfg.tasks}: {len(ev)} kernels, span {(t1 - t0) / 1e3:.3f} ms, busy "
          f"{busy / 1e3:.3f} ms, idle gaps {gaps / 1e3:.3f} ms "
          f"(mean gap {gaps / max(1, len(ev) - 1):.2f} us)")
    tot = {}
    for e in ev:
        k = e.name[:100]
        c, t = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, t + (e.time_range.end - e.time_range.start))
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:args.top]:
        print(f"{t / 1e3:9.3f} ms {100 * t / busy:5.1f}% x{c:4d} avg {t / c:7.2f} us  {k}")
    if args.timeline:
        with open(args.timeline, "w") as f:
            prev = t0
            for e in ev:
                f.write(f"{(e.time_range.start - t0):9.2f} gap {e.time_range.start - prev:6.2f} "
                        f"dur {e.time_range.end - e.time_range.start:8.2f}  {e.name[:90]}\n")
                prev = e.time_range.end


if __name__ == "__main__":
    main()
