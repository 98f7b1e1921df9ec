"""Op-level breakdown of one eager (not graphed) task-batched MAML shard
(C4): device time attributed to the aten / autograd op that launched it, so
the network's glue can be told apart from its GEMMs.

    python tools/maml_ops.py [--tasks 32] [--net gemm]
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
    ap.add_argument("--net", default="gemm")
    ap.add_argument("--rows", type=int, default=45)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = maml.MamlConfig(tasks=args.tasks, net=args.net)
    phi = maml.init_params(0, dev)
    inner = maml.TaskBatchInner(args.tasks, dev, cfg)
    data = [maml.task_data(0, t, dev, cfg.seed) for t in range(args.tasks)]
    for _ in range(2):
        maml.meta_grad_batched(phi, data, cfg, inner)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        maml.meta_grad_batched(phi, data, cfg, inner)
        torch.cuda.synchronize()
    ka = prof.key_averages()
    rows = [(e.key, e.count, e.self_device_time_total) for e in ka if e.self_device_time_total > 0]
    tot = sum(r[2] for r in rows)
    print(f"self device time {tot / 1e3:.2f} ms")
    for k, c, t in sorted(rows, key=lambda r: -r[2])[:args.rows]:
        print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% x{c:5d}  {k[:100]}")
    print("\ninclusive device time per autograd node / forward op")
    inc = [(e.key, e.count, e.device_time_total) for e in ka
           if e.key.startswith("autograd::engine::evaluate_function") or e.key.startswith("maml")]
    for k, c, t in sorted(inc, key=lambda r: -r[2])[:args.rows]:
        print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% x{c:5d}  {k[:110]}")


if __name__ == "__main__":
    main()
