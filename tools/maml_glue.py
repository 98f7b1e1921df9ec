"""Where the MAML step's glue kernels (adds, copies, reductions) come from:
one eager task-batched shard under torch.profiler with shapes and Python
stacks; aten::add / copy_ / sum / cat grouped by (op, input shapes, the
nearest maml.py frame or autograd node).

    python tools/maml_glue.py [--tasks 4]
"""
import argparse
import collections
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_06934_b200 import maml  # noqa: E402

GLUE = ("aten::add", "aten::add_", "aten::copy_", "aten::sum", "aten::cat", "aten::clone",
        "aten::mul", "aten::fill_", "aten::zero_", "aten::contiguous", "aten::zeros")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", type=int, default=4)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = maml.MamlConfig(tasks=args.tasks)
    phi = maml.init_params(0, dev)
    inner = maml.TaskBatchInner(args.tasks, dev, cfg)
    data = [maml.task_data(0, t, dev, cfg.seed) for t in range(args.tasks)]
    for _ in range(2):
        maml.meta_grad_batched(phi, data, cfg, inner)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True,
                 with_stack=True) as prof:
        maml.meta_grad_batched(phi, data, cfg, inner)
        torch.cuda.synchronize()
    # parent autograd node of each op
    evs = prof.events()
    groups = collections.defaultdict(lambda: [0, 0.0])
    for e in evs:
        if e.name not in GLUE or e.device_type != torch.autograd.DeviceType.CPU:
            continue
        dt = e.self_device_time_total if hasattr(e, "self_device_time_total") else 0
        if dt <= 0:
            dt = e.device_time_total
        if dt <= 0:
            continue
        p, node = e.cpu_parent, ""
        while p is not None:
            if p.name.startswith("autograd::engine::evaluate_function"):
                node = p.name.split(": ")[-1]
                break
            p = p.cpu_parent
        frame = ""
        for f in (e.stack or []):
            if "maml.py" in f or "functional.py" in f:
                frame = f.split("/")[-1]
                break
        key = (e.name, str(e.input_shapes)[:90], node or frame)
        groups[key][0] += 1
        groups[key][1] += dt
    tot = sum(v[1] for v in groups.values())
    print(f"glue device time {tot / 1e3:.3f} ms")
    for k, (c, t) in sorted(groups.items(), key=lambda kv: -kv[1][1])[:60]:
        print(f"{t / 1e3:8.3f} ms x{c:4d}  {k[0]:12s} {k[2][:40]:40s} {k[1]}")


if __name__ == "__main__":
    main()
