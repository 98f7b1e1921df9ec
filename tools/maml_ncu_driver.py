"""ncu target: one eager task-batched MAML shard (C4, fused network) after
warm-up, inside cudaProfilerStart/Stop so `ncu --profile-from-start off`
captures only the measured step's kernels.

    ncu --profile-from-start off --set full -k regex:'bnpool|im2col|col2im|gemm_nt' \
        -c 12 python tools/maml_ncu_driver.py --tasks 32
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
    torch.cuda.profiler.start()
    maml.meta_grad_batched(phi, data, cfg, inner)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
