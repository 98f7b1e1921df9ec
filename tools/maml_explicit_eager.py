"""Run the explicit MAML schedule eagerly (no CUDA graph) a few times, for
ncu: every kernel is a separate launch ncu can select and replay.

    ncu ... python tools/maml_explicit_eager.py --tasks 4 [--serial]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_06934_b200 import maml, maml_explicit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tasks", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--serial", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
torch.backends.cuda.matmul.allow_tf32 = False
cfg = maml.MamlConfig(tasks=args.tasks)
eng = maml_explicit.ExplicitMaml(args.tasks, cfg, dev, concurrent=not args.serial)
phi = maml.init_params(0, dev)
for r in range(args.reps):
    eng.load_seeded(r, range(args.tasks))
    mg, loss = eng.meta_grad(phi)
torch.cuda.synchronize()
print("ok", float(loss))
