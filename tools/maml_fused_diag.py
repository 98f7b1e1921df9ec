"""Diagnostic: meta-gradient of the failing config under each network form
vs float64 (gemm form, plain-torch inner step)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import maml  # noqa
torch.backends.cuda.matmul.allow_tf32 = False
DEV = "cuda:0"
ntask = int(sys.argv[1]) if len(sys.argv) > 1 else 3
step = int(sys.argv[2]) if len(sys.argv) > 2 else 2
phi = maml.init_params(0, DEV)
def torch_inner_for(cfg):
    def f(g, b, theta):
        b1 = g if b is None else cfg.inner_momentum * b + g
        return theta - cfg.inner_lr * b1, b1
    return f
cfg64 = maml.MamlConfig(tasks=ntask, inner_steps=3, net="gemm")
data64 = [[a.double() if a.is_floating_point() else a for a in maml.task_data(step, t, DEV)] for t in range(ntask)]
for t in range(ntask):
    mg64, _ = maml.meta_grad_data(phi.double(), [data64[t]], cfg64, torch_inner_for(cfg64))
    for net in ("gemm", "fused"):
        cfg = maml.MamlConfig(tasks=ntask, inner_steps=3, net=net)
        inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
        mg, _ = maml.meta_grad_tasks(phi, [t], step, cfg, inner)
        print("task", t, net, "per-task rel err", float((mg.double() - mg64).norm() / mg64.norm()), flush=True)
mg64, _ = maml.meta_grad_data(phi.double(), data64, cfg64, torch_inner_for(cfg64))
for net in ("gemm", "fused"):
    cfg = maml.MamlConfig(tasks=ntask, inner_steps=3, net=net)
    data = [maml.task_data(step, t, DEV, cfg.seed) for t in range(ntask)]
    mg, _ = maml.meta_grad_batched(phi, data, cfg, maml.TaskBatchInner(ntask, DEV, cfg))
    print(net, "batched rel err", float((mg.double() - mg64).norm() / mg64.norm()), flush=True)
