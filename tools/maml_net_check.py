"""Precision check of the two task-batched MAML network forms on the GPU
against a float64 CPU run (pure torch inner SGD-momentum; no library)."""
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_06934_b200 import maml  # noqa: E402

torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
T = 3
sizes = maml.sizes_of(maml.CONV4_SHAPES)
blk = [T * n for n in sizes]


def run(net, dev, dt, steps=3):
    phi = maml.init_params(0, "cpu").to(dev, dt)
    data = [maml.task_data(2, t, "cpu") for t in range(T)]
    xs = torch.stack([d[0] for d in data], 1).flatten(1, 2).to(dev, dt)
    ys = torch.stack([d[1] for d in data]).to(dev)
    xq = torch.stack([d[2] for d in data], 1).flatten(1, 2).to(dev, dt)
    yq = torch.stack([d[3] for d in data]).to(dev)

    def loss_of(theta, x, y):
        params = [p.view(T, *s) for p, s in zip(torch.split(theta, blk), maml.CONV4_SHAPES)]
        logits = maml.conv4_forward_tasks(params, x, T, net)
        return F.cross_entropy(logits.reshape(-1, 5), y.reshape(-1), reduction="sum") / y.shape[1]

    phi_v = phi.clone().requires_grad_(True)
    theta, b = maml.theta0_tasks(torch.split(phi_v, sizes), T), None
    for _ in range(steps):
        (g,) = torch.autograd.grad(loss_of(theta, xs, ys), theta, create_graph=True)
        b = g if b is None else 0.9 * b + g
        theta = theta - 0.1 * b
    (mg,) = torch.autograd.grad(loss_of(theta, xq, yq), phi_v)
    return mg.double().cpu()


ref = run("cudnn", "cpu", torch.float64)
for net in ("cudnn", "gemm"):
    for dt in (torch.float32, torch.float64):
        m = run(net, "cuda", dt)
        print(net, dt, "rel err vs cpu f64:", float((m - ref).norm() / ref.norm()), flush=True)
