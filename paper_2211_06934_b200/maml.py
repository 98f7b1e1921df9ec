"""Task-sharded MAML meta-batch.

PAPER.md: MAML needs a "large task-level batch size"; TorchOpt
distributes the differentiable-optimization tasks of a meta-batch to GPU
workers that run in parallel under a synchronous coordinator (P:269-271,
App. C; 5.2x on 8 GPUs). B200-native equivalent: SPMD, one
process per GPU; rank r of W owns tasks [r*T/W, (r+1)*T/W) of the T-task
meta-batch, runs each task's inner loop locally, sums its meta-gradients in
task order, and ONE all-reduce (NCCL over NVLink/NVSwitch) combines them;
every replica then applies the same outer Adam step, so replicas stay
identical without a coordinator (synchronous semantics).

Per task (reading Z16): 4-conv64 + BN (batch statistics) + ReLU + maxpool,
fc -> 5 ways; 5-way 5-shot support, 15 queries per class, 28x28x1 inputs
N(0,1) seeded by (outer step, task id), labels fixed by class; 5 inner SGD
momentum steps (lr 0.1, mu 0.9) through the fused differentiable SGD op with
apply_updates fused; second-order meta-gradient (create_graph=True, Z15).
The network forward/backward runs in PyTorch (cuDNN): it is the task's loss,
not the method; the optimizer step and its VJP run in libdiffopt.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

WAYS, SHOTS, QUERIES, HW = 5, 5, 15, 28
CONV4_SHAPES = ([(64, 1, 3, 3), (64,), (64,), (64,)]
                + [(64, 64, 3, 3), (64,), (64,), (64,)] * 3
                + [(WAYS, 64), (WAYS,)])  # 18 leaves, 112,261 elements


def conv4_forward(params, x):
    """params: 18 tensors in CONV4_SHAPES order; x: [B, 1, 28, 28]."""
    h = x
    for blk in range(4):
        w, b, gam, bet = params[4 * blk: 4 * blk + 4]
        h = F.conv2d(h, w, b, padding=1)
        h = F.batch_norm(h, None, None, gam, bet, training=True)
        h = F.max_pool2d(F.relu(h), 2)
    h = h.flatten(1)
    return F.linear(h, params[16], params[17])


def init_params(seed, device):
    """Deterministic phi (same on every rank)."""
    gen = torch.Generator().manual_seed(seed)
    out = []
    for s in CONV4_SHAPES:
        if len(s) == 4:
            fan_in = s[1] * s[2] * s[3]
            out.append(torch.randn(s, generator=gen) * (2.0 / fan_in) ** 0.5)
        elif len(s) == 2:
            out.append(torch.randn(s, generator=gen) * (1.0 / s[1]) ** 0.5)
        else:
            out.append(torch.zeros(s))
    # BN weights = 1
    for blk in range(4):
        out[4 * blk + 2] = torch.ones(64)
    return torch.cat([p.reshape(-1) for p in out]).to(device)


def task_seed(outer_step, task_id, seed=0):
    return ((seed * 1_000_003 + outer_step) * 1_000_033 + task_id) & 0x7FFFFFFFFFFFFFFF


def task_data(outer_step, task_id, device, seed=0):
    """Seeded synthetic 5-way task, generated on `device` by a generator
    keyed on (seed, step, task) only -- never on the rank layout. (CPU and
    CUDA generators draw different streams; each is reproducible.)"""
    device = torch.device(device)
    gen = torch.Generator(device=device).manual_seed(task_seed(outer_step, task_id, seed))
    xs = torch.randn(WAYS * SHOTS, 1, HW, HW, generator=gen, device=device)
    xq = torch.randn(WAYS * QUERIES, 1, HW, HW, generator=gen, device=device)
    # class-dependent mean shift so the task is learnable
    proto = torch.randn(WAYS, 1, HW, HW, generator=gen, device=device)
    ys = torch.arange(WAYS, device=device).repeat_interleave(SHOTS)
    yq = torch.arange(WAYS, device=device).repeat_interleave(QUERIES)
    return xs + proto[ys], ys, xq + proto[yq], yq


@dataclass
class MamlConfig:
    tasks: int = 32
    inner_steps: int = 5
    inner_lr: float = 0.1
    inner_momentum: float = 0.9
    nesterov: bool = False
    outer_lr: float = 1e-3
    seed: int = 0


class FusedSgdInner:
    """Inner step through libdiffopt.so (SgdStep with apply_updates fused)."""

    def __init__(self, sizes, device, cfg: MamlConfig):
        from . import _lib as L
        from .functional import SgdStep, StepConfig

        self.tree = L.Tree.from_sizes(sizes, device=device)
        self.step_cfg = StepConfig(self.tree)
        self.fn = SgdStep
        self.cfg = cfg

    def __call__(self, g, b, theta):
        c = self.cfg
        return self.fn.apply(g, b, theta, c.inner_lr, c.inner_momentum, c.nesterov, self.step_cfg)


class FusedAdamOuter:
    """Outer (non-differentiable) Adam on phi through opt_adam_fwd with
    apply fused and in-place state (G9 of SURVEY §2.2)."""

    def __init__(self, n, device, lr):
        from . import _lib as L

        self.L = L
        self.tree = L.Tree(numel=n, device=device)
        self.mu = torch.zeros(n, device=device)
        self.nu = torch.zeros(n, device=device)
        self.t = 0
        self.lr = lr

    def __call__(self, phi, grad):
        self.t += 1
        self.L.opt_adam_fwd(self.tree, self.t, (self.lr, 0.9, 0.999, 1e-8, 0.0), 0, 0, grad,
                            self.mu, self.nu, None, self.mu, self.nu, phi, phi)
        return phi


def task_range(world, rank, tasks):
    return range(rank * tasks // world, (rank + 1) * tasks // world)


def sizes_of(shapes):
    return [int(torch.Size(s).numel()) for s in shapes]


def meta_grad_tasks(phi, task_ids, outer_step, cfg: MamlConfig, inner):
    """Sum over task_ids (in order) of d L_query(theta_K(phi)) / d phi, and
    the summed query loss. phi: flat leaf tensor (no grad needed on entry)."""
    data = [task_data(outer_step, tid, phi.device, cfg.seed) for tid in task_ids]
    return meta_grad_data(phi, data, cfg, inner)


def meta_grad_data(phi, data, cfg: MamlConfig, inner):
    """meta_grad_tasks on pre-generated task data [(xs, ys, xq, yq), ...]."""
    sizes = sizes_of(CONV4_SHAPES)
    phi_v = phi.detach().requires_grad_(True)
    total = torch.zeros_like(phi)
    loss_sum = torch.zeros((), device=phi.device)
    for xs, ys, xq, yq in data:
        theta, b = phi_v, None
        for _ in range(cfg.inner_steps):
            params = [p.view(s) for p, s in zip(torch.split(theta, sizes), CONV4_SHAPES)]
            loss = F.cross_entropy(conv4_forward(params, xs), ys)
            (g,) = torch.autograd.grad(loss, theta, create_graph=True)
            theta, b = inner(g, b, theta)
        params = [p.view(s) for p, s in zip(torch.split(theta, sizes), CONV4_SHAPES)]
        qloss = F.cross_entropy(conv4_forward(params, xq), yq)
        (mg,) = torch.autograd.grad(qloss, phi_v)
        total += mg
        loss_sum += qloss.detach()
    return total, loss_sum


class GraphedShard:
    """One rank's share of the meta-batch captured as a single CUDA graph
    (all inner loops, query losses, second-order backward and the local
    meta-gradient sum): per outer step only the task data and phi are
    copied into static buffers and the graph is replayed, removing the
    per-kernel launch cost that dominates these tiny convolutions.
    Call it like meta_grad_tasks."""

    def __init__(self, task_ids, cfg: MamlConfig, inner, device, warmup=2):
        self.ids, self.cfg, self.inner = list(task_ids), cfg, inner
        self.phi = torch.zeros(sum(sizes_of(CONV4_SHAPES)), device=device)
        self.data = [task_data(0, t, device, cfg.seed) for t in self.ids]
        side = torch.cuda.Stream(device)
        side.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                meta_grad_data(self.phi, self.data, cfg, inner)
        torch.cuda.current_stream(device).wait_stream(side)
        from . import _lib as L

        self.graph = torch.cuda.CUDAGraph()
        n0 = L.opt_launch_count()
        with torch.cuda.graph(self.graph):
            self.mg, self.loss = meta_grad_data(self.phi, self.data, cfg, inner)
        self.launches_per_replay = L.opt_launch_count() - n0  # captured library kernels

    def __call__(self, phi, task_ids, outer_step, cfg, inner):
        assert list(task_ids) == self.ids
        self.phi.copy_(phi)
        for tid, bufs in zip(self.ids, self.data):
            for dst, src in zip(bufs, task_data(outer_step, tid, phi.device, cfg.seed)):
                dst.copy_(src)
        self.graph.replay()
        return self.mg, self.loss


def outer_step(phi, outer_step_idx, cfg: MamlConfig, inner, outer, world=1, rank=0, group=None,
               shard=None):
    """One synchronous meta-update over the cfg.tasks-task meta-batch.
    ``shard`` (optional) replaces meta_grad_tasks, e.g. a GraphedShard."""
    import torch.distributed as dist

    ids = task_range(world, rank, cfg.tasks)
    run = shard if shard is not None else meta_grad_tasks
    mg, loss = run(phi, ids, outer_step_idx, cfg, inner)
    buf = torch.cat([mg, loss.reshape(1)])
    if world > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)  # the one exchange step
    buf.mul_(1.0 / cfg.tasks)
    mg, loss = buf[:-1].contiguous(), buf[-1]
    phi = outer(phi, mg)
    return phi, loss, mg
