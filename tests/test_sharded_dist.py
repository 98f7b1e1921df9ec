"""Element-sharded optimizer step (NEXT-2) with the gloo backend on CPU,
world size 2: the sharded step (reduce-scatter, local step on the shard,
all-gather) equals the unsharded step on the averaged gradient, every rank
ends with the same parameters, and the shards tile the tree. The local
step here is a plain-torch Adam test reference (the product uses the fused
CUDA kernel)."""
import os
import tempfile

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_06934_b200 import sharded


def torch_adam(hp):
    lr, b1, b2, eps, _ = hp

    def step(g, m, v, p, p_out, t):
        m.mul_(b1).add_((1 - b1) * g)
        v.mul_(b2).add_((1 - b2) * g * g)
        mh = m / (1 - b1 ** t)
        vh = v / (1 - b2 ** t)
        p_out.copy_(p - lr * mh / (vh.sqrt() + eps))

    return step


def _grads(rank, n_pad, t):
    gen = torch.Generator().manual_seed(1000 * t + rank)
    return torch.randn(n_pad, generator=gen)


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    opt = sharded.ShardedAdam(n, world, rank, "cpu", lr=1e-2,
                              local_step=torch_adam((1e-2, 0.9, 0.999, 1e-8, 0.0)))
    params = torch.zeros(opt.n_pad)
    params[:n] = torch.linspace(-1, 1, n)
    for t in range(1, 4):
        opt.step(params, _grads(rank, opt.n_pad, t))
    torch.save(params, f"{out}.{rank}")
    dist.destroy_process_group()


def test_shard_sizes_tile_the_tree():
    for n in (1, 7, 1000, 112261):
        for w in (1, 2, 3, 8):
            s = sharded.shard_size(n, w)
            assert s % 4 == 0 and s * w >= n and (s - 4) * w < n + 4 * w


def test_gloo_sharded_step_equals_unsharded():
    n, world = 1001, 2
    ref_opt = sharded.ShardedAdam(n, 1, 0, "cpu", lr=1e-2,
                                  local_step=torch_adam((1e-2, 0.9, 0.999, 1e-8, 0.0)))
    n_pad = sharded.shard_size(n, world) * world
    ref = torch.zeros(n_pad)
    ref[:n] = torch.linspace(-1, 1, n)
    ref_opt.n_pad = n_pad
    ref_opt.shard = n_pad
    ref_opt.m, ref_opt.v = torch.zeros(n_pad), torch.zeros(n_pad)
    ref_opt.g, ref_opt.p_out = torch.empty(n_pad), torch.empty(n_pad)
    for t in range(1, 4):
        g = sum(_grads(r, n_pad, t) for r in range(world)) / world
        ref_opt.step(ref, g)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "p")
        mp.spawn(_worker, args=(world, 29700 + os.getpid() % 1000, n, out), nprocs=world,
                 join=True)
        p0, p1 = torch.load(f"{out}.0"), torch.load(f"{out}.1")
    assert torch.equal(p0, p1)
    torch.testing.assert_close(p0, ref, rtol=1e-6, atol=1e-7)
