"""Element-sharded optimizer step (">= 1B trees:
reduce-scatter + local fwd + all-gather").

For a data-parallel job whose optimizer state (m, v: 8 B/element fp32) does
not fit next to the model on every GPU, each of the W ranks owns a
contiguous 1/W shard of the flat tree (ZeRO-1 layout):
  1. reduce_scatter the full gradient -> this rank's shard (sum, then 1/W),
  2. the fused Adam step with apply_updates on the shard only (one
     libdiffopt.so launch; m, v exist for the shard only),
  3. all_gather the updated parameter shards -> the full parameters.
Over NVLink/NVSwitch both collectives are NCCL's; the per-rank HBM traffic
of the step drops by W. The local step is injectable so the sharding logic
is tested with the gloo backend on CPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L


def shard_size(n, world):
    per = -(-int(n) // world)
    return -(-per // 4) * 4  # 16-byte aligned shards


class ShardedAdam:
    def __init__(self, n, world, rank, device, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8,
                 local_step=None, group=None):
        self.n, self.world, self.rank, self.dev = int(n), int(world), int(rank), device
        self.shard = shard_size(n, world)
        self.n_pad = self.shard * world
        self.hp = (lr, b1, b2, eps, 0.0)
        self.m = torch.zeros(self.shard, device=device)
        self.v = torch.zeros(self.shard, device=device)
        self.g = torch.empty(self.shard, device=device)
        self.p_out = torch.empty(self.shard, device=device)
        self.t = 0
        self.group = group
        self.local_step = local_step or self._fused
        self.tree = None if local_step else L.Tree(numel=self.shard, device=device)

    def _fused(self, g, m, v, p, p_out, t):
        L.opt_adam_fwd(self.tree, t, self.hp, L.OPT_F32, L.OPT_COMPUTE_DEFAULT, g, m, v, None,
                       m, v, p, p_out)

    def step(self, params, grads):
        """params, grads: flat tensors of n_pad elements (padding is zero);
        params is updated in place (every rank ends with the same values)."""
        assert params.numel() == self.n_pad and grads.numel() == self.n_pad
        self.t += 1
        if self.world > 1:
            dist.reduce_scatter_tensor(self.g, grads, op=dist.ReduceOp.SUM, group=self.group)
            self.g.mul_(1.0 / self.world)
        else:
            self.g.copy_(grads)
        lo = self.rank * self.shard
        p_local = params[lo:lo + self.shard]
        self.local_step(self.g, self.m, self.v, p_local, self.p_out, self.t)
        if self.world > 1:
            dist.all_gather_into_tensor(params, self.p_out, group=self.group)
        else:
            params.copy_(self.p_out)
        return params
