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


class PeerShardedAdam:
    """ZeRO-1 Adam with the reduce-scatter, the fused step and the all-gather
    in ONE kernel over peer memory (opt_adam_fwd_peers): every rank maps its
    peers' gradient, parameter and flag buffers with CUDA IPC once (handles
    exchanged through the process group), then each step rank r reads the
    W gradient slices of its shard over NVLink, steps its m, v, and stores
    the new parameter slice into all W parameter copies. Cross-rank ordering
    is on the device, with no host round trip: a one-warp signal/wait launch
    (opt_peer_signal_wait) before the step ("my gradient of step t is
    written"; wait for every peer's) and after it ("my stores of step t
    are done"; wait for every peer's), epochs in peer-mapped flag arrays.
    step() only enqueues work on the current stream.

    grads / params: this rank's full (n_pad) buffers, allocated here so
    they can be shared: write gradients into ``self.grads`` and read the
    parameters from ``self.params`` (stream-ordered after step())."""

    def __init__(self, n, world, rank, device, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, group=None,
                 average=True, grad_scale=None, timeout_s=20.0):
        from torch.multiprocessing.reductions import reduce_tensor

        if world > L.OPT_MAX_PEERS:
            raise ValueError(f"world {world} > OPT_MAX_PEERS {L.OPT_MAX_PEERS}")
        self.n, self.world, self.rank, self.dev = int(n), int(world), int(rank), device
        self.shard = shard_size(n, world)
        self.n_pad = self.shard * world
        self.hp = (lr, b1, b2, eps, 0.0)
        self.scale = grad_scale if grad_scale is not None else (1.0 / world if average else 1.0)
        self.timeout_s = float(timeout_s)
        self.grads = torch.zeros(self.n_pad, device=device)
        self.params = torch.zeros(self.n_pad, device=device)
        self.flags = torch.zeros(2 * L.OPT_MAX_PEERS, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.m = torch.zeros(self.shard, device=device)
        self.v = torch.zeros(self.shard, device=device)
        self.t = 0
        self.group = group
        torch.cuda.synchronize(device)  # zeroed flags visible before any peer maps them
        mine = (reduce_tensor(self.grads), reduce_tensor(self.params), reduce_tensor(self.flags))
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, mine, group=group)
        else:
            handles = [mine]
        self.g_peers, self.p_peers, self.f_peers = [], [], []
        for w, hs in enumerate(handles):
            if w == rank:
                bufs = (self.grads, self.params, self.flags)
            else:  # peer's buffers mapped into this process (kept alive here)
                bufs = tuple(h[0](*h[1]) for h in hs)
            self.g_peers.append(bufs[0])
            self.p_peers.append(bufs[1])
            self.f_peers.append(bufs[2])
        if world > 1:  # every rank has mapped every peer before the first signal
            dist.barrier(group=group)

    def step(self):
        """Enqueue one synchronous sharded step on self.grads -> self.params
        (all ranks) on the current stream."""
        self.t += 1
        L.opt_peer_signal_wait(self.world, self.rank, L.PEER_READY, self.f_peers, self.t,
                               self.status, self.timeout_s)
        L.opt_adam_fwd_peers(self.world, self.g_peers, self.p_peers, self.rank * self.shard,
                             self.shard, self.t, self.hp, self.scale, self.m, self.v, self.params)
        L.opt_peer_signal_wait(self.world, self.rank, L.PEER_DONE, self.f_peers, self.t,
                               self.status, self.timeout_s)
        return self.params

    def check(self):
        """Raise if a device-side wait timed out (synchronises)."""
        if int(self.status.item()):
            raise RuntimeError("PeerShardedAdam: a peer did not signal within "
                               f"{self.timeout_s} s (device-side barrier timed out)")
