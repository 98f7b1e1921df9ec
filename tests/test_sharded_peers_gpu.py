"""GPU tests of the fused peer-memory sharded Adam step (opt_adam_fwd_peers,
SURVEY §8(f) NEXT-2): reduce-scatter + step + all-gather in one kernel.

* W virtual ranks in one process (W buffers on one device, the W calls in
  sequence): every parameter copy is bitwise identical to the others and
  equals the fused single-GPU Adam step (opt_adam_fwd with apply) on the
  averaged gradient to fp32 rounding (two kernels may contract the same
  expressions into FMAs differently), for W = 1, 2, 3, 8, ragged sizes.
* Two real processes on one GPU: the buffers of the other process are mapped
  by CUDA IPC (handles exchanged over a gloo process group) exactly as on a
  multi-GPU node; three steps match the virtual-rank run bitwise."""
import os
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
HP = (1e-2, 0.9, 0.999, 1e-8, 0.0)


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06934_b200 import _lib

    return _lib


def virtual(L, grads, p0, steps):
    """The W ranks' calls in sequence in one process (same kernel as the
    multi-process run): returns rank 0's parameter copy."""
    from paper_2211_06934_b200.sharded import shard_size

    W = len(grads[0])
    shard = p0.numel() // W
    copies = [p0.clone() for _ in range(W)]
    state = [(torch.zeros(shard, device=DEV), torch.zeros(shard, device=DEV)) for _ in range(W)]
    for t in range(steps):
        for r in range(W):
            L.opt_adam_fwd_peers(W, grads[t], copies, r * shard, shard, t + 1, HP, 1.0 / W,
                                 state[r][0], state[r][1], copies[r])
    torch.cuda.synchronize()
    return copies[0]


def reference(L, grads, params, steps):
    """Fused single-GPU Adam (opt_adam_fwd with apply) on the averaged gradient."""
    W = len(grads[0])
    n = params.numel()
    tree = L.Tree(numel=n, device=DEV)
    m, v, p = torch.zeros(n, device=DEV), torch.zeros(n, device=DEV), params.clone()
    for t in range(steps):
        g = grads[t][0].clone()
        for w in range(1, W):
            g = g + grads[t][w]
        g = g * (1.0 / W)
        L.opt_adam_fwd(tree, t + 1, HP, 0, 1, g, m, v, None, m, v, p, p)
    return p


@pytest.mark.parametrize("W,n", [(1, 1000), (2, 4096), (3, 10001), (8, 2 ** 18 + 7)])
def test_virtual_ranks_equal_single_gpu_step(L, W, n):
    from paper_2211_06934_b200.sharded import shard_size

    shard = shard_size(n, W)
    n_pad = shard * W
    gen = torch.Generator(device=DEV).manual_seed(W)
    p0 = torch.zeros(n_pad, device=DEV)
    p0[:n] = torch.randn(n, device=DEV, generator=gen)
    steps = 3
    grads = [[torch.zeros(n_pad, device=DEV) for _ in range(W)] for _ in range(steps)]
    for t in range(steps):
        for w in range(W):
            grads[t][w][:n] = torch.randn(n, device=DEV, generator=gen)
    copies = [p0.clone() for _ in range(W)]
    state = [(torch.zeros(shard, device=DEV), torch.zeros(shard, device=DEV)) for _ in range(W)]
    for t in range(steps):
        for r in range(W):  # each "rank" in turn: disjoint shards
            L.opt_adam_fwd_peers(W, grads[t], copies, r * shard, shard, t + 1, HP, 1.0 / W,
                                 state[r][0], state[r][1], copies[r])
        torch.cuda.synchronize()
    ref = reference(L, grads, p0, steps)
    for w in range(W):
        assert torch.equal(copies[w], copies[0]), f"copy {w} differs from copy 0"
    torch.testing.assert_close(copies[0], ref, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("W", [2, 3, 8])
def test_device_flags_virtual_ranks_on_streams(L, W):
    """The device-side barrier (opt_peer_signal_wait) with W virtual ranks in
    one process, each on its own stream and never synchronised by the host:
    ready-wait, fused step, done-wait per rank per step. Ranks that run ahead
    block on the device until the others signal; the result is bitwise the
    serialised run's, and no wait times out."""
    from paper_2211_06934_b200.sharded import shard_size

    n, steps = 30_011, 3
    shard = shard_size(n, W)
    n_pad = shard * W
    gen = torch.Generator(device=DEV).manual_seed(40 + W)
    p0 = torch.zeros(n_pad, device=DEV)
    p0[:n] = torch.randn(n, device=DEV, generator=gen)
    grads = [[torch.zeros(n_pad, device=DEV) for _ in range(W)] for _ in range(steps)]
    for t in range(steps):
        for w in range(W):
            grads[t][w][:n] = torch.randn(n, device=DEV, generator=gen)
    ref = virtual(L, grads, p0, steps)
    copies = [p0.clone() for _ in range(W)]
    gbuf = [torch.zeros(n_pad, device=DEV) for _ in range(W)]
    flags = [torch.zeros(2 * L.OPT_MAX_PEERS, dtype=torch.int64, device=DEV) for _ in range(W)]
    status = torch.zeros(1, dtype=torch.int32, device=DEV)
    state = [(torch.zeros(shard, device=DEV), torch.zeros(shard, device=DEV)) for _ in range(W)]
    streams = [torch.cuda.Stream(DEV) for _ in range(W)]
    torch.cuda.synchronize()
    for t in range(steps):
        for r in reversed(range(W)):  # enqueue the last rank first: it must wait on the device
            with torch.cuda.stream(streams[r]):
                gbuf[r].copy_(grads[t][r])  # "my gradient of step t"
                L.opt_peer_signal_wait(W, r, L.PEER_READY, flags, t + 1, status, 20.0)
                L.opt_adam_fwd_peers(W, gbuf, copies, r * shard, shard, t + 1, HP, 1.0 / W,
                                     state[r][0], state[r][1], copies[r])
                L.opt_peer_signal_wait(W, r, L.PEER_DONE, flags, t + 1, status, 20.0)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    for w in range(W):
        assert torch.equal(copies[w], ref), f"copy {w}"
    assert all(int(f[:W].min()) == steps and int(f[8:8 + W].min()) == steps for f in flags)


def test_device_flags_timeout_is_reported_not_hung(L):
    """A peer that never signals: the wait gives up after timeout_s and sets
    the status word instead of hanging the stream."""
    flags = [torch.zeros(2 * L.OPT_MAX_PEERS, dtype=torch.int64, device=DEV) for _ in range(2)]
    status = torch.zeros(1, dtype=torch.int32, device=DEV)
    L.opt_peer_signal_wait(2, 0, L.PEER_READY, flags, 1, status, 0.05)
    torch.cuda.synchronize()
    assert int(status.item()) == 1
    assert int(flags[1][0]) == 1 and int(flags[0][0]) == 1  # rank 0 did publish its epoch


def test_bad_arguments_rejected(L):
    z = torch.zeros(16, device=DEV)
    with pytest.raises(L.DiffoptError):
        L.opt_adam_fwd_peers(0, [], [], 0, 16, 1, HP, 1.0, z, z, z)
    with pytest.raises(L.DiffoptError):
        L.opt_adam_fwd_peers(1, [z], [z], 2, 8, 1, HP, 1.0, z, z, z)  # lo not a multiple of 4
    with pytest.raises(L.DiffoptError):
        L.opt_adam_fwd_peers(9, [z] * 9, [z] * 9, 0, 16, 1, HP, 1.0, z, z, z)


def _worker(rank, world, init_file, n, steps, out_dir):
    import torch.distributed as dist

    from paper_2211_06934_b200.sharded import PeerShardedAdam

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    opt = PeerShardedAdam(n, world, rank, torch.device(DEV), lr=HP[0])
    gen = torch.Generator(device=DEV).manual_seed(100)
    opt.params[:n] = torch.randn(n, device=DEV, generator=gen)
    for t in range(steps):
        g = torch.Generator(device=DEV).manual_seed(1000 * t + rank)
        opt.grads[:n] = torch.randn(n, device=DEV, generator=g)
        opt.step()  # enqueues only: device-side signal/wait, no host sync
    opt.check()
    np.save(os.path.join(out_dir, f"p{rank}.npy"), opt.params.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_cuda_ipc(L):
    import torch.multiprocessing as mp

    from paper_2211_06934_b200.sharded import shard_size

    n, world, steps = 50_003, 2, 3
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_worker, args=(r, world, os.path.join(d, "init"), n, steps, d))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=240)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
        outs = [np.load(os.path.join(d, f"p{r}.npy")) for r in range(world)]
    shard = shard_size(n, world)
    n_pad = shard * world
    p0 = torch.zeros(n_pad, device=DEV)
    p0[:n] = torch.randn(n, device=DEV, generator=torch.Generator(device=DEV).manual_seed(100))
    grads = []
    for t in range(steps):
        row = []
        for r in range(world):
            g = torch.zeros(n_pad, device=DEV)
            g[:n] = torch.randn(n, device=DEV,
                                generator=torch.Generator(device=DEV).manual_seed(1000 * t + r))
            row.append(g)
        grads.append(row)
    ref = virtual(L, grads, p0, steps).cpu().numpy()
    for r in range(world):
        assert np.array_equal(outs[r], ref), f"rank {r}"


def _maml_worker(rank, world, init_file, out_dir):
    import torch.distributed as dist

    from paper_2211_06934_b200 import maml

    torch.cuda.set_device(0)
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    cfg = maml.MamlConfig(tasks=4, inner_steps=2)
    phi = maml.init_params(0, DEV)
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
    outer = maml.PeerAdamOuter(phi.numel(), world, rank, torch.device(DEV), cfg.outer_lr,
                               cfg.tasks)
    losses, phis = [], []
    for step in range(2):
        phi, loss, _ = maml.outer_step(phi, step, cfg, inner, outer, world, rank)
        losses.append(float(loss))
        phis.append(phi.cpu().numpy())
    np.save(os.path.join(out_dir, f"phi{rank}.npy"), np.stack(phis))
    np.save(os.path.join(out_dir, f"loss{rank}.npy"), np.array(losses))
    dist.barrier()
    dist.destroy_process_group()


def test_maml_outer_step_with_fused_peer_allreduce(L):
    """Two ranks x 2 tasks with the meta-gradient all-reduce fused into the
    outer Adam step (maml.PeerAdamOuter) == one process computing the same
    two local sums, adding them in rank order and taking the fused
    single-GPU Adam step. Step 1 starts from identical inputs: updates agree
    to fp32 rounding. Step 2 starts from phis that differ by that rounding,
    and Adam maps near-zero meta-gradient entries to +-lr-sized updates, so
    there only the replicas' identity and the losses are held tight."""
    import torch.multiprocessing as mp

    from paper_2211_06934_b200 import maml

    world = 2
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_maml_worker, args=(r, world, os.path.join(d, "init"), d))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
        phis = [np.load(os.path.join(d, f"phi{r}.npy")) for r in range(world)]
        losses = [np.load(os.path.join(d, f"loss{r}.npy")) for r in range(world)]
    assert np.array_equal(phis[0], phis[1])  # replicas identical
    assert np.array_equal(losses[0], losses[1])
    # reference in one process with the same summation: the two ranks' local
    # meta-gradient sums (same kernels, same tasks), added in rank order,
    # scaled by 1/tasks, then the fused single-GPU Adam step with apply
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = maml.MamlConfig(tasks=4, inner_steps=2)
    phi = maml.init_params(0, DEV)
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
    tree = L.Tree(numel=phi.numel(), device=DEV)
    m, v = torch.zeros_like(phi), torch.zeros_like(phi)
    ref_losses, refs = [], []
    for step in range(2):
        parts = [maml.meta_grad_tasks(phi, maml.task_range(world, r, cfg.tasks), step, cfg, inner)
                 for r in range(world)]
        g = (parts[0][0] + parts[1][0]) * (1.0 / cfg.tasks)
        ref_losses.append(float((parts[0][1] + parts[1][1]) / cfg.tasks))
        L.opt_adam_fwd(tree, step + 1, (cfg.outer_lr, 0.9, 0.999, 1e-8, 0.0), 0, 1, g, m, v, None,
                       m, v, phi, phi)
        refs.append(phi.cpu().numpy())
    phi0 = maml.init_params(0, "cpu").numpy()
    upd, ref_upd = phis[0][0] - phi0, refs[0] - phi0
    assert np.abs(upd - ref_upd).max() <= 1e-5 * np.abs(ref_upd).max() + 1e-8
    np.testing.assert_allclose(losses[0], ref_losses, rtol=1e-5)
    assert np.all(np.isfinite(phis[0][1]))
