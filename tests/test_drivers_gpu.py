"""GPU tests of the drivers above the C ABI: the K-step unrolled sweep (row
a9) against the oracle sweep, the autograd wiring (functional API, P:246
torch.autograd.Function) against the oracle VJP, and the MAML meta-batch
(row a10) with the fused inner step against a plain-torch inner step."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_close, assert_sum_close, dev_f32, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_06934_b200 as p

    return p


SWEEP_CASES = [("adam", (1e-2, 0.9, 0.999, 1e-8, 0.0)), ("rmsprop", (1e-2, 0.99, 1e-8)),
               ("sgd", (0.1, 0.9, False)), ("sgd", (0.1, 0.9, True))]


@pytest.mark.parametrize("kind,hp", SWEEP_CASES)
@pytest.mark.parametrize("K", [1, 5])
@pytest.mark.parametrize("fuse", [False, True])
def test_sweep_matches_oracle(pkg, kind, hp, K, fuse):
    """K-step sweep vs the oracle's sweep; fuse=True (Adam) runs the NEXT-2
    fused-glue kernels (opt_adam_quad_fwd / opt_adam_quad_rev)."""
    if fuse and kind != "adam":
        pytest.skip("glue fusion is Adam-only")
    from paper_2211_06934_b200.unroll import QuadraticSweep, NH

    leaves = [7, 4096, 333, 5000, 1]
    n = sum(leaves)
    q = synth.quadratic_problem(0xC3, n)
    tree = pkg.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    sw = QuadraticSweep(tree, kind, hp, K, DEV, fuse_glue=fuse and kind == "adam")
    a, th0, phi, y = (dev_f32(q[k]) for k in ("a", "theta0", "phi", "y"))
    thK, phib, th0b, hyper = sw.run(a, th0, phi, y)
    torch.cuda.synchronize()
    ohp = list(hp[:2]) + [1.0 if hp[2] else 0.0] if kind == "sgd" else list(hp)
    ref = oracle.sweep_quadratic(kind, q["a"], q["theta0"], q["phi"], q["y"], K, ohp, prec=1)
    assert_close("thetaK", host(thK), ref["thetaK"], rtol=1e-5, atol=1e-6,
                 scale=np.abs(ref["thetaK"]) + np.abs(q["theta0"]))
    assert_close("phi_bar", host(phib), ref["phi_bar"], scale=ref["bar_abs"])
    assert_close("theta0_bar", host(th0b), ref["theta0_bar"], scale=ref["bar_abs"])
    hs = host(hyper).sum(0)
    nh = NH[kind]
    assert_sum_close("hyper", hs[:nh], ref["hyper_bar"][:nh], ref["hyper_abs"][:nh])
    assert sw.launches_per_sweep == (2 if sw.fuse else 4) * K + 1


@pytest.mark.parametrize("kind,hp", SWEEP_CASES[:2])
@pytest.mark.parametrize("K,c", [(5, 2), (7, 3), (6, 1), (5, 5)])
def test_checkpointed_sweep_is_bitwise_full_storage(pkg, kind, hp, K, c):
    """NEXT-2: recomputing segments from checkpoints reproduces the full-
    storage sweep bitwise (same deterministic kernels on the same inputs),
    with the launch count the class reports and less saved state."""
    from paper_2211_06934_b200.unroll import QuadraticSweep

    leaves = [7, 4096, 333, 5000, 1]
    q = synth.quadratic_problem(0xC4, sum(leaves))
    tree = pkg.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    args = [dev_f32(q[k]) for k in ("a", "theta0", "phi", "y")]
    full = QuadraticSweep(tree, kind, hp, K, DEV)
    ref = [t.clone() for t in full.run(*args)]
    ck = QuadraticSweep(tree, kind, hp, K, DEV, checkpoint_every=c)
    n0 = pkg._lib.opt_launch_count()
    out = ck.run(*args)
    torch.cuda.synchronize()
    assert pkg._lib.opt_launch_count() - n0 == ck.launches_per_sweep
    for a, b in zip(ref, out):
        assert torch.equal(a, b)
    assert ck.saved_bytes() <= full.saved_bytes()


@pytest.mark.parametrize("c", [5, 2])
def test_fused_glue_sweep_equals_unfused(pkg, c):
    """NEXT-2: the fused-glue sweep (2 launches per step) gives the unfused
    sweep's results (same arithmetic; FMA contraction may differ by an ulp)
    with the launch count it reports, also with checkpointed recompute."""
    from paper_2211_06934_b200.unroll import QuadraticSweep

    leaves = [7, 4096, 333, 5000, 1]
    q = synth.quadratic_problem(0xC5, sum(leaves))
    tree = pkg.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    args = [dev_f32(q[k]) for k in ("a", "theta0", "phi", "y")]
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    ref = [t.clone() for t in QuadraticSweep(tree, "adam", hp, 5, DEV, checkpoint_every=c,
                                             fuse_glue=False).run(*args)]
    sw = QuadraticSweep(tree, "adam", hp, 5, DEV, checkpoint_every=c, fuse_glue=True)
    n0 = pkg._lib.opt_launch_count()
    out = sw.run(*args)
    torch.cuda.synchronize()
    assert pkg._lib.opt_launch_count() - n0 == sw.launches_per_sweep
    for name, a, b in zip(("thetaK", "phi_bar", "theta0_bar"), ref[:3], out[:3]):
        # phi_bar sums -a g_bar over the steps and can cancel: absolute scale
        torch.testing.assert_close(b, a, rtol=1e-5, atol=1e-6 * float(a.abs().max()), msg=name)
    # hyper sums: theta_bar feeds them and differs by rounding; each side is
    # pinned to the oracle by test_sweep_matches_oracle (Sigma|term| bar)
    torch.testing.assert_close(out[3].sum(0), ref[3].sum(0), rtol=1e-4, atol=1e-9)


def test_sweep_bytes_accounting(pkg):
    from paper_2211_06934_b200.unroll import QuadraticSweep

    tree = pkg.Tree(numel=1024, device=DEV)
    sw = QuadraticSweep(tree, "adam", (1e-2, 0.9, 0.999, 1e-8, 0.0), 5, DEV, fuse_glue=False)
    # K=5 Adam: fwd 5x16 + (20 + 4x28) ; outer 16 ; reverse 5x(24 incl.) ...
    per = sw.alg_bytes() // 1024
    assert per == 500  # 212 forward + 16 outer + 272 reverse
    fused = QuadraticSweep(tree, "adam", (1e-2, 0.9, 0.999, 1e-8, 0.0), 5, DEV, fuse_glue=True)
    assert fused.alg_bytes() // 1024 == 400  # 172 forward + 16 outer + 212 reverse


# ------------------------------------------------- autograd / functional
def test_adam_autograd_matches_oracle(pkg):
    """AdamStep.apply forward + torch.autograd backward (through the C ABI)
    equals the oracle's step and VJP, including the lr hyper-gradient."""
    x = synth.state_tree(0xF1, [1000, 37])
    g = dev_f32(x["g"]).requires_grad_(True)
    m = dev_f32(x["m"]).requires_grad_(True)
    v = dev_f32(x["v"]).requires_grad_(True)
    lr = torch.tensor(1e-2, dtype=torch.float64, requires_grad=True)
    cfg = pkg.functional.StepConfig(pkg.Tree(numel=g.numel(), device=DEV))
    u, m1, v1 = pkg.AdamStep.apply(g, m, v, None, lr, 0.9, 0.999, 1e-8, 5, 0.0, cfg)
    du, dm1, dv1 = dev_f32(x["du"]), dev_f32(x["dm1"]), dev_f32(x["dv1"])
    loss = (u * du).sum() + (m1 * dm1).sum() + (v1 * dv1).sum()
    gg, gm, gv, glr = torch.autograd.grad(loss, [g, m, v, lr])
    r = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 5, 1e-2, 0.9, 0.999,
                        1e-8, prec=1)
    mag = oracle.adam_mag(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 5, 1e-2, 0.9, 0.999,
                          1e-8)
    for name, got in (("dg", gg), ("dm", gm), ("dv", gv)):
        assert_close(name, host(got), r[name], scale=np.maximum(np.abs(r[name]), mag[name]))
    assert_sum_close("dlr", [float(glr)], [r["dhp"][0]], [mag["dhp"][0]])


def test_listing1_functional_api_two_steps(pkg):
    """Listing 1: opt.init / opt.update(inplace=False) /
    apply_updates over a 3-leaf tree for two steps, meta-gradient w.r.t. a
    meta-parameter scaling the inner loss; compared with the same program
    on plain torch ops in float64 (independent composed implementation)."""
    torch.manual_seed(0)
    shapes = [(5, 3), (7,), (2, 2, 2)]
    params0 = [torch.randn(s, device=DEV) for s in shapes]
    target = [torch.randn(s, device=DEV) for s in shapes]

    def run(use_fused, dtype):
        meta = torch.tensor(1.5, device=DEV, dtype=dtype, requires_grad=True)
        params = [p.to(dtype).clone().requires_grad_(True) for p in params0]
        if use_fused:
            opt = pkg.adam(lr=0.1)
            layout = pkg.FlatTree.of(params)
            flat = layout.flatten(params)
            state = opt.init(params)
            for _ in range(2):
                ps = layout.views(flat)
                inner = meta * sum(((p - t) ** 2).sum() for p, t in zip(ps, target))
                (gflat,) = torch.autograd.grad(inner, flat, create_graph=True)
                upd, state = opt.update(gflat, state, inplace=False)
                flat = pkg.apply_updates(flat, upd)
            ps = layout.views(flat)
        else:
            ps = params
            m = [torch.zeros_like(p) for p in ps]
            v = [torch.zeros_like(p) for p in ps]
            for t in (1, 2):
                inner = meta * sum(((p - tt.to(dtype)) ** 2).sum() for p, tt in zip(ps, target))
                gs = torch.autograd.grad(inner, ps, create_graph=True)
                m = [0.9 * mm + 0.1 * gg for mm, gg in zip(m, gs)]
                v = [0.999 * vv + 0.001 * gg * gg for vv, gg in zip(v, gs)]
                ps = [p - 0.1 * (mm / (1 - 0.9 ** t)) / ((vv / (1 - 0.999 ** t)).sqrt() + 1e-8)
                      for p, mm, vv in zip(ps, m, v)]
        outer = sum((p.to(torch.float64) ** 2).sum() for p in ps)
        (gmeta,) = torch.autograd.grad(outer, meta)
        return float(outer), float(gmeta)

    o_f, g_f = run(True, torch.float32)
    o_r, g_r = run(False, torch.float64)
    assert o_f == pytest.approx(o_r, rel=1e-5)
    assert g_f == pytest.approx(g_r, rel=1e-3, abs=1e-6)


def test_inplace_differentiable_rejected(pkg):
    opt = pkg.adam(lr=0.1)
    p = torch.randn(8, device=DEV, requires_grad=True)
    state = opt.init(p)
    g = (p * 2).detach().requires_grad_(True)
    with pytest.raises(RuntimeError):
        opt.update(g, state, inplace=True)


# ---------------------------------------------------------------- MAML
def test_maml_fused_inner_matches_torch_inner(pkg):
    """One outer step of a 2-task, 2-inner-step meta-batch: the fused CUDA
    SGD-momentum step (create_graph second-order path) gives the same
    meta-gradient as a plain-torch differentiable SGD-momentum step."""
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=2, inner_steps=2)
    phi = maml.init_params(0, DEV)
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)

    def torch_inner(g, b, theta):
        b1 = g if b is None else cfg.inner_momentum * b + g
        return theta - cfg.inner_lr * b1, b1

    torch.backends.cudnn.deterministic = True
    # TF32 convolutions would round ~1e-3 and turn 1e-7 differences between
    # two fp32 SGD implementations into percent-level meta-gradient noise
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    mg_f, loss_f = maml.meta_grad_tasks(phi, range(2), 0, cfg, inner)
    mg_t, loss_t = maml.meta_grad_tasks(phi, range(2), 0, cfg, torch_inner)
    assert float(loss_f) == pytest.approx(float(loss_t), rel=1e-5)
    err = (mg_f - mg_t).norm() / mg_t.norm()
    assert float(err) < 1e-4
    outer = maml.FusedAdamOuter(phi.numel(), DEV, 1e-3)
    phi2 = phi.clone()
    outer(phi2, mg_f)
    assert torch.isfinite(phi2).all() and not torch.equal(phi2, phi)


@pytest.mark.parametrize("net", ["gemm", "fused"])
@pytest.mark.parametrize("batched", [False, True])
def test_maml_meta_gradient_fp32_accuracy(pkg, batched, net):
    """The production MAML path (fp32 SGEMM network, fused CUDA inner step;
    per-task loop or task-batched) against the same meta-gradient computed
    in float64 with a plain-torch inner step: relative error < 2e-4 (fp32
    rounding through 3 second-order inner steps; cuDNN's fp32 convolutions
    miss this by ~2%, tools/maml_net_check.py)."""
    from paper_2211_06934_b200 import maml

    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = maml.MamlConfig(tasks=2, inner_steps=3, net=net)
    phi = maml.init_params(0, DEV)

    def torch_inner(g, b, theta):
        b1 = g if b is None else cfg.inner_momentum * b + g
        return theta - cfg.inner_lr * b1, b1

    if batched:
        data32 = [maml.task_data(1, t, DEV) for t in range(2)]
        mg, loss = maml.meta_grad_batched(phi, data32, cfg, maml.TaskBatchInner(2, DEV, cfg))
    else:
        inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
        mg, loss = maml.meta_grad_tasks(phi, range(2), 1, cfg, inner)
    data = [[a.double() if a.is_floating_point() else a for a in maml.task_data(1, t, DEV)]
            for t in range(2)]
    cfg64 = maml.MamlConfig(tasks=2, inner_steps=3, net="gemm")  # float64 torch network
    mg64, loss64 = maml.meta_grad_data(phi.double(), data, cfg64, torch_inner)
    err = float((mg.double() - mg64).norm() / mg64.norm())
    assert err < 2e-4, err
    assert float(loss) == pytest.approx(float(loss64), rel=1e-5)
    # reading N5: the conv biases feed batch norms, so their meta-gradient is
    # 0 (float64: rounding-sized); the task-batched fused network leaves
    # them out and returns exact zeros
    offs = [0]
    for shp in maml.CONV4_SHAPES:
        offs.append(offs[-1] + int(torch.Size(shp).numel()))
    for leaf in (1, 5, 9, 13):
        blk64 = mg64[offs[leaf]:offs[leaf + 1]]
        assert float(blk64.abs().max()) <= 1e-9 * float(mg64.norm())
        if batched and net == "fused":
            assert not mg[offs[leaf]:offs[leaf + 1]].any()


@pytest.mark.parametrize("net", ["gemm", "fused"])
def test_maml_per_task_fp32_accuracy(pkg, net):
    """Per-task second-order meta-gradients (3 inner steps) over 8 (step,
    task) pairs against float64: the typical error is fp32 rounding (~2e-6
    measured); decision flips (see test_maml_task_batched_equals_per_task)
    are rare, so the median must be < 1e-5 and at least 6 of 8 < 1e-4."""
    from paper_2211_06934_b200 import maml

    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = maml.MamlConfig(tasks=1, inner_steps=3, net=net)
    cfg64 = maml.MamlConfig(tasks=1, inner_steps=3, net="gemm")
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
    phi = maml.init_params(0, DEV)

    def torch_inner(g, b, theta):
        b1 = g if b is None else cfg.inner_momentum * b + g
        return theta - cfg.inner_lr * b1, b1

    errs = []
    for step, task in [(0, 0), (0, 1), (1, 2), (1, 3), (3, 0), (3, 2), (4, 0), (4, 3)]:
        mg, _ = maml.meta_grad_tasks(phi, [task], step, cfg, inner)
        d = [a.double() if a.is_floating_point() else a for a in maml.task_data(step, task, DEV)]
        mg64, _ = maml.meta_grad_data(phi.double(), [d], cfg64, torch_inner)
        errs.append(float((mg.double() - mg64).norm() / mg64.norm()))
    errs.sort()
    assert errs[3] < 1e-5 and errs[5] < 1e-4, errs


@pytest.mark.parametrize("streams", [1, 3])
def test_maml_graphed_shard_equals_eager(pkg, streams):
    """The CUDA-graph replay of a rank's task shard gives the eager result,
    for two different outer steps (fresh task data through static buffers),
    with the tasks captured on one stream or as parallel graph branches."""
    from paper_2211_06934_b200 import maml

    ntask = 4
    cfg = maml.MamlConfig(tasks=ntask, inner_steps=2)
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.allow_tf32 = False
    shard = maml.GraphedShard(range(ntask), cfg, inner, DEV, streams=streams)
    assert shard.nstreams == streams
    phi = maml.init_params(0, DEV)
    for step in (0, 3):
        mg_e, loss_e = maml.meta_grad_tasks(phi, range(ntask), step, cfg, inner)
        mg_g, loss_g = shard(phi, range(ntask), step, cfg, inner)
        torch.testing.assert_close(mg_g, mg_e, rtol=1e-4, atol=1e-6)
        assert float(loss_g) == pytest.approx(float(loss_e), rel=1e-5)
        phi = phi + 1e-3 * mg_e


@pytest.mark.parametrize("net", ["cudnn", "gemm", "fused"])
def test_maml_task_batched_equals_per_task(pkg, net):
    """The task-batched network (grouped convolutions, per-(task, channel)
    batch norm, one fused inner step over all tasks) gives the per-task
    loop's meta-gradient and loss; eager and CUDA-graph replay.
    The network has discontinuous decisions (ReLU sign, window argmax): where
    one lies within rounding distance, two fp32 evaluations with different
    GEMM shapes can route differently and the second-order meta-gradient
    jumps (1e-4..2e-2). tools/maml_fused_diag.py measured that on (step,
    task) pairs for the gemm and fused forms alike (profiles/
    r01f_maml_decision_flips.txt); step 1's tasks have none, so the two
    summation orders are compared there. test_maml_per_task_fp32_accuracy
    covers the statistics over many pairs."""
    from paper_2211_06934_b200 import maml

    ntask, step = 3, 1
    cfg = maml.MamlConfig(tasks=ntask, inner_steps=3, net=net)
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), DEV, cfg)
    inner_b = maml.TaskBatchInner(ntask, DEV, cfg)
    phi = maml.init_params(0, DEV)
    mg_e, loss_e = maml.meta_grad_tasks(phi, range(ntask), step, cfg, inner)
    data = [maml.task_data(step, t, DEV, cfg.seed) for t in range(ntask)]
    mg_b, loss_b = maml.meta_grad_batched(phi, data, cfg, inner_b)
    # two fp32 evaluations (different GEMM / BN reduction orders) of a
    # 3-step second-order meta-gradient: ~1e-4 apart (each ~1e-4 from fp64,
    # test_maml_meta_gradient_fp32_accuracy)
    assert float((mg_b - mg_e).norm()) <= 5e-4 * float(mg_e.norm())
    assert float(loss_b) == pytest.approx(float(loss_e), rel=1e-5)
    shard = maml.GraphedShard(range(ntask), cfg, inner, DEV, batched=True)
    mg_g, loss_g = shard(phi, range(ntask), step, cfg, inner)
    assert float((mg_g - mg_e).norm()) <= 5e-4 * float(mg_e.norm())
    assert float(loss_g) == pytest.approx(float(loss_e), rel=1e-5)


def test_functional_per_leaf_lr_and_adamw_meta_gradients(pkg):
    """Listing-1 loop with AdamW weight decay and learnable per-leaf learning
    rates (lr_leaf requires grad): the meta-gradients w.r.t. lr_leaf and the
    weight decay match the same program written with plain float64 torch
    ops (independent composed implementation)."""
    torch.manual_seed(1)
    shapes = [(6, 4), (9,), (3, 3)]
    p0 = [torch.randn(s, device=DEV) for s in shapes]
    tgt = [torch.randn(s, device=DEV) for s in shapes]
    lr0 = torch.tensor([0.05, 0.02, 0.1])

    def run(fused):
        dt = torch.float32 if fused else torch.float64
        lr_leaf = lr0.to(DEV, dt).clone().requires_grad_(True)
        wd = torch.tensor(0.01, dtype=torch.float64, requires_grad=True)
        params = [p.to(dt).clone().requires_grad_(True) for p in p0]
        if fused:
            layout = pkg.FlatTree.of(params)
            flat = layout.flatten(params)
            opt = pkg.adam(lr=1e-3, weight_decay=wd, decoupled=True, lr_leaf=lr_leaf)
            state = opt.init(params)
            for _ in range(2):
                ps = layout.views(flat)
                inner = sum(((p - t) ** 2).sum() for p, t in zip(ps, tgt))
                (g,) = torch.autograd.grad(inner, flat, create_graph=True)
                upd, state = opt.update(g, state, params=flat)
                flat = pkg.apply_updates(flat, upd)
            ps = layout.views(flat)
        else:
            ps = params
            m = [torch.zeros_like(p) for p in ps]
            v = [torch.zeros_like(p) for p in ps]
            for t in (1, 2):
                inner = sum(((p - tt.to(dt)) ** 2).sum() for p, tt in zip(ps, tgt))
                gs = torch.autograd.grad(inner, ps, create_graph=True)
                m = [0.9 * a + 0.1 * b for a, b in zip(m, gs)]
                v = [0.999 * a + 0.001 * b * b for a, b in zip(v, gs)]
                ps = [p - lr_leaf[i] * ((mm / (1 - 0.9 ** t)) / ((vv / (1 - 0.999 ** t)).sqrt()
                                                                 + 1e-8) + wd * p)
                      for i, (p, mm, vv) in enumerate(zip(ps, m, v))]
        outer = sum((p.double() ** 2).sum() for p in ps)
        glr, gwd = torch.autograd.grad(outer, [lr_leaf, wd])
        return glr.double().cpu(), float(gwd)

    glr_f, gwd_f = run(True)
    glr_r, gwd_r = run(False)
    torch.testing.assert_close(glr_f, glr_r, rtol=2e-4, atol=1e-5)
    assert gwd_f == pytest.approx(gwd_r, rel=2e-4, abs=1e-6)


def test_functional_centered_momentum_rmsprop_meta_gradients(pkg):
    """Listing-1 loop with centred momentum RMSProp (weight decay, learnable
    per-leaf lr, learnable alpha / eps / momentum): meta-gradients equal the
    same program written with plain float64 torch ops
    (torch.optim.RMSprop's update rule, composed)."""
    torch.manual_seed(2)
    shapes = [(5, 4), (7,), (2, 3)]
    p0 = [torch.randn(s, device=DEV) for s in shapes]
    tgt = [torch.randn(s, device=DEV) for s in shapes]
    lr0 = torch.tensor([0.03, 0.01, 0.05])

    def run(fused):
        dt = torch.float32 if fused else torch.float64
        lr_leaf = lr0.to(DEV, dt).clone().requires_grad_(True)
        mk = lambda x: torch.tensor(x, dtype=torch.float64, requires_grad=True)
        alpha, eps, mom, wd = mk(0.9), mk(1e-3), mk(0.8), mk(0.02)
        params = [p.to(dt).clone().requires_grad_(True) for p in p0]
        if fused:
            layout = pkg.FlatTree.of(params)
            flat = layout.flatten(params)
            opt = pkg.rmsprop(lr=1e-2, alpha=alpha, eps=eps, momentum=mom, centered=True,
                              weight_decay=wd, lr_leaf=lr_leaf)
            state = opt.init(params)
            for _ in range(3):
                ps = layout.views(flat)
                inner = sum(((p - t) ** 4).sum() for p, t in zip(ps, tgt))
                (g,) = torch.autograd.grad(inner, flat, create_graph=True)
                upd, state = opt.update(g, state, params=flat)
                flat = pkg.apply_updates(flat, upd)
            ps = layout.views(flat)
        else:
            ps = params
            v = [torch.zeros_like(p) for p in ps]
            a = [torch.zeros_like(p) for p in ps]
            b = [torch.zeros_like(p) for p in ps]
            for _ in range(3):
                inner = sum(((p - tt.to(dt)) ** 4).sum() for p, tt in zip(ps, tgt))
                gs = torch.autograd.grad(inner, ps, create_graph=True)
                gs = [gg + wd * p for gg, p in zip(gs, ps)]
                v = [alpha * x + (1 - alpha) * gg * gg for x, gg in zip(v, gs)]
                a = [alpha * x + (1 - alpha) * gg for x, gg in zip(a, gs)]
                b = [mom * x + gg / ((vv - aa * aa).sqrt() + eps)
                     for x, gg, vv, aa in zip(b, gs, v, a)]
                ps = [p - lr_leaf[i] * bb for i, (p, bb) in enumerate(zip(ps, b))]
        outer = sum((p.double() ** 2).sum() for p in ps)
        grads = torch.autograd.grad(outer, [lr_leaf, alpha, eps, mom, wd])
        return [x.double().cpu() for x in grads]

    got, ref = run(True), run(False)
    for name, x, y in zip(("lr_leaf", "alpha", "eps", "momentum", "wd"), got, ref):
        torch.testing.assert_close(x, y, rtol=5e-4, atol=1e-5, msg=name)


@pytest.mark.parametrize("packed", [False, True])
def test_host_streamed_step_equals_device_step(pkg, packed):
    """offload.HostStreamedAdam (pinned host arrays, chunked H2D / kernels /
    D2H on three streams) gives the device-resident step's outputs bitwise
    per element, and the chunk-ordered hyper-gradient sum to rounding --
    with six separate host arrays per direction, and with the arrays as rows
    of one buffer (alloc_host(): one opt_copy_rows DMA per chunk and
    direction)."""
    from paper_2211_06934_b200.offload import HostStreamedAdam, IN_KEYS, OUT_KEYS

    leaves = [70000, 4096, 333, 120000]
    n = sum(leaves)
    x = synth.state_tree(0xF5, leaves)
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.0)
    L = pkg._lib
    if packed:
        h_in, h_out = HostStreamedAdam.alloc_host(n)
        for k in IN_KEYS:
            h_in[k].copy_(torch.from_numpy(x[k]))
        for k in OUT_KEYS:
            h_out[k].fill_(float("nan"))
    else:
        h_in = {k: torch.from_numpy(x[k]).pin_memory() for k in IN_KEYS}
        h_out = {k: torch.empty(n).pin_memory() for k in OUT_KEYS}
    hs = HostStreamedAdam(n, DEV, chunks=5)
    assert (hs._rows([h_in[k] for k in IN_KEYS], n) is not None) == packed
    h_dhp = hs.run(h_in, h_out, 4, hp)
    torch.cuda.synchronize()
    d = {k: dev_f32(x[k]) for k in IN_KEYS}
    o = {k: torch.empty(n, device=DEV) for k in OUT_KEYS}
    tree = L.Tree(numel=n, device=DEV)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_fwd(tree, 4, hp, 0, 0, d["g"], d["m"], d["v"], o["u"], o["m1"], o["v1"])
    L.opt_adam_bwd(tree, 4, hp, 0, 0, d["g"], d["m"], d["v"], d["du"], d["dm1"], d["dv1"],
                   o["dg"], o["dm"], o["dv"], dhp, None, tree.workspace(DEV))
    for k in OUT_KEYS:
        assert torch.equal(h_out[k], o[k].cpu()), k
    ref = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 4, *hp)
    np.testing.assert_allclose(h_dhp.numpy(), host(dhp), rtol=1e-9,
                               atol=1e-12 * ref["dhp_abs"].max())
    # the chunk rows are summed on the device in chunk order (opt_sum_rows)
    rows = hs.dhp.cpu().numpy()
    want = np.zeros(4)
    for r in rows:
        want += r
    np.testing.assert_array_equal(h_dhp.numpy(), want)
    # back-to-back calls (the next call's host->device copies may start while
    # the previous call's results stream out): three more steps on new
    # gradients, no synchronisation in between; the last one checked
    # (each call gets its own host input buffers: a host array may not be
    # rewritten while an enqueued copy still reads it)
    ins = []
    for rep in range(3):
        hi = HostStreamedAdam.alloc_host(n)[0] if packed else {
            k: torch.empty(n).pin_memory() for k in IN_KEYS}
        for k in IN_KEYS:
            hi[k].copy_(h_in[k])
        hi["g"].mul_((-0.5) ** (rep + 1))
        ins.append(hi)
    for hi in ins:
        hs.run(hi, h_out, 4, hp, inputs_on_host=True)
    torch.cuda.synchronize()
    d["g"].copy_(ins[-1]["g"])
    L.opt_adam_fwd(tree, 4, hp, 0, 0, d["g"], d["m"], d["v"], o["u"], o["m1"], o["v1"])
    L.opt_adam_bwd(tree, 4, hp, 0, 0, d["g"], d["m"], d["v"], d["du"], d["dm1"], d["dv1"],
                   o["dg"], o["dm"], o["dv"], dhp, None, tree.workspace(DEV))
    for k in OUT_KEYS:
        assert torch.equal(h_out[k], o[k].cpu()), k
    # default mode: inputs written into host memory by device work still
    # queued on the current stream (a device->host copy), then run(): the
    # uploads must wait for it
    hi = ins[0]
    g_dev = torch.full((n,), 0.25, device=DEV)
    torch.cuda._sleep(2_000_000)  # keep the stream busy so an early upload would see stale data
    hi["g"].copy_(g_dev, non_blocking=True)
    hs.run(hi, h_out, 4, hp)
    torch.cuda.synchronize()
    d["g"].fill_(0.25)
    L.opt_adam_fwd(tree, 4, hp, 0, 0, d["g"], d["m"], d["v"], o["u"], o["m1"], o["v1"])
    L.opt_adam_bwd(tree, 4, hp, 0, 0, d["g"], d["m"], d["v"], d["du"], d["dm1"], d["dv1"],
                   o["dg"], o["dm"], o["dv"], dhp, None, tree.workspace(DEV))
    for k in OUT_KEYS:
        assert torch.equal(h_out[k], o[k].cpu()), k


def test_host_streamed_c2_bench_config(pkg):
    """The e2e configuration bench.py times: the C2 tree (11,689,512
    elements) through HostStreamedAdam with 12 chunks, packed host rows
    (opt_copy_rows) and back-to-back pipelined calls: every output element
    bitwise equal to the device-resident fused step, the chunk-ordered
    hyper-gradient sums equal to the whole-tree launch's to rounding."""
    from paper_2211_06934_b200.offload import HostStreamedAdam, IN_KEYS, OUT_KEYS

    leaves = synth.RESNET18_LEAVES
    n = int(sum(leaves))
    x = synth.state_tree(0xC2, leaves)
    hp, t = (1e-3, 0.9, 0.999, 1e-8, 0.0), 10
    L = pkg._lib
    h_in, h_out = HostStreamedAdam.alloc_host(n)
    for k in IN_KEYS:
        h_in[k].copy_(torch.from_numpy(x[k]))
    hs = HostStreamedAdam(n, DEV, chunks=12)
    for _ in range(3):
        h_dhp = hs.run(h_in, h_out, t, hp, inputs_on_host=True)
    torch.cuda.synchronize()
    d = {k: dev_f32(x[k]) for k in IN_KEYS}
    o = {k: torch.empty(n, device=DEV) for k in OUT_KEYS}
    tree = L.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_fwd(tree, t, hp, 0, 0, d["g"], d["m"], d["v"], o["u"], o["m1"], o["v1"])
    L.opt_adam_bwd(tree, t, hp, 0, 0, d["g"], d["m"], d["v"], d["du"], d["dm1"], d["dv1"],
                   o["dg"], o["dm"], o["dv"], dhp, None, tree.workspace(DEV))
    for k in OUT_KEYS:
        assert torch.equal(h_out[k], o[k].cpu()), k
    full = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], t, *hp)
    np.testing.assert_allclose(h_dhp.numpy(), host(dhp), rtol=1e-9,
                               atol=1e-12 * full["dhp_abs"].max())


def test_sum_rows_fixed_order(pkg):
    """opt_sum_rows: column sums in row order, bitwise equal to a sequential
    fp64 sum of the same rows; rows = 0 writes zeros."""
    L = pkg._lib
    rng = np.random.default_rng(3)
    for rows, cols in ((1, 4), (7, 4), (33, 5), (1000, 3), (65, 70)):
        x = rng.standard_normal((rows, cols)) * 10.0 ** rng.integers(-8, 8, (rows, cols))
        out = torch.empty(cols, dtype=torch.float64, device=DEV)
        L.opt_sum_rows(rows, cols, torch.from_numpy(x).to(DEV), out)
        # lane l sums rows l, l+32, ... then a xor tree: compare to the same order in numpy
        lanes = np.zeros((32, cols))
        for r in range(rows):
            lanes[r % 32] += x[r]
        for o in (16, 8, 4, 2, 1):
            lanes = lanes + lanes[np.arange(32) ^ o]
        np.testing.assert_array_equal(host(out), lanes[0])
        np.testing.assert_allclose(host(out), x.sum(0), rtol=1e-12, atol=1e-12 * np.abs(x).sum())
    out = torch.full((3,), 5.0, dtype=torch.float64, device=DEV)
    L.opt_sum_rows(0, 3, None, out)
    assert torch.all(out == 0)


def test_sharded_adam_fused_local_step(pkg):
    """ShardedAdam's fused shard step (world = 1: the whole padded tree is
    the shard) equals three plain opt_adam_fwd steps with apply."""
    from paper_2211_06934_b200 import sharded

    n = 70001
    opt = sharded.ShardedAdam(n, 1, 0, DEV, lr=1e-2)
    p = torch.zeros(opt.n_pad, device=DEV)
    p[:n] = torch.linspace(-1, 1, n, device=DEV)
    ref = p.clone()
    L = pkg._lib
    tree = L.Tree(numel=opt.n_pad, device=DEV)
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    for t in range(1, 4):
        g = torch.randn(opt.n_pad, device=DEV, generator=torch.Generator(device=DEV).manual_seed(t))
        opt.step(p, g)
        L.opt_adam_fwd(tree, t, (1e-2, 0.9, 0.999, 1e-8, 0.0), 0, 0, g, m, v, None, m, v, ref, ref)
    assert torch.equal(p, ref)


# ------------------------------------------- functional API input handling
@pytest.mark.parametrize("kind", ["adam", "rmsprop", "sgd", "rmsprop_cm", "adamw"])
def test_bf16_state_autograd_cotangents_are_widened(pkg, kind):
    """bfloat16 state through the autograd Functions: the
    cotangent autograd hands a bf16 state output is bf16; the Function must
    widen it to float32 before the C call (diffopt.h reads cotangents as
    float). Checked bitwise against a direct C-ABI call with the widened
    cotangents, plus a 2-step Listing-1 meta-gradient within bf16 rounding
    of the fp32-state run."""
    torch.manual_seed(3)
    n = 4097
    tree = pkg.Tree(numel=n, device=DEV)
    cfg = pkg.functional.StepConfig(tree)
    g = torch.randn(n, device=DEV) * 1e-2
    s0 = (torch.rand(n, device=DEV) * 1e-4).to(torch.bfloat16).requires_grad_(True)
    s1 = (torch.rand(n, device=DEV) * 1e-4).to(torch.bfloat16).requires_grad_(True)
    du, dn0, dn1 = (torch.randn(n, device=DEV) for _ in range(3))
    gg = g.clone().requires_grad_(True)
    L = pkg._lib
    if kind == "adam":
        hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
        u, a, b = pkg.AdamStep.apply(gg, s0, s1, None, *hp[:4], 3, 0.0, cfg)
        loss = (u * du).sum() + (a.float() * dn0).sum() + (b.float() * dn1).sum()
        got = torch.autograd.grad(loss, [gg, s0, s1])
        ref = [torch.empty(n, device=DEV) for _ in range(3)]
        L.opt_adam_bwd(tree, 3, hp, L.OPT_BF16, L.OPT_COMPUTE_DEFAULT, g, s0.detach(),
                       s1.detach(), du, dn0.bfloat16().float(), dn1.bfloat16().float(), *ref)
    elif kind == "rmsprop":
        hp = (1e-2, 0.99, 1e-8)
        u, a = pkg.RmsPropStep.apply(gg, s0, None, *hp, cfg)
        loss = (u * du).sum() + (a.float() * dn0).sum()
        got = torch.autograd.grad(loss, [gg, s0])
        ref = [torch.empty(n, device=DEV) for _ in range(2)]
        L.opt_rmsprop_bwd(tree, hp, L.OPT_BF16, L.OPT_COMPUTE_DEFAULT, g, s0.detach(), du,
                          dn0.bfloat16().float(), *ref)
    elif kind == "sgd":
        hp = (1e-1, 0.9, True)
        u, a = pkg.SgdStep.apply(gg, s0, None, *hp, cfg)
        loss = (u * du).sum() + (a.float() * dn0).sum()
        got = torch.autograd.grad(loss, [gg, s0])
        ref = [torch.empty(n, device=DEV) for _ in range(2)]
        L.opt_sgd_bwd(tree, hp, L.OPT_BF16, L.OPT_COMPUTE_DEFAULT, g, s0.detach(), du,
                      dn0.bfloat16().float(), *ref)
    elif kind == "rmsprop_cm":
        hp = (1e-2, 0.9, 1e-3, 0.5, True)
        ext = L._ext()
        gavg = (torch.randn(n, device=DEV) * 1e-3).to(torch.bfloat16).requires_grad_(True)
        u, a, c, b = pkg.functional.RmsCmStep.apply(gg, s0, gavg, s1, None, *hp[:4], 0.0, None,
                                                    (True, False, False), cfg)
        loss = ((u * du).sum() + (a.float() * dn0).sum() + (c.float() * dn1).sum()
                + (b.float() * du).sum())
        got = torch.autograd.grad(loss, [gg, s0, gavg, s1])
        ref = [torch.empty(n, device=DEV) for _ in range(4)]
        L.opt_rmsprop_cm_bwd(tree, hp, ext, L.OPT_BF16, L.OPT_COMPUTE_DEFAULT, g, s0.detach(),
                             gavg.detach(), s1.detach(), None, du, dn0.bfloat16().float(),
                             dn1.bfloat16().float(), du.bfloat16().float(), *ref, None)
    else:  # adamw through the _ex path
        hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
        p = torch.randn(n, device=DEV)
        u, a, b = pkg.functional.StepEx.apply(gg, s0, s1, p, hp[0], 0.1, None, hp[1:4], "adam",
                                              3, (True, False, False, 0.0, False), cfg)
        loss = (u * du).sum() + (a.float() * dn0).sum() + (b.float() * dn1).sum()
        got = torch.autograd.grad(loss, [gg, s0, s1])
        ref = [torch.empty(n, device=DEV) for _ in range(3)]
        ext = L._ext(0.1, True, False, None)
        L.opt_adam_bwd_ex(tree, 3, hp, ext, L.OPT_BF16, L.OPT_COMPUTE_DEFAULT, g, s0.detach(),
                          s1.detach(), p, du, dn0.bfloat16().float(), dn1.bfloat16().float(),
                          *ref, None)
    torch.cuda.synchronize()
    assert torch.equal(got[0], ref[0]), "gradient cotangent"
    for x, y in zip(got[1:], ref[1:]):
        # the gradient of a bf16 leaf is bf16: autograd rounds the fp32 VJP
        assert x.dtype == torch.bfloat16
        assert torch.equal(x, y.bfloat16())


@pytest.mark.parametrize("make", ["adam", "rmsprop", "sgd"])
def test_listing1_bf16_state_meta_gradient(pkg, make):
    """Two Listing-1 steps with bf16 optimizer state: the meta-gradient is
    within bf16 rounding (1e-2, reading Z9) of the fp32-state run."""
    torch.manual_seed(4)
    shapes = [(33, 7), (129,), (4, 4, 4)]
    p0 = [torch.randn(s, device=DEV) for s in shapes]
    tgt = [torch.randn(s, device=DEV) for s in shapes]

    def run(sd):
        meta = torch.tensor(1.5, device=DEV, requires_grad=True)
        params = [p.clone().requires_grad_(True) for p in p0]
        opt = {"adam": lambda: pkg.adam(lr=0.05, state_dtype=sd),
               "rmsprop": lambda: pkg.rmsprop(lr=0.01, state_dtype=sd),
               "sgd": lambda: pkg.sgd(lr=0.05, momentum=0.9, state_dtype=sd)}[make]()
        layout = pkg.FlatTree.of(params)
        flat = layout.flatten(params)
        state = opt.init(params)
        for _ in range(2):
            ps = layout.views(flat)
            # meta shifts the target (a loss scale would cancel in Adam/RMSProp)
            inner = sum(((p - meta * t) ** 2).sum() for p, t in zip(ps, tgt))
            (g,) = torch.autograd.grad(inner, flat, create_graph=True)
            upd, state = opt.update(g, state)
            flat = pkg.apply_updates(flat, upd)
        outer = (flat.double() ** 2).sum()
        (gm,) = torch.autograd.grad(outer, meta)
        assert all(s is None or s.dtype == (torch.bfloat16 if sd == pkg._lib.OPT_BF16
                                            else torch.float32) for s in state.slots)
        return float(outer), float(gm)

    o32, g32 = run(pkg._lib.OPT_F32)
    o16, g16 = run(pkg._lib.OPT_BF16)
    assert np.isfinite(g16)
    assert o16 == pytest.approx(o32, rel=1e-2)
    assert abs(g32) > 1e-2
    assert g16 == pytest.approx(g32, rel=1e-2)


def test_update_accepts_flat_gradient_of_multi_leaf_tree(pkg):
    """update() with the 1-D flat gradient autograd returns for a flat
    parameter buffer of a many-leaf tree takes it as the flat buffer (no
    per-element flatten); equals the leaf-list path bitwise."""
    import time
    sizes = [300_000, 7, 200_000, 1]
    params = [torch.randn(s, device=DEV) for s in sizes]
    opt = pkg.adam(lr=1e-2)
    layout = pkg.FlatTree.of(params)
    flat_g = torch.randn(sum(sizes), device=DEV)
    st = opt.init(params)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u1, _ = opt.update(flat_g, st)
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 1.0
    u2, _ = opt.update(layout.views(flat_g), st)
    assert torch.equal(u1, u2)


def test_fixed_lr_leaf_with_learnable_weight_decay_large_tree(pkg):
    """A fixed (non-learnable) lr_leaf plus a learnable weight decay on a
    >1M-element tree: the library sums per leaf whenever lr_leaf is given,
    so the Function must size the per-leaf workspace."""
    sizes = [1_500_000, 300_001, 17]
    tree = pkg.Tree.from_sizes(sizes, device=DEV)
    cfg = pkg.functional.StepConfig(tree)
    n = tree.numel
    g = (torch.randn(n, device=DEV) * 1e-2).requires_grad_(True)
    p = torch.randn(n, device=DEV)
    lr_leaf = torch.tensor([1e-2, 2e-2, 3e-2], device=DEV)
    wd = torch.tensor(0.1, dtype=torch.float64, requires_grad=True)
    u, a, b = pkg.functional.StepEx.apply(g, None, None, p, 1e-2, wd, lr_leaf, (0.9, 0.999, 1e-8),
                                          "adam", 1, (True, False, False, 0.0, False), cfg)
    (gwd,) = torch.autograd.grad(u.sum(), [wd])
    # AdamW: u = -lr_l (g / (|g| + eps) + wd p) at t = 1, so du/dwd = -lr_l p
    lrs = torch.repeat_interleave(lr_leaf.double(), torch.tensor(sizes, device=DEV))
    want = float(-(lrs * p.double()).sum())
    assert float(gwd) == pytest.approx(want, rel=1e-5, abs=1e-3)
