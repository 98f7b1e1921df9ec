"""GPU tests of the hand-scheduled second-order MAML step (row a10,
paper_2211_06934_b200/maml_explicit.py) and the forward-mode kernels it
adds to libmamlnet.so (include/mamlnet.h, ABI v2).

Kernel checks compare the fp32 kernels with float64 forward-mode AD
(torch.func.jvp / forward-over-reverse) of the PyTorch composition; the
header formulas are pinned the same way on CPU (tests/test_mamlnet_math.py).
The meta-gradient checks compare the whole schedule with an INDEPENDENT
float64 MAML written in this file from torch.nn.functional ops and
torch.autograd.grad(create_graph=True) -- no code of the product's network,
inner step or driver -- per task, and with the product's autograd path."""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
EPS = 1e-5


@pytest.fixture(scope="module")
def mx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    from paper_2211_06934_b200 import maml_explicit as m

    return m


def close(got, ref, tol=2e-5):
    """fp32 kernel vs float64 reference: |d| <= tol * (|ref| + max|ref|/10)."""
    got, ref = got.double().cpu(), ref.double().cpu()
    scale = float(ref.abs().max()) + 1e-30
    bad = (got - ref).abs() > tol * (ref.abs() + 0.1 * scale)
    assert not bool(bad.any()), (f"{int(bad.sum())}/{ref.numel()} off; max abs err "
                                 f"{float((got - ref).abs().max()):.3e}, scale {scale:.3e}")


def ref_block(x, gamma, beta):
    """relu(max_pool2d(batch_norm(x))), per-(task, channel) statistics, on
    [T, C, B, H, W] (float64 PyTorch ops)."""
    T, C, B, H, W = x.shape
    z = F.batch_norm(x.reshape(1, T * C, -1), None, None, gamma.reshape(-1), beta.reshape(-1),
                     training=True, eps=EPS)
    p = F.max_pool2d(z.reshape(T * C * B, 1, H, W), 2)
    return F.relu(p).reshape(T, C, B, H // 2, W // 2)


GEOS = [(2, 64, 5, 28, 28), (2, 64, 25, 14, 14), (2, 64, 5, 7, 7), (4, 64, 25, 3, 3),
        (3, 5, 7, 9, 6), (1, 3, 2, 2, 2), (2, 3, 25, 28, 28), (1, 2, 75, 14, 14)]


def _block_case(geo, seed):
    gen = torch.Generator().manual_seed(seed)
    T, C, B, H, W = geo
    r = lambda *s: torch.randn(*s, generator=gen, dtype=torch.float64)
    x = r(*geo) * 2 + 0.5
    gamma = torch.rand(T, C, generator=gen, dtype=torch.float64) + 0.5
    beta = r(T, C) * 0.3
    dp = r(T, C, B, H // 2, W // 2)
    return x, gamma, beta, dp, r(*geo), r(T, C), r(T, C), r(T, C, B, H // 2, W // 2)


def _fwd_gpu(N, x, gamma, beta):
    T, C, B, H, W = x.shape
    xf, gf, bf = (t.float().to(DEV).contiguous() for t in (x, gamma, beta))
    out = torch.empty(T, C, B, H // 2, W // 2, device=DEV)
    code = torch.empty(out.shape, dtype=torch.uint8, device=DEV)
    mean, rstd = torch.empty(T * C, device=DEV), torch.empty(T * C, device=DEV)
    N.net_bnpool_fwd(T * C, B, H, W, xf, gf, bf, EPS, out, code, mean, rstd)
    return xf, gf, bf, code, mean, rstd


@pytest.mark.parametrize("geo", GEOS)
def test_bnpool_jvp_and_bwd_jvp_against_forward_mode_ad(mx, geo):
    from torch.func import jvp, vjp

    from paper_2211_06934_b200 import _net as N

    x, gamma, beta, dp, xd, gd, bd, dpd = _block_case(geo, 21)
    T, C, B, H, W = geo
    _, ref_outd = jvp(ref_block, (x, gamma, beta), (xd, gd, bd))

    def bwd(dp_, x_, g_):
        return vjp(lambda a, c, b_: ref_block(a, c, b_), x_, g_, beta)[1](dp_)

    _, (rdxd, rdgd, rdbd) = jvp(bwd, (dp, x, gamma), (dpd, xd, gd))
    xf, gf, bf, code, mean, rstd = _fwd_gpu(N, x, gamma, beta)
    xdf, gdf, bdf, dpf, dpdf = (t.float().to(DEV).contiguous() for t in (xd, gd, bd, dp, dpd))
    outd = torch.empty(T, C, B, H // 2, W // 2, device=DEV)
    s1, s2 = torch.empty(T * C, device=DEV), torch.empty(T * C, device=DEV)
    N.net_bnpool_jvp(T * C, B, H, W, xf, xdf, gf, gdf, bdf, code, mean, rstd, outd, s1, s2)
    close(outd, ref_outd)
    # the backward's own outputs (dgamma, dbeta) are inputs of its JVP
    dx = torch.empty_like(xf)
    dg, db = torch.empty(T * C, device=DEV), torch.empty(T * C, device=DEV)
    N.net_bnpool_bwd(T * C, B, H, W, dpf, code, xf, gf, mean, rstd, dx, dg, db)
    dxd = torch.empty_like(xf)
    base_g, base_b = torch.randn(T * C, device=DEV), torch.randn(T * C, device=DEV)
    acc_g, acc_b = base_g.clone(), base_b.clone()  # accumulated into (+=)
    N.net_bnpool_bwd_jvp(T * C, B, H, W, dpf, dpdf, code, xf, xdf, gf, gdf, mean, rstd, dg, db,
                         s1, s2, dxd, acc_g, acc_b)
    close(dxd, rdxd, tol=5e-5)
    close(acc_g - base_g, rdgd.reshape(-1), tol=5e-5)
    close(acc_b - base_b, rdbd.reshape(-1), tol=5e-5)


@pytest.mark.parametrize("T,B", [(3, 25), (2, 75), (5, 1)])
def test_fc_xent_and_jvp_against_float64(mx, T, B):
    from torch.func import grad, jvp

    from paper_2211_06934_b200 import _net as N

    C, J = 64, 5
    gen = torch.Generator().manual_seed(22)
    r = lambda *s: torch.randn(*s, generator=gen, dtype=torch.float64)
    h4, W, b, h4d, Wd, bd = r(T, C, B), r(T, J, C) * 0.3, r(T, J), r(T, C, B), r(T, J, C), r(T, J)
    y = torch.randint(0, J, (T, B), generator=gen)

    def loss_fn(hh, WW, bb):
        logits = hh.transpose(1, 2) @ WW.transpose(1, 2) + bb[:, None, :]
        return F.cross_entropy(logits.reshape(-1, J), y.reshape(-1), reduction="none") \
            .view(T, B).mean(1)

    rl = loss_fn(h4, W, b)
    rg = grad(lambda *a: loss_fn(*a).sum(), argnums=(0, 1, 2))(h4, W, b)
    _, rt = jvp(grad(lambda *a: loss_fn(*a).sum(), argnums=(0, 1, 2)), (h4, W, b), (h4d, Wd, bd))
    g = lambda t: t.float().to(DEV).contiguous()
    yd = y.to(DEV)
    loss, prob = torch.empty(T, device=DEV), torch.empty(T, B, J, device=DEV)
    dW, db, dh4 = torch.empty(T, J, C, device=DEV), torch.empty(T, J, device=DEV), torch.empty(
        T, C, B, device=DEV)
    N.net_fc_xent(T, B, C, J, g(h4), g(W), g(b), yd, loss, prob, dW, db, dh4)
    close(loss, rl)
    close(dh4, rg[0])
    close(dW, rg[1])
    close(db, rg[2])
    aW, ab = torch.ones(T, J, C, device=DEV), torch.ones(T, J, device=DEV)
    dh4d = torch.empty(T, C, B, device=DEV)
    N.net_fc_xent_jvp(T, B, C, J, g(h4), g(h4d), g(W), g(Wd), g(bd), yd, prob, aW, ab, dh4d)
    close(dh4d, rt[0])
    close(aW - 1, rt[1], tol=5e-5)
    close(ab - 1, rt[2], tol=5e-5)


@pytest.mark.parametrize("T,M,P,N_", [(2, 64, 9, 19600), (4, 64, 576, 4900), (3, 64, 576, 225),
                                      (1, 5, 7, 33), (2, 64, 576, 0)])
@pytest.mark.parametrize("pairs,acc", [(1, False), (1, True), (2, False), (2, True)])
def test_gemm_nt2_pairs_and_accumulate(mx, T, M, P, N_, pairs, acc):
    from paper_2211_06934_b200 import _net as N

    gen = torch.Generator(device=DEV).manual_seed(23)
    A, B = (torch.randn(T, M, N_, device=DEV, generator=gen),
            torch.randn(T, P, N_, device=DEV, generator=gen))
    A2, B2 = (torch.randn(T, M, N_, device=DEV, generator=gen),
              torch.randn(T, P, N_, device=DEV, generator=gen)) if pairs == 2 else (None, None)
    C0 = torch.randn(T, M, P, device=DEV, generator=gen)
    Cm = C0.clone()
    wb = N.net_gemm_nt2_workspace_bytes(T, M, P, N_, pairs, acc)
    ws = torch.empty((wb + 3) // 4, device=DEV) if wb else None
    N.net_gemm_nt2(T, M, P, N_, A, B, A2, B2, Cm, acc, ws)
    ref = (C0.double() if acc else 0) + A.double() @ B.double().transpose(1, 2)
    if pairs == 2:
        ref = ref + A2.double() @ B2.double().transpose(1, 2)
    err = float((Cm.double() - ref).abs().max()) if N_ or acc else float(Cm.abs().max())
    assert err <= 1e-5 * max(N_, 1) ** 0.5 + 1e-5
    Cr = C0.clone()
    N.net_gemm_nt2(T, M, P, N_, A, B, A2, B2, Cr, acc, ws)
    assert torch.equal(Cr, Cm)  # fixed-order reduce: bitwise reproducible


def test_task_sum_is_the_broadcast_adjoint(mx):
    from paper_2211_06934_b200 import _net as N

    e = mx.ExplicitMaml(3, mx.MamlConfig(tasks=3, inner_steps=1), DEV)
    x = torch.randn(3 * e.n, device=DEV)
    out = torch.empty(e.n, device=DEV)
    N.net_task_sum(3, len(mx.CONV4_SHAPES), e.h_off, e.d_off, x, out)
    ref = torch.zeros(e.n, dtype=torch.float64, device=DEV)
    ref.index_add_(0, e.bcast, x.double())       # adjoint of the theta_0 gather
    assert float((out.double() - ref).abs().max()) <= 1e-6 * float(ref.abs().max())


# ------------------------------------------------ independent float64 MAML
def ref_conv4(params, x):
    """4 x [conv3x3 -> batch norm (batch statistics) -> ReLU -> 2x2 max-pool],
    fc -> 5 ways, torch.nn.functional only (reading Z16). params: 18 tensors."""
    h = x
    for blk in range(4):
        w, b, gam, bet = params[4 * blk: 4 * blk + 4]
        h = F.conv2d(h, w, b, padding=1)
        h = F.batch_norm(h, None, None, gam, bet, training=True, eps=EPS)
        h = F.max_pool2d(F.relu(h), 2)
    return F.linear(h.flatten(1), params[16], params[17])


def ref_codes(params, x):
    """The network's discontinuous decisions in float64, per conv block: for
    every 2x2 pooling window, the position (dy*2 + dx) of the batch-norm
    output's maximum if it is > 0 (ReLU on), else 255 -- the code layout the
    kernels save ([C, B*H2*W2] per task; include/mamlnet.h)."""
    h, out = x, []
    for blk in range(4):
        w, b, gam, bet = params[4 * blk: 4 * blk + 4]
        z = F.batch_norm(F.conv2d(h, w, b, padding=1), None, None, gam, bet, training=True,
                         eps=EPS)
        B, C, H, W = z.shape
        H2, W2 = H // 2, W // 2
        zw = z[:, :, :2 * H2, :2 * W2].reshape(B, C, H2, 2, W2, 2).permute(1, 0, 2, 4, 3, 5) \
            .reshape(C, B * H2 * W2, 4)
        best, k = zw.max(-1)
        out.append(torch.where(best > 0, k, torch.full_like(k, 255)).to(torch.uint8))
        h = F.max_pool2d(F.relu(z), 2)
    return out


def ref_meta_grad(phi_leaves, xs, ys, xq, yq, steps, lr, mom, codes=None, nesterov=False):
    """float64 second-order MAML meta-gradient of ONE task: `steps` SGD
    momentum steps b' = mom*b + g, theta' = theta - lr*b' (b_0 = 0) on the
    support loss with create_graph=True, then d L_query / d phi. codes (a
    list): receives ref_codes of the support set at theta_0..theta_{K-1}
    and of the query set at theta_K."""
    phi = [p.detach().clone().requires_grad_(True) for p in phi_leaves]
    theta, buf = phi, None
    for _ in range(steps):
        if codes is not None:
            codes.append(ref_codes([t.detach() for t in theta], xs))
        loss = F.cross_entropy(ref_conv4(theta, xs), ys)
        grads = torch.autograd.grad(loss, theta, create_graph=True)
        buf = list(grads) if buf is None else [mom * b + g for b, g in zip(buf, grads)]
        step = [g + mom * b for g, b in zip(grads, buf)] if nesterov else buf
        theta = [t - lr * st for t, st in zip(theta, step)]
    if codes is not None:
        codes.append(ref_codes([t.detach() for t in theta], xq))
    qloss = F.cross_entropy(ref_conv4(theta, xq), yq)
    return (torch.cat([g.reshape(-1) for g in torch.autograd.grad(qloss, phi)]),
            float(qloss.detach()))


BIAS_LEAVES = (1, 5, 9, 13)  # conv biases: inert (reading N5)


def ref_meta_grad_adam(phi_leaves, xs, ys, xq, yq, steps, lr, b1, b2, eps, codes=None):
    """float64 second-order MAML meta-gradient of ONE task with an Adam inner
    loop (bias-corrected, eps outside the sqrt, zero initial moments; reading
    Z1), torch ops and create_graph only. The inert conv biases are left out
    (held at their values): their exactly-zero gradients would put sqrt(0)'s
    infinite slope times 0 into autograd's second derivative, the 0/0 the
    library resolves by convention (reading Z6); their meta-gradient is 0."""
    phi = [p.detach().clone().requires_grad_(i not in BIAS_LEAVES)
           for i, p in enumerate(phi_leaves)]
    live = [i for i in range(len(phi)) if i not in BIAS_LEAVES]
    net = lambda th, x: ref_conv4([None if i in BIAS_LEAVES else t for i, t in enumerate(th)], x)
    theta = phi
    m = [torch.zeros_like(p) for p in phi]
    v = [torch.zeros_like(p) for p in phi]
    for k in range(steps):
        if codes is not None:
            codes.append(ref_codes([t.detach() for t in theta], xs))
        gl = torch.autograd.grad(F.cross_entropy(net(theta, xs), ys), [theta[i] for i in live],
                                 create_graph=True)
        new_t, new_m, new_v = list(theta), list(m), list(v)
        for i, g in zip(live, gl):
            m1 = b1 * m[i] + (1 - b1) * g
            v1 = b2 * v[i] + (1 - b2) * g * g
            u = -lr * (m1 / (1 - b1 ** (k + 1))) / (torch.sqrt(v1 / (1 - b2 ** (k + 1))) + eps)
            new_t[i], new_m[i], new_v[i] = theta[i] + u, m1, v1
        theta, m, v = new_t, new_m, new_v
    if codes is not None:
        codes.append(ref_codes([t.detach() for t in theta], xq))
    qloss = F.cross_entropy(net(theta, xq), yq)
    gq = torch.autograd.grad(qloss, [phi[i] for i in live])
    out = [torch.zeros_like(p) for p in phi]
    for i, g in zip(live, gq):
        out[i] = g
    return torch.cat([g.reshape(-1) for g in out]), float(qloss.detach())


def _phi_leaves(mx, phi):
    sizes = mx.sizes_of(mx.CONV4_SHAPES)
    return [p.view(s) for p, s in zip(torch.split(phi, sizes), mx.CONV4_SHAPES)]


def _engine_codes(eng, t):
    """The codes the engine's kernels saved for task t, in ref_codes' order."""
    return [[a.code[l][t] for l in range(4)] for a in eng.acts] + \
        [[eng.acts_q.code[l][t] for l in range(4)]]


def _per_task_meta_grads(eng):
    """Task t's meta-gradient: its slice of theta_bar_0 (leaf-major buffer)."""
    T = eng.T
    parts = [eng.theta_bar[T * int(eng.off[l]):T * int(eng.off[l + 1])].view(T, -1)
             for l in range(len(eng.off) - 1)]
    return torch.cat(parts, 1)


def _flip_aware_check(eng, data, phi, K, strict=2e-5, min_clean=None, only=None):
    """Per task of an engine that has just run meta_grad on `data`: if every
    routing decision the fp32 kernels took (ReLU on/off, 2x2 argmax, every
    block, every inner step and the query pass) equals float64's, the
    network is the same smooth function on both sides and the meta-gradient
    and query loss must agree to fp32 rounding (`strict`, relative). Tasks
    with a decision inside rounding distance (a 'decision flip', DESIGN.md
    §8) are reported and counted, not compared. Returns (clean errors,
    flipped task indices)."""
    leaves64 = _phi_leaves(eng_mod(), phi.double())
    per = _per_task_meta_grads(eng)
    errs, flipped = [], []
    for t, (xs, ys, xq, yq) in enumerate(data):
        if only is not None and t not in only:
            continue
        codes = []
        if eng.cfg.inner_opt == "adam":
            ref, rloss = ref_meta_grad_adam(leaves64, xs.double(), ys, xq.double(), yq, K,
                                            eng.cfg.inner_lr, eng.cfg.adam_b1, eng.cfg.adam_b2,
                                            eng.cfg.adam_eps, codes)
        else:
            ref, rloss = ref_meta_grad(leaves64, xs.double(), ys, xq.double(), yq, K,
                                       eng.cfg.inner_lr, eng.cfg.inner_momentum, codes,
                                       eng.cfg.nesterov)
        same = all(torch.equal(a.reshape(-1), b.reshape(-1)) for ca, cb in
                   zip(_engine_codes(eng, t), codes) for a, b in zip(ca, cb))
        if not same:
            flipped.append(t)
            continue
        err = float((per[t].double() - ref).norm() / ref.norm())
        lerr = abs(float(eng.acts_q.loss[t]) - rloss) / abs(rloss)
        assert err < strict and lerr < 1e-5, (t, err, lerr)
        errs.append(err)
    if min_clean is not None:
        assert len(errs) >= min_clean, (errs, flipped)
    return errs, flipped


def eng_mod():
    from paper_2211_06934_b200 import maml_explicit

    return maml_explicit


def test_explicit_adam_inner_vs_independent_float64(mx):
    """The explicit schedule with a differentiable ADAM inner loop (the
    paper's MetaAdam use: opt_adam_fwd forward, opt_adam_bwd -- rows a3/a4 --
    in the reverse sweep) vs the independent float64 MAML with Adam steps,
    per task, strict where the routing decisions match; conv-bias
    meta-gradients exactly 0. eps = 1e-2: with eps = 1e-8 Adam's slope
    d u/d g = -lr eps / (|g| + eps)^2 (t = 1) turns the ~1e-9 absolute fp32
    error of near-zero gradient elements into percent-level changes of the
    second-order meta-gradient in ANY fp32 evaluation (measured: 0.6-680% at
    eps 1e-8, 1e-4 at 1e-3, 1.3-8e-6 at 1e-2 / 1e-1 where the routing
    matches; profiles/r02bb_adam_inner_conditioning.txt); the float64
    schedule pin (tests/test_maml_explicit_math.py) covers eps = 1e-8."""
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=1, inner_steps=3, inner_opt="adam", inner_lr=0.01,
                          adam_eps=1e-2)
    eng = mx.ExplicitMaml(1, cfg, DEV)
    phi = maml.init_params(0, DEV)
    clean = 0
    for step, task in [(0, 0), (1, 2), (3, 1), (4, 3), (2, 0), (5, 1)]:
        d = maml.task_data(step, task, DEV)
        mg, _ = mx.meta_grad_explicit(phi, [d], cfg, eng)
        errs, _ = _flip_aware_check(eng, [d], phi, 3)
        clean += len(errs)
        sizes = mx.sizes_of(mx.CONV4_SHAPES)
        offs = [0]
        for sz in sizes:
            offs.append(offs[-1] + sz)
        for leaf in BIAS_LEAVES:
            assert not mg[offs[leaf]:offs[leaf + 1]].any()
    assert clean >= 2, clean


def test_explicit_nesterov_vs_independent_float64(mx):
    """The explicit schedule with Nesterov inner momentum (opt_sgd_fwd/bwd
    carry it) vs the independent float64 MAML with Nesterov steps, per task,
    strict where the routing decisions match."""
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=1, inner_steps=2, nesterov=True)
    eng = mx.ExplicitMaml(1, cfg, DEV)
    phi = maml.init_params(0, DEV)
    clean = 0
    for step, task in [(0, 0), (1, 2), (3, 1), (4, 3), (2, 0), (5, 1), (6, 2), (7, 3)]:
        d = maml.task_data(step, task, DEV)
        mx.meta_grad_explicit(phi, [d], cfg, eng)
        errs, _ = _flip_aware_check(eng, [d], phi, 2)
        clean += len(errs)
    assert clean >= 2, clean


def test_explicit_per_task_vs_independent_float64(mx):
    """Per task (3 inner steps, 8 (step, task) pairs, one task per batch):
    the explicit schedule's meta-gradient and query loss vs the independent
    float64 MAML, strict (2e-5 relative) wherever every routing decision
    matches float64's; decision flips are detected, not tolerated by a
    looser bar (most pairs have none)."""
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=1, inner_steps=3)
    eng = mx.ExplicitMaml(1, cfg, DEV)
    phi = maml.init_params(0, DEV)
    clean = 0
    for step, task in [(0, 0), (0, 1), (1, 2), (1, 3), (3, 0), (3, 2), (4, 0), (4, 3)]:
        d = maml.task_data(step, task, DEV)
        mx.meta_grad_explicit(phi, [d], cfg, eng)
        errs, _ = _flip_aware_check(eng, [d], phi, 3)
        clean += len(errs)
    assert clean >= 5, clean


def test_explicit_task_batch_vs_independent_float64(mx):
    """8 tasks in one batch, all 5 inner steps (the C4 recipe): every task's
    meta-gradient (its slice of theta_bar_0) and query loss vs the
    independent float64 MAML, strict where the routing decisions match; the
    summed meta-gradient is the fixed-order task fold of those slices, and
    the conv-bias meta-gradients are exactly zero (reading N5)."""
    from paper_2211_06934_b200 import maml

    T = 8
    cfg = maml.MamlConfig(tasks=T, inner_steps=5)
    phi = maml.init_params(0, DEV)
    data = [maml.task_data(2, t, DEV) for t in range(T)]
    eng = mx.ExplicitMaml(T, cfg, DEV)
    mg, loss = mx.meta_grad_explicit(phi, data, cfg, eng)
    _flip_aware_check(eng, data, phi, 5, min_clean=2)
    per = _per_task_meta_grads(eng)
    fold = per[0].clone()
    for t in range(1, T):
        fold += per[t]
    assert torch.equal(fold, mg)
    assert float(loss) == pytest.approx(float(eng.acts_q.loss.sum()), rel=1e-6)
    sizes = mx.sizes_of(mx.CONV4_SHAPES)
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    for leaf in (1, 5, 9, 13):
        assert not mg[offs[leaf]:offs[leaf + 1]].any()


@pytest.mark.parametrize("tasks,check", [(32, tuple(range(32))), (4, (0, 1, 2, 3))])
def test_bench_shard_vs_independent_float64(mx, tasks, check):
    """The shards bench.py times, as CUDA graphs with their default task
    groups: 32 tasks (the 1-GPU C4 step: one chain, separate im2col) and 4
    tasks (the 8-GPU shard: four single-task chains, fused next-layer
    columns, captured under the cuBLAS SM-count hint). Seeded outer-step-0
    data as the bench draws it; every task's meta-gradient and query loss vs
    the independent float64 MAML (flip-aware, strict 2e-5; at least half the
    tasks decision-clean), and the shard's meta-gradient equals the
    fixed-order fold of the per-task slices."""
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=tasks)
    phi = maml.init_params(0, DEV)
    shard = mx.ExplicitShard(range(tasks), cfg, DEV)
    assert len(shard.engs) == mx.default_groups(tasks)
    mg, loss = shard(phi, range(tasks), 0, cfg)
    torch.cuda.synchronize()
    data = [maml.task_data(0, t, DEV) for t in range(tasks)]
    clean, off = 0, 0
    for eng in shard.engs:
        part = data[off:off + eng.T]
        only = [t - off for t in check if off <= t < off + eng.T]
        errs, _ = _flip_aware_check(eng, part, phi, cfg.inner_steps, only=only)
        clean += len(errs)
        off += eng.T
    assert clean >= len(check) // 2, clean
    total = None
    for eng in shard.engs:  # group order, each group's fold in task order
        per = _per_task_meta_grads(eng)
        g = per[0].clone()
        for t in range(1, eng.T):
            g += per[t]
        total = g if total is None else total + g
    assert torch.equal(total, mg)


def test_explicit_equals_autograd_path(mx):
    """The explicit schedule and the product's autograd (create_graph) path
    compute the same meta-gradient up to fp32 rounding (8 tasks, 2 steps)."""
    from paper_2211_06934_b200 import maml

    T = 8
    cfg = maml.MamlConfig(tasks=T, inner_steps=2)
    phi = maml.init_params(0, DEV)
    data = [maml.task_data(1, t, DEV) for t in range(T)]
    mg_e, loss_e = mx.meta_grad_explicit(phi, data, cfg)
    mg_a, loss_a = maml.meta_grad_batched(phi, data, cfg, maml.TaskBatchInner(T, DEV, cfg))
    assert float((mg_e - mg_a).norm() / mg_a.norm()) < 1e-4
    assert float(loss_e) == pytest.approx(float(loss_a), rel=1e-5)


@pytest.mark.parametrize("groups", [1, 2])
def test_explicit_shard_graph_replay(mx, groups):
    """The CUDA-graph shard replays the eager schedule bit for bit on fresh
    task data -- with one task group, and with two groups on parallel graph
    branches against two eager engines summed in group order -- and the
    schedule is a few hundred library launches per group."""
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=4)
    shard = mx.ExplicitShard(range(4), cfg, DEV, groups=groups)
    assert 0 < shard.launches_per_replay <= 400 * groups, shard.launches_per_replay
    phi = maml.init_params(0, DEV)
    cuts = [4 * i // groups for i in range(groups + 1)]
    engs = [mx.ExplicitMaml(cuts[i + 1] - cuts[i], cfg, DEV) for i in range(groups)]
    for step in (0, 3, 4, 5):  # 4 and 5: inputs prefetched during the previous replay
        mg_g, loss_g = shard(phi, range(4), step, cfg)
        mg_e = loss_e = None
        for i, e in enumerate(engs):
            m, l = mx.meta_grad_explicit(phi, [maml.task_data(step, t, DEV)
                                               for t in range(cuts[i], cuts[i + 1])], cfg, e)
            mg_e = m if mg_e is None else mg_e + m
            loss_e = l if loss_e is None else loss_e + l
        assert torch.equal(mg_g, mg_e)
        assert torch.equal(loss_g, loss_e)
        phi = phi - 1e-3 * mg_e


def test_seeded_load_and_serial_schedule_are_bitwise_equal(mx):
    """load_seeded draws maml.task_data's values into the static buffers
    bit for bit, and the side-stream schedule computes exactly what the
    single-stream one does (same kernels on the same inputs)."""
    from paper_2211_06934_b200 import maml

    T = 3
    cfg = maml.MamlConfig(tasks=T, inner_steps=2)
    phi = maml.init_params(0, DEV)
    a = mx.ExplicitMaml(T, cfg, DEV)
    b = mx.ExplicitMaml(T, cfg, DEV, concurrent=False)
    a.load_seeded(7, [4, 9, 2])
    b.load([maml.task_data(7, t, DEV) for t in (4, 9, 2)])
    for x, y in ((a.xs, b.xs), (a.xq, b.xq), (a.labels_s, b.labels_s), (a.labels_q, b.labels_q)):
        assert torch.equal(x, y)
    mga, la = a.meta_grad(phi)
    mgb, lb = b.meta_grad(phi)
    torch.cuda.synchronize()
    assert torch.equal(mga, mgb) and torch.equal(la, lb)
    # next-layer columns fused into the norm/pool launches (chains of <= 8
    # tasks) or written by a separate im2col: the same values, bitwise
    assert a.fuse_cols
    c = mx.ExplicitMaml(T, cfg, DEV)
    c.fuse_cols = False
    c.load_seeded(7, [4, 9, 2])
    mgc, lc = c.meta_grad(phi)
    torch.cuda.synchronize()
    assert torch.equal(mga, mgc) and torch.equal(la, lc)


@pytest.mark.parametrize("geo", [(2, 64, 25, 28, 28), (1, 64, 75, 14, 14), (2, 64, 5, 7, 7),
                                 (3, 5, 7, 9, 6), (1, 3, 2, 2, 2), (1, 2, 64, 64, 64)])
def test_bnpool_fused_columns_equal_separate_im2col(mx, geo):
    """net_bnpool_fwd_cols / net_bnpool_jvp_cols (ABI v3): the pooled output
    and tangent are bitwise those of net_bnpool_fwd / net_bnpool_jvp, and the
    fused columns are bitwise net_im2col3x3 of them (a gather of the same
    values) -- the padding taps stay as the caller left them (zero)."""
    from paper_2211_06934_b200 import _net as N

    x, gamma, beta, dp, xd, gd, bd, dpd = _block_case(geo, 33)
    T, C, B, H, W = geo
    H2, W2 = H // 2, W // 2
    xf, gf, bf, code, mean, rstd = _fwd_gpu(N, x, gamma, beta)
    out = torch.empty(T, C, B, H2, W2, device=DEV)
    code2 = torch.empty(out.shape, dtype=torch.uint8, device=DEV)
    mean2, rstd2 = torch.empty(T * C, device=DEV), torch.empty(T * C, device=DEV)
    cols = torch.zeros(T * C, 9, B, H2, W2, device=DEV)
    N.net_bnpool_fwd_cols(T * C, B, H, W, xf, gf, bf, EPS, out, code2, mean2, rstd2, cols)
    ref_out = torch.empty_like(out)
    N.net_bnpool_fwd(T * C, B, H, W, xf, gf, bf, EPS, ref_out, code, mean, rstd)
    assert torch.equal(out, ref_out) and torch.equal(code2, code)
    assert torch.equal(mean2, mean) and torch.equal(rstd2, rstd)
    ref_cols = torch.full_like(cols, float("nan"))
    N.net_im2col3x3(T * C, B, H2, W2, ref_out, ref_cols)
    assert torch.equal(cols, ref_cols)
    # tangent
    xdf, gdf, bdf = (t.float().to(DEV).contiguous() for t in (xd, gd, bd))
    outd, ref_outd = torch.empty_like(out), torch.empty_like(out)
    s1, s2, r1, r2 = (torch.empty(T * C, device=DEV) for _ in range(4))
    tcols = torch.zeros_like(cols)
    N.net_bnpool_jvp_cols(T * C, B, H, W, xf, xdf, gf, gdf, bdf, code, mean, rstd, outd, s1, s2,
                          tcols)
    N.net_bnpool_jvp(T * C, B, H, W, xf, xdf, gf, gdf, bdf, code, mean, rstd, ref_outd, r1, r2)
    assert torch.equal(outd, ref_outd) and torch.equal(s1, r1) and torch.equal(s2, r2)
    N.net_im2col3x3(T * C, B, H2, W2, ref_outd, ref_cols)
    assert torch.equal(tcols, ref_cols)
    with pytest.raises(RuntimeError):
        N.net_bnpool_fwd_cols(T * C, B, H, W, xf, gf, bf, EPS, out, code2, mean2, rstd2, None)
