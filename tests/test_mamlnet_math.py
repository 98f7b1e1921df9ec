"""CPU checks (float64, no GPU) of the MAML network library's contract
(include/mamlnet.h): the closed-form VJP and VJP-of-VJP it states for the
batch-norm + 2x2 max-pool + ReLU block are restated here from the header
and compared with PyTorch autograd's first and second derivatives of the
composition relu(max_pool2d(batch_norm(x))) -- an independent derivation.
Also: the library loads and exports every symbol the header declares, and
rejects bad geometry before launching anything."""
import os
import re

import pytest
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EPS = 1e-5


def block_ref(x, gamma, beta):
    """The composition with PyTorch ops. x [G, B, H, W]; per-group stats."""
    G, B, H, W = x.shape
    z = F.batch_norm(x.reshape(1, G, B * H * W), None, None, gamma, beta, training=True, eps=EPS)
    return F.relu(F.max_pool2d(z.reshape(G * B, 1, H, W), 2)).reshape(G, B, H // 2, W // 2)


def stats(x):
    G = x.shape[0]
    xf = x.reshape(G, -1)
    mean = xf.mean(1)
    rstd = 1.0 / torch.sqrt(((xf - mean[:, None]) ** 2).mean(1) + EPS)
    return mean, rstd


def routed(x, gamma, beta, dp):
    """dy: the pooled cotangent routed to each active window's maximum."""
    G, B, H, W = x.shape
    mean, rstd = stats(x)
    z = gamma[:, None, None, None] * (x - mean[:, None, None, None]) * rstd[:, None, None, None] \
        + beta[:, None, None, None]
    H2, W2 = H // 2, W // 2
    zw = z[:, :, :2 * H2, :2 * W2].reshape(G, B, H2, 2, W2, 2).permute(0, 1, 2, 4, 3, 5)
    zw = zw.reshape(G, B, H2, W2, 4)
    best, k = zw.max(-1)
    on = best > 0
    onehot = F.one_hot(k, 4).to(x.dtype) * on[..., None].to(x.dtype)
    dyw = onehot * dp[..., None]
    dy = torch.zeros_like(x)
    dy[:, :, :2 * H2, :2 * W2] = dyw.reshape(G, B, H2, W2, 2, 2).permute(0, 1, 2, 4, 3, 5) \
        .reshape(G, B, 2 * H2, 2 * W2)
    return dy, onehot


def header_bwd(x, gamma, beta, dp):
    """net_bnpool_bwd as include/mamlnet.h states it."""
    G = x.shape[0]
    n = x[0].numel()
    mean, rstd = stats(x)
    xh = (x - mean[:, None, None, None]) * rstd[:, None, None, None]
    dy, _ = routed(x, gamma, beta, dp)
    dbeta = dy.reshape(G, -1).sum(1)
    dgamma = (dy * xh).reshape(G, -1).sum(1)
    e = lambda v: v[:, None, None, None]
    dx = e(gamma * rstd) * (dy - e(dbeta / n) - xh * e(dgamma / n))
    return dx, dgamma, dbeta


def header_bwd2(x, gamma, beta, dp, gdx, gdgamma, gdbeta):
    """net_bnpool_bwd2 as include/mamlnet.h states it."""
    G, B, H, W = x.shape
    n = x[0].numel()
    e = lambda v: v[:, None, None, None]
    s = lambda v: v.reshape(G, -1).sum(1)
    mean, rstd = stats(x)
    r = rstd
    xh = (x - e(mean)) * e(r)
    dy, onehot = routed(x, gamma, beta, dp)
    _, dgamma, dbeta = header_bwd(x, gamma, beta, dp)
    A, Bm = dbeta / n, dgamma / n
    G1, Gx = s(gdx), s(gdx * xh)
    GD = s(gdx * dy) - A * G1
    h = -e(gamma * r) * (dy * e(Gx / n) + e(Bm) * gdx) + e(gdgamma) * dy
    mh = s(h) / n
    mhx = s(h * xh) / n
    g_x = e(r) * (h - e(mh) - xh * e(mhx)) - e(gamma * r * r / n * (GD - Bm * Gx)) * xh
    g_dy = e(gamma * r) * (gdx - e(G1 / n) - xh * e(Gx / n)) + e(gdgamma) * xh + e(gdbeta)
    H2, W2 = H // 2, W // 2
    gw = g_dy[:, :, :2 * H2, :2 * W2].reshape(G, B, H2, 2, W2, 2).permute(0, 1, 2, 4, 3, 5) \
        .reshape(G, B, H2, W2, 4)
    g_dp = (gw * onehot).sum(-1)
    g_gamma = r * (GD - Bm * Gx)
    return g_dp, g_x, g_gamma


SHAPES = [(3, 2, 6, 6), (4, 3, 7, 7), (2, 5, 3, 3), (3, 2, 4, 5), (2, 1, 2, 2)]


def inputs(shape, seed):
    gen = torch.Generator().manual_seed(seed)
    G, B, H, W = shape
    x = torch.randn(shape, generator=gen, dtype=torch.float64) * 1.7 + 0.3
    gamma = torch.rand(G, generator=gen, dtype=torch.float64) + 0.5
    beta = torch.randn(G, generator=gen, dtype=torch.float64) * 0.3
    dp = torch.randn(G, B, H // 2, W // 2, generator=gen, dtype=torch.float64)
    return x, gamma, beta, dp


@pytest.mark.parametrize("shape", SHAPES)
def test_forward_matches_composition(shape):
    x, gamma, beta, dp = inputs(shape, 1)
    mean, rstd = stats(x)
    z = gamma[:, None, None, None] * (x - mean[:, None, None, None]) * rstd[:, None, None, None] \
        + beta[:, None, None, None]
    G, B, H, W = shape
    ref = block_ref(x, gamma, beta)
    mine = F.relu(F.max_pool2d(z.reshape(G * B, 1, H, W), 2)).reshape(ref.shape)
    torch.testing.assert_close(mine, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("shape", SHAPES)
def test_header_vjp_matches_autograd(shape):
    x, gamma, beta, dp = inputs(shape, 2)
    xs, gs, bs = (t.clone().requires_grad_(True) for t in (x, gamma, beta))
    ref = torch.autograd.grad(block_ref(xs, gs, bs), (xs, gs, bs), dp)
    mine = header_bwd(x, gamma, beta, dp)
    for a, b in zip(mine, ref):
        torch.testing.assert_close(a, b, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("which", ["all", "gdx", "gdgamma", "gdbeta"])
def test_header_second_derivative_matches_autograd(shape, which):
    x, gamma, beta, dp = inputs(shape, 3)
    gen = torch.Generator().manual_seed(4)
    gdx = torch.randn(x.shape, generator=gen, dtype=torch.float64)
    gdg = torch.randn(x.shape[0], generator=gen, dtype=torch.float64)
    gdb = torch.randn(x.shape[0], generator=gen, dtype=torch.float64)
    if which != "all":  # one cotangent at a time: each term is pinned alone
        gdx, gdg, gdb = (t if nm == which else torch.zeros_like(t)
                         for t, nm in ((gdx, "gdx"), (gdg, "gdgamma"), (gdb, "gdbeta")))
    xs, gs, bs, dps = (t.clone().requires_grad_(True) for t in (x, gamma, beta, dp))
    dx, dg, db = torch.autograd.grad(block_ref(xs, gs, bs), (xs, gs, bs), dps, create_graph=True)
    S = (dx * gdx).sum() + (dg * gdg).sum() + (db * gdb).sum()
    ref_dp, ref_x, ref_g = torch.autograd.grad(S, (dps, xs, gs), allow_unused=True)
    g_dp, g_x, g_gamma = header_bwd2(x, gamma, beta, dp, gdx, gdg, gdb)
    torch.testing.assert_close(g_dp, ref_dp, rtol=1e-9, atol=1e-11)
    torch.testing.assert_close(g_x, ref_x, rtol=1e-9, atol=1e-11)
    torch.testing.assert_close(g_gamma, ref_g, rtol=1e-9, atol=1e-11)


def test_second_derivative_wrt_beta_is_zero():
    """dx, dgamma, dbeta do not depend on beta except through the piecewise-
    constant routing: the header's bwd2 has no beta output."""
    x, gamma, beta, dp = inputs((3, 2, 6, 6), 5)
    xs, gs, bs = (t.clone().requires_grad_(True) for t in (x, gamma, beta))
    dx, dg, db = torch.autograd.grad(block_ref(xs, gs, bs), (xs, gs, bs), dp, create_graph=True)
    S = dx.sum() + dg.sum() + db.sum()
    (gb,) = torch.autograd.grad(S, (bs,), allow_unused=True)
    assert gb is None or float(gb.abs().max()) < 1e-10


def test_conv_bias_before_batch_norm_is_inert():
    """Reading N5: the fused network leaves the conv bias out
    because a training-mode batch norm follows. In float64 with PyTorch's
    own conv2d and batch_norm: the block's output with and without a
    per-channel bias agrees to rounding, and the first and second
    derivatives w.r.t. the bias vanish (BN's input gradient sums to zero
    over every channel group)."""
    g = torch.Generator().manual_seed(11)
    x = torch.randn(6, 3, 10, 10, generator=g, dtype=torch.float64)
    w = torch.randn(4, 3, 3, 3, generator=g, dtype=torch.float64, requires_grad=True)
    b = (3 * torch.randn(4, generator=g, dtype=torch.float64)).requires_grad_(True)
    gam = (torch.rand(4, generator=g, dtype=torch.float64) + 0.5).requires_grad_(True)
    bet = torch.randn(4, generator=g, dtype=torch.float64, requires_grad=True)

    def net(bias):
        y = F.conv2d(x, w, bias, padding=1)
        z = F.batch_norm(y, None, None, gam, bet, training=True, eps=EPS)
        return F.relu(F.max_pool2d(z, 2))

    out_b, out_0 = net(b), net(None)
    torch.testing.assert_close(out_b, out_0, rtol=0, atol=1e-12)
    dp = torch.randn(out_b.shape, generator=g, dtype=torch.float64)
    gw, gb = torch.autograd.grad(out_b, (w, b), dp, create_graph=True)
    assert float(gb.abs().max()) < 1e-11 * float(dp.abs().sum())
    (ggb,) = torch.autograd.grad((gw * torch.randn(gw.shape, generator=g, dtype=torch.float64))
                                 .sum(), (b,), allow_unused=True)
    assert ggb is None or float(ggb.abs().max()) < 1e-9


# ------------------------------------------- forward-mode (JVP) formulas
def header_jvp(x, gamma, beta, xd, gd, bd):
    """net_bnpool_jvp as include/mamlnet.h states it: (outd, s1, s2)."""
    G, B, H, W = x.shape
    e = lambda v: v[:, None, None, None]
    mean, r = stats(x)
    xh = (x - e(mean)) * e(r)
    a = xd.reshape(G, -1).mean(1)
    b = (xh * xd).reshape(G, -1).mean(1)
    xhd = e(r) * (xd - e(a) - xh * e(b))
    zd = e(gd) * xh + e(gamma) * xhd + e(bd)
    _, onehot = routed(x, gamma, beta, torch.zeros(G, B, H // 2, W // 2, dtype=x.dtype))
    H2, W2 = H // 2, W // 2
    zw = zd[:, :, :2 * H2, :2 * W2].reshape(G, B, H2, 2, W2, 2).permute(0, 1, 2, 4, 3, 5) \
        .reshape(G, B, H2, W2, 4)
    return (zw * onehot).sum(-1), a, b


def header_bwd_jvp(x, gamma, beta, dp, xd, gd, dpd):
    """net_bnpool_bwd_jvp as include/mamlnet.h states it: (dxd, dgammad, dbetad)."""
    G = x.shape[0]
    n = x[0].numel()
    e = lambda v: v[:, None, None, None]
    s = lambda v: v.reshape(G, -1).sum(1)
    mean, r = stats(x)
    xh = (x - e(mean)) * e(r)
    _, a, b = header_jvp(x, gamma, beta, xd, gd, torch.zeros_like(gd))
    xhd = e(r) * (xd - e(a) - xh * e(b))
    dy, _ = routed(x, gamma, beta, dp)
    dyd, _ = routed(x, gamma, beta, dpd)
    _, dgamma, dbeta = header_bwd(x, gamma, beta, dp)
    A, Bm = dbeta / n, dgamma / n
    dbetad = s(dyd)
    dgammad = s(dyd * xh + dy * xhd)
    D = dy - e(A) - xh * e(Bm)
    Dd = dyd - e(dbetad / n) - xhd * e(Bm) - xh * e(dgammad / n)
    dxd = e(gd * r - gamma * r * r * b) * D + e(gamma * r) * Dd
    return dxd, dgammad, dbetad


def _tangents(shape, seed):
    gen = torch.Generator().manual_seed(seed)
    G, B, H, W = shape
    return (torch.randn(shape, generator=gen, dtype=torch.float64),
            torch.randn(G, generator=gen, dtype=torch.float64),
            torch.randn(G, generator=gen, dtype=torch.float64),
            torch.randn(G, B, H // 2, W // 2, generator=gen, dtype=torch.float64))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("which", ["all", "xd", "gd", "bd"])
def test_header_jvp_matches_forward_mode_ad(shape, which):
    """net_bnpool_jvp's formula vs torch.func.jvp of the composition, each
    tangent alone and together (an independent forward-mode derivation)."""
    from torch.func import jvp

    x, gamma, beta, _ = inputs(shape, 6)
    xd, gd, bd, _ = _tangents(shape, 7)
    if which != "all":
        xd, gd, bd = (t if nm == which else torch.zeros_like(t)
                      for t, nm in ((xd, "xd"), (gd, "gd"), (bd, "bd")))
    _, ref = jvp(block_ref, (x, gamma, beta), (xd, gd, bd))
    mine, _, _ = header_jvp(x, gamma, beta, xd, gd, bd)
    torch.testing.assert_close(mine, ref, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("which", ["all", "dpd", "xd", "gd"])
def test_header_bwd_jvp_matches_forward_over_reverse_ad(shape, which):
    """net_bnpool_bwd_jvp's formula vs torch.func.jvp of the VJP map
    (dp, x, gamma) -> (dx, dgamma, dbeta): forward-over-reverse AD."""
    from torch.func import jvp, vjp

    x, gamma, beta, dp = inputs(shape, 8)
    xd, gd, _, dpd = _tangents(shape, 9)
    if which != "all":
        xd, gd, dpd = (t if nm == which else torch.zeros_like(t)
                       for t, nm in ((xd, "xd"), (gd, "gd"), (dpd, "dpd")))

    def bwd(dp_, x_, g_):
        return vjp(lambda a, c: block_ref(a, c, beta), x_, g_)[1](dp_)

    _, (rx, rg) = jvp(bwd, (dp, x, gamma), (dpd, xd, gd))
    _, rb = jvp(lambda dp_, x_, g_: torch.func.vjp(lambda bb: block_ref(x_, g_, bb), beta)[1](dp_)[0],
                (dp, x, gamma), (dpd, xd, gd))
    dxd, dgd, dbd = header_bwd_jvp(x, gamma, beta, dp, xd, gd, dpd)
    torch.testing.assert_close(dxd, rx, rtol=1e-9, atol=1e-11)
    torch.testing.assert_close(dgd, rg, rtol=1e-9, atol=1e-11)
    torch.testing.assert_close(dbd, rb, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("shape", SHAPES[:3])
def test_bwd_jvp_is_the_adjoint_of_bwd2(shape):
    """<w, J t> = <J^T w, t>: the forward-mode tangent of the backward
    (header_bwd_jvp) against the reverse-mode second derivative
    (header_bwd2, itself pinned to autograd above) -- the two derivations
    of the same Jacobian must be adjoint."""
    x, gamma, beta, dp = inputs(shape, 10)
    xd, gd, _, dpd = _tangents(shape, 11)
    gen = torch.Generator().manual_seed(12)
    gdx = torch.randn(x.shape, generator=gen, dtype=torch.float64)
    gdg = torch.randn(x.shape[0], generator=gen, dtype=torch.float64)
    gdb = torch.randn(x.shape[0], generator=gen, dtype=torch.float64)
    dxd, dgd, dbd = header_bwd_jvp(x, gamma, beta, dp, xd, gd, dpd)
    lhs = (gdx * dxd).sum() + (gdg * dgd).sum() + (gdb * dbd).sum()
    g_dp, g_x, g_gamma = header_bwd2(x, gamma, beta, dp, gdx, gdg, gdb)
    rhs = (g_dp * dpd).sum() + (g_x * xd).sum() + (g_gamma * gd).sum()
    assert abs(float(lhs - rhs)) <= 1e-10 * (abs(float(lhs)) + 1.0)


def header_fc_xent(h4, Wfc, bfc, labels):
    """net_fc_xent as include/mamlnet.h states it: h4 [T, C, B]."""
    feat = h4.transpose(1, 2)                                  # [T, B, C]
    logits = feat @ Wfc.transpose(1, 2) + bfc[:, None, :]
    prob = torch.softmax(logits, -1)
    B = h4.shape[2]
    loss = -torch.log(prob.gather(-1, labels[..., None])[..., 0]).mean(1)
    dl = (prob - F.one_hot(labels, Wfc.shape[1]).to(h4.dtype)) / B
    dW = dl.transpose(1, 2) @ feat
    db = dl.sum(1)
    dh4 = (dl @ Wfc).transpose(1, 2)
    return loss, prob, dW, db, dh4


def header_fc_xent_jvp(h4, Wfc, bfc, labels, h4d, Wd, bd):
    """net_fc_xent_jvp as include/mamlnet.h states it: (dWd, dbd, dh4d)."""
    _, prob, _, _, _ = header_fc_xent(h4, Wfc, bfc, labels)
    feat, featd = h4.transpose(1, 2), h4d.transpose(1, 2)
    B = h4.shape[2]
    ld = featd @ Wfc.transpose(1, 2) + feat @ Wd.transpose(1, 2) + bd[:, None, :]
    dld = prob * (ld - (prob * ld).sum(-1, keepdim=True)) / B
    dl = (prob - F.one_hot(labels, Wfc.shape[1]).to(h4.dtype)) / B
    dWd = dld.transpose(1, 2) @ feat + dl.transpose(1, 2) @ featd
    dbd = dld.sum(1)
    dh4d = (dld @ Wfc + dl @ Wd).transpose(1, 2)
    return dWd, dbd, dh4d


def _head_inputs(seed, T=3, B=7, C=6, J=5):
    gen = torch.Generator().manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=gen, dtype=torch.float64)
    labels = torch.randint(0, J, (T, B), generator=gen)
    return r(T, C, B), r(T, J, C), r(T, J), labels, r(T, C, B), r(T, J, C), r(T, J)


def test_header_fc_xent_matches_autograd():
    h4, W, b, y, _, _, _ = _head_inputs(13)
    hs, Ws, bs = (t.clone().requires_grad_(True) for t in (h4, W, b))
    logits = hs.transpose(1, 2) @ Ws.transpose(1, 2) + bs[:, None, :]
    lref = F.cross_entropy(logits.reshape(-1, W.shape[1]), y.reshape(-1), reduction="none") \
        .view(y.shape).mean(1)
    gh, gW, gb = torch.autograd.grad(lref.sum(), (hs, Ws, bs))
    loss, _, dW, db, dh4 = header_fc_xent(h4, W, b, y)
    torch.testing.assert_close(loss, lref.detach(), rtol=1e-12, atol=1e-12)
    for a, r in ((dW, gW), (db, gb), (dh4, gh)):
        torch.testing.assert_close(a, r, rtol=1e-10, atol=1e-12)


def test_header_fc_xent_jvp_matches_forward_over_reverse_ad():
    from torch.func import grad, jvp

    h4, W, b, y, h4d, Wd, bd = _head_inputs(14)

    def loss_fn(hh, WW, bb):
        logits = hh.transpose(1, 2) @ WW.transpose(1, 2) + bb[:, None, :]
        return F.cross_entropy(logits.reshape(-1, WW.shape[1]), y.reshape(-1),
                               reduction="none").view(y.shape).mean(1).sum()

    _, (rh, rW, rb) = jvp(grad(loss_fn, argnums=(0, 1, 2)), (h4, W, b), (h4d, Wd, bd))
    dWd, dbd, dh4d = header_fc_xent_jvp(h4, W, b, y, h4d, Wd, bd)
    for a, r in ((dWd, rW), (dbd, rb), (dh4d, rh)):
        torch.testing.assert_close(a, r, rtol=1e-10, atol=1e-12)


# ------------------------------------------------------------- the library
def declared():
    src = open(os.path.join(ROOT, "include", "mamlnet.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(net_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def N():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2211_06934_b200 import _net

    return _net


def test_header_symbols_exported(N):
    syms = declared()
    assert len(syms) == 19
    assert set(syms) == set(N.EXPORTS)
    for s in syms:
        assert hasattr(N.lib, s)
    assert N.net_abi_version() == 3


def test_bad_geometry_rejected_before_launch(N):
    n0 = N.net_launch_count()
    with pytest.raises(RuntimeError, match="bad geometry"):
        N.net_bnpool_fwd(4, 2, 1, 5, 16, 16, 16, 1e-5, 16, 16, 16, 16, stream=0)  # H < 2
    with pytest.raises(RuntimeError, match="eps"):
        N.net_bnpool_fwd(4, 2, 4, 4, 16, 16, 16, -1.0, 16, 16, 16, 16, stream=0)
    with pytest.raises(RuntimeError, match="NULL"):
        N.net_bnpool_bwd(4, 2, 4, 4, None, 16, 16, 16, 16, 16, 16, 16, 16, stream=0)
    with pytest.raises(RuntimeError, match="bad geometry"):
        N.net_im2col3x3(-1, 2, 4, 4, 16, 16, stream=0)
    N.net_im2col3x3(0, 2, 4, 4, None, None, stream=0)  # empty: valid, nothing launched
    assert N.net_launch_count() == n0
