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
    assert len(syms) == 10
    assert set(syms) == set(N.EXPORTS)
    for s in syms:
        assert hasattr(N.lib, s)
    assert N.net_abi_version() == 1


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
