"""GPU tests of libmamlnet.so (include/mamlnet.h) through its autograd
wrappers in maml.py: im2col / col2im against the PyTorch-op versions
(_Im2Col / _Col2Im) and adjointness; the batch-norm + pool + ReLU block's
forward, VJP and VJP-of-VJP against PyTorch autograd of the composition in
float64 (tests/test_mamlnet_math.py pins the header formulas the same way
on CPU), at the network's real geometries and ragged ones."""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def maml():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06934_b200 import maml as m

    return m


def ref_block(x, gamma, beta):
    """relu(max_pool2d(batch_norm(x))) with per-(task, channel) statistics on
    the [T, C, B, H, W] layout, PyTorch ops."""
    T, C, B, H, W = x.shape
    z = F.batch_norm(x.reshape(1, T * C, -1), None, None, gamma.reshape(-1), beta.reshape(-1),
                     training=True, eps=1e-5)
    p = F.max_pool2d(z.reshape(T * C * B, 1, H, W), 2)
    return F.relu(p).reshape(T, C, B, H // 2, W // 2)


def close(got, ref, tol=2e-5):
    """fp32 kernel vs float64 reference: |d| <= tol * (|ref| + max|ref|/10)."""
    got, ref = got.double().cpu(), ref.double().cpu()
    scale = float(ref.abs().max()) + 1e-30
    bad = (got - ref).abs() > tol * (ref.abs() + 0.1 * scale)
    assert not bool(bad.any()), (f"{int(bad.sum())}/{ref.numel()} off; max abs err "
                                 f"{float((got - ref).abs().max()):.3e}, scale {scale:.3e}")


GEOS = [(2, 64, 5, 28, 28), (2, 64, 5, 14, 14), (2, 64, 5, 7, 7), (2, 64, 5, 3, 3),
        (3, 5, 7, 9, 6), (1, 3, 2, 2, 2), (4, 2, 75, 14, 14),
        (2, 3, 25, 28, 28), (1, 2, 75, 14, 14),  # clusters of 8 / 4 CTAs per group
        (1, 2, 64, 64, 64)]  # group slice too large for shared memory: 2-pass fallback


def block_inputs(geo, seed):
    gen = torch.Generator().manual_seed(seed)
    T, C, B, H, W = geo
    x = torch.randn(geo, generator=gen, dtype=torch.float64) * 2 + 0.5
    gamma = torch.rand(T, C, generator=gen, dtype=torch.float64) + 0.5
    beta = torch.randn(T, C, generator=gen, dtype=torch.float64) * 0.3
    dp = torch.randn(T, C, B, H // 2, W // 2, generator=gen, dtype=torch.float64)
    return x, gamma, beta, dp


@pytest.mark.parametrize("geo", GEOS)
def test_bnpool_forward_and_vjp(maml, geo):
    x, gamma, beta, dp = block_inputs(geo, 1)
    xs, gs, bs = (t.clone().requires_grad_(True) for t in (x, gamma, beta))
    ref = ref_block(xs, gs, bs)
    rdx, rdg, rdb = torch.autograd.grad(ref, (xs, gs, bs), dp)
    xf, gf, bf = (t.float().to(DEV).requires_grad_(True) for t in (x, gamma, beta))
    out = maml._BnPool.apply(xf, gf, bf)
    close(out, ref.detach())
    dx, dg, db = torch.autograd.grad(out, (xf, gf, bf), dp.float().to(DEV))
    close(dx, rdx)
    close(dg, rdg)
    close(db, rdb)


@pytest.mark.parametrize("geo", GEOS)
def test_bnpool_second_derivative(maml, geo):
    x, gamma, beta, dp = block_inputs(geo, 2)
    gen = torch.Generator().manual_seed(3)
    gdx = torch.randn(x.shape, generator=gen, dtype=torch.float64)
    gdg = torch.randn(gamma.shape, generator=gen, dtype=torch.float64)
    gdb = torch.randn(gamma.shape, generator=gen, dtype=torch.float64)

    def second(fn, dev, dt):
        xx, gg, bb, dd = (t.to(dev, dt).requires_grad_(True) for t in (x, gamma, beta, dp))
        dx, dg, db = torch.autograd.grad(fn(xx, gg, bb), (xx, gg, bb), dd, create_graph=True)
        c = [t.to(dev, dt) for t in (gdx, gdg, gdb)]
        S = (dx * c[0]).sum() + (dg * c[1]).sum() + (db * c[2]).sum()
        return torch.autograd.grad(S, (dd, xx, gg))

    ref = second(ref_block, "cpu", torch.float64)
    got = second(maml._BnPool.apply, DEV, torch.float32)
    for name, a, b in zip(("g_dp", "g_x", "g_gamma"), got, ref):
        close(a, b, tol=5e-5)


def test_bnpool_second_derivative_partial_cotangents(maml):
    """Only dx carries a cotangent (dgamma, dbeta unused): the NULL paths."""
    x, gamma, beta, dp = block_inputs((2, 4, 5, 14, 14), 4)
    w = torch.randn(x.shape, dtype=torch.float64, generator=torch.Generator().manual_seed(5))

    def run(fn, dt, dev):
        xx, gg, bb, dd = (t.to(dev, dt).requires_grad_(True) for t in (x, gamma, beta, dp))
        (dx,) = torch.autograd.grad(fn(xx, gg, bb), (xx,), dd, create_graph=True)
        return torch.autograd.grad((dx * w.to(dev, dt)).sum(), (dd, xx, gg))

    for a, b in zip(run(maml._BnPool.apply, torch.float32, DEV), run(ref_block, torch.float64,
                                                                       "cpu")):
        close(a, b, tol=5e-5)


@pytest.mark.parametrize("geo", [(2, 1, 5, 28, 28), (2, 64, 5, 14, 14), (3, 4, 2, 7, 7),
                                 (2, 64, 3, 3, 3), (1, 2, 1, 1, 5),
                                 # n % 4 == 0 (float4 im2col) with 4-runs crossing rows and
                                 # images: HW = 15, and H = 1 (the row index wraps at once)
                                 (2, 3, 4, 3, 5), (1, 2, 4, 1, 3)])
def test_im2col_col2im(maml, geo):
    gen = torch.Generator(device=DEV).manual_seed(6)
    h = torch.randn(geo, device=DEV, generator=gen)
    cols = maml._Im2ColK.apply(h)
    assert torch.equal(cols, maml._Im2Col.apply(h))  # a gather: bit-exact
    T, C, B, H, W = geo
    c = torch.randn(cols.shape, device=DEV, generator=gen)
    dh = maml._Col2ImK.apply(c, tuple(geo))
    ref = maml._Col2Im.apply(c.double(), tuple(geo))
    close(dh, ref, tol=1e-6)
    # adjoint pair: <im2col(h), c> = <h, col2im(c)>
    lhs = float((cols.double() * c.double()).sum())
    rhs = float((h.double() * dh.double()).sum())
    assert lhs == pytest.approx(rhs, rel=1e-5)


def test_im2col_double_backward_routes_through_kernels(maml):
    """Second order through the conv: grad of grad uses _Im2ColK again."""
    gen = torch.Generator().manual_seed(7)
    h = torch.randn(2, 3, 2, 6, 6, generator=gen, dtype=torch.float64)
    w = torch.randn(2, 4, 3, 3, 3, generator=gen, dtype=torch.float64)
    b = torch.randn(2, 4, generator=gen, dtype=torch.float64)

    def f(hh, ww, bb, fused):
        out = maml._conv3x3_tasks(hh, ww, bb, maml._Im2ColK.apply if fused else None)
        (gh,) = torch.autograd.grad((out ** 2).sum(), (hh,), create_graph=True)
        return torch.autograd.grad((gh ** 3).sum(), (hh, ww, bb))

    ref = f(*(t.clone().requires_grad_(True) for t in (h, w, b)), False)
    got = f(*(t.float().to(DEV).requires_grad_(True) for t in (h, w, b)), True)
    for a, r in zip(got, ref):
        close(a, r, tol=1e-4)


def test_fused_network_forward_equals_gemm_form(maml):
    T = 3
    sizes = maml.sizes_of(maml.CONV4_SHAPES)
    phi = maml.init_params(0, DEV)
    theta = maml.theta0_tasks(torch.split(phi, sizes), T)
    theta = theta + 0.01 * torch.randn(theta.shape, device=DEV,
                                       generator=torch.Generator(device=DEV).manual_seed(8))
    params = [p.view(T, *s) for p, s in zip(torch.split(theta, [T * n for n in sizes]),
                                            maml.CONV4_SHAPES)]
    x = torch.randn(25, T, 28, 28, device=DEV, generator=torch.Generator(device=DEV).manual_seed(9))
    a = maml.conv4_forward_tasks(params, x, T, "fused")
    b = maml.conv4_forward_tasks([p.double() for p in params], x.double(), T, "gemm")
    close(a, b, tol=1e-4)


@pytest.mark.parametrize("shape", [(4, 64, 576, 14700), (32, 64, 576, 4900), (3, 64, 9, 58800),
                                   (2, 5, 7, 33), (1, 64, 576, 1), (2, 70, 130, 1000),
                                   (4, 64, 576, 225),
                                   # 64 x 9 (first conv layer's weight gradient): many splits,
                                   # one split (straight to C), ragged n
                                   (32, 64, 9, 19600), (1, 64, 9, 100), (2, 64, 9, 33)])
def test_gemm_nt_against_float64(maml, shape):
    """net_gemm_nt (split-K fp32) vs the float64 product; ragged tiles,
    N not a multiple of the k-chunk, several split counts; deterministic."""
    T, M, P, n = shape
    gen = torch.Generator(device=DEV).manual_seed(10)
    a = torch.randn(T, M, n, device=DEV, generator=gen)
    b = torch.randn(T, P, n, device=DEV, generator=gen)
    c = maml._gemm_nt(a, b)
    ref = torch.bmm(a.double(), b.double().transpose(1, 2))
    # fp32 accumulation over n terms of unit variance: error ~ sqrt(n) * 2^-24 * sqrt(n)
    tol = 4 * n * 2.0 ** -24 * 8
    err = float((c.double() - ref).abs().max())
    assert err <= tol * max(1.0, float(ref.abs().max()) / n ** 0.5), (err, tol)
    assert torch.equal(c, maml._gemm_nt(a, b))  # fixed split order: bitwise reproducible


def test_gemm_nt_empty_contraction(maml):
    from paper_2211_06934_b200 import _net as N

    c = torch.full((2, 3, 4), 7.0, device=DEV)
    a = torch.empty(2, 3, 0, device=DEV)
    N.net_gemm_nt(2, 3, 4, 0, a, a, c)
    assert torch.equal(c, torch.zeros_like(c))


def test_task_conv_second_order(maml):
    """The fused convolution (im2col kernel, cuBLAS forward, split-K weight
    gradient) differentiated twice vs the PyTorch-op form in float64."""
    gen = torch.Generator().manual_seed(11)
    h = torch.randn(3, 4, 5, 7, 7, generator=gen, dtype=torch.float64)
    w = torch.randn(3, 6, 4, 3, 3, generator=gen, dtype=torch.float64)
    b = torch.randn(3, 6, generator=gen, dtype=torch.float64)

    def f(hh, ww, bb, fused):
        conv = maml._conv3x3_tasks_fused if fused else maml._conv3x3_tasks
        out = conv(hh, ww, bb)
        gh, gw, gb = torch.autograd.grad((out ** 2).sum(), (hh, ww, bb), create_graph=True)
        return torch.autograd.grad((gh ** 2).sum() + (gw ** 3).sum() + (gb * out.sum()).sum(),
                                   (hh, ww, bb))

    ref = f(*(t.clone().requires_grad_(True) for t in (h, w, b)), False)
    got = f(*(t.float().to(DEV).requires_grad_(True) for t in (h, w, b)), True)
    for a, r in zip(got, ref):
        close(a, r, tol=1e-4)


@pytest.mark.parametrize("geo,second_order", [((32, 64, 25, 28, 28), True),
                                              ((32, 64, 75, 28, 28), False)])
def test_bnpool_full_size_32_tasks(maml, geo, second_order):
    """The 28x28 layer at the bench's 32 tasks (2048 groups of 19,600 /
    58,800 elements: groups above 16K elements are split over 2 / 4-CTA
    clusters, the finer-last-wave plan): forward, VJP and (support size)
    VJP-of-VJP against the float64 composition, computed on the GPU."""
    gen = torch.Generator(device=DEV).manual_seed(8)
    T, C, B, H, W = geo
    x = torch.randn(geo, device=DEV, generator=gen, dtype=torch.float64) * 2 + 0.5
    gamma = torch.rand(T, C, device=DEV, generator=gen, dtype=torch.float64) + 0.5
    beta = torch.randn(T, C, device=DEV, generator=gen, dtype=torch.float64) * 0.3
    dp = torch.randn(T, C, B, H // 2, W // 2, device=DEV, generator=gen, dtype=torch.float64)
    gdx = torch.randn(geo, device=DEV, generator=gen, dtype=torch.float64)

    def run(fn, dt):
        xx, gg, bb, dd = (t.to(dt).requires_grad_(True) for t in (x, gamma, beta, dp))
        out = fn(xx, gg, bb)
        dx, dg, db = torch.autograd.grad(out, (xx, gg, bb), dd, create_graph=second_order)
        res = [out.detach(), dx.detach(), dg.detach(), db.detach()]
        if second_order:
            res += list(torch.autograd.grad((dx * gdx.to(dt)).sum(), (dd, xx, gg)))
        return res

    got = run(maml._BnPool.apply, torch.float32)
    ref = run(ref_block, torch.float64)
    for a, b in zip(got, ref):
        close(a, b, tol=5e-5)
