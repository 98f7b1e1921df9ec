"""GPU tests of the implicit-gradient solvers:
one fused CG iteration against the oracle's textbook iteration, full CG and
Neumann solves against dense/closed-form references, and the IFT
meta-gradient against the closed-form best response."""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import DEV, assert_close, dev_f32, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_06934_b200 as p

    return p


@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_cg_iteration_matches_oracle(pkg, n):
    L = pkg._lib
    rng = np.random.default_rng(n)
    x, r, p, Ap = (rng.standard_normal(n).astype(np.float32) for _ in range(4))
    dx, dr, dp, dAp = (dev_f32(a) for a in (x, r, p, Ap))
    state = torch.zeros(8, dtype=torch.float64, device=DEV)
    ws = L.Tree(numel=n, device=DEV).workspace(DEV)
    rr = float(r.astype(np.float64) @ r.astype(np.float64))
    state[0] = rr
    L.opt_cg_alpha(n, dp, dAp, state, ws)
    L.opt_cg_update(n, dx, dr, dp, dAp, state, ws)
    L.opt_cg_direction(n, dp, dr, state)
    x1, r1, p1, s = oracle.cg_iter(x, r, p, Ap, rr)
    st = host(state)
    abs_pap = float(np.abs(p.astype(np.float64) * Ap).sum())
    assert abs(st[1] - s["pAp"]) <= 1e-12 * abs_pap + 1e-300
    assert st[2] == pytest.approx(s["alpha"], rel=1e-6)
    assert st[0] == pytest.approx(s["rr_new"], rel=1e-5)
    assert st[3] == pytest.approx(s["beta"], rel=1e-5)
    a = abs(s["alpha"])
    assert_close("x", host(dx), x1, scale=np.abs(x) + a * np.abs(p))
    assert_close("r", host(dr), r1, scale=np.abs(r) + a * np.abs(Ap))
    assert_close("p", host(dp), p1, scale=np.abs(r1) + abs(s["beta"]) * np.abs(p) + a * np.abs(Ap))


def test_cg_solve_spd_matches_dense_solve(pkg):
    n = 512
    rng = np.random.default_rng(3)
    M = rng.standard_normal((n, n))
    A = M.T @ M / n + np.eye(n)
    b = rng.standard_normal(n)
    At = torch.tensor(A, dtype=torch.float32, device=DEV)
    cg = pkg.implicit.CG(n, DEV)
    x = cg.solve(lambda v: At @ v, torch.tensor(b, dtype=torch.float32, device=DEV),
                 max_iter=200, tol=1e-6, check_every=5)
    ref = np.linalg.solve(A, b)
    assert np.linalg.norm(host(x) - ref) <= 1e-4 * np.linalg.norm(ref)
    assert cg.residual_ratio() <= 1e-5
    assert cg.iters < 200


def test_neumann_closed_form(pkg):
    b = torch.tensor([1.0, -4.0, 0.5, 2.0, 3.0], device=DEV)
    x = pkg.implicit.neumann_solve(lambda v: 2.0 * v, b, K=20, alpha=0.25)
    ref = b.double().cpu().numpy() / 2 * (1 - 0.5 ** 21)
    np.testing.assert_allclose(host(x), ref, rtol=1e-6)
    x = pkg.implicit.neumann_solve(lambda v: v, b, K=5, alpha=1.0)
    np.testing.assert_allclose(host(x), host(b), rtol=0)


@pytest.mark.parametrize("lam", [0.0, 0.5, 1.0, 10.0])
@pytest.mark.parametrize("solver", ["cg", "neumann"])
def test_ift_meta_gradient_closed_form(pkg, lam, solver):
    """Inner loss 1/2 (theta - phi)^2 + lam/2 theta^2: F = (1+lam) theta - phi,
    theta* = phi/(1+lam), so d(sum theta*)/d phi = 1/(1+lam) per element
    (SPEC implicit-diff example; S:575 closed form)."""
    n = 1000
    phi = torch.linspace(-2, 2, n, device=DEV, requires_grad=True)

    def F(th, ph):
        return (1 + lam) * th - ph

    kw = dict(max_iter=20, tol=1e-7) if solver == "cg" else dict(K=60, alpha=1.0 / (1 + lam) * 0.9)

    @pkg.implicit.custom_root(F, solver=solver, **kw)
    def solve(ph):  # any inner solver; here the exact minimiser
        return ph / (1 + lam)

    theta = solve(phi)
    (g,) = torch.autograd.grad(theta.sum(), phi)
    np.testing.assert_allclose(host(g), np.full(n, 1 / (1 + lam)), rtol=1e-5)
