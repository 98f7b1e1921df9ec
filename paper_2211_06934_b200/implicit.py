"""Implicit-gradient (IG) mode (§2.2).

At a stationary point F(theta*, phi) = 0 the implicit function theorem gives
the best-response derivative without unrolling: for a cotangent v of theta*,
    (dF/dtheta)^T u = v,   dL/dphi = -(dF/dphi)^T u.
The linear solve is matrix-free: conjugate gradient (iMAML) or a truncated
Neumann series. The matrix-vector products are autograd VJPs through
F (the caller's model); every other vector operation of each iteration runs
in libdiffopt.so's fused kernels with device-resident scalars (no host
synchronisation except an optional convergence check every few iterations).
"""
from __future__ import annotations

import torch

from . import _lib as L


class CG:
    """Conjugate gradient on flat fp32 vectors of n elements."""

    def __init__(self, n, device):
        self.n, self.dev = int(n), device
        e = lambda: torch.empty(self.n, device=device)
        self.x, self.r, self.p = e(), e(), e()
        self.state = torch.zeros(8, dtype=torch.float64, device=device)
        self.ws = L.Tree(numel=max(self.n, 1), device=device).workspace(device)
        self.iters = 0

    def solve(self, matvec, b, max_iter=100, tol=1e-5, check_every=10, x0=None):
        """x with ||A x - b|| <= tol ||b|| (checked every `check_every`
        iterations, the only host syncs) or after max_iter iterations."""
        n = self.n
        b = b.contiguous()
        Ax0 = None
        if x0 is None:
            self.x.zero_()
        else:
            self.x.copy_(x0)
            Ax0 = matvec(self.x).contiguous()
        L.opt_cg_init(n, b, Ax0, self.r, self.p, self.state, self.ws)
        self.iters = 0
        for it in range(max_iter):
            Ap = matvec(self.p).contiguous()
            L.opt_cg_alpha(n, self.p, Ap, self.state, self.ws)
            L.opt_cg_update(n, self.x, self.r, self.p, Ap, self.state, self.ws)
            self.iters = it + 1
            if check_every and (it + 1) % check_every == 0:
                rr, rr0 = self.state[0].item(), self.state[4].item()
                if rr <= tol * tol * rr0:
                    break
            L.opt_cg_direction(n, self.p, self.r, self.state)
        return self.x

    def residual_ratio(self):
        rr, rr0 = self.state[0].item(), self.state[4].item()
        return (rr / rr0) ** 0.5 if rr0 > 0 else 0.0


def neumann_solve(matvec, b, K=10, alpha=1.0):
    """x = alpha sum_{k=0}^{K} (I - alpha A)^k b  (spectral radius of
    I - alpha A below 1 is the caller's choice of alpha)."""
    b = b.contiguous()
    n = b.numel()
    v = torch.zeros_like(b)
    x = torch.zeros_like(b)
    L.opt_neumann_step(n, v, b, x, -alpha)  # v = x = alpha b
    for _ in range(K):
        Av = matvec(v).contiguous()
        L.opt_neumann_step(n, v, Av, x, alpha)
    return x


def implicit_grad(F, theta_star, phi, v, solver="cg", **kw):
    """dL/dphi for L depending on theta* through v = dL/dtheta*, by the IFT
    on the optimality condition F(theta, phi) = 0 (flat tensors)."""
    th = theta_star.detach().requires_grad_(True)
    ph = phi.detach().requires_grad_(True)
    Fv = F(th, ph)

    def matvec(w):  # (dF/dtheta)^T w
        (jt,) = torch.autograd.grad(Fv, th, grad_outputs=w, retain_graph=True)
        return jt

    if solver == "cg":
        u = CG(th.numel(), th.device).solve(matvec, v.detach(), **kw).clone()
    else:
        u = neumann_solve(matvec, v.detach(), **kw)
    (gphi,) = torch.autograd.grad(Fv, ph, grad_outputs=u)
    return -gphi


class _Root(torch.autograd.Function):
    @staticmethod
    def forward(ctx, phi, solve, F, solver, kw):
        theta = solve(phi.detach())
        ctx.save_for_backward(theta, phi)
        ctx.F, ctx.solver, ctx.kw = F, solver, kw
        return theta

    @staticmethod
    def backward(ctx, v):
        theta, phi = ctx.saved_tensors
        with torch.enable_grad():
            g = implicit_grad(ctx.F, theta, phi, v.contiguous(), ctx.solver, **ctx.kw)
        return g, None, None, None, None


def custom_root(F, solver="cg", **kw):
    """Listing 2 shape: wrap an inner solver theta* = solve(phi)
    so that gradients w.r.t. phi flow by the implicit function theorem on
    F(theta, phi) = 0 instead of through the solver's iterations."""

    def deco(solve):
        def wrapped(phi):
            return _Root.apply(phi, solve, F, solver, kw)

        return wrapped

    return deco
