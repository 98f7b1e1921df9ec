"""K-step unrolled differentiable optimization with the reverse meta-gradient
sweep (§2.2 "Explicit Gradient (EG) over
unrolled optimization", Listing 1).

Forward, k = 0..K-1 (t = k+1):  g_k = grad L_in(theta_k, phi);
    (theta_{k+1}, s_{k+1}) = fwd(g_k, s_k) with apply_updates fused.
Reverse (theta_bar_K = dL_out/dtheta_K, state cotangents 0), k = K-1..0:
    (g_bar_k, s_bar_k, h_k) = bwd(g_k, s_k; theta_bar_{k+1}, s_bar_{k+1})
    theta_bar_k = theta_bar_{k+1} + H_k g_bar_k ; phi_bar -= (dg_k/dphi)^T g_bar_k
    hyper_bar += h_k
Saved per step: g_k and s_k ("store some intermediate data that can be
reused during the back-propagation"). The inner loss of the benchmark
(DESIGN.md input recipe, C3) is the diagonal quadratic
L_in = 1/2 sum a (theta - phi)^2, L_out = 1/2 ||theta_K - y||^2; its
gradient and Hessian-vector product run in the library's glue kernels. Every
array op of the sweep is a libdiffopt.so launch on the current stream.
"""
from __future__ import annotations

import torch

from . import _lib as L

NSLOT = {"adam": 2, "rmsprop": 1, "sgd": 1}
NH = {"adam": 4, "rmsprop": 3, "sgd": 2}


class QuadraticSweep:
    """Buffers and launches of one K-step sweep over a flat tree of n
    elements. All state fp32 (or bf16 state with state_dtype=OPT_BF16)."""

    def __init__(self, tree: L.Tree, kind: str, hp, K: int, device,
                 compute=L.OPT_COMPUTE_DEFAULT, state_dtype=L.OPT_F32):
        if kind not in NSLOT:
            raise ValueError(kind)
        if kind == "sgd" and float(hp[1]) == 0.0:
            raise ValueError("sweep needs a stateful optimizer (momentum > 0 for sgd)")
        self.tree, self.kind, self.hp, self.K = tree, kind, tuple(hp), int(K)
        self.dev, self.compute, self.sd = device, compute, state_dtype
        n = tree.numel
        e = lambda dt=torch.float32: torch.empty(n, dtype=dt, device=device)
        sdt = torch.bfloat16 if state_dtype == L.OPT_BF16 else torch.float32
        ns = NSLOT[kind]
        self.g = [e() for _ in range(K)]                       # saved g_k
        self.s = [[None] * ns] + [[e(sdt) for _ in range(ns)] for _ in range(K)]  # s_0 = 0
        self.theta = [e(), e()]
        self.theta_bar, self.phi_bar, self.g_bar = e(), e(), e()
        self.s_bar = [e() for _ in range(ns)]
        self.ones = torch.ones(n, device=device)
        self.hyper = torch.empty(K, NH[kind], dtype=torch.float64, device=device)
        self.ws = tree.workspace(device)
        self.launches_per_sweep = 4 * K + 2

    # ---- one optimizer step with fused apply: theta_out = theta_in + u
    def _fwd(self, k, th_in, th_out):
        t, s_in, s_out, g = k + 1, self.s[k], self.s[k + 1], self.g[k]
        if self.kind == "adam":
            L.opt_adam_fwd(self.tree, t, self.hp, self.sd, self.compute, g, s_in[0], s_in[1],
                           None, s_out[0], s_out[1], th_in, th_out)
        elif self.kind == "rmsprop":
            L.opt_rmsprop_fwd(self.tree, self.hp, self.sd, self.compute, g, s_in[0], None,
                              s_out[0], th_in, th_out)
        else:
            L.opt_sgd_fwd(self.tree, self.hp, self.sd, self.compute, g, s_in[0], None, s_out[0],
                          th_in, th_out)

    def _bwd(self, k):
        t, s_in, g = k + 1, self.s[k], self.g[k]
        last, first = k == self.K - 1, k == 0
        sb_in = [None] * len(self.s_bar) if last else self.s_bar   # s_bar_K = 0
        sb_out = [None] * len(self.s_bar) if first else self.s_bar  # s_bar_0 unused
        if self.kind == "adam":
            L.opt_adam_bwd(self.tree, t, self.hp, self.sd, self.compute, g, s_in[0], s_in[1],
                           self.theta_bar, sb_in[0], sb_in[1], self.g_bar, sb_out[0], sb_out[1],
                           self.hyper[k], None, self.ws)
        elif self.kind == "rmsprop":
            L.opt_rmsprop_bwd(self.tree, self.hp, self.sd, self.compute, g, s_in[0],
                              self.theta_bar, sb_in[0], self.g_bar, sb_out[0], self.hyper[k],
                              None, self.ws)
        else:
            L.opt_sgd_bwd(self.tree, self.hp, self.sd, self.compute, g, s_in[0], self.theta_bar,
                          sb_in[0], self.g_bar, sb_out[0], self.hyper[k], None, self.ws)

    def run(self, a, theta0, phi, y):
        """Enqueue the whole sweep; returns device tensors (theta_K,
        phi_bar, theta0_bar, hyper[K, NH]) without synchronising."""
        n = self.tree.numel
        th = [theta0] + [self.theta[k % 2] for k in range(self.K)]
        for k in range(self.K):
            L.opt_quadratic_grad(n, a, th[k], phi, self.g[k])
            self._fwd(k, th[k], th[k + 1])
        thK = th[self.K]
        # outer loss 1/2 ||theta_K - y||^2: theta_bar_K = 1 * (theta_K - y)
        L.opt_quadratic_grad(n, self.ones, thK, y, self.theta_bar)
        for k in range(self.K - 1, -1, -1):
            self._bwd(k)
            L.opt_quadratic_rev(n, a, self.g_bar, self.theta_bar, self.phi_bar,
                                init_phi=(k == self.K - 1))
        return thK, self.phi_bar, self.theta_bar, self.hyper

    def alg_bytes(self):
        """Algorithmic bytes of one sweep: every array argument of every
        launch read or written once."""
        n, K, ns = self.tree.numel, self.K, NSLOT[self.kind]
        sb = 2 if self.sd == L.OPT_BF16 else 4
        total = 0
        for k in range(K):
            total += 16                                     # a, theta_k, phi -> g_k
            total += 4 + 4 + (ns * sb if k > 0 else 0)      # g_k, theta_k, s_k (NULL at k=0)
            total += ns * sb + 4                            # -> s_{k+1}, theta_{k+1}
        total += 16                                         # ones, theta_K, y -> theta_bar_K
        for k in range(K - 1, -1, -1):
            total += 4 + (ns * sb if k > 0 else 0)          # g_k, s_k
            total += 4 + (0 if k == K - 1 else 4 * ns)      # theta_bar, s_bar_{k+1}
            total += 4 + (0 if k == 0 else 4 * ns)          # -> g_bar, s_bar_k
            total += 12 + 8 + (0 if k == K - 1 else 4)      # a, g_bar, theta_bar (+phi_bar) -> both
        return n * total
