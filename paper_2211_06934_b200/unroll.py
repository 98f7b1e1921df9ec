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
    elements. All state fp32 (or bf16 state with state_dtype=OPT_BF16).

    ``checkpoint_every = c`` (NEXT-2, memory-saving recompute for long
    unrolls): only (theta_k, s_k) at segment starts k = 0, c, 2c, ... are kept
    from the forward pass; the reverse sweep recomputes each earlier segment's
    c steps from its checkpoint (the same deterministic kernels, so the
    recomputed g_k, s_k are bitwise those of the first pass) and then
    reverses it. Saved state drops from K x (g + state) to
    ceil(K/c) x (theta + state) + c x (g + state) for one extra forward over
    the first K - c steps. c = K (default) is plain full storage."""

    def __init__(self, tree: L.Tree, kind: str, hp, K: int, device,
                 compute=L.OPT_COMPUTE_DEFAULT, state_dtype=L.OPT_F32, checkpoint_every=None,
                 fuse_glue=None):
        if kind not in NSLOT:
            raise ValueError(kind)
        if kind == "sgd" and float(hp[1]) == 0.0:
            raise ValueError("sweep needs a stateful optimizer (momentum > 0 for sgd)")
        self.tree, self.kind, self.hp, self.K = tree, kind, tuple(hp), int(K)
        self.dev, self.compute, self.sd = device, compute, state_dtype
        c = int(checkpoint_every or K)
        if not 1 <= c <= K:
            raise ValueError("checkpoint_every must be in [1, K]")
        self.c = c
        self.nseg = -(-K // c)
        n = tree.numel
        e = lambda dt=torch.float32: torch.empty(n, dtype=dt, device=device)
        sdt = torch.bfloat16 if state_dtype == L.OPT_BF16 else torch.float32
        ns = NSLOT[kind]
        es = lambda: [e(sdt) for _ in range(ns)]
        self.g_seg = [e() for _ in range(c)]                 # g_k of the segment in reverse
        self.s_seg = [None] + [es() for _ in range(c)]       # s_seg[r+1] = state after step r
        self.th_ck = [None] + [e() for _ in range(self.nseg - 1)]   # theta at segment starts
        self.s_ck = [[None] * ns] + [es() for _ in range(self.nseg - 1)]
        self.g_tmp = e() if self.nseg > 1 else None
        self.s_pp = [es(), es()] if self.nseg > 1 else None
        self.theta = [e(), e()]
        self.thK_buf = e()
        self.theta_bar, self.phi_bar, self.g_bar = e(), e(), e()
        self.s_bar = [e() for _ in range(ns)]
        self.ones = torch.ones(n, device=device)
        self.hyper = torch.empty(K, NH[kind], dtype=torch.float64, device=device)
        self.ws = tree.workspace(device)
        recompute = K - self._seg_len(self.nseg - 1)
        # NEXT-2 glue fusion (Adam): the quadratic-loss gradient is computed
        # inside the step (opt_adam_quad_fwd) and its reverse inside the VJP
        # (opt_adam_quad_rev): 2 launches per step instead of 4
        self.fuse = (kind == "adam") if fuse_glue is None else bool(fuse_glue)
        if self.fuse and kind != "adam":
            raise ValueError("fused glue is implemented for adam")
        per = 1 if self.fuse else 2
        self.launches_per_sweep = 2 * per * K + 1 + per * recompute

    def _seg_len(self, j):
        return min(self.c, self.K - j * self.c)

    # ---- one optimizer step with fused apply: theta_out = theta_in + u
    def _fwd(self, k, g, s_in, s_out, th_in, th_out):
        t = k + 1
        if self.kind == "adam":
            L.opt_adam_fwd(self.tree, t, self.hp, self.sd, self.compute, g, s_in[0], s_in[1],
                           None, s_out[0], s_out[1], th_in, th_out)
        elif self.kind == "rmsprop":
            L.opt_rmsprop_fwd(self.tree, self.hp, self.sd, self.compute, g, s_in[0], None,
                              s_out[0], th_in, th_out)
        else:
            L.opt_sgd_fwd(self.tree, self.hp, self.sd, self.compute, g, s_in[0], None, s_out[0],
                          th_in, th_out)

    def _bwd(self, k, g, s_in):
        t = k + 1
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

    def _quad_rev(self, k, a, g, s_in):
        last, first = k == self.K - 1, k == 0
        sb_in = [None, None] if last else self.s_bar
        sb_out = [None, None] if first else self.s_bar
        L.opt_adam_quad_rev(self.tree, k + 1, self.hp, self.sd, self.compute, a, g, s_in[0],
                            s_in[1], self.theta_bar, sb_in[0], sb_in[1], sb_out[0], sb_out[1],
                            self.phi_bar, last, self.hyper[k], self.ws)

    def _segment_fwd(self, j, a, phi, theta_start, keep):
        """Steps of segment j from its checkpoint. keep=True stores g_k and the
        states in the segment buffers (for the reverse); otherwise only the
        end-of-segment checkpoint is written. Returns theta at segment end."""
        n, c = self.tree.numel, self.c
        k0, length = j * c, self._seg_len(j)
        th_in, s_in = theta_start, self.s_ck[j]
        for r in range(length):
            k = k0 + r
            end = r == length - 1
            g = self.g_seg[r] if keep else self.g_tmp
            if keep:
                s_out = self.s_seg[r + 1]
            elif end:
                s_out = self.s_ck[j + 1]
            else:
                s_out = self.s_pp[r % 2]
            if k == self.K - 1:
                th_out = self.thK_buf
            elif end and not keep and j + 1 < self.nseg:
                th_out = self.th_ck[j + 1]
            else:
                th_out = self.theta[r % 2]
            if self.fuse:
                L.opt_adam_quad_fwd(self.tree, k + 1, self.hp, self.sd, self.compute, a, phi,
                                    th_in, s_in[0], s_in[1], g, s_out[0], s_out[1], th_out)
            else:
                L.opt_quadratic_grad(n, a, th_in, phi, g)
                self._fwd(k, g, s_in, s_out, th_in, th_out)
            th_in, s_in = th_out, s_out
        return th_in

    def run(self, a, theta0, phi, y):
        """Enqueue the whole sweep; returns device tensors (theta_K,
        phi_bar, theta0_bar, hyper[K, NH]) without synchronising."""
        n = self.tree.numel
        th = theta0
        for j in range(self.nseg):  # forward: checkpoints, last segment kept whole
            th = self._segment_fwd(j, a, phi, theta0 if j == 0 else self.th_ck[j],
                                   keep=(j == self.nseg - 1))
        thK = th
        # outer loss 1/2 ||theta_K - y||^2: theta_bar_K = 1 * (theta_K - y)
        L.opt_quadratic_grad(n, self.ones, thK, y, self.theta_bar)
        for j in range(self.nseg - 1, -1, -1):
            if j < self.nseg - 1:  # recompute this segment's g_k, s_k
                self._segment_fwd(j, a, phi, theta0 if j == 0 else self.th_ck[j], keep=True)
            for r in range(self._seg_len(j) - 1, -1, -1):
                k = j * self.c + r
                s_in = self.s_ck[j] if r == 0 else self.s_seg[r]
                if self.fuse:
                    self._quad_rev(k, a, self.g_seg[r], s_in)
                else:
                    self._bwd(k, self.g_seg[r], s_in)
                    L.opt_quadratic_rev(n, a, self.g_bar, self.theta_bar, self.phi_bar,
                                        init_phi=(k == self.K - 1))
        return thK, self.phi_bar, self.theta_bar, self.hyper

    def saved_bytes(self):
        """Bytes of per-step storage the sweep holds for the reverse pass."""
        n, ns = self.tree.numel, NSLOT[self.kind]
        sb = 2 if self.sd == L.OPT_BF16 else 4
        return n * (self.c * (4 + ns * sb) + (self.nseg - 1) * (4 + ns * sb))

    def alg_bytes(self):
        """Algorithmic bytes of one sweep: every array argument of every
        launch read or written once."""
        n, K, ns = self.tree.numel, self.K, NSLOT[self.kind]
        sb = 2 if self.sd == L.OPT_BF16 else 4
        total = 0
        if self.fuse:
            for k in range(K):   # a, theta_k, phi, s_k -> g_k, s_{k+1}, theta_{k+1}
                total += 12 + (ns * sb if k > 0 else 0) + 4 + ns * sb + 4
            total += 16          # ones, theta_K, y -> theta_bar_K
            for k in range(K - 1, -1, -1):
                total += 4 + 4 + (ns * sb if k > 0 else 0)   # a, g_k, s_k
                total += 4 + (0 if k == K - 1 else 4 * ns)   # theta_bar, s_bar_{k+1}
                total += 0 if k == K - 1 else 4              # phi_bar (read)
                total += (0 if k == 0 else 4 * ns) + 4 + 4   # -> s_bar_k, theta_bar, phi_bar
            return n * total
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
