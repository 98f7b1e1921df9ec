"""Hand-scheduled second-order MAML meta-gradient.

The autograd form (maml.meta_grad_batched, create_graph=True) records the
network's backward as a graph and differentiates it again, which costs ~890
kernels per 4-task outer step, a quarter of them PyTorch adds, copies and
reductions that sum cotangents autograd could not fuse. Here the whole
meta-gradient is an explicit schedule of libmamlnet.so / libdiffopt.so /
cuBLAS calls (~370 per outer step at any task count), captured in one CUDA
graph by ExplicitShard:

Inner loop (MAML; 5 SGD-momentum steps, the optimizer of row a7):
    for k = 0..K-1:  g_k = grad L_s(theta_k)        (forward + backward, saved)
                     b_{k+1} = mu b_k + g_k;  theta_{k+1} = theta_k - lr b_{k+1}
                     (Nesterov: theta_{k+1} = theta_k - lr (g_k + mu b_{k+1}))
                     (ONE fused opt_sgd_fwd launch with apply, all T tasks)
Outer reverse sweep (row a9's recurrence with the SGD VJP of row a7):
    theta_bar_K = grad L_q(theta_K);  b_bar_K = 0
    for k = K-1..0:  (v, b_bar_k) = opt_sgd_bwd(u_bar = theta_bar_{k+1}, b_bar_{k+1})
                     (plain: v = b_bar' - lr u_bar; Nesterov: v = -lr u_bar + B,
                      B = b_bar' - lr mu u_bar; b_bar_k = mu v or mu B)
                     theta_bar_k = theta_bar_{k+1} + H_k v     (H_k = Hessian of L_s at theta_k)
    phi_bar = sum over tasks of theta_bar_0           (theta_0 = phi for every task)

The Hessian-vector product is forward-over-reverse: the tangent v of theta
rides through the saved forward pass and the saved backward pass (Pearlmutter's
R-operator), every tangent computed once and every sum landing in a GEMM
accumulator or a kernel's `+=` epilogue, so there is no cotangent glue:
    conv:      Ry = RW.cols + W.Rcols;   R(dW) = Rdy.cols^T + dy.Rcols^T (+= theta_bar)
               R(dcols) = RW^T.dy + W^T.Rdy;   Rdh = col2im(R dcols)
    norm/pool: net_bnpool_jvp / net_bnpool_bwd_jvp (include/mamlnet.h)
    head:      net_fc_xent_jvp
Conv biases feed training-mode batch norms and are inert (reading N5): their
gradients, tangents and meta-gradients are exactly zero and never touched.

Launch-count and sharing details: chains of <= 8 tasks get
the next layer's im2col columns from the norm/pool launch itself
(net_bnpool_fwd_cols / net_bnpool_jvp_cols); a shard of several concurrent
chains is captured with a cuBLAS SM-count hint of half the GPU.

Layout: the T tasks' parameters are one leaf-major flat buffer (leaf l is a
[T, size_l] block; conv weight l is [T, 64, Cin*9], the im2col row order),
activations task-major [T, C, B, H, W] (maml.conv4_forward_tasks' "fused"
form). Every intermediate of the K inner steps is kept (about 1 GB per step
at 32 tasks): nothing is recomputed in the reverse sweep.
"""
from __future__ import annotations

import contextlib

import numpy as np
import torch

from . import _lib as L
from . import _net as N
from .maml import BN_EPS, CONV4_SHAPES, HW, WAYS, MamlConfig, _wgrad_uses_split_k, sizes_of

C = 64                      # channels of every conv block
LAYER_H = (28, 14, 7, 3)    # input spatial size of conv block l (3x3, padding 1)
LAYER_CIN = (1, 64, 64, 64)


class _Acts:
    """Saved forward/backward intermediates of one gradient evaluation."""

    def __init__(self, T, B, dev, with_cols=True):
        self.B = B
        self.cols = [None] * 4      # cols[0] is the image's (shared, set by the caller)
        self.y, self.code, self.mean, self.rstd, self.h, self.dh, self.dy = ([None] * 4 for _ in
                                                                               range(7))
        for l, H in enumerate(LAYER_H):
            n = B * H * H
            if l > 0 and with_cols:  # zeroed once: fused producers never write the padding taps
                self.cols[l] = torch.zeros(T, LAYER_CIN[l] * 9, n, device=dev)
            self.y[l] = torch.empty(T, C, n, device=dev)
            self.dy[l] = torch.empty(T, C, n, device=dev)
            H2 = H // 2
            self.h[l] = torch.empty(T, C, B * H2 * H2, device=dev)
            self.dh[l] = torch.empty(T, C, B * H2 * H2, device=dev)
            self.code[l] = torch.empty(T, C, B * H2 * H2, dtype=torch.uint8, device=dev)
            self.mean[l] = torch.empty(T * C, device=dev)
            self.rstd[l] = torch.empty(T * C, device=dev)
        self.prob = torch.empty(T, B, WAYS, device=dev)
        self.loss = torch.empty(T, device=dev)


class ExplicitMaml:
    """Meta-gradient of T tasks through K inner SGD-momentum steps, run as
    an explicit kernel schedule (module docstring). Buffers are allocated
    once for (T, n_support, n_query); meta_grad() only launches work on the
    current stream (graph-capturable)."""

    def __init__(self, T, cfg: MamlConfig, device, n_support=WAYS * 5, n_query=WAYS * 15,
                 concurrent=True):
        dev = torch.device(device)
        if dev.type != "cuda":
            raise ValueError("ExplicitMaml runs on a CUDA device (libmamlnet.so / libdiffopt.so)")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.T, self.cfg, self.dev = int(T), cfg, dev
        self.K = int(cfg.inner_steps)
        # next-layer im2col fused into the norm/pool producers (forward and
        # tangent) for chains of <= 8 tasks: one launch fewer per layer on the
        # dependency chain (4 tasks 5.10 -> 4.99 ms, 8: 8.42 -> 8.24, 16 equal);
        # a 32-task chain keeps the separate float4 im2col (26.6 vs 26.9 ms)
        # (profiles/r02bf_fused_cols.txt)
        self.fuse_cols = self.T <= 8
        sizes = sizes_of(CONV4_SHAPES)
        self.n = sum(sizes)
        self.off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.h_off = torch.from_numpy(self.off.copy())          # host copy (net_task_sum)
        self.d_off = self.h_off.to(dev)
        self.tree = L.Tree(numel=self.T * self.n, device=dev)
        # plain or Nesterov momentum: opt_sgd_fwd / opt_sgd_bwd carry the
        # difference (u = -lr b' or -lr (g + mu b'); the VJP gives v = g_bar)
        self.hp = (cfg.inner_lr, cfg.inner_momentum, bool(cfg.nesterov))
        if cfg.inner_opt not in ("sgd", "adam"):
            raise ValueError(f"inner_opt {cfg.inner_opt!r}: 'sgd' or 'adam'")
        self.adam = cfg.inner_opt == "adam"
        self.hp_adam = (cfg.inner_lr, cfg.adam_b1, cfg.adam_b2, cfg.adam_eps, 0.0)
        Tn = self.T * self.n
        # theta_0..theta_K, b_1..b_K, g_0..g_{K-1}; conv-bias slices of g stay 0
        self.theta = [torch.empty(Tn, device=dev) for _ in range(self.K + 1)]
        self.b = [None] + [torch.empty(Tn, device=dev) for _ in range(self.K)]
        if self.adam:  # Adam inner loop: m, v per step (step 0: zero state = NULL)
            self.mu = [None] + [torch.empty(Tn, device=dev) for _ in range(self.K)]
            self.nu = [None] + [torch.empty(Tn, device=dev) for _ in range(self.K)]
            self.mu_bar = torch.empty(Tn, device=dev)
            self.nu_bar = torch.empty(Tn, device=dev)
        self.g = [torch.zeros(Tn, device=dev) for _ in range(self.K)]
        self.theta_bar = torch.zeros(Tn, device=dev)
        self.b_bar = torch.empty(Tn, device=dev)
        self.v = torch.empty(Tn, device=dev)
        self.mg = torch.empty(self.n, device=dev)
        # theta_0 = phi broadcast to every task: one gather
        idx = [self.off[l] + np.tile(np.arange(sizes[l]), self.T) for l in range(len(sizes))]
        self.bcast = torch.from_numpy(np.concatenate(idx)).to(dev)
        # saved intermediates: one set per inner step (support), one for the query
        self.Bs, self.Bq = int(n_support), int(n_query)
        self.acts = [_Acts(self.T, self.Bs, dev) for _ in range(self.K)]
        self.acts_q = _Acts(self.T, self.Bq, dev)
        self.cols1_s = torch.empty(self.T, 9, self.Bs * HW * HW, device=dev)
        self.cols1_q = torch.empty(self.T, 9, self.Bq * HW * HW, device=dev)
        # tangent scratch (reused by every HVP) and the input-gradient scratch
        self.tan = _Acts(self.T, self.Bs, dev)
        self.s1 = [torch.empty(self.T * C, device=dev) for _ in range(4)]
        self.s2 = [torch.empty(self.T * C, device=dev) for _ in range(4)]
        nmax = max(self.Bs, self.Bq) * LAYER_H[1] ** 2
        self.dcols = torch.empty(self.T * C * 9 * nmax, device=dev)
        self.rdc = [None] + [torch.empty(self.T, C * 9, self.Bs * H * H, device=dev)
                             for H in LAYER_H[1:]]
        # off-chain work (weight gradients, the tangent terms that need only v)
        # runs on a side stream that forks from and joins the current one
        self.concurrent = bool(concurrent)
        self.side = torch.cuda.Stream(dev) if self.concurrent else None
        self.labels_s = torch.empty(self.T, self.Bs, dtype=torch.int64, device=dev)
        self.labels_q = torch.empty(self.T, self.Bq, dtype=torch.int64, device=dev)
        self.xs = torch.empty(self.T, 1, self.Bs, HW, HW, device=dev)
        self.xq = torch.empty(self.T, 1, self.Bq, HW, HW, device=dev)
        # split-K workspace: the largest of every weight-gradient call
        need = 0
        for B in (self.Bs, self.Bq):
            for l, H in enumerate(LAYER_H):
                for npairs in (1, 2):
                    for acc in (0, 1):
                        need = max(need, N.net_gemm_nt2_workspace_bytes(
                            self.T, C, LAYER_CIN[l] * 9, B * H * H, npairs, acc))
        self.ws = torch.empty(max(1, (need + 3) // 4), device=dev)

    # ----------------------------------------------------------- views
    def leaf(self, buf, l):
        """Leaf l of a leaf-major T-task buffer as [T, *shape]."""
        a, b = self.T * int(self.off[l]), self.T * int(self.off[l + 1])
        return buf[a:b].view(self.T, *CONV4_SHAPES[l])

    def _w(self, buf, l):    # conv weight of block l as [T, 64, Cin*9]
        return self.leaf(buf, 4 * l).reshape(self.T, C, LAYER_CIN[l] * 9)

    def _gamma(self, buf, l):
        return self.leaf(buf, 4 * l + 2)

    def _beta(self, buf, l):
        return self.leaf(buf, 4 * l + 3)

    # ------------------------------------------------------ contractions
    def _wgrad(self, dy, cols, out, dy2=None, cols2=None, accumulate=False):
        """out (+)= dy.cols^T (+ dy2.cols2^T): the weight-gradient shape."""
        T, M, n = dy.shape
        P = cols.shape[1]
        if _wgrad_uses_split_k(T, M, P):
            N.net_gemm_nt2(T, M, P, n, dy, cols, dy2, cols2, out, accumulate, self.ws)
            return
        if accumulate:
            out.baddbmm_(dy, cols.transpose(1, 2))
        else:
            torch.bmm(dy, cols.transpose(1, 2), out=out)
        if dy2 is not None:
            out.baddbmm_(dy2, cols2.transpose(1, 2))

    def _dcols(self, l, n):
        return self.dcols[:self.T * LAYER_CIN[l] * 9 * n].view(self.T, LAYER_CIN[l] * 9, n)

    # ------------------------------------------------------------ streams
    def _fork(self):
        """Side stream waits for everything enqueued so far on the current one."""
        if self.concurrent:
            self.side.wait_stream(torch.cuda.current_stream(self.dev))

    def _on_side(self):
        return torch.cuda.stream(self.side) if self.concurrent else contextlib.nullcontext()

    def _mark(self):
        e = torch.cuda.Event()
        e.record(torch.cuda.current_stream(self.dev))
        return e

    def _join(self):
        if self.concurrent:
            torch.cuda.current_stream(self.dev).wait_stream(self.side)

    # ----------------------------------------------------------- gradient
    def _grad(self, theta, cols1, labels, A: _Acts, g):
        """Forward + backward of the T tasks' losses at theta; saves A,
        writes the gradient into g (conv-bias slices untouched) and the
        per-task losses into A.loss. The weight gradients (off the
        backward's dependency chain) run on the side stream."""
        T, B = self.T, A.B
        A.cols[0] = cols1
        for l, H in enumerate(LAYER_H):
            torch.bmm(self._w(theta, l), A.cols[l], out=A.y[l])
            args = (T * C, B, H, H, A.y[l], self._gamma(theta, l), self._beta(theta, l), BN_EPS,
                    A.h[l], A.code[l], A.mean[l], A.rstd[l])
            if l < 3 and self.fuse_cols:  # the next layer's columns from the same launch
                N.net_bnpool_fwd_cols(*args, A.cols[l + 1])
            else:
                N.net_bnpool_fwd(*args)
                if l < 3:
                    N.net_im2col3x3(T * C, B, H // 2, H // 2, A.h[l], A.cols[l + 1])
        N.net_fc_xent(T, B, C, WAYS, A.h[3], self.leaf(theta, 16), self.leaf(theta, 17), labels,
                      A.loss, A.prob, self.leaf(g, 16), self.leaf(g, 17), A.dh[3])
        for l in range(3, -1, -1):
            H = LAYER_H[l]
            N.net_bnpool_bwd(T * C, B, H, H, A.dh[l], A.code[l], A.y[l], self._gamma(theta, l),
                             A.mean[l], A.rstd[l], A.dy[l], self._gamma(g, l), self._beta(g, l))
            self._fork()
            with self._on_side():
                self._wgrad(A.dy[l], A.cols[l], self._w(g, l))
            if l > 0:
                dc = self._dcols(l, B * H * H)
                torch.bmm(self._w(theta, l).transpose(1, 2), A.dy[l], out=dc)
                N.net_col2im3x3(T * C, B, LAYER_H[l - 1] // 2, LAYER_H[l - 1] // 2, dc, A.dh[l - 1])
        self._join()

    # ------------------------------------------------------ Hessian-vector
    def _hvp(self, theta, g, A: _Acts, v, acc):
        """acc += H(theta) v for the support loss whose gradient pass saved A
        and g (forward-over-reverse; module docstring). The dependency chain
        (tangents through the layers and back) stays on the current stream;
        the terms that need only v and saved values (RW.cols, RW^T.dy) and
        the weight-gradient tangents go to the side stream."""
        T, B, R = self.T, A.B, self.tan
        cur = torch.cuda.current_stream(self.dev)
        self._fork()
        ey, edc = [None] * 4, [None] * 4
        with self._on_side():
            for l in range(4):
                torch.bmm(self._w(v, l), A.cols[l], out=R.y[l])
                ey[l] = self._mark()
            for l in range(3, 0, -1):
                torch.bmm(self._w(v, l).transpose(1, 2), A.dy[l], out=self.rdc[l])
                edc[l] = self._mark()
        for l, H in enumerate(LAYER_H):        # forward tangents
            cur.wait_event(ey[l])
            if l > 0:
                R.y[l].baddbmm_(self._w(theta, l), R.cols[l])
            args = (T * C, B, H, H, A.y[l], R.y[l], self._gamma(theta, l), self._gamma(v, l),
                    self._beta(v, l), A.code[l], A.mean[l], A.rstd[l], R.h[l], self.s1[l],
                    self.s2[l])
            if l < 3 and self.fuse_cols:  # tangent columns of the next layer, same launch
                N.net_bnpool_jvp_cols(*args, R.cols[l + 1])
            else:
                N.net_bnpool_jvp(*args)
                if l < 3:
                    N.net_im2col3x3(T * C, B, H // 2, H // 2, R.h[l], R.cols[l + 1])
        N.net_fc_xent_jvp(T, B, C, WAYS, A.h[3], R.h[3], self.leaf(theta, 16), self.leaf(v, 16),
                          self.leaf(v, 17), self.labels_s, A.prob, self.leaf(acc, 16),
                          self.leaf(acc, 17), R.dh[3])
        for l in range(3, -1, -1):             # backward tangents
            H = LAYER_H[l]
            N.net_bnpool_bwd_jvp(T * C, B, H, H, A.dh[l], R.dh[l], A.code[l], A.y[l], R.y[l],
                                 self._gamma(theta, l), self._gamma(v, l), A.mean[l], A.rstd[l],
                                 self._gamma(g, l), self._beta(g, l), self.s1[l], self.s2[l],
                                 R.dy[l], self._gamma(acc, l), self._beta(acc, l))
            self._fork()
            with self._on_side():
                if l == 0:
                    self._wgrad(R.dy[0], A.cols[0], self._w(acc, 0), accumulate=True)
                else:
                    self._wgrad(R.dy[l], A.cols[l], self._w(acc, l), A.dy[l], R.cols[l],
                                accumulate=True)
            if l > 0:
                cur.wait_event(edc[l])
                dc = self.rdc[l]
                dc.baddbmm_(self._w(theta, l).transpose(1, 2), R.dy[l])
                N.net_col2im3x3(T * C, B, LAYER_H[l - 1] // 2, LAYER_H[l - 1] // 2, dc,
                                R.dh[l - 1])
        self._join()

    # -------------------------------------------------------- meta-gradient
    def meta_grad(self, phi):
        """Sum over the T tasks of d L_query(theta_K(phi)) / d phi, and the
        summed query loss, for the task data in self.xs/labels_s/xq/labels_q
        (written by load()). Returns views of internal buffers."""
        T, K = self.T, self.K
        if phi.dtype != torch.float32 or phi.device != self.dev or phi.numel() != self.n:
            raise ValueError(f"ExplicitMaml.meta_grad: phi must be float32 on {self.dev} with "
                             f"{self.n} elements (got {phi.dtype}, {phi.device}, {phi.numel()})")
        torch.index_select(phi.reshape(-1), 0, self.bcast, out=self.theta[0])
        N.net_im2col3x3(T, self.Bs, HW, HW, self.xs, self.cols1_s)
        N.net_im2col3x3(T, self.Bq, HW, HW, self.xq, self.cols1_q)
        F32, CD = L.OPT_F32, L.OPT_COMPUTE_DEFAULT
        for k in range(K):
            self._grad(self.theta[k], self.cols1_s, self.labels_s, self.acts[k], self.g[k])
            if self.adam:  # (u, m', v') = Adam_t(g, m, v), t = k + 1; theta' = theta + u
                L.opt_adam_fwd(self.tree, k + 1, self.hp_adam, F32, CD, self.g[k], self.mu[k],
                               self.nu[k], None, self.mu[k + 1], self.nu[k + 1], self.theta[k],
                               self.theta[k + 1])
            else:
                L.opt_sgd_fwd(self.tree, self.hp, F32, CD, self.g[k], self.b[k], None,
                              self.b[k + 1], self.theta[k], self.theta[k + 1])
        self._grad(self.theta[K], self.cols1_q, self.labels_q, self.acts_q, self.theta_bar)
        for k in range(K - 1, -1, -1):
            if self.adam:  # Adam VJP (row a4): v = g_bar; m_bar, v_bar carried backwards
                last, first = k == K - 1, k == 0
                L.opt_adam_bwd(self.tree, k + 1, self.hp_adam, F32, CD, self.g[k], self.mu[k],
                               self.nu[k], self.theta_bar, None if last else self.mu_bar,
                               None if last else self.nu_bar, self.v,
                               None if first else self.mu_bar, None if first else self.nu_bar)
            else:
                L.opt_sgd_bwd(self.tree, self.hp, F32, CD, self.g[k], self.b[k], self.theta_bar,
                              self.b_bar if k < K - 1 else None, self.v,
                              self.b_bar if k > 0 else None)
            self._hvp(self.theta[k], self.g[k], self.acts[k], self.v, self.theta_bar)
        N.net_task_sum(T, len(CONV4_SHAPES), self.h_off, self.d_off, self.theta_bar, self.mg)
        return self.mg, self.acts_q.loss.sum()

    def load(self, data):
        """Copy T tasks' (xs, ys, xq, yq) into the static input buffers."""
        if len(data) != self.T:
            raise ValueError(f"ExplicitMaml.load: {len(data)} tasks for an engine of {self.T}")
        for t, (xs, ys, xq, yq) in enumerate(data):
            self.xs[t, 0].copy_(xs.view(self.Bs, HW, HW))
            self.xq[t, 0].copy_(xq.view(self.Bq, HW, HW))
            self.labels_s[t].copy_(ys)
            self.labels_q[t].copy_(yq)


    def load_seeded(self, outer_step, task_ids, seed=0, xs_out=None, xq_out=None):
        """maml.task_data(outer_step, t, seed) for every task, drawn straight
        into the static buffers (or xs_out / xq_out of the same shapes; the
        same generator draws in the same order, so bitwise the same data,
        without the per-task temporaries and copies). Labels are the fixed
        class-major ones."""
        from .maml import QUERIES, SHOTS, task_seed

        assert len(task_ids) == self.T and self.Bs == WAYS * SHOTS and self.Bq == WAYS * QUERIES
        if not getattr(self, "_labels_set", False):
            ar = torch.arange(WAYS, device=self.dev)
            self.labels_s.copy_(ar.repeat_interleave(SHOTS).expand(self.T, -1))
            self.labels_q.copy_(ar.repeat_interleave(QUERIES).expand(self.T, -1))
            self._labels_set = True
        if not hasattr(self, "_proto"):
            self._proto = torch.empty(WAYS, 1, HW, HW, device=self.dev)
        XS = self.xs if xs_out is None else xs_out
        XQ = self.xq if xq_out is None else xq_out
        proto = torch.empty(WAYS, 1, HW, HW, device=self.dev) if xs_out is not None else self._proto
        for t, tid in enumerate(task_ids):
            gen = torch.Generator(device=self.dev).manual_seed(task_seed(outer_step, tid, seed))
            xs = XS[t, 0].view(self.Bs, 1, HW, HW)
            xq = XQ[t, 0].view(self.Bq, 1, HW, HW)
            torch.randn(xs.shape, generator=gen, device=self.dev, out=xs)
            torch.randn(xq.shape, generator=gen, device=self.dev, out=xq)
            torch.randn(proto.shape, generator=gen, device=self.dev, out=proto)
            xs.view(WAYS, SHOTS, HW, HW).add_(proto.view(WAYS, 1, HW, HW))
            xq.view(WAYS, QUERIES, HW, HW).add_(proto.view(WAYS, 1, HW, HW))


def meta_grad_explicit(phi, data, cfg: MamlConfig, engine: ExplicitMaml | None = None):
    """maml.meta_grad_batched's result through the explicit schedule."""
    eng = engine or ExplicitMaml(len(data), cfg, phi.device)
    eng.load(data)
    mg, loss = eng.meta_grad(phi.detach().contiguous())
    return mg.clone(), loss.clone()


def _cublas_sm_target(n):
    """cublasSetSmCountTarget on the current thread's PyTorch cuBLAS handle
    (n = 0 restores the device's own count); returns False if the library
    entry point is not available. A heuristics hint only: cuBLAS picks its
    tile shape / split-K as if the GPU had n SMs."""
    import ctypes
    import glob
    import os

    for cand in ["libcublas.so.12"] + glob.glob(
            os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cublas", "lib",
                         "libcublas.so.12")):
        try:
            lib = ctypes.CDLL(cand)
            fn = lib.cublasSetSmCountTarget
            break
        except (OSError, AttributeError):
            continue
    else:
        return False
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    fn.restype = ctypes.c_int
    return fn(ctypes.c_void_p(torch.cuda.current_blas_handle()), int(n)) == 0


def default_groups(tasks):
    """Task groups (concurrent graph chains) for a shard of `tasks` tasks,
    from the measured sweeps on one B200 (profiles/r02ab_task_groups.txt;
    with the cuBLAS SM hint and 8K norm/pool slices, profiles/r02ca_*):
    <= 16 tasks -> up to 4 chains (16 tasks: 14.47 ms vs 14.72 with 2),
    more -> 1 (32 tasks: 26.6 ms vs 27.7-27.8 with 2 or 4)."""
    if tasks <= 16:
        return max(1, min(tasks, 4))
    return 1


class ExplicitShard:
    """One rank's task shard as ONE CUDA graph of the explicit schedule
    (the maml.GraphedShard interface: call it like maml.meta_grad_tasks).
    Per outer step only phi and the task data are copied in.

    groups = G > 1 splits the shard into G contiguous task groups, each its
    own ExplicitMaml on its own pair of streams, captured as parallel
    branches of the graph: at a few tasks per GPU most kernels are
    latency-bound, so two independent chains overlap where one cannot. The
    group meta-gradients are summed in group order after the join."""

    batched = True

    def __init__(self, task_ids, cfg: MamlConfig, device, warmup=2, concurrent=True, groups=None):
        self.ids, self.cfg = list(task_ids), cfg
        if groups is None:
            groups = default_groups(len(self.ids))
        n, G = len(self.ids), max(1, min(int(groups), len(self.ids)))
        cuts = [n * i // G for i in range(G + 1)]
        self.groups = [self.ids[cuts[i]:cuts[i + 1]] for i in range(G)]
        self.nstreams = G
        self.engs = [ExplicitMaml(len(g), cfg, device, concurrent=concurrent) for g in self.groups]
        # with several groups, the dependency chains run on high-priority
        # streams so the side streams' off-chain work fills in behind them
        # (graph nodes keep the priority; measured: 4 tasks 5.53 -> 5.44 ms;
        # one chain of 32 tasks is 1.5% slower this way, so not there)
        self.streams = [torch.cuda.Stream(device, priority=-1 if G > 1 else 0)
                        for _ in self.groups]
        self.phi = torch.zeros(self.engs[0].n, device=device)
        self._load(0)
        # with concurrent chains, cuBLAS sizes each product as if it had half
        # the GPU (its kernel choices are baked into the graph; the handle is
        # restored after capture). Measured: 4 tasks 4.99 -> 4.91 ms, 8: 8.25
        # -> 8.11, 16 (2 chains): 14.90 -> 14.75 (a quarter of the GPU: 4.91 /
        # 8.69) (profiles/r02bm_cublas_sm_target.txt)
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        self.cublas_sm_target = sms // 2 if G >= 2 else 0
        hinted = self.cublas_sm_target > 0 and _cublas_sm_target(self.cublas_sm_target)
        try:
            side = torch.cuda.Stream(device)
            side.wait_stream(torch.cuda.current_stream(device))
            with torch.cuda.stream(side):
                for _ in range(warmup):
                    self._body()
            torch.cuda.current_stream(device).wait_stream(side)
            n0 = L.opt_launch_count() + N.net_launch_count()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.mg, self.loss = self._body()
            self.launches_per_replay = L.opt_launch_count() + N.net_launch_count() - n0
        finally:
            if hinted:
                _cublas_sm_target(0)
        # next step's task data, drawn on a side stream while this step's
        # graph replays (input pipelining; bitwise the same draws)
        self.stage = [(torch.empty_like(e.xs), torch.empty_like(e.xq)) for e in self.engs]
        self.pf_stream = torch.cuda.Stream(device)
        self.pf_step, self.pf_done, self.copied = None, None, None

    def _prefetch(self, outer_step):
        if self.copied is not None:
            self.pf_stream.wait_event(self.copied)  # the stage buffers were consumed
        with torch.cuda.stream(self.pf_stream):
            for eng, ids, (sx, sq) in zip(self.engs, self.groups, self.stage):
                eng.load_seeded(outer_step, ids, self.cfg.seed, sx, sq)
            self.pf_done = torch.cuda.Event()
            self.pf_done.record(self.pf_stream)
        self.pf_step = outer_step

    def _load(self, outer_step):
        for eng, ids in zip(self.engs, self.groups):
            eng.load_seeded(outer_step, ids, self.cfg.seed)

    def _body(self):
        if len(self.engs) == 1:
            return self.engs[0].meta_grad(self.phi)
        cur = torch.cuda.current_stream()
        parts = []
        for eng, st in zip(self.engs, self.streams):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                parts.append(eng.meta_grad(self.phi))
        for st in self.streams:
            cur.wait_stream(st)
        mg, loss = parts[0][0].clone(), parts[0][1].clone()
        for m, l in parts[1:]:  # group order
            mg += m
            loss += l
        return mg, loss

    def __call__(self, phi, task_ids, outer_step, cfg, inner=None):
        assert list(task_ids) == self.ids
        cur = torch.cuda.current_stream(self.phi.device)
        if self.pf_step == outer_step:  # drawn during the previous replay
            cur.wait_event(self.pf_done)
            for eng, (sx, sq) in zip(self.engs, self.stage):
                eng.xs.copy_(sx)
                eng.xq.copy_(sq)
        else:
            self._load(outer_step)
        self.copied = torch.cuda.Event()
        self.copied.record(cur)
        self.phi.copy_(phi)
        self.graph.replay()
        self._prefetch(outer_step + 1)  # the outer loop's next step
        return self.mg, self.loss
