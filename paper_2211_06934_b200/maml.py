"""Task-sharded MAML meta-batch.

PAPER.md: MAML needs a "large task-level batch size"; TorchOpt
distributes the differentiable-optimization tasks of a meta-batch to GPU
workers that run in parallel under a synchronous coordinator (P:269-271,
App. C; 5.2x on 8 GPUs). B200-native equivalent: SPMD, one
process per GPU; rank r of W owns tasks [r*T/W, (r+1)*T/W) of the T-task
meta-batch, runs each task's inner loop locally, sums its meta-gradients in
task order, and ONE all-reduce (NCCL over NVLink/NVSwitch) combines them;
every replica then applies the same outer Adam step, so replicas stay
identical without a coordinator (synchronous semantics).

Per task (reading Z16): 4-conv64 + BN (batch statistics) + ReLU + maxpool,
fc -> 5 ways; 5-way 5-shot support, 15 queries per class, 28x28x1 inputs
N(0,1) seeded by (outer step, task id), labels fixed by class; 5 inner SGD
momentum steps (lr 0.1, mu 0.9) through the fused differentiable SGD op with
apply_updates fused; second-order meta-gradient (create_graph=True, Z15).
The network forward/backward runs in PyTorch (cuDNN): it is the task's loss,
not the method; the optimizer step and its VJP run in libdiffopt.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

WAYS, SHOTS, QUERIES, HW = 5, 5, 15, 28
CONV4_SHAPES = ([(64, 1, 3, 3), (64,), (64,), (64,)]
                + [(64, 64, 3, 3), (64,), (64,), (64,)] * 3
                + [(WAYS, 64), (WAYS,)])  # 18 leaves, 112,261 elements


def conv4_forward(params, x):
    """params: 18 tensors in CONV4_SHAPES order; x: [B, 1, 28, 28]."""
    h = x
    for blk in range(4):
        w, b, gam, bet = params[4 * blk: 4 * blk + 4]
        h = F.conv2d(h, w, b, padding=1)
        h = F.batch_norm(h, None, None, gam, bet, training=True)
        h = F.max_pool2d(F.relu(h), 2)
    h = h.flatten(1)
    return F.linear(h, params[16], params[17])


def init_params(seed, device):
    """Deterministic phi (same on every rank)."""
    gen = torch.Generator().manual_seed(seed)
    out = []
    for s in CONV4_SHAPES:
        if len(s) == 4:
            fan_in = s[1] * s[2] * s[3]
            out.append(torch.randn(s, generator=gen) * (2.0 / fan_in) ** 0.5)
        elif len(s) == 2:
            out.append(torch.randn(s, generator=gen) * (1.0 / s[1]) ** 0.5)
        else:
            out.append(torch.zeros(s))
    # BN weights = 1
    for blk in range(4):
        out[4 * blk + 2] = torch.ones(64)
    return torch.cat([p.reshape(-1) for p in out]).to(device)


def task_seed(outer_step, task_id, seed=0):
    return ((seed * 1_000_003 + outer_step) * 1_000_033 + task_id) & 0x7FFFFFFFFFFFFFFF


def task_data(outer_step, task_id, device, seed=0):
    """Seeded synthetic 5-way task, generated on `device` by a generator
    keyed on (seed, step, task) only -- never on the rank layout. (CPU and
    CUDA generators draw different streams; each is reproducible.)"""
    device = torch.device(device)
    gen = torch.Generator(device=device).manual_seed(task_seed(outer_step, task_id, seed))
    xs = torch.randn(WAYS * SHOTS, 1, HW, HW, generator=gen, device=device)
    xq = torch.randn(WAYS * QUERIES, 1, HW, HW, generator=gen, device=device)
    # class-dependent mean shift so the task is learnable
    proto = torch.randn(WAYS, 1, HW, HW, generator=gen, device=device)
    ys = torch.arange(WAYS, device=device).repeat_interleave(SHOTS)
    yq = torch.arange(WAYS, device=device).repeat_interleave(QUERIES)
    return xs + proto[ys], ys, xq + proto[yq], yq


@dataclass
class MamlConfig:
    tasks: int = 32
    inner_steps: int = 5
    inner_lr: float = 0.1
    inner_momentum: float = 0.9
    nesterov: bool = False
    outer_lr: float = 1e-3
    seed: int = 0
    net: str = "fused"  # network form (conv4_forward_tasks)
    # inner optimizer of the explicit step (maml_explicit): "sgd" (momentum /
    # Nesterov, the C4 recipe) or "adam" (differentiable Adam inner loop,
    # MetaAdam-style; inner_lr is its lr)
    inner_opt: str = "sgd"
    adam_b1: float = 0.9
    adam_b2: float = 0.999
    adam_eps: float = 1e-8


class FusedSgdInner:
    """Inner step through libdiffopt.so (SgdStep with apply_updates fused)."""

    def __init__(self, sizes, device, cfg: MamlConfig):
        from . import _lib as L
        from .functional import SgdStep, StepConfig

        self.tree = L.Tree.from_sizes(sizes, device=device)
        self.step_cfg = StepConfig(self.tree)
        self.fn = SgdStep
        self.cfg = cfg

    def __call__(self, g, b, theta):
        c = self.cfg
        return self.fn.apply(g, b, theta, c.inner_lr, c.inner_momentum, c.nesterov, self.step_cfg)


class FusedAdamOuter:
    """Outer (non-differentiable) Adam on phi through opt_adam_fwd with
    apply fused and in-place state (G9 of SURVEY §2.2)."""

    def __init__(self, n, device, lr):
        from . import _lib as L

        self.L = L
        self.tree = L.Tree(numel=n, device=device)
        self.mu = torch.zeros(n, device=device)
        self.nu = torch.zeros(n, device=device)
        self.t = 0
        self.lr = lr

    def __call__(self, phi, grad):
        self.t += 1
        self.L.opt_adam_fwd(self.tree, self.t, (self.lr, 0.9, 0.999, 1e-8, 0.0), 0, 0, grad,
                            self.mu, self.nu, None, self.mu, self.nu, phi, phi)
        return phi


def task_range(world, rank, tasks):
    return range(rank * tasks // world, (rank + 1) * tasks // world)


def sizes_of(shapes):
    return [int(torch.Size(s).numel()) for s in shapes]


def meta_grad_tasks(phi, task_ids, outer_step, cfg: MamlConfig, inner):
    """Sum over task_ids (in order) of d L_query(theta_K(phi)) / d phi, and
    the summed query loss. phi: flat leaf tensor (no grad needed on entry)."""
    data = [task_data(outer_step, tid, phi.device, cfg.seed) for tid in task_ids]
    return meta_grad_data(phi, data, cfg, inner)


def _task_logits(theta, x, net):
    """One task's logits; net as in conv4_forward_tasks (T = 1)."""
    sizes = sizes_of(CONV4_SHAPES)
    if net in ("gemm", "fused"):
        params = [p.view(1, *s) for p, s in zip(torch.split(theta, sizes), CONV4_SHAPES)]
        return conv4_forward_tasks(params, x.view(x.shape[0], 1, HW, HW), 1, net)[0]
    params = [p.view(s) for p, s in zip(torch.split(theta, sizes), CONV4_SHAPES)]
    return conv4_forward(params, x)


def meta_grad_data(phi, data, cfg: MamlConfig, inner):
    """meta_grad_tasks on pre-generated task data [(xs, ys, xq, yq), ...]."""
    sizes = sizes_of(CONV4_SHAPES)
    phi_v = phi.detach().requires_grad_(True)
    total = torch.zeros_like(phi)
    loss_sum = torch.zeros((), device=phi.device, dtype=phi.dtype)
    for xs, ys, xq, yq in data:
        theta, b = phi_v, None
        for _ in range(cfg.inner_steps):
            loss = F.cross_entropy(_task_logits(theta, xs, cfg.net), ys)
            (g,) = torch.autograd.grad(loss, theta, create_graph=True)
            theta, b = inner(g, b, theta)
        qloss = F.cross_entropy(_task_logits(theta, xq, cfg.net), yq)
        (mg,) = torch.autograd.grad(qloss, phi_v)
        total += mg
        loss_sum += qloss.detach()
    return total, loss_sum


# ---------------------------------------------------- task-batched form
def theta0_tasks(phi_leaves, T):
    """theta_0 of T tasks, leaf-major: leaf l becomes a [T, size_l] block
    (every task starts from phi; the backward of the broadcast is the sum
    over tasks of the meta-gradients)."""
    return torch.cat([p.reshape(1, -1).expand(T, -1).reshape(-1) for p in phi_leaves])


class _Im2Col(torch.autograd.Function):
    """3x3 / padding-1 im2col of the task-major layout: h [T, C, B, H, W] ->
    columns [T, C*9, B*H*W], row cin*9 + 3i + j = h shifted by (i-1, j-1)
    (zero outside). Its adjoint is _Col2Im and each one's backward is the
    other, so the pair is differentiable to any order (MAML's second-order
    meta-gradient differentiates through the convolution backward)."""

    @staticmethod
    def forward(ctx, h):
        T, C, B, H, W = h.shape
        ctx.shape = tuple(h.shape)
        hp = F.pad(h, (1, 1, 1, 1))
        cols = torch.stack([hp[..., i:i + H, j:j + W] for i in range(3) for j in range(3)], 2)
        return cols.view(T, C * 9, B * H * W)

    @staticmethod
    def backward(ctx, dcols):
        return _Col2Im.apply(dcols, ctx.shape)


class _Col2Im(torch.autograd.Function):
    """Adjoint of _Im2Col: dh[y + i - 1, x + j - 1] += cols_(i,j)[y, x]."""

    @staticmethod
    def forward(ctx, cols, shape):
        T, C, B, H, W = shape
        c = cols.reshape(T, C, 9, B, H, W)
        dh = cols.new_zeros(shape)
        for k in range(9):
            di, dj = k // 3 - 1, k % 3 - 1
            ya, yb, xa, xb = max(0, di), min(H, H + di), max(0, dj), min(W, W + dj)
            dh[..., ya:yb, xa:xb] += c[:, :, k, :, ya - di:yb - di, xa - dj:xb - dj]
        return dh

    @staticmethod
    def backward(ctx, dh):
        return _Im2Col.apply(dh), None


def _conv3x3_tasks(h, w, b, im2col=None):
    """Task-batched 3x3 conv (padding 1) as one batched GEMM: h [T, Cin, B,
    H, W], w [T, Cout, Cin, 3, 3], b [T, Cout] -> [T, Cout, B, H, W]."""
    T, Cin, B, H, W = h.shape
    cols = (im2col or _Im2Col.apply)(h)
    out = torch.baddbmm(b.unsqueeze(-1), w.reshape(T, w.shape[1], Cin * 9), cols)
    return out.view(T, -1, B, H, W)


# ------------------------------------- fused network layers (libmamlnet.so)
BN_EPS = 1e-5  # F.batch_norm's default


class _Im2ColK(torch.autograd.Function):
    """_Im2Col with both directions in libmamlnet.so (net_im2col3x3 /
    net_col2im3x3): one pass each instead of pad + 9 slices + stack and
    9 read-modify-write passes."""

    @staticmethod
    def forward(ctx, h):
        from . import _net as N

        if h.dtype != torch.float32 or not h.is_cuda:
            raise TypeError("_Im2ColK: libmamlnet.so takes fp32 CUDA tensors")
        h = h.contiguous()
        T, C, B, H, W = h.shape
        ctx.shape = tuple(h.shape)
        cols = h.new_empty(T, C * 9, B * H * W)
        N.net_im2col3x3(T * C, B, H, W, h, cols)
        return cols

    @staticmethod
    def backward(ctx, dcols):
        return _Col2ImK.apply(dcols, ctx.shape)


class _Col2ImK(torch.autograd.Function):
    @staticmethod
    def forward(ctx, cols, shape):
        from . import _net as N

        T, C, B, H, W = shape
        cols = cols.contiguous()
        dh = cols.new_empty(shape)
        N.net_col2im3x3(T * C, B, H, W, cols, dh)
        return dh

    @staticmethod
    def backward(ctx, dh):
        return _Im2ColK.apply(dh), None


def _gemm_nt(a, b):
    """C[t] = a[t] @ b[t]^T through net_gemm_nt (split-K fp32)."""
    from . import _net as N

    a, b = a.contiguous(), b.contiguous()
    T, M, n = a.shape
    P = b.shape[1]
    c = a.new_empty(T, M, P)
    wb = N.net_gemm_nt_workspace_bytes(T, M, P, n)
    ws = a.new_empty((wb + 3) // 4) if wb else None
    N.net_gemm_nt(T, M, P, n, a, b, c, ws)
    return c


def _wgrad_uses_split_k(T, M, P):
    """net_gemm_nt when the output alone cannot fill the GPU (measured on
    B200, profiles/r01f_gemm_nt_bench.jsonl: split-K wins up to ~16 tasks and
    for the 9-column first layer at any T; cuBLAS's SIMT SGEMM wins once
    T x 64 x 576 gives >= 148 output tiles of 64 x 64)."""
    return P <= 16 or T * ((M + 63) // 64) * ((P + 63) // 64) < 148


def _wgrad_fwd(a, b):
    """a @ b^T, long contraction: split-K kernel or cuBLAS by shape."""
    T, M, n = a.shape
    P = b.shape[1]
    if _wgrad_uses_split_k(T, M, P):
        return _gemm_nt(a, b)
    return torch.bmm(a, b.transpose(1, 2))


def _conv_fwd(w, cols, bias):
    """bias + w @ cols (w [T, Co, K], cols [T, K, n])."""
    if bias is None:
        return torch.bmm(w, cols)
    return torch.baddbmm(bias.unsqueeze(-1), w, cols)


class _ConvBwd(torch.autograd.Function):
    """The task-batched convolution's VJP as ONE node: (dy, w, cols) ->
    (gw = dy cols^T, gcols = w^T dy, gb = sum dy). Its own VJP (needed once,
    by the second-order meta-gradient) writes the cotangent of dy with two
    accumulating GEMMs, d_dy = gb_bar + gw_bar cols + w gcols_bar, instead of
    three autograd nodes whose contributions are summed by separate
    elementwise adds over the dy-sized tensor.

    cols enters as a plain (detached) tensor and h, the image cols was
    built from, as the differentiable input: the cotangent gw_bar reaches
    h as col2im(gw_bar^T dy), so autograd adds it to the conv's other
    contribution (col2im of w^T dy_meta through the im2col node) on h, 9x
    smaller than cols, instead of summing the two 9x-expanded cols
    cotangents (col2im is linear: the same sum, one add of |h| elements)."""

    @staticmethod
    def forward(ctx, dy, w, cols, h, need_w, need_cols, need_b, hshape):
        ctx.save_for_backward(dy, w, cols)
        ctx.set_materialize_grads(False)  # unused outputs: no GEMMs on zero cotangents
        ctx.hshape = hshape
        gw = _wgrad_fwd(dy, cols) if need_w else None
        gc = torch.bmm(w.transpose(1, 2), dy) if need_cols else None
        gb = dy.sum(-1) if need_b else None
        return gw, gc, gb

    @staticmethod
    @torch.autograd.function.once_differentiable
    def backward(ctx, ggw, ggc, ggb):
        dy, w, cols = ctx.saved_tensors
        d_dy = d_w = d_h = None
        if ctx.needs_input_grad[0]:
            bias = ggb.unsqueeze(-1) if ggb is not None else None
            pairs = ([(ggw, cols)] if ggw is not None else []) + ([(w, ggc)] if ggc is not None else [])
            for a, b in pairs:
                if d_dy is None:
                    d_dy = torch.baddbmm(bias, a, b) if bias is not None else torch.bmm(a, b)
                else:
                    d_dy.baddbmm_(a, b)
            if d_dy is None:
                d_dy = bias.expand(dy.shape).contiguous() if bias is not None else None
        if ctx.needs_input_grad[1] and ggc is not None:
            d_w = _wgrad_fwd(dy, ggc)
        if ctx.needs_input_grad[3] and ggw is not None:
            d_h = _Col2ImK.apply(torch.bmm(ggw.transpose(1, 2), dy), ctx.hshape)
        return d_dy, d_w, None, d_h, None, None, None, None


class _TaskConvGemm(torch.autograd.Function):
    """bias + w @ cols for the task-batched convolution (cuBLAS batched
    SGEMM); backward: one _ConvBwd node (weight gradient through the
    split-K kernel or cuBLAS, input gradient, bias gradient), differentiable
    once for the second-order meta-gradient. h: the image cols = im2col(h)
    was built from (not read here; handed to _ConvBwd as its differentiable
    image input)."""

    @staticmethod
    def forward(ctx, w, cols, bias, h):
        ctx.save_for_backward(w, cols, h)
        return _conv_fwd(w, cols, bias)

    @staticmethod
    def backward(ctx, dy):
        w, cols, h = ctx.saved_tensors
        nw, nc, nb = ctx.needs_input_grad[:3]
        gw, gc, gb = _ConvBwd.apply(dy.contiguous(), w, cols.detach(), h, nw, nc, nb,
                                    tuple(h.shape))
        return gw, gc, gb, None


def _conv3x3_tasks_fused(h, w, b, bn_follows=False):
    """_conv3x3_tasks with libmamlnet.so im2col/col2im and split-K weight
    gradients. bn_follows: a training-mode batch norm over (task, channel)
    groups consumes the output. It subtracts the group mean, so a
    per-channel bias is inert: BN(y + b) = BN(y) in exact arithmetic, the
    bias gradient is identically zero (BN's input gradient sums to zero
    over the group: sum dx = gamma*r*(sum dy - n*A - Bm*sum xh) = 0), and
    the network output does not depend on b. The bias is then left out of
    the GEMM (no broadcast copy into the output, no reduction for its
    gradient; reading N5 in DESIGN.md): its meta-gradient is exactly 0 and
    the outputs differ from the biased form by rounding only."""
    T, Cin, B, H, W = h.shape
    out = _TaskConvGemm.apply(w.reshape(T, w.shape[1], Cin * 9), _Im2ColK.apply(h),
                              None if bn_follows else b, h)
    return out.view(T, -1, B, H, W)


class _BnPool(torch.autograd.Function):
    """relu(max_pool2d(batch_norm(x), 2)) with per-(task, channel) batch
    statistics, one kernel (net_bnpool_fwd). x [T, C, B, H, W], gamma/beta
    [T, C]. Backward: _BnPoolBwd (itself differentiable once, for the
    second-order meta-gradient)."""

    @staticmethod
    def forward(ctx, x, gamma, beta):
        from . import _net as N

        if x.dtype != torch.float32 or not x.is_cuda:
            raise TypeError("_BnPool: libmamlnet.so takes fp32 CUDA tensors")
        x = x.contiguous()
        T, C, B, H, W = x.shape
        out = x.new_empty(T, C, B, H // 2, W // 2)
        code = torch.empty(out.shape, dtype=torch.uint8, device=x.device)
        mean, rstd = x.new_empty(T * C), x.new_empty(T * C)
        N.net_bnpool_fwd(T * C, B, H, W, x, gamma.contiguous(), beta.contiguous(), BN_EPS, out,
                         code, mean, rstd)
        ctx.save_for_backward(x, gamma, code, mean, rstd)
        return out

    @staticmethod
    def backward(ctx, dp):
        x, gamma, code, mean, rstd = ctx.saved_tensors
        dx, dgamma, dbeta = _BnPoolBwd.apply(dp, x, gamma, code, mean, rstd)
        return dx, dgamma.view_as(gamma), dbeta.view_as(gamma)


class _BnPoolBwd(torch.autograd.Function):
    """VJP of _BnPool (net_bnpool_bwd) as a function of (dp, x, gamma); its
    own VJP is net_bnpool_bwd2 (include/mamlnet.h)."""

    @staticmethod
    def forward(ctx, dp, x, gamma, code, mean, rstd):
        from . import _net as N

        dp = dp.contiguous()
        T, C, B, H, W = x.shape
        dx = torch.empty_like(x)
        dgamma, dbeta = x.new_empty(T * C), x.new_empty(T * C)
        N.net_bnpool_bwd(T * C, B, H, W, dp, code, x, gamma.contiguous(), mean, rstd, dx, dgamma,
                         dbeta)
        ctx.save_for_backward(dp, x, gamma, code, mean, rstd, dgamma, dbeta)
        return dx, dgamma, dbeta

    @staticmethod
    @torch.autograd.function.once_differentiable
    def backward(ctx, gdx, gdgamma, gdbeta):
        from . import _net as N

        dp, x, gamma, code, mean, rstd, dgamma, dbeta = ctx.saved_tensors
        T, C, B, H, W = x.shape
        g_dp, g_x = torch.empty_like(dp), torch.empty_like(x)
        g_gamma = x.new_empty(T * C)
        c = lambda t: None if t is None else t.contiguous()
        N.net_bnpool_bwd2(T * C, B, H, W, c(gdx), c(gdgamma), c(gdbeta), dp, code, x,
                          gamma.contiguous(), mean, rstd, dgamma, dbeta, g_dp, g_x, g_gamma)
        return g_dp, g_x, g_gamma.view_as(gamma), None, None, None


def _bn_tasks(h, gamma, beta):
    """Training-mode batch norm with per-(task, channel) batch statistics on
    the [T, C, B, H, W] layout: F.batch_norm on the [1, T*C, B*H*W] view."""
    T, C = h.shape[:2]
    y = F.batch_norm(h.reshape(1, T * C, -1), None, None, gamma.reshape(-1), beta.reshape(-1),
                     training=True)
    return y.view_as(h)


def _pool_relu_tasks(h):
    """relu(max_pool2d(., 2)) (= max_pool2d(relu(.)), floor mode) on the
    [T, C, B, H, W] layout as a 2x2 window max."""
    T, C, B, H, W = h.shape
    H2, W2 = H // 2, W // 2
    if H != 2 * H2 or W != 2 * W2:
        h = h[..., :2 * H2, :2 * W2]
    return F.relu(h.reshape(T, C, B, H2, 2, W2, 2).amax(dim=(4, 6)))


def conv4_forward_tasks(params, x, T, net="cudnn"):
    """The T networks of a task batch as ONE network: params are the 18
    leaves with a leading task dim [T, *shape]; x: [B, T, 28, 28] (channel t
    = task t). Task t's logits depend on task t's parameters and images only
    and equal conv4_forward(params[t], x[:, t:t+1]). Returns [T, B, WAYS].
      net="cudnn": grouped convolutions (groups = T) and F.batch_norm over
                   the T*64 channels (= per (task, channel) statistics);
      net="gemm" : activations kept task-major [T, C, B, H, W], every conv
                   one batched GEMM over the T tasks (_conv3x3_tasks), BN
                   statistics per (task, channel) (_bn_tasks), 2x2 window
                   max (_pool_relu_tasks). On B200, cuDNN's fp32 convolution
                   algorithms lose ~2% on this second-order meta-gradient
                   while the SGEMM form keeps fp32 accuracy (~3e-6 vs a
                   float64 run, tools/maml_net_check.py);
      net="fused": the gemm form with im2col/col2im and the whole
                   batch-norm + pool + ReLU block (forward, VJP and the VJP's
                   VJP) in libmamlnet.so kernels (_Im2ColK, _BnPool)."""
    if net == "fused":
        h = x.permute(1, 0, 2, 3).unsqueeze(1).contiguous()  # [T, 1, B, 28, 28]
        for blk in range(4):
            w, b, gam, bet = params[4 * blk: 4 * blk + 4]
            h = _BnPool.apply(_conv3x3_tasks_fused(h, w, b, bn_follows=True), gam, bet)
        h = h.reshape(T, 64, -1).transpose(1, 2)  # [T, B, 64]
    elif net == "gemm":
        h = x.permute(1, 0, 2, 3).unsqueeze(1)  # [T, 1, B, 28, 28]
        for blk in range(4):
            w, b, gam, bet = params[4 * blk: 4 * blk + 4]
            h = _pool_relu_tasks(_bn_tasks(_conv3x3_tasks(h, w, b), gam, bet))
        h = h.reshape(T, 64, -1).transpose(1, 2)  # [T, B, 64]
    else:
        h = x
        for blk in range(4):
            w, b, gam, bet = params[4 * blk: 4 * blk + 4]
            h = F.conv2d(h, w.reshape(-1, *w.shape[2:]), b.reshape(-1), padding=1, groups=T)
            h = F.batch_norm(h, None, None, gam.reshape(-1), bet.reshape(-1), training=True)
            h = F.max_pool2d(F.relu(h), 2)
        h = h.reshape(h.shape[0], T, -1).transpose(0, 1)  # [T, B, 64]
    return torch.baddbmm(params[17].unsqueeze(1), h, params[16].transpose(1, 2))


class TaskBatchInner(FusedSgdInner):
    """The inner SGD-momentum step of all T tasks of a batch: one fused
    differentiable libdiffopt.so launch over the T x 112,261 flat buffer."""

    def __init__(self, T, device, cfg: MamlConfig):
        super().__init__([T * n for n in sizes_of(CONV4_SHAPES)], device, cfg)
        self.T = T


def meta_grad_batched(phi, data, cfg: MamlConfig, inner: TaskBatchInner):
    """meta_grad_data for a batch of tasks run as one task-batched network
    (conv4_forward_tasks): Sum_t d L_query,t(theta_K,t(phi)) / d phi and the
    summed query loss. Each task's inner loop is the same recurrence as in
    meta_grad_data (its loss is a mean over its own images); only the
    summation order of the meta-gradient over tasks differs."""
    T = len(data)
    assert inner.T == T
    sizes = sizes_of(CONV4_SHAPES)
    blk = [T * n for n in sizes]
    xs = torch.stack([d[0] for d in data], 1).flatten(1, 2)
    ys = torch.stack([d[1] for d in data])
    xq = torch.stack([d[2] for d in data], 1).flatten(1, 2)
    yq = torch.stack([d[3] for d in data])

    def loss_of(theta, x, y):
        params = [p.view(T, *s) for p, s in zip(torch.split(theta, blk), CONV4_SHAPES)]
        logits = conv4_forward_tasks(params, x, T, cfg.net)
        return F.cross_entropy(logits.reshape(-1, WAYS), y.reshape(-1), reduction="sum") / y.shape[1]

    phi_v = phi.detach().requires_grad_(True)
    theta, b = theta0_tasks(torch.split(phi_v, sizes), T), None
    for _ in range(cfg.inner_steps):
        (g,) = torch.autograd.grad(loss_of(theta, xs, ys), theta, create_graph=True)
        theta, b = inner(g, b, theta)
    qloss = loss_of(theta, xq, yq)
    (mg,) = torch.autograd.grad(qloss, phi_v)
    return mg, qloss.detach()


class GraphedShard:
    """One rank's share of the meta-batch captured as a single CUDA graph
    (all inner loops, query losses, second-order backward and the local
    meta-gradient sum): per outer step only the task data and phi are
    copied into static buffers and the graph is replayed, removing the
    per-kernel launch cost that dominates these tiny convolutions.
    With ``streams = S > 1`` the tasks are captured on S forked streams, so
    the graph holds S independent branches that the GPU runs concurrently
    (one task's small convolutions leave most SMs idle); the per-task
    meta-gradients are summed in task order after the join (the same sum as
    the sequential version). With ``batched=True`` the shard's tasks run as
    task-batched networks (meta_grad_batched: batched GEMM convolutions, one
    fused inner step per group), ~T x fewer kernels per replay; with
    ``streams = S > 1`` as S contiguous task groups on concurrent graph
    branches (at a few tasks per GPU each kernel underfills the SMs, so
    concurrent groups recover the idle capacity), summed in group order.
    Call it like meta_grad_tasks."""

    def __init__(self, task_ids, cfg: MamlConfig, inner, device, warmup=2, streams=1,
                 batched=False):
        self.ids, self.cfg, self.inner = list(task_ids), cfg, inner
        self.batched = bool(batched)
        self.nstreams = max(1, min(int(streams), len(self.ids)))
        if self.batched:
            # contiguous task groups, one task-batched network per graph branch
            n, S = len(self.ids), self.nstreams
            cuts = [n * i // S for i in range(S + 1)]
            self.groups = [(cuts[i], cuts[i + 1]) for i in range(S) if cuts[i + 1] > cuts[i]]
            self.nstreams = len(self.groups)
            self.inners = [TaskBatchInner(b - a, device, cfg) for a, b in self.groups]
            self.inner = self.inners[0]
        self.phi = torch.zeros(sum(sizes_of(CONV4_SHAPES)), device=device)
        self.data = [task_data(0, t, device, cfg.seed) for t in self.ids]
        self.streams = [torch.cuda.Stream(device) for _ in range(self.nstreams)]
        side = torch.cuda.Stream(device)
        side.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream(device).wait_stream(side)
        from . import _lib as L

        def ours():  # launches of this repo's kernels (libdiffopt.so + libmamlnet.so)
            n = L.opt_launch_count()
            if cfg.net == "fused":
                from . import _net as N

                n += N.net_launch_count()
            return n

        self.graph = torch.cuda.CUDAGraph()
        n0 = ours()
        with torch.cuda.graph(self.graph):
            self.mg, self.loss = self._body()
        self.launches_per_replay = ours() - n0  # captured library kernels

    def _body(self):
        if self.batched and self.nstreams == 1:
            return meta_grad_batched(self.phi, self.data, self.cfg, self.inner)
        if self.nstreams == 1:
            return meta_grad_data(self.phi, self.data, self.cfg, self.inner)
        cur = torch.cuda.current_stream()
        parts = []
        if self.batched:  # task groups as concurrent graph branches
            for s, (a, b), inner in zip(self.streams, self.groups, self.inners):
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    parts.append(meta_grad_batched(self.phi, self.data[a:b], self.cfg, inner))
        for k, d in enumerate(self.data if not self.batched else []):
            s = self.streams[k % self.nstreams]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                parts.append(meta_grad_data(self.phi, [d], self.cfg, self.inner))
        for s in self.streams:
            cur.wait_stream(s)
        total = torch.zeros_like(self.phi)
        loss = torch.zeros((), device=self.phi.device)
        for mg, l in parts:  # task order
            total += mg
            loss += l
        return total, loss

    def __call__(self, phi, task_ids, outer_step, cfg, inner):
        assert list(task_ids) == self.ids
        self.phi.copy_(phi)
        for tid, bufs in zip(self.ids, self.data):
            for dst, src in zip(bufs, task_data(outer_step, tid, phi.device, cfg.seed)):
                dst.copy_(src)
        self.graph.replay()
        return self.mg, self.loss


class PeerAdamOuter:
    """Outer Adam with the meta-gradient all-reduce FUSED into the step
    (sharded.PeerShardedAdam / opt_adam_fwd_peers): rank r sums the W ranks'
    local meta-gradient sums for its 1/W shard of phi straight from their
    memory (CUDA IPC; NVLink on a multi-GPU node), applies Adam with the
    1/tasks scaling, and stores the new phi slice into every rank's copy.
    Replaces FusedAdamOuter + the NCCL all-reduce of the meta-gradient; the
    scalar query loss is still all-reduced (4 bytes)."""

    fused_allreduce = True

    def __init__(self, n, world, rank, device, lr, tasks, group=None):
        from .sharded import PeerShardedAdam

        self.n = int(n)
        self.opt = PeerShardedAdam(n, world, rank, device, lr=lr, group=group,
                                   grad_scale=1.0 / tasks)

    def step_from_local(self, phi, mg_local):
        self.opt.params[:self.n].copy_(phi)  # replicas are identical; keeps phi's storage
        self.opt.grads[:self.n].copy_(mg_local)
        self.opt.step()
        phi.copy_(self.opt.params[:self.n])
        return phi


def outer_step(phi, outer_step_idx, cfg: MamlConfig, inner, outer, world=1, rank=0, group=None,
               shard=None, allreduce_events=None):
    """One synchronous meta-update over the cfg.tasks-task meta-batch.
    ``shard`` (optional) replaces meta_grad_tasks, e.g. a GraphedShard.
    ``allreduce_events`` (optional list) receives a (start, end) CUDA event
    pair recorded around the exchange step on the current stream."""
    import torch.distributed as dist

    ids = task_range(world, rank, cfg.tasks)
    run = shard if shard is not None else meta_grad_tasks
    mg, loss = run(phi, ids, outer_step_idx, cfg, inner)
    if getattr(outer, "fused_allreduce", False):
        loss = loss.reshape(1).clone()
        if world > 1:
            dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)
        phi = outer.step_from_local(phi, mg)
        return phi, loss[0] / cfg.tasks, None
    buf = torch.cat([mg, loss.reshape(1)])
    if allreduce_events is not None:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    if world > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)  # the one exchange step
    if allreduce_events is not None:
        ev[1].record()
        allreduce_events.append(ev)
    buf.mul_(1.0 / cfg.tasks)
    mg, loss = buf[:-1].contiguous(), buf[-1]
    phi = outer(phi, mg)
    return phi, loss, mg
