"""Differentiable optimizer steps as torch.autograd.Functions over flat buffers,
and the functional API of PAPER.md Listing 1:

    opt = adam(lr=1e-3)
    state = opt.init(params)
    updates, state = opt.update(grads, state, inplace=False)
    params = apply_updates(params, updates)

Every forward and backward is one call into libdiffopt.so (the C ABI); this
module only allocates outputs (torch caching allocator), picks the current
stream and wires autograd ("we define the forward and backward
behavior using torch.autograd.Function"). Hyper-parameters may be Python
floats or CPU scalar tensors; a tensor that requires grad receives the
kernel's hyper-gradient sum.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch
from torch.autograd.function import once_differentiable

from . import _lib as L

_WS = {}


def _workspace(tree: L.Tree, device, per_leaf=False):
    """Per (device, stream, tree size) zeroed workspace, reused across calls
    (the library leaves it zero-filled)."""
    stream = torch.cuda.current_stream(device).cuda_stream
    nbytes = tree.workspace_bytes(per_leaf)
    key = (str(device), stream, nbytes)
    ws = _WS.get(key)
    if ws is None:
        ws = tree.workspace(device, per_leaf)
        _WS[key] = ws
    return ws


def _f(x):
    return float(x.detach().item()) if isinstance(x, torch.Tensor) else float(x)


def _needs(x):
    return isinstance(x, torch.Tensor) and x.requires_grad


def _hp_grad(x, val):
    if not _needs(x):
        return None
    return val.to(device=x.device, dtype=x.dtype).reshape(x.shape)


def _state_dtype(t):
    if t is None:
        return None
    if t.dtype == torch.bfloat16:
        return L.OPT_BF16
    if t.dtype == torch.float32:
        return L.OPT_F32
    raise TypeError(f"state must be float32 or bfloat16, got {t.dtype}")


def _sd(*states, default=L.OPT_F32):
    for s in states:
        if s is not None:
            return _state_dtype(s)
    return default


def _empty_state(like, sd):
    return torch.empty_like(like, dtype=torch.bfloat16 if sd == L.OPT_BF16 else torch.float32)


def _contig(t):
    return None if t is None else t.contiguous()


def _cot(t):
    """A cotangent as a contiguous float32 buffer. Autograd hands the VJP of a
    bfloat16 state output a bfloat16 cotangent; the C ABI reads every
    cotangent as float (diffopt.h), so it is widened here (exactly)."""
    if t is None:
        return None
    if t.dtype != torch.float32:
        t = t.float()
    return t.contiguous()


def _check_args(cfg, g, states=(), f32=(), lr_leaf=None):
    """Validate what the kernels assume before raw pointers leave Python:
    float32 CUDA buffers of exactly tree.numel elements on one device
    (state may be bfloat16), lr_leaf float32 with one entry per leaf."""
    n = cfg.tree.numel
    if not isinstance(g, torch.Tensor) or not g.is_cuda:
        raise TypeError("the gradient must be a CUDA tensor (there is no CPU path)")
    if g.dtype != torch.float32:
        raise TypeError(f"the gradient must be float32, got {g.dtype}")
    if g.numel() != n:
        raise ValueError(f"the gradient has {g.numel()} elements, the tree {n}")
    d = cfg.tree.d_offsets
    if d is not None and d.device != g.device:
        raise ValueError(f"the tree's offsets live on {d.device}, the gradient on {g.device}")
    for kind, ts in (("state", states), ("buffer", f32)):
        for t in ts:
            if t is None:
                continue
            if t.device != g.device:
                raise ValueError(f"a {kind} tensor is on {t.device}, the gradient on {g.device}")
            ok = (torch.float32, torch.bfloat16) if kind == "state" else (torch.float32,)
            if t.dtype not in ok:
                raise TypeError(f"a {kind} tensor has dtype {t.dtype}; allowed: {ok}")
            if t.numel() != n:
                raise ValueError(f"a {kind} tensor has {t.numel()} elements, the tree {n}")
    if lr_leaf is not None:
        if lr_leaf.device != g.device or lr_leaf.dtype != torch.float32:
            raise TypeError("lr_leaf must be a float32 tensor on the gradient's device")
        if lr_leaf.numel() != cfg.tree.n_leaves:
            raise ValueError("lr_leaf must have one entry per leaf")


@dataclass
class StepConfig:
    tree: L.Tree
    compute: int = L.OPT_COMPUTE_DEFAULT
    state_dtype: Optional[int] = None   # None: follow the input state (fp32 if none)


# ------------------------------------------------------------------ Adam
class AdamStep(torch.autograd.Function):
    """(g, mu, nu[, params]) -> (updates or params + updates, mu', nu')."""

    @staticmethod
    def forward(ctx, g, mu, nu, params, lr, b1, b2, eps, step, eps_root, cfg):
        g, mu, nu, params = _contig(g), _contig(mu), _contig(nu), _contig(params)
        _check_args(cfg, g, (mu, nu), (params,))
        with torch.cuda.device(g.device):
            return AdamStep._fwd(ctx, g, mu, nu, params, lr, b1, b2, eps, step, eps_root, cfg)

    @staticmethod
    def _fwd(ctx, g, mu, nu, params, lr, b1, b2, eps, step, eps_root, cfg):
        sd = cfg.state_dtype if cfg.state_dtype is not None else _sd(mu, nu)
        hp = (_f(lr), _f(b1), _f(b2), _f(eps), float(eps_root))
        out = torch.empty_like(g)
        mu1, nu1 = _empty_state(g, sd), _empty_state(g, sd)
        fused = params is not None
        L.opt_adam_fwd(cfg.tree, step, hp, sd, cfg.compute, g, mu, nu,
                       None if fused else out, mu1, nu1,
                       params if fused else None, out if fused else None)
        ctx.save_for_backward(g, mu, nu)
        ctx.meta = (hp, step, sd, cfg, fused, (lr, b1, b2, eps), mu is None, nu is None)
        return out, mu1, nu1

    @staticmethod
    @once_differentiable
    def backward(ctx, d_out, d_mu1, d_nu1):
        g, mu, nu = ctx.saved_tensors
        with torch.cuda.device(g.device):
            return AdamStep._bwd(ctx, g, mu, nu, d_out, d_mu1, d_nu1)

    @staticmethod
    def _bwd(ctx, g, mu, nu, d_out, d_mu1, d_nu1):
        hp, step, sd, cfg, fused, hps, mu_none, nu_none = ctx.meta
        want_hp = any(_needs(x) for x in hps)
        d_g = torch.empty_like(g)
        d_mu = None if mu_none or not ctx.needs_input_grad[1] else torch.empty_like(g)
        d_nu = None if nu_none or not ctx.needs_input_grad[2] else torch.empty_like(g)
        d_hp = torch.empty(4, dtype=torch.float64, device=g.device) if want_hp else None
        ws = _workspace(cfg.tree, g.device) if want_hp else None
        L.opt_adam_bwd(cfg.tree, step, hp, sd, cfg.compute, g, mu, nu, _cot(d_out),
                       _cot(d_mu1), _cot(d_nu1), d_g, d_mu, d_nu, d_hp, None, ws)
        d_params = d_out if fused else None
        hg = [None] * 4 if d_hp is None else [_hp_grad(x, d_hp[k]) for k, x in enumerate(hps)]
        return (d_g, d_mu, d_nu, d_params, *hg, None, None, None)


# --------------------------------------------------------------- RMSProp
class RmsPropStep(torch.autograd.Function):
    """(g, nu[, params]) -> (updates or params + updates, nu')."""

    @staticmethod
    def forward(ctx, g, nu, params, lr, alpha, eps, cfg):
        g, nu, params = _contig(g), _contig(nu), _contig(params)
        _check_args(cfg, g, (nu,), (params,))
        with torch.cuda.device(g.device):
            return RmsPropStep._fwd(ctx, g, nu, params, lr, alpha, eps, cfg)

    @staticmethod
    def _fwd(ctx, g, nu, params, lr, alpha, eps, cfg):
        sd = cfg.state_dtype if cfg.state_dtype is not None else _sd(nu)
        hp = (_f(lr), _f(alpha), _f(eps))
        out = torch.empty_like(g)
        nu1 = _empty_state(g, sd)
        fused = params is not None
        L.opt_rmsprop_fwd(cfg.tree, hp, sd, cfg.compute, g, nu, None if fused else out, nu1,
                          params if fused else None, out if fused else None)
        ctx.save_for_backward(g, nu)
        ctx.meta = (hp, sd, cfg, fused, (lr, alpha, eps), nu is None)
        return out, nu1

    @staticmethod
    @once_differentiable
    def backward(ctx, d_out, d_nu1):
        g, nu = ctx.saved_tensors
        with torch.cuda.device(g.device):
            return RmsPropStep._bwd(ctx, g, nu, d_out, d_nu1)

    @staticmethod
    def _bwd(ctx, g, nu, d_out, d_nu1):
        hp, sd, cfg, fused, hps, nu_none = ctx.meta
        want_hp = any(_needs(x) for x in hps)
        d_g = torch.empty_like(g)
        d_nu = None if nu_none or not ctx.needs_input_grad[1] else torch.empty_like(g)
        d_hp = torch.empty(3, dtype=torch.float64, device=g.device) if want_hp else None
        ws = _workspace(cfg.tree, g.device) if want_hp else None
        L.opt_rmsprop_bwd(cfg.tree, hp, sd, cfg.compute, g, nu, _cot(d_out), _cot(d_nu1),
                          d_g, d_nu, d_hp, None, ws)
        hg = [None] * 3 if d_hp is None else [_hp_grad(x, d_hp[k]) for k, x in enumerate(hps)]
        return (d_g, d_nu, d_out if fused else None, *hg, None)


# ------------------------------------------------------------------- SGD
class SgdStep(torch.autograd.Function):
    """(g, mom[, params]) -> (updates or params + updates, mom')."""

    @staticmethod
    def forward(ctx, g, mom, params, lr, momentum, nesterov, cfg):
        g, mom, params = _contig(g), _contig(mom), _contig(params)
        _check_args(cfg, g, (mom,), (params,))
        with torch.cuda.device(g.device):
            return SgdStep._fwd(ctx, g, mom, params, lr, momentum, nesterov, cfg)

    @staticmethod
    def _fwd(ctx, g, mom, params, lr, momentum, nesterov, cfg):
        sd = cfg.state_dtype if cfg.state_dtype is not None else _sd(mom)
        hp = (_f(lr), _f(momentum), bool(nesterov))
        out = torch.empty_like(g)
        has_state = hp[1] != 0.0
        mom1 = _empty_state(g, sd) if has_state else None
        fused = params is not None
        L.opt_sgd_fwd(cfg.tree, hp, sd, cfg.compute, g, mom, None if fused else out, mom1,
                      params if fused else None, out if fused else None)
        ctx.save_for_backward(g, mom)
        ctx.meta = (hp, sd, cfg, fused, (lr, momentum), mom is None)
        if mom1 is None:
            mom1 = g.new_zeros(0)
        return out, mom1

    @staticmethod
    @once_differentiable
    def backward(ctx, d_out, d_mom1):
        g, mom = ctx.saved_tensors
        with torch.cuda.device(g.device):
            return SgdStep._bwd(ctx, g, mom, d_out, d_mom1)

    @staticmethod
    def _bwd(ctx, g, mom, d_out, d_mom1):
        hp, sd, cfg, fused, hps, mom_none = ctx.meta
        want_hp = any(_needs(x) for x in hps)
        if d_mom1 is not None and d_mom1.numel() == 0:
            d_mom1 = None
        d_g = torch.empty_like(g)
        d_mom = None if mom_none or not ctx.needs_input_grad[1] else torch.empty_like(g)
        d_hp = torch.empty(2, dtype=torch.float64, device=g.device) if want_hp else None
        ws = _workspace(cfg.tree, g.device) if want_hp else None
        L.opt_sgd_bwd(cfg.tree, hp, sd, cfg.compute, g, mom, _cot(d_out), _cot(d_mom1),
                      d_g, d_mom, d_hp, None, ws)
        hg = [None] * 2 if d_hp is None else [_hp_grad(x, d_hp[k]) for k, x in enumerate(hps)]
        return (d_g, d_mom, d_out if fused else None, *hg, None, None)


# ---------------------------------------------- variants (NEXT-1, *_ex ABI)
_EX_NH = {"adam": 5, "rmsprop": 4, "sgd": 3}


class StepEx(torch.autograd.Function):
    """Any of the three optimizers with weight decay (L2 / AdamW), maximize
    and per-leaf learning rates (``lr_leaf``: a float32 CUDA tensor of
    n_leaves entries that may require grad -- Meta-SGD/MGRL-style learnable
    per-leaf lr). Inputs: (g, s0, s1, params, hyper tuple, wd, lr_leaf).
    Outputs: (params + u if ``fused`` else u, s0', s1'). ``hps`` are the
    optimizer's hyper-parameters after lr (adam: b1, b2, eps; rmsprop: alpha,
    eps; sgd: momentum)."""

    @staticmethod
    def forward(ctx, g, s0, s1, params, lr, wd, lr_leaf, hps, kind, step, opts, cfg):
        decoupled, maximize, nesterov, eps_root, fused = opts
        g, s0, s1, params = _contig(g), _contig(s0), _contig(s1), _contig(params)
        _check_args(cfg, g, (s0, s1), (params,), None if lr_leaf is None else lr_leaf)
        with torch.cuda.device(g.device):
            return StepEx._fwd(ctx, g, s0, s1, params, lr, wd, lr_leaf, hps, kind, step, opts,
                               cfg)

    @staticmethod
    def _fwd(ctx, g, s0, s1, params, lr, wd, lr_leaf, hps, kind, step, opts, cfg):
        decoupled, maximize, nesterov, eps_root, fused = opts
        sd = cfg.state_dtype if cfg.state_dtype is not None else _sd(s0, s1)
        ext = L._ext(_f(wd), decoupled, maximize, None if lr_leaf is None else lr_leaf.detach())
        out = torch.empty_like(g)
        n0 = _empty_state(g, sd)
        if kind == "adam":
            hp = (_f(lr), _f(hps[0]), _f(hps[1]), _f(hps[2]), float(eps_root))
            n1 = _empty_state(g, sd)
            L.opt_adam_fwd_ex(cfg.tree, step, hp, ext, sd, cfg.compute, g, s0, s1, params,
                              None if fused else out, n0, n1, out if fused else None)
        elif kind == "rmsprop":
            hp = (_f(lr), _f(hps[0]), _f(hps[1]))
            n1 = g.new_zeros(0)
            L.opt_rmsprop_fwd_ex(cfg.tree, hp, ext, sd, cfg.compute, g, s0, params,
                                 None if fused else out, n0, out if fused else None)
        else:
            hp = (_f(lr), _f(hps[0]), bool(nesterov))
            n1 = g.new_zeros(0)
            L.opt_sgd_fwd_ex(cfg.tree, hp, ext, sd, cfg.compute, g, s0, params,
                             None if fused else out, n0, out if fused else None)
        ctx.save_for_backward(g, s0, s1, params, lr_leaf)
        ctx.meta = (kind, hp, ext, sd, cfg, fused, (lr,) + tuple(hps) + (wd,), step)
        return out, n0, n1

    @staticmethod
    @once_differentiable
    def backward(ctx, d_out, d_n0, d_n1):
        g, s0, s1, params, lr_leaf = ctx.saved_tensors
        with torch.cuda.device(g.device):
            return StepEx._bwd(ctx, g, s0, s1, params, lr_leaf, d_out, d_n0, d_n1)

    @staticmethod
    def _bwd(ctx, g, s0, s1, params, lr_leaf, d_out, d_n0, d_n1):
        kind, hp, ext, sd, cfg, fused, hyp, step = ctx.meta
        nh = _EX_NH[kind]
        want_leaf = lr_leaf is not None and lr_leaf.requires_grad
        want_hp = want_leaf or any(_needs(x) for x in hyp)
        d_g = torch.empty_like(g)
        d_s0 = None if s0 is None else torch.empty_like(g)
        d_s1 = None if (s1 is None or kind != "adam") else torch.empty_like(g)
        d_p = None if params is None else torch.empty_like(g)
        d_hp = torch.empty(nh, dtype=torch.float64, device=g.device) if want_hp else None
        d_leaf = (torch.empty(cfg.tree.n_leaves * nh, dtype=torch.float64, device=g.device)
                  if want_leaf else None)
        # the library sums per leaf whenever lr_leaf is given (even a fixed one)
        ws = _workspace(cfg.tree, g.device, per_leaf=lr_leaf is not None) if want_hp else None
        d_out = _cot(d_out)
        if d_n1 is not None and d_n1.numel() == 0:
            d_n1 = None
        if kind == "adam":
            L.opt_adam_bwd_ex(cfg.tree, step, hp, ext, sd, cfg.compute, g, s0, s1, params, d_out,
                              _cot(d_n0), _cot(d_n1), d_g, d_s0, d_s1, d_p, d_hp, d_leaf, ws)
        elif kind == "rmsprop":
            L.opt_rmsprop_bwd_ex(cfg.tree, hp, ext, sd, cfg.compute, g, s0, params, d_out,
                                 _cot(d_n0), d_g, d_s0, d_p, d_hp, d_leaf, ws)
        else:
            L.opt_sgd_bwd_ex(cfg.tree, hp, ext, sd, cfg.compute, g, s0, params, d_out,
                             _cot(d_n0), d_g, d_s0, d_p, d_hp, d_leaf, ws)
        if d_p is not None and fused:
            d_p = d_p + d_out  # identity of the fused apply_updates
        lr, *rest = hyp
        hg = [None] * len(hyp)
        if d_hp is not None:
            hg = [_hp_grad(x, d_hp[k]) for k, x in enumerate(hyp[:-1])] + [
                _hp_grad(hyp[-1], d_hp[nh - 1])]
        d_lrl = None
        if want_leaf:
            d_lrl = d_leaf.view(-1, nh)[:, 0].to(lr_leaf.dtype)
        hps_grad = None  # hyper-parameters after lr are passed as a tuple (no grads)
        return (d_g, d_s0, d_s1, d_p, hg[0], hg[-1], d_lrl, hps_grad, None, None, None, None)


class RmsCmStep(torch.autograd.Function):
    """Centred and/or momentum RMSProp (NEXT-1, reading N4) with weight
    decay, maximize and per-leaf lr: (g, nu, gavg, buf, params, lr, alpha,
    eps, momentum, wd, lr_leaf) -> (params + u if fused else u, nu', gavg',
    buf'). Differentiable in every tensor input and hyper-parameter."""

    @staticmethod
    def forward(ctx, g, nu, gavg, buf, params, lr, alpha, eps, mom, wd, lr_leaf, opts, cfg):
        g, nu, gavg, buf, params = (_contig(x) for x in (g, nu, gavg, buf, params))
        _check_args(cfg, g, (nu, gavg, buf), (params,), lr_leaf)
        with torch.cuda.device(g.device):
            return RmsCmStep._fwd(ctx, g, nu, gavg, buf, params, lr, alpha, eps, mom, wd,
                                  lr_leaf, opts, cfg)

    @staticmethod
    def _fwd(ctx, g, nu, gavg, buf, params, lr, alpha, eps, mom, wd, lr_leaf, opts, cfg):
        centered, maximize, fused = opts
        sd = cfg.state_dtype if cfg.state_dtype is not None else _sd(nu, gavg, buf)
        ext = L._ext(_f(wd), False, maximize, None if lr_leaf is None else lr_leaf.detach())
        hp = (_f(lr), _f(alpha), _f(eps), _f(mom), bool(centered))
        out = torch.empty_like(g)
        n_nu, n_buf = _empty_state(g, sd), _empty_state(g, sd)
        n_gavg = _empty_state(g, sd) if centered else g.new_zeros(0)
        L.opt_rmsprop_cm_fwd(cfg.tree, hp, ext, sd, cfg.compute, g, nu, gavg, buf, params,
                             None if fused else out, n_nu, n_gavg if centered else None, n_buf,
                             out if fused else None)
        ctx.save_for_backward(g, nu, gavg, buf, params, lr_leaf)
        ctx.meta = (hp, ext, sd, cfg, fused, centered, (lr, alpha, eps, mom, wd))
        return out, n_nu, n_gavg, n_buf

    @staticmethod
    @once_differentiable
    def backward(ctx, d_out, d_nu1, d_gavg1, d_buf1):
        g, nu, gavg, buf, params, lr_leaf = ctx.saved_tensors
        with torch.cuda.device(g.device):
            return RmsCmStep._bwd(ctx, g, nu, gavg, buf, params, lr_leaf, d_out, d_nu1, d_gavg1,
                                  d_buf1)

    @staticmethod
    def _bwd(ctx, g, nu, gavg, buf, params, lr_leaf, d_out, d_nu1, d_gavg1, d_buf1):
        hp, ext, sd, cfg, fused, centered, hyp = ctx.meta
        want_leaf = lr_leaf is not None and lr_leaf.requires_grad
        want_hp = want_leaf or any(_needs(x) for x in hyp)
        d_g = torch.empty_like(g)
        d_nu = None if nu is None else torch.empty_like(g)
        d_gavg = None if (gavg is None or not centered) else torch.empty_like(g)
        d_buf = None if buf is None else torch.empty_like(g)
        d_p = None if params is None else torch.empty_like(g)
        d_hp = torch.empty(5, dtype=torch.float64, device=g.device) if want_hp else None
        d_leaf = (torch.empty(cfg.tree.n_leaves * 5, dtype=torch.float64, device=g.device)
                  if want_leaf else None)
        ws = _workspace(cfg.tree, g.device, per_leaf=lr_leaf is not None) if want_hp else None
        if d_gavg1 is not None and d_gavg1.numel() == 0:
            d_gavg1 = None
        L.opt_rmsprop_cm_bwd(cfg.tree, hp, ext, sd, cfg.compute, g, nu, gavg, buf, params,
                             _cot(d_out), _cot(d_nu1), _cot(d_gavg1), _cot(d_buf1),
                             d_g, d_nu, d_gavg, d_buf, d_p, d_hp, d_leaf, ws)
        if d_p is not None and fused:
            d_p = d_p + d_out  # identity of the fused apply_updates
        hg = [None] * 5 if d_hp is None else [_hp_grad(x, d_hp[k]) for k, x in enumerate(hyp)]
        d_lrl = d_leaf.view(-1, 5)[:, 0].to(lr_leaf.dtype) if want_leaf else None
        return (d_g, d_nu, d_gavg, d_buf, d_p, *hg, d_lrl, None, None)


class ApplyUpdates(torch.autograd.Function):
    """params + updates (row a8); backward is the identity for both."""

    @staticmethod
    def forward(ctx, params, updates):
        p, u = params.contiguous(), updates.contiguous()
        if not (p.is_cuda and u.is_cuda) or p.device != u.device:
            raise TypeError("apply_updates needs params and updates on one CUDA device")
        if p.dtype != torch.float32 or u.dtype != torch.float32:
            raise TypeError("apply_updates needs float32 params and updates")
        out = torch.empty_like(p)
        with torch.cuda.device(p.device):
            L.opt_apply_updates(p.numel(), p, u, out)
        return out

    @staticmethod
    @once_differentiable
    def backward(ctx, d):
        return d, d


# ------------------------------------------------ functional (Listing 1)
class FlatTree:
    """Host description of a tensor tree flattened to one buffer per role
    (leaves in depth-first order). ``views(flat)`` returns the leaf
    views of a flat buffer via one ``split`` whose autograd backward is a
    single concatenation (no per-leaf scatter)."""

    def __init__(self, shapes, device):
        self.shapes = [tuple(s) for s in shapes]
        self.sizes = [int(torch.Size(s).numel()) for s in self.shapes]
        self.tree = L.Tree.from_sizes(self.sizes, device=device)
        self.device = device

    @classmethod
    def of(cls, tensors):
        tensors = list(tensors)
        return cls([t.shape for t in tensors], tensors[0].device)

    def flatten(self, tensors):
        return torch.cat([t.reshape(-1) for t in tensors])

    def views(self, flat):
        return [p.view(s) for p, s in zip(torch.split(flat, self.sizes), self.shapes)]


@dataclass
class OptState:
    step: int
    slots: tuple          # flat state buffers (or None = zero state)
    layout: FlatTree


class GradientTransformation:
    """init/update pair. ``update`` accepts a flat gradient
    buffer or a sequence of leaf gradients (flattened once into one buffer)."""

    def __init__(self, kind, hp, n_slots, compute=L.OPT_COMPUTE_DEFAULT, state_dtype=L.OPT_F32,
                 ext=None):
        self.kind, self.hp, self.n_slots = kind, hp, n_slots
        self.compute, self.state_dtype = compute, state_dtype
        self.ext = ext  # None or dict(weight_decay, decoupled, maximize, lr_leaf) (NEXT-1)

    def init(self, params):
        """Zero state. Slots are None until the first update: the
        kernel reads a NULL state as zeros (no HBM read)."""
        if isinstance(params, torch.Tensor):
            layout = FlatTree([params.shape], params.device)
        else:
            layout = FlatTree.of(params)
        return OptState(0, (None,) * self.n_slots, layout)

    def update(self, grads, state: OptState, inplace: bool = False, params=None):
        differentiable = torch.is_grad_enabled()
        if inplace and differentiable and _any_requires_grad(grads, state):
            # in-place update would destroy the state the VJP needs
            raise RuntimeError("inplace=True is not allowed with a differentiable update")
        layout = state.layout
        flat = grads if _is_flat(grads, layout) else layout.flatten(grads)
        cfg = StepConfig(layout.tree, self.compute, self.state_dtype)
        t = state.step + 1
        flat_p = None
        if params is not None:
            flat_p = params if _is_flat(params, layout) else layout.flatten(params)
        if self.kind == "rmsprop_cm":
            return self._update_cm(flat, state, flat_p, cfg, t, inplace, differentiable)
        if self.ext is not None:
            return self._update_ex(flat, state, flat_p, cfg, t, inplace, differentiable)
        if self.kind == "adam":
            lr, b1, b2, eps, eps_root = self.hp
            out, m1, v1 = AdamStep.apply(flat, state.slots[0], state.slots[1], None, lr, b1,
                                         b2, eps, t, eps_root, cfg)
            slots = (m1, v1)
        elif self.kind == "rmsprop":
            lr, alpha, eps = self.hp
            out, v1 = RmsPropStep.apply(flat, state.slots[0], None, lr, alpha, eps, cfg)
            slots = (v1,)
        else:
            lr, mom, nest = self.hp
            out, b1 = SgdStep.apply(flat, state.slots[0] if state.slots else None, None, lr,
                                    mom, nest, cfg)
            slots = (b1 if _f(mom) != 0.0 else None,)
        if inplace and not differentiable:
            for old, new in zip(state.slots, slots):
                if old is not None and new is not None:
                    old.copy_(new)
        return out, OptState(t, slots, layout)

    def _update_ex(self, flat, state, flat_p, cfg, t, inplace, differentiable):
        e = self.ext
        if _f(e["weight_decay"]) != 0.0 and flat_p is None:
            raise ValueError("weight_decay needs update(..., params=...)")
        lr_leaf = e.get("lr_leaf")
        if lr_leaf is not None and lr_leaf.numel() != cfg.tree.n_leaves:
            raise ValueError("lr_leaf must have one entry per leaf")
        if self.kind == "adam":
            lr, b1, b2, eps, eps_root = self.hp
            hps, nest = (b1, b2, eps), False
        elif self.kind == "rmsprop":
            lr, alpha, eps = self.hp
            hps, nest, eps_root = (alpha, eps), False, 0.0
        else:
            lr, mom, nest = self.hp
            hps, eps_root = (mom,), 0.0
        s0 = state.slots[0] if state.slots else None
        s1 = state.slots[1] if len(state.slots) > 1 else None
        opts = (bool(e.get("decoupled", False)), bool(e.get("maximize", False)), bool(nest),
                eps_root, False)
        out, n0, n1 = StepEx.apply(flat, s0, s1, flat_p, lr, e["weight_decay"], lr_leaf, hps,
                                   self.kind, t, opts, cfg)
        slots = (n0, n1) if self.kind == "adam" else (n0,)
        if inplace and not differentiable:
            for old, new in zip(state.slots, slots):
                if old is not None and new is not None:
                    old.copy_(new)
        return out, OptState(t, slots, state.layout)


    def _update_cm(self, flat, state, flat_p, cfg, t, inplace, differentiable):
        e = self.ext or dict(weight_decay=0.0, maximize=False, lr_leaf=None)
        if _f(e["weight_decay"]) != 0.0 and flat_p is None:
            raise ValueError("weight_decay needs update(..., params=...)")
        lr_leaf = e.get("lr_leaf")
        if lr_leaf is not None and lr_leaf.numel() != cfg.tree.n_leaves:
            raise ValueError("lr_leaf must have one entry per leaf")
        lr, alpha, eps, mom, centered = self.hp
        nu, gavg, buf = state.slots
        out, n_nu, n_gavg, n_buf = RmsCmStep.apply(
            flat, nu, gavg, buf, flat_p, lr, alpha, eps, mom, e["weight_decay"], lr_leaf,
            (bool(centered), bool(e.get("maximize", False)), False), cfg)
        slots = (n_nu, n_gavg if centered else None, n_buf)
        if inplace and not differentiable:
            for old, new in zip(state.slots, slots):
                if old is not None and new is not None:
                    old.copy_(new)
        return out, OptState(t, slots, state.layout)


def _is_flat(x, layout):
    """A 1-D tensor of tree.numel elements is already the flat buffer (e.g. the
    gradient autograd returns for a flat parameter buffer); a single tensor of
    another shape is the one leaf of a one-leaf tree; sequences are leaves."""
    if not isinstance(x, torch.Tensor):
        return False
    if x.dim() == 1 and x.numel() == layout.tree.numel:
        return True
    if len(layout.sizes) == 1:
        return True  # flatten() of one tensor would iterate its first dimension
    raise ValueError(f"a single tensor of shape {tuple(x.shape)} is not the flat buffer of a "
                     f"{len(layout.sizes)}-leaf tree ({layout.tree.numel} elements)")


def _any_requires_grad(grads, state):
    ts = [grads] if isinstance(grads, torch.Tensor) else list(grads)
    ts += [s for s in state.slots if s is not None]
    return any(t.requires_grad for t in ts)


def _check_unit(name, x):
    v = _f(x)
    if not (0.0 <= v < 1.0):
        raise ValueError(f"{name} must be in [0, 1), got {v}")


def _check_lr(lr):
    if not _f(lr) > 0.0:
        raise ValueError(f"lr must be > 0, got {_f(lr)}")


def _ext_opts(weight_decay, decoupled, maximize, lr_leaf):
    if _f(weight_decay) < 0.0:
        raise ValueError("weight_decay must be >= 0")
    if _f(weight_decay) == 0.0 and not decoupled and not maximize and lr_leaf is None:
        return None
    return dict(weight_decay=weight_decay, decoupled=decoupled, maximize=maximize,
                lr_leaf=lr_leaf)


def adam(lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, eps_root=0.0, weight_decay=0.0, decoupled=False,
         maximize=False, lr_leaf=None, compute=L.OPT_COMPUTE_DEFAULT, state_dtype=L.OPT_F32):
    """Adam (defaults; validation S:189). weight_decay/decoupled
    (AdamW)/maximize/lr_leaf are the NEXT-1 variants (reading N1)."""
    _check_lr(lr)
    _check_unit("b1", b1)
    _check_unit("b2", b2)
    if not _f(eps) > 0.0:
        raise ValueError("eps must be > 0")
    return GradientTransformation("adam", (lr, b1, b2, eps, eps_root), 2, compute, state_dtype,
                                  _ext_opts(weight_decay, decoupled, maximize, lr_leaf))


def rmsprop(lr=1e-2, alpha=0.99, eps=1e-8, weight_decay=0.0, maximize=False, lr_leaf=None,
            centered=False, momentum=0.0, compute=L.OPT_COMPUTE_DEFAULT, state_dtype=L.OPT_F32):
    """RMSProp; ``centered`` / ``momentum`` select the torch.optim
    RMSprop forms (NEXT-1, reading N4: opt_rmsprop_cm_fwd/bwd, state = square
    average, gradient average, momentum buffer)."""
    _check_lr(lr)
    _check_unit("alpha", alpha)
    _check_unit("momentum", momentum)
    if not _f(eps) >= 0.0:
        raise ValueError("eps must be >= 0")
    if centered or _f(momentum) != 0.0:
        return GradientTransformation("rmsprop_cm", (lr, alpha, eps, momentum, bool(centered)), 3,
                                      compute, state_dtype,
                                      _ext_opts(weight_decay, False, maximize, lr_leaf))
    return GradientTransformation("rmsprop", (lr, alpha, eps), 1, compute, state_dtype,
                                  _ext_opts(weight_decay, False, maximize, lr_leaf))


def sgd(lr, momentum=0.0, nesterov=False, weight_decay=0.0, maximize=False, lr_leaf=None,
        compute=L.OPT_COMPUTE_DEFAULT, state_dtype=L.OPT_F32):
    """SGD with optional (Nesterov) momentum."""
    _check_lr(lr)
    _check_unit("momentum", momentum)
    return GradientTransformation("sgd", (lr, momentum, nesterov), 1, compute, state_dtype,
                                  _ext_opts(weight_decay, False, maximize, lr_leaf))


def apply_updates(params, updates):
    """params + updates, leafwise or on flat buffers."""
    if isinstance(params, torch.Tensor):
        if params.shape != updates.shape:
            raise ValueError("params and updates differ in shape")
        return ApplyUpdates.apply(params, updates)
    params = list(params)
    if isinstance(updates, torch.Tensor):  # flat updates for a leaf tuple
        layout = FlatTree.of(params)
        return layout.views(ApplyUpdates.apply(layout.flatten(params), updates))
    updates = list(updates)
    if len(params) != len(updates):
        raise ValueError("TreeDef mismatch between params and updates")
    return [ApplyUpdates.apply(p, u) for p, u in zip(params, updates)]
