"""Thin ctypes binding of include/diffopt.h (argument marshalling only).

Every function here has the name of the C entry point it calls and forwards
device pointers (``tensor.data_ptr()``), sizes, hyper-parameters and the
current CUDA stream. All arithmetic happens in libdiffopt.so. There is no CPU
fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DIFFOPT_LIB") or os.path.join(HERE, "libdiffopt.so")  # env: tuning sweeps

OPT_OK, OPT_EINVAL, OPT_EALIGN, OPT_ECUDA, OPT_EWORKSPACE = 0, 1, 2, 3, 4
OPT_F32, OPT_BF16 = 0, 1
OPT_COMPUTE_DEFAULT, OPT_COMPUTE_F32, OPT_COMPUTE_F64 = 0, 1, 2

EXPORTS = [
    "opt_workspace_bytes", "opt_adam_fwd", "opt_adam_bwd", "opt_rmsprop_fwd", "opt_rmsprop_bwd",
    "opt_sgd_fwd", "opt_sgd_bwd", "opt_apply_updates", "opt_quadratic_grad", "opt_quadratic_rev",
    "opt_status_string", "opt_last_error", "opt_abi_version", "opt_launch_count",
]


class opt_tree(ctypes.Structure):
    _fields_ = [("numel", ctypes.c_int64), ("n_leaves", ctypes.c_int64),
                ("h_offsets", ctypes.c_void_p), ("d_offsets", ctypes.c_void_p)]


class opt_adam_hp(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("lr", "b1", "b2", "eps", "eps_root")]


class opt_rmsprop_hp(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("lr", "alpha", "eps")]


class opt_sgd_hp(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("momentum", ctypes.c_double), ("nesterov", ctypes.c_int)]


class DiffoptError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_status_name(code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2211_06934_b200/build.py` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, I, sz, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_double
    T = ctypes.POINTER(opt_tree)
    L.opt_workspace_bytes.argtypes = [T, I]
    L.opt_workspace_bytes.restype = sz
    L.opt_adam_fwd.argtypes = [T, i64, ctypes.POINTER(opt_adam_hp), I, I] + [P] * 9
    L.opt_adam_bwd.argtypes = [T, i64, ctypes.POINTER(opt_adam_hp), I, I] + [P] * 12 + [sz, P]
    L.opt_rmsprop_fwd.argtypes = [T, ctypes.POINTER(opt_rmsprop_hp), I, I] + [P] * 7
    L.opt_rmsprop_bwd.argtypes = [T, ctypes.POINTER(opt_rmsprop_hp), I, I] + [P] * 9 + [sz, P]
    L.opt_sgd_fwd.argtypes = [T, ctypes.POINTER(opt_sgd_hp), I, I] + [P] * 7
    L.opt_sgd_bwd.argtypes = [T, ctypes.POINTER(opt_sgd_hp), I, I] + [P] * 9 + [sz, P]
    L.opt_apply_updates.argtypes = [i64, P, P, P, P]
    L.opt_quadratic_grad.argtypes = [i64, P, P, P, P, P]
    L.opt_quadratic_rev.argtypes = [i64, P, P, P, P, I, P]
    L.opt_status_string.argtypes = [I]
    L.opt_status_string.restype = ctypes.c_char_p
    L.opt_last_error.restype = ctypes.c_char_p
    L.opt_abi_version.restype = I
    L.opt_launch_count.restype = i64
    for name in ("opt_adam_fwd", "opt_adam_bwd", "opt_rmsprop_fwd", "opt_rmsprop_bwd",
                 "opt_sgd_fwd", "opt_sgd_bwd", "opt_apply_updates", "opt_quadratic_grad",
                 "opt_quadratic_rev"):
        getattr(L, name).restype = I
    return L


lib = _load()


def _status_name(code):
    return lib.opt_status_string(int(code)).decode()


def _check(rc):
    if rc != OPT_OK:
        raise DiffoptError(rc, lib.opt_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


_HP_CACHE = {}


def _hp(cls, hp):
    """ctypes struct for a hyper-parameter tuple, cached by value."""
    if isinstance(hp, cls):
        return hp
    key = (cls, tuple(hp))
    h = _HP_CACHE.get(key)
    if h is None:
        if cls is opt_sgd_hp:
            h = cls(float(hp[0]), float(hp[1]), int(bool(hp[2])))
        else:
            h = cls(*[float(x) for x in hp])
        if len(_HP_CACHE) > 4096:
            _HP_CACHE.clear()
        _HP_CACHE[key] = h
    return h


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream):
    if stream is None:
        if _raw_stream is not None:  # cheaper than building a torch.cuda.Stream object
            return _raw_stream(torch.cuda.current_device())
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Tree:
    """A flattened tensor tree: numel and leaf offsets (host + device copy).

    ``offsets`` is [0, n_0, n_0+n_1, ..., numel]."""

    def __init__(self, numel=None, offsets=None, device=None):
        if offsets is None:
            offsets = [0, int(numel)]
        self.h_offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        self.numel = int(self.h_offsets[-1])
        self.n_leaves = len(self.h_offsets) - 1
        self.sizes = np.diff(self.h_offsets).tolist()
        self.d_offsets = None
        if device is not None and torch.device(device).type == "cuda":
            self.d_offsets = torch.from_numpy(self.h_offsets).to(device)
        self.c = opt_tree(self.numel, self.n_leaves, self.h_offsets.ctypes.data,
                          _ptr(self.d_offsets))

    @classmethod
    def from_sizes(cls, sizes, device=None):
        off = np.zeros(len(sizes) + 1, dtype=np.int64)
        off[1:] = np.cumsum(np.asarray(sizes, dtype=np.int64))
        return cls(offsets=off, device=device)

    def workspace_bytes(self, per_leaf=False):
        n = lib.opt_workspace_bytes(ctypes.byref(self.c), int(bool(per_leaf)))
        if n == 0:
            raise DiffoptError(OPT_EINVAL, lib.opt_last_error().decode())
        return int(n)

    def workspace(self, device, per_leaf=False):
        """Zero-filled workspace (diffopt.h: zero once; calls leave it zero)."""
        nbytes = self.workspace_bytes(per_leaf)
        return torch.zeros((nbytes + 7) // 8, dtype=torch.float64, device=device)


def _ws(ws):
    if ws is None:
        return None, 0
    return ws.data_ptr(), ws.numel() * ws.element_size()


# ------------------------------------------------------------- entry points
def opt_adam_fwd(tree, step, hp, state_dtype, compute, g, mu, nu, updates, mu_out, nu_out,
                 params=None, params_out=None, stream=None):
    h = _hp(opt_adam_hp, hp)
    _check(lib.opt_adam_fwd(ctypes.byref(tree.c), int(step), ctypes.byref(h), int(state_dtype),
                            int(compute), _ptr(g), _ptr(mu), _ptr(nu), _ptr(updates),
                            _ptr(mu_out), _ptr(nu_out), _ptr(params), _ptr(params_out),
                            _stream(stream)))


def opt_adam_bwd(tree, step, hp, state_dtype, compute, g, mu, nu, d_updates, d_mu_out,
                 d_nu_out, d_g, d_mu, d_nu, d_hp=None, d_hp_leaf=None, workspace=None,
                 stream=None):
    h = _hp(opt_adam_hp, hp)
    wp, wb = _ws(workspace)
    _check(lib.opt_adam_bwd(ctypes.byref(tree.c), int(step), ctypes.byref(h), int(state_dtype),
                            int(compute), _ptr(g), _ptr(mu), _ptr(nu), _ptr(d_updates),
                            _ptr(d_mu_out), _ptr(d_nu_out), _ptr(d_g), _ptr(d_mu), _ptr(d_nu),
                            _ptr(d_hp), _ptr(d_hp_leaf), wp, wb, _stream(stream)))


class Prepared:
    """A C-ABI call with every argument already marshalled (tensor pointers,
    hyper-parameter struct, tree, workspace, stream resolved once): calling
    it costs one ctypes call, for launch-bound small trees (C1) called in a
    loop on fixed buffers. `step` stays a per-call argument (Adam's bias
    correction); everything else, including the stream, is fixed at
    preparation time, so the buffers must outlive the object."""

    __slots__ = ("fn", "head", "tail", "keep")

    def __init__(self, fn, head, tail, keep):
        self.fn, self.head, self.tail, self.keep = fn, head, tail, keep

    def __call__(self, step):
        rc = self.fn(*self.head, int(step), *self.tail)
        if rc != OPT_OK:
            _check(rc)


def prepare_adam_fwd(tree, hp, state_dtype, compute, g, mu, nu, updates, mu_out, nu_out,
                     params=None, params_out=None, stream=None):
    """opt_adam_fwd pre-marshalled: returns f with f(step) == opt_adam_fwd(tree, step, ...)."""
    h = _hp(opt_adam_hp, hp)
    tail = (ctypes.byref(h), int(state_dtype), int(compute), _ptr(g), _ptr(mu), _ptr(nu),
            _ptr(updates), _ptr(mu_out), _ptr(nu_out), _ptr(params), _ptr(params_out),
            _stream(stream))
    return Prepared(lib.opt_adam_fwd, (ctypes.byref(tree.c),), tail, (tree, h))


def prepare_adam_bwd(tree, hp, state_dtype, compute, g, mu, nu, d_updates, d_mu_out, d_nu_out,
                     d_g, d_mu, d_nu, d_hp=None, d_hp_leaf=None, workspace=None, stream=None):
    """opt_adam_bwd pre-marshalled: returns f with f(step) == opt_adam_bwd(tree, step, ...)."""
    h = _hp(opt_adam_hp, hp)
    wp, wb = _ws(workspace)
    tail = (ctypes.byref(h), int(state_dtype), int(compute), _ptr(g), _ptr(mu), _ptr(nu),
            _ptr(d_updates), _ptr(d_mu_out), _ptr(d_nu_out), _ptr(d_g), _ptr(d_mu), _ptr(d_nu),
            _ptr(d_hp), _ptr(d_hp_leaf), wp, wb, _stream(stream))
    return Prepared(lib.opt_adam_bwd, (ctypes.byref(tree.c),), tail, (tree, h, workspace))


def opt_rmsprop_fwd(tree, hp, state_dtype, compute, g, nu, updates, nu_out, params=None,
                    params_out=None, stream=None):
    h = _hp(opt_rmsprop_hp, hp)
    _check(lib.opt_rmsprop_fwd(ctypes.byref(tree.c), ctypes.byref(h), int(state_dtype),
                               int(compute), _ptr(g), _ptr(nu), _ptr(updates), _ptr(nu_out),
                               _ptr(params), _ptr(params_out), _stream(stream)))


def opt_rmsprop_bwd(tree, hp, state_dtype, compute, g, nu, d_updates, d_nu_out, d_g, d_nu,
                    d_hp=None, d_hp_leaf=None, workspace=None, stream=None):
    h = _hp(opt_rmsprop_hp, hp)
    wp, wb = _ws(workspace)
    _check(lib.opt_rmsprop_bwd(ctypes.byref(tree.c), ctypes.byref(h), int(state_dtype),
                               int(compute), _ptr(g), _ptr(nu), _ptr(d_updates), _ptr(d_nu_out),
                               _ptr(d_g), _ptr(d_nu), _ptr(d_hp), _ptr(d_hp_leaf), wp, wb,
                               _stream(stream)))


def opt_sgd_fwd(tree, hp, state_dtype, compute, g, mom, updates, mom_out, params=None,
                params_out=None, stream=None):
    h = _hp(opt_sgd_hp, hp)
    _check(lib.opt_sgd_fwd(ctypes.byref(tree.c), ctypes.byref(h), int(state_dtype), int(compute),
                           _ptr(g), _ptr(mom), _ptr(updates), _ptr(mom_out), _ptr(params),
                           _ptr(params_out), _stream(stream)))


def opt_sgd_bwd(tree, hp, state_dtype, compute, g, mom, d_updates, d_mom_out, d_g, d_mom,
                d_hp=None, d_hp_leaf=None, workspace=None, stream=None):
    h = _hp(opt_sgd_hp, hp)
    wp, wb = _ws(workspace)
    _check(lib.opt_sgd_bwd(ctypes.byref(tree.c), ctypes.byref(h), int(state_dtype), int(compute),
                           _ptr(g), _ptr(mom), _ptr(d_updates), _ptr(d_mom_out), _ptr(d_g),
                           _ptr(d_mom), _ptr(d_hp), _ptr(d_hp_leaf), wp, wb, _stream(stream)))


def opt_apply_updates(numel, params, updates, out, stream=None):
    _check(lib.opt_apply_updates(int(numel), _ptr(params), _ptr(updates), _ptr(out),
                                 _stream(stream)))


lib.opt_sum_rows.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_void_p]
lib.opt_sum_rows.restype = ctypes.c_int
EXPORTS.append("opt_sum_rows")


def opt_sum_rows(rows, cols, inp, out, stream=None):
    _check(lib.opt_sum_rows(int(rows), int(cols), _ptr(inp), _ptr(out), _stream(stream)))


lib.opt_copy_rows.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                              ctypes.c_size_t, ctypes.c_size_t, ctypes.c_void_p]
lib.opt_copy_rows.restype = ctypes.c_int
EXPORTS.append("opt_copy_rows")


def opt_copy_rows(dst, dpitch, src, spitch, width_bytes, rows, stream=None):
    """dst / src: raw addresses (int) or tensors (their data_ptr())."""
    _check(lib.opt_copy_rows(_ptr(dst), int(dpitch), _ptr(src), int(spitch), int(width_bytes),
                             int(rows), _stream(stream)))


def opt_quadratic_grad(numel, a, theta, phi, g, stream=None):
    _check(lib.opt_quadratic_grad(int(numel), _ptr(a), _ptr(theta), _ptr(phi), _ptr(g),
                                  _stream(stream)))


def opt_quadratic_rev(numel, a, g_bar, theta_bar, phi_bar, init_phi=False, stream=None):
    _check(lib.opt_quadratic_rev(int(numel), _ptr(a), _ptr(g_bar), _ptr(theta_bar),
                                 _ptr(phi_bar), int(bool(init_phi)), _stream(stream)))


def opt_launch_count():
    return int(lib.opt_launch_count())


def opt_abi_version():
    return int(lib.opt_abi_version())


# ---------------------------------------------- optimizer variants (NEXT-1)
class opt_ext(ctypes.Structure):
    _fields_ = [("weight_decay", ctypes.c_double), ("decoupled", ctypes.c_int),
                ("maximize", ctypes.c_int), ("lr_leaf", ctypes.c_void_p)]


def _ext(weight_decay=0.0, decoupled=False, maximize=False, lr_leaf=None):
    e = opt_ext(float(weight_decay), int(bool(decoupled)), int(bool(maximize)), _ptr(lr_leaf))
    e._keep = lr_leaf  # the struct holds a raw device pointer: keep the tensor alive with it
    return e


def _setup_ex():
    P, i64, I, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    T, E = ctypes.POINTER(opt_tree), ctypes.POINTER(opt_ext)
    lib.opt_adam_fwd_ex.argtypes = [T, i64, ctypes.POINTER(opt_adam_hp), E, I, I] + [P] * 9
    lib.opt_adam_bwd_ex.argtypes = [T, i64, ctypes.POINTER(opt_adam_hp), E, I, I] + [P] * 14 + [sz, P]
    lib.opt_rmsprop_fwd_ex.argtypes = [T, ctypes.POINTER(opt_rmsprop_hp), E, I, I] + [P] * 7
    lib.opt_rmsprop_bwd_ex.argtypes = [T, ctypes.POINTER(opt_rmsprop_hp), E, I, I] + [P] * 11 + [sz, P]
    lib.opt_sgd_fwd_ex.argtypes = [T, ctypes.POINTER(opt_sgd_hp), E, I, I] + [P] * 7
    lib.opt_sgd_bwd_ex.argtypes = [T, ctypes.POINTER(opt_sgd_hp), E, I, I] + [P] * 11 + [sz, P]
    for name in ("opt_adam_fwd_ex", "opt_adam_bwd_ex", "opt_rmsprop_fwd_ex", "opt_rmsprop_bwd_ex",
                 "opt_sgd_fwd_ex", "opt_sgd_bwd_ex"):
        getattr(lib, name).restype = I


_setup_ex()
EXPORTS += ["opt_adam_fwd_ex", "opt_adam_bwd_ex", "opt_rmsprop_fwd_ex", "opt_rmsprop_bwd_ex",
            "opt_sgd_fwd_ex", "opt_sgd_bwd_ex"]


def opt_adam_fwd_ex(tree, step, hp, ext, state_dtype, compute, g, mu, nu, params, updates,
                    mu_out, nu_out, params_out=None, stream=None):
    _check(lib.opt_adam_fwd_ex(ctypes.byref(tree.c), int(step), ctypes.byref(_hp(opt_adam_hp, hp)),
                               ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g), _ptr(mu),
                               _ptr(nu), _ptr(params), _ptr(updates), _ptr(mu_out), _ptr(nu_out),
                               _ptr(params_out), _stream(stream)))


def opt_adam_bwd_ex(tree, step, hp, ext, state_dtype, compute, g, mu, nu, params, d_updates,
                    d_mu_out, d_nu_out, d_g, d_mu, d_nu, d_params, d_hp=None, d_hp_leaf=None,
                    workspace=None, stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_adam_bwd_ex(ctypes.byref(tree.c), int(step), ctypes.byref(_hp(opt_adam_hp, hp)),
                               ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g), _ptr(mu),
                               _ptr(nu), _ptr(params), _ptr(d_updates), _ptr(d_mu_out),
                               _ptr(d_nu_out), _ptr(d_g), _ptr(d_mu), _ptr(d_nu), _ptr(d_params),
                               _ptr(d_hp), _ptr(d_hp_leaf), wp, wb, _stream(stream)))


def opt_rmsprop_fwd_ex(tree, hp, ext, state_dtype, compute, g, nu, params, updates, nu_out,
                       params_out=None, stream=None):
    _check(lib.opt_rmsprop_fwd_ex(ctypes.byref(tree.c), ctypes.byref(_hp(opt_rmsprop_hp, hp)),
                                  ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g),
                                  _ptr(nu), _ptr(params), _ptr(updates), _ptr(nu_out),
                                  _ptr(params_out), _stream(stream)))


def opt_rmsprop_bwd_ex(tree, hp, ext, state_dtype, compute, g, nu, params, d_updates, d_nu_out,
                       d_g, d_nu, d_params, d_hp=None, d_hp_leaf=None, workspace=None,
                       stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_rmsprop_bwd_ex(ctypes.byref(tree.c), ctypes.byref(_hp(opt_rmsprop_hp, hp)),
                                  ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g),
                                  _ptr(nu), _ptr(params), _ptr(d_updates), _ptr(d_nu_out),
                                  _ptr(d_g), _ptr(d_nu), _ptr(d_params), _ptr(d_hp),
                                  _ptr(d_hp_leaf), wp, wb, _stream(stream)))


def opt_sgd_fwd_ex(tree, hp, ext, state_dtype, compute, g, mom, params, updates, mom_out,
                   params_out=None, stream=None):
    _check(lib.opt_sgd_fwd_ex(ctypes.byref(tree.c), ctypes.byref(_hp(opt_sgd_hp, hp)),
                              ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g),
                              _ptr(mom), _ptr(params), _ptr(updates), _ptr(mom_out),
                              _ptr(params_out), _stream(stream)))


def opt_sgd_bwd_ex(tree, hp, ext, state_dtype, compute, g, mom, params, d_updates, d_mom_out,
                   d_g, d_mom, d_params, d_hp=None, d_hp_leaf=None, workspace=None, stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_sgd_bwd_ex(ctypes.byref(tree.c), ctypes.byref(_hp(opt_sgd_hp, hp)),
                              ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g),
                              _ptr(mom), _ptr(params), _ptr(d_updates), _ptr(d_mom_out),
                              _ptr(d_g), _ptr(d_mom), _ptr(d_params), _ptr(d_hp),
                              _ptr(d_hp_leaf), wp, wb, _stream(stream)))


# ---------------------------------- fused inner-loss glue (NEXT-2, C3)
lib.opt_adam_quad_fwd.argtypes = ([ctypes.POINTER(opt_tree), ctypes.c_int64,
                                   ctypes.POINTER(opt_adam_hp), ctypes.c_int, ctypes.c_int]
                                  + [ctypes.c_void_p] * 10)
lib.opt_adam_quad_rev.argtypes = ([ctypes.POINTER(opt_tree), ctypes.c_int64,
                                   ctypes.POINTER(opt_adam_hp), ctypes.c_int, ctypes.c_int]
                                  + [ctypes.c_void_p] * 10 + [ctypes.c_int, ctypes.c_void_p,
                                                              ctypes.c_void_p, ctypes.c_size_t,
                                                              ctypes.c_void_p])
lib.opt_adam_quad_fwd.restype = ctypes.c_int
lib.opt_adam_quad_rev.restype = ctypes.c_int
EXPORTS += ["opt_adam_quad_fwd", "opt_adam_quad_rev"]


def opt_adam_quad_fwd(tree, step, hp, state_dtype, compute, a, phi, theta, mu, nu, g_out, mu_out,
                      nu_out, theta_out, stream=None):
    _check(lib.opt_adam_quad_fwd(ctypes.byref(tree.c), int(step),
                                 ctypes.byref(_hp(opt_adam_hp, hp)), int(state_dtype),
                                 int(compute), _ptr(a), _ptr(phi), _ptr(theta), _ptr(mu),
                                 _ptr(nu), _ptr(g_out), _ptr(mu_out), _ptr(nu_out),
                                 _ptr(theta_out), _stream(stream)))


def opt_adam_quad_rev(tree, step, hp, state_dtype, compute, a, g, mu, nu, theta_bar, d_mu_out,
                      d_nu_out, d_mu, d_nu, phi_bar, init_phi, d_hp=None, workspace=None,
                      stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_adam_quad_rev(ctypes.byref(tree.c), int(step),
                                 ctypes.byref(_hp(opt_adam_hp, hp)), int(state_dtype),
                                 int(compute), _ptr(a), _ptr(g), _ptr(mu), _ptr(nu),
                                 _ptr(theta_bar), _ptr(d_mu_out), _ptr(d_nu_out), _ptr(d_mu),
                                 _ptr(d_nu), _ptr(phi_bar), int(bool(init_phi)), _ptr(d_hp), wp,
                                 wb, _stream(stream)))


# ------------------------------ RMSProp centred / momentum (NEXT-1, N4)
class opt_rmsprop_cm_hp(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("alpha", ctypes.c_double), ("eps", ctypes.c_double),
                ("momentum", ctypes.c_double), ("centered", ctypes.c_int)]


def _rms_cm_hp(hp):
    lr, alpha, eps, momentum, centered = hp
    return opt_rmsprop_cm_hp(float(lr), float(alpha), float(eps), float(momentum),
                             int(bool(centered)))


_T, _E = ctypes.POINTER(opt_tree), ctypes.POINTER(opt_ext)
lib.opt_rmsprop_cm_fwd.argtypes = [_T, ctypes.POINTER(opt_rmsprop_cm_hp), _E, ctypes.c_int,
                                   ctypes.c_int] + [ctypes.c_void_p] * 11
lib.opt_rmsprop_cm_bwd.argtypes = [_T, ctypes.POINTER(opt_rmsprop_cm_hp), _E, ctypes.c_int,
                                   ctypes.c_int] + [ctypes.c_void_p] * 17 + [ctypes.c_size_t,
                                                                             ctypes.c_void_p]
lib.opt_rmsprop_cm_fwd.restype = ctypes.c_int
lib.opt_rmsprop_cm_bwd.restype = ctypes.c_int
EXPORTS += ["opt_rmsprop_cm_fwd", "opt_rmsprop_cm_bwd"]


def opt_rmsprop_cm_fwd(tree, hp, ext, state_dtype, compute, g, nu, gavg, buf, params, updates,
                       nu_out, gavg_out, buf_out, params_out=None, stream=None):
    """hp = (lr, alpha, eps, momentum, centered)."""
    _check(lib.opt_rmsprop_cm_fwd(ctypes.byref(tree.c), ctypes.byref(_rms_cm_hp(hp)),
                                  ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g),
                                  _ptr(nu), _ptr(gavg), _ptr(buf), _ptr(params), _ptr(updates),
                                  _ptr(nu_out), _ptr(gavg_out), _ptr(buf_out), _ptr(params_out),
                                  _stream(stream)))


def opt_rmsprop_cm_bwd(tree, hp, ext, state_dtype, compute, g, nu, gavg, buf, params, d_updates,
                       d_nu_out, d_gavg_out, d_buf_out, d_g, d_nu, d_gavg, d_buf, d_params,
                       d_hp=None, d_hp_leaf=None, workspace=None, stream=None):
    """d_hp (5 doubles) = (lr, alpha, eps, momentum, weight_decay)."""
    wp, wb = _ws(workspace)
    _check(lib.opt_rmsprop_cm_bwd(ctypes.byref(tree.c), ctypes.byref(_rms_cm_hp(hp)),
                                  ctypes.byref(ext), int(state_dtype), int(compute), _ptr(g),
                                  _ptr(nu), _ptr(gavg), _ptr(buf), _ptr(params), _ptr(d_updates),
                                  _ptr(d_nu_out), _ptr(d_gavg_out), _ptr(d_buf_out), _ptr(d_g),
                                  _ptr(d_nu), _ptr(d_gavg), _ptr(d_buf), _ptr(d_params),
                                  _ptr(d_hp), _ptr(d_hp_leaf), wp, wb, _stream(stream)))


# ------------------------------------------------ zero-order ES (NEXT-3)
lib.opt_es_perturb.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                               ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p]
lib.opt_es_perturb.restype = ctypes.c_int
lib.opt_es_grad.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                            ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
lib.opt_es_grad.restype = ctypes.c_int
EXPORTS += ["opt_es_perturb", "opt_es_grad"]


def es_row_stride(numel):
    return (int(numel) + 3) & ~3


def opt_es_perturb(numel, n_samples, sample0, antithetic, sigma, seed, theta, out, stream=None):
    _check(lib.opt_es_perturb(int(numel), int(n_samples), int(sample0), int(bool(antithetic)),
                              float(sigma), int(seed), _ptr(theta), _ptr(out), _stream(stream)))


def opt_es_grad(numel, n_samples, antithetic, sigma, seed, f_values, grad, stream=None):
    _check(lib.opt_es_grad(int(numel), int(n_samples), int(bool(antithetic)), float(sigma),
                           int(seed), _ptr(f_values), _ptr(grad), _stream(stream)))


# ---------------------------------------- implicit-gradient solvers (NEXT-4)
_P, _i64, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
lib.opt_cg_init.argtypes = [_i64] + [_P] * 6 + [_sz, _P]
lib.opt_cg_alpha.argtypes = [_i64] + [_P] * 4 + [_sz, _P]
lib.opt_cg_update.argtypes = [_i64] + [_P] * 6 + [_sz, _P]
lib.opt_cg_direction.argtypes = [_i64, _P, _P, _P, _P]
lib.opt_neumann_step.argtypes = [_i64, _P, _P, _P, ctypes.c_double, _P]
for _n in ("opt_cg_init", "opt_cg_alpha", "opt_cg_update", "opt_cg_direction",
           "opt_neumann_step"):
    getattr(lib, _n).restype = ctypes.c_int
EXPORTS += ["opt_cg_init", "opt_cg_alpha", "opt_cg_update", "opt_cg_direction",
            "opt_neumann_step"]


def opt_cg_init(n, b, Ax0, r, p, state, workspace, stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_cg_init(int(n), _ptr(b), _ptr(Ax0), _ptr(r), _ptr(p), _ptr(state), wp, wb,
                           _stream(stream)))


def opt_cg_alpha(n, p, Ap, state, workspace, stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_cg_alpha(int(n), _ptr(p), _ptr(Ap), _ptr(state), wp, wb, _stream(stream)))


def opt_cg_update(n, x, r, p, Ap, state, workspace, stream=None):
    wp, wb = _ws(workspace)
    _check(lib.opt_cg_update(int(n), _ptr(x), _ptr(r), _ptr(p), _ptr(Ap), _ptr(state), wp, wb,
                             _stream(stream)))


def opt_cg_direction(n, p, r, state, stream=None):
    _check(lib.opt_cg_direction(int(n), _ptr(p), _ptr(r), _ptr(state), _stream(stream)))


def opt_neumann_step(n, v, Av, x, alpha, stream=None):
    _check(lib.opt_neumann_step(int(n), _ptr(v), _ptr(Av), _ptr(x), float(alpha),
                                _stream(stream)))


# ------------------------- sharded Adam step over peer memory (NEXT-2, fused)
OPT_MAX_PEERS = 8


class opt_peers(ctypes.Structure):
    _fields_ = [("g", ctypes.c_void_p * OPT_MAX_PEERS),
                ("params", ctypes.c_void_p * OPT_MAX_PEERS)]


lib.opt_adam_fwd_peers.argtypes = [ctypes.c_int, ctypes.POINTER(opt_peers), _i64, _i64, _i64,
                                   ctypes.POINTER(opt_adam_hp), ctypes.c_double, _P, _P, _P, _P]
lib.opt_adam_fwd_peers.restype = ctypes.c_int
EXPORTS += ["opt_adam_fwd_peers"]


class opt_peer_flags(ctypes.Structure):
    _fields_ = [("f", ctypes.c_void_p * OPT_MAX_PEERS)]


lib.opt_peer_signal_wait.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(opt_peer_flags), ctypes.c_uint64,
                                     ctypes.c_double, _P, _P]
lib.opt_peer_signal_wait.restype = ctypes.c_int
EXPORTS += ["opt_peer_signal_wait"]
PEER_READY, PEER_DONE = 0, 1


def opt_peer_signal_wait(world, rank, slot, flag_peers, epoch, status, timeout_s=20.0,
                         stream=None):
    """flag_peers: per-rank int64 device tensors of 2*OPT_MAX_PEERS (IPC-mapped
    for remote ranks); status: a device int32 tensor (set to 1 on timeout)."""
    fl = opt_peer_flags()
    for w in range(min(int(world), OPT_MAX_PEERS, len(flag_peers))):
        fl.f[w] = _ptr(flag_peers[w])
    _check(lib.opt_peer_signal_wait(int(world), int(rank), int(slot), ctypes.byref(fl),
                                    int(epoch), float(timeout_s), _ptr(status), _stream(stream)))


def opt_adam_fwd_peers(world, g_peers, params_peers, lo, n_shard, step, hp, grad_scale, mu, nu,
                       params, stream=None):
    """g_peers / params_peers: per-rank tensors (or device pointers) valid in
    this process (CUDA-IPC mapped for remote ranks)."""
    pr = opt_peers()
    for w in range(min(int(world), OPT_MAX_PEERS, len(g_peers))):  # the C side validates world
        pr.g[w] = _ptr(g_peers[w])
        pr.params[w] = _ptr(params_peers[w])
    h = _hp(opt_adam_hp, hp)
    _check(lib.opt_adam_fwd_peers(int(world), ctypes.byref(pr), int(lo), int(n_shard), int(step),
                                  ctypes.byref(h), float(grad_scale), _ptr(mu), _ptr(nu),
                                  _ptr(params), _stream(stream)))
