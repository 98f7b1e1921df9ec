"""Scalar CPU oracle for the differentiable optimizer step (ctypes wrapper).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs (``cpu_baseline`` and ``--impl reference``)
may import this package. The product package ``paper_2211_06934_b200`` never
imports it and shares no code with it (see ``oracle/oracle.hpp`` header for
the formulas and their citations into PAPER.md / SPEC.md).

Every function takes numpy arrays holding the exact fp32 inputs the GPU path
sees (bf16 state as uint16 bit patterns) and returns float64 arrays.
``prec=1`` evaluates in x87 long double.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SOURCES = [os.path.join(_HERE, "oracle.cpp"), os.path.join(_HERE, "oracle.hpp")]


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2, no fast-math, OpenMP)."""
    newest = max(os.path.getmtime(s) for s in SOURCES)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-fopenmp",
           "-fno-fast-math", "-o", LIB_PATH, SOURCES[0]]
    subprocess.check_call(cmd)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        I = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [I]
        L.oracle_set_num_threads.restype = I
        L.oracle_has_openmp.restype = I
        L.oracle_adam_fwd.argtypes = [i64, i64, P, I, I, P, P, P, P, P, P]
        L.oracle_adam_vjp.argtypes = [i64, i64, P, I, I, P, P, P, P, P, P, P, P, P, P, P, i64, P, P]
        L.oracle_rmsprop_fwd.argtypes = [i64, P, I, I, P, P, P, P]
        L.oracle_rmsprop_vjp.argtypes = [i64, P, I, I, P, P, P, P, P, P, P, P, i64, P, P]
        L.oracle_sgd_fwd.argtypes = [i64, P, I, I, P, P, P, P]
        L.oracle_sgd_vjp.argtypes = [i64, P, I, I, P, P, P, P, P, P, P, P, i64, P, P]
        L.oracle_bf16_rne.argtypes = [i64, P, P]
        L.oracle_sweep_quadratic.argtypes = [I, i64, i64, P, I, P, P, P, P, P, P, P, P, P, P, P]
        L.oracle_adam_fwd_cplx.argtypes = [i64, i64] + [P] * 14
        L.oracle_rmsprop_fwd_cplx.argtypes = [i64] + [P] * 10
        L.oracle_sgd_fwd_cplx.argtypes = [i64, P, P, I] + [P] * 8
        L.oracle_sweep_forward_cplx.argtypes = [I, i64, i64, P, P, I, P, P, P, P, P, P, P]
        _lib = L
    return _lib


def set_num_threads(n: int) -> int:
    """Threads for the chunked loops (0 = all cores). Returns the count used."""
    return lib().oracle_set_num_threads(int(n))


def _p(a):
    return None if a is None else a.ctypes.data


def _f32(a):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=np.float32)


def _state(a, bf16):
    if a is None:
        return None
    if bf16:
        a = np.ascontiguousarray(a)
        assert a.dtype == np.uint16, "bf16 state is passed as uint16 bit patterns"
        return a
    return np.ascontiguousarray(a, dtype=np.float32)


def _out(n, want=True):
    return np.empty(n, dtype=np.float64) if want else None


def _hp(vals):
    return np.ascontiguousarray(vals, dtype=np.float64)


def _offsets(offsets):
    if offsets is None:
        return 0, None
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    return len(off) - 1, off


# ------------------------------------------------------------------ Adam
def adam_fwd(g, m, v, t, lr, b1, b2, eps, eps_root=0.0, state_bf16=False, prec=0):
    """(u, m', v') of one Adam step. m/v None = zero state."""
    g = _f32(g)
    n = g.size
    m, v = _state(m, state_bf16), _state(v, state_bf16)
    hp = _hp([lr, b1, b2, eps, eps_root])
    u, m1, v1 = _out(n), _out(n), _out(n)
    lib().oracle_adam_fwd(n, int(t), _p(hp), int(state_bf16), int(prec), _p(g), _p(m), _p(v),
                          _p(u), _p(m1), _p(v1))
    return u, m1, v1


def adam_vjp(g, m, v, du, dm1, dv1, t, lr, b1, b2, eps, eps_root=0.0, state_bf16=False,
             prec=0, offsets=None):
    """VJP of the Adam step. Returns dict with dg, dm, dv (arrays), dhp (4:
    lr, b1, b2, eps), dhp_abs (Sigma|term|), and dhp_leaf (n_leaves x 4) if
    offsets is given."""
    g = _f32(g)
    n = g.size
    m, v = _state(m, state_bf16), _state(v, state_bf16)
    du, dm1, dv1 = _f32(du), _f32(dm1), _f32(dv1)
    hp = _hp([lr, b1, b2, eps, eps_root])
    dg, dm, dv = _out(n), _out(n), _out(n)
    dhp, dhp_abs = np.zeros(4), np.zeros(4)
    nl, off = _offsets(offsets)
    leaf = np.zeros((nl, 4)) if off is not None else None
    lib().oracle_adam_vjp(n, int(t), _p(hp), int(state_bf16), int(prec), _p(g), _p(m), _p(v),
                          _p(du), _p(dm1), _p(dv1), _p(dg), _p(dm), _p(dv), _p(dhp),
                          _p(dhp_abs), nl, _p(off), _p(leaf))
    return dict(dg=dg, dm=dm, dv=dv, dhp=dhp, dhp_abs=dhp_abs, dhp_leaf=leaf)


# --------------------------------------------------------------- RMSProp
def rmsprop_fwd(g, v, lr, alpha, eps, state_bf16=False, prec=0):
    """(u, v') of one RMSProp step."""
    g = _f32(g)
    n = g.size
    v = _state(v, state_bf16)
    hp = _hp([lr, alpha, eps])
    u, v1 = _out(n), _out(n)
    lib().oracle_rmsprop_fwd(n, _p(hp), int(state_bf16), int(prec), _p(g), _p(v), _p(u), _p(v1))
    return u, v1


def rmsprop_vjp(g, v, du, dv1, lr, alpha, eps, state_bf16=False, prec=0, offsets=None):
    """VJP of the RMSProp step; dhp = (lr, alpha, eps)."""
    g = _f32(g)
    n = g.size
    v = _state(v, state_bf16)
    du, dv1 = _f32(du), _f32(dv1)
    hp = _hp([lr, alpha, eps])
    dg, dv = _out(n), _out(n)
    dhp, dhp_abs = np.zeros(3), np.zeros(3)
    nl, off = _offsets(offsets)
    leaf = np.zeros((nl, 3)) if off is not None else None
    lib().oracle_rmsprop_vjp(n, _p(hp), int(state_bf16), int(prec), _p(g), _p(v), _p(du),
                             _p(dv1), _p(dg), _p(dv), _p(dhp), _p(dhp_abs), nl, _p(off),
                             _p(leaf))
    return dict(dg=dg, dv=dv, dhp=dhp, dhp_abs=dhp_abs, dhp_leaf=leaf)


# ------------------------------------------------------------------- SGD
def sgd_fwd(g, b, lr, momentum, nesterov=False, state_bf16=False, prec=0):
    """(u, b') of one SGD(-momentum) step."""
    g = _f32(g)
    n = g.size
    b = _state(b, state_bf16)
    hp = _hp([lr, momentum, 1.0 if nesterov else 0.0])
    u, b1 = _out(n), _out(n)
    lib().oracle_sgd_fwd(n, _p(hp), int(state_bf16), int(prec), _p(g), _p(b), _p(u), _p(b1))
    return u, b1


def sgd_vjp(g, b, du, db1, lr, momentum, nesterov=False, state_bf16=False, prec=0,
            offsets=None):
    """VJP of the SGD step; dhp = (lr, momentum)."""
    g = _f32(g)
    n = g.size
    b = _state(b, state_bf16)
    du, db1 = _f32(du), _f32(db1)
    hp = _hp([lr, momentum, 1.0 if nesterov else 0.0])
    dg, db = _out(n), _out(n)
    dhp, dhp_abs = np.zeros(2), np.zeros(2)
    nl, off = _offsets(offsets)
    leaf = np.zeros((nl, 2)) if off is not None else None
    lib().oracle_sgd_vjp(n, _p(hp), int(state_bf16), int(prec), _p(g), _p(b), _p(du), _p(db1),
                         _p(dg), _p(db), _p(dhp), _p(dhp_abs), nl, _p(off), _p(leaf))
    return dict(dg=dg, db=db, dhp=dhp, dhp_abs=dhp_abs, dhp_leaf=leaf)


def bf16_rne(x):
    """Round-to-nearest-even of float64 values to bf16 bit patterns (Z9)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.size, dtype=np.uint16)
    lib().oracle_bf16_rne(x.size, _p(x), _p(out))
    return out


def bf16_to_f64(bits):
    """Exact value of bf16 bit patterns."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ------------------------------------------------------ K-step sweep (a9)
KIND = {"adam": 0, "rmsprop": 1, "sgd": 2}


def sweep_quadratic(kind, a, theta0, phi, y, K, hp, prec=0):
    """Row a9: K unrolled steps on L_in = 1/2 sum a (theta-phi)^2 and the
    reverse sweep of L_out = 1/2 ||theta_K - y||^2. ``hp`` is the optimizer's
    hyper-parameter list (adam: lr,b1,b2,eps,eps_root; rmsprop: lr,alpha,eps;
    sgd: lr,momentum,nesterov). Returns dict phi_bar, theta0_bar, hyper_bar(4),
    loss, thetaK."""
    a, theta0, phi, y = _f32(a), _f32(theta0), _f32(phi), _f32(y)
    n = a.size
    hp = _hp(list(hp) + [0.0] * (5 - len(hp)))
    pb, tb, tk, ba = _out(n), _out(n), _out(n), _out(n)
    hyp, habs = np.zeros(4), np.zeros(4)
    loss = np.zeros(1)
    lib().oracle_sweep_quadratic(KIND[kind], n, int(K), _p(hp), int(prec), _p(a), _p(theta0),
                                 _p(phi), _p(y), _p(pb), _p(tb), _p(hyp), _p(loss), _p(tk), _p(ba),
                                 _p(habs))
    return dict(phi_bar=pb, theta0_bar=tb, hyper_bar=hyp, loss=float(loss[0]), thetaK=tk,
                bar_abs=ba, hyper_abs=habs)


# --------------------------------------------------- complex-step helpers
def _cparts(x, n):
    if x is None:
        return None, None
    x = np.broadcast_to(np.asarray(x, dtype=np.complex128), (n,))
    return np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)


def adam_fwd_complex(g, m, v, t, hp):
    """Forward Adam map in complex128 (hp: 5 complex). Returns (u, m', v')."""
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 5)
    gr, gi = _cparts(g, n)
    mr, mi = _cparts(m, n)
    vr, vi = _cparts(v, n)
    outs = [np.empty(n) for _ in range(6)]
    lib().oracle_adam_fwd_cplx(n, int(t), _p(hr), _p(hi), _p(gr), _p(gi), _p(mr), _p(mi),
                               _p(vr), _p(vi), *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(3))


def rmsprop_fwd_complex(g, v, hp):
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 3)
    gr, gi = _cparts(g, n)
    vr, vi = _cparts(v, n)
    outs = [np.empty(n) for _ in range(4)]
    lib().oracle_rmsprop_fwd_cplx(n, _p(hr), _p(hi), _p(gr), _p(gi), _p(vr), _p(vi),
                                  *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(2))


def sgd_fwd_complex(g, b, hp, nesterov=False):
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 2)
    gr, gi = _cparts(g, n)
    br, bi = _cparts(b, n)
    outs = [np.empty(n) for _ in range(4)]
    lib().oracle_sgd_fwd_cplx(n, _p(hr), _p(hi), int(nesterov), _p(gr), _p(gi), _p(br), _p(bi),
                              *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(2))


def sweep_forward_complex(kind, a, theta0, phi, K, hp, nesterov=False):
    """theta_K of the K-step map in complex128 (per element)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.size
    nhp = 5 if kind == "adam" else 3
    hp = list(hp) + [0.0] * (nhp - len(hp))
    hr, hi = _cparts(hp, nhp)
    tr, ti = _cparts(theta0, n)
    pr, pi = _cparts(phi, n)
    o_r, o_i = np.empty(n), np.empty(n)
    lib().oracle_sweep_forward_cplx(KIND[kind], n, int(K), _p(hr), _p(hi), int(nesterov), _p(a),
                                    _p(tr), _p(ti), _p(pr), _p(pi), _p(o_r), _p(o_i))
    return o_r + 1j * o_i


# ------------------------------------------------ magnitude twins (Z10)
def _mag_lib():
    L = lib()
    P, i64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.oracle_adam_mag.argtypes = [i64, i64, P, I, P, P, P, P, P, P, P, P, P]
    L.oracle_rmsprop_mag.argtypes = [i64, P, I, P, P, P, P, P, P, P]
    L.oracle_sgd_mag.argtypes = [i64, P, I, P, P, P, P, P, P, P]
    L.oracle_ex_mag.argtypes = [I, i64, i64, P, P, P, i64, P, I] + [P] * 10
    return L


def adam_mag(g, m, v, du, dm1, dv1, t, lr, b1, b2, eps, eps_root=0.0, state_bf16=False):
    """Magnitude twins (fp32 error scales, reading Z10) of u, m', v', dg, dm,
    dv, of the four hyper-gradient terms per element ('h', 4 x n) and of
    their sums ('dhp', Sigma of the per-element scales)."""
    g = _f32(g)
    n = g.size
    m, v = _state(m, state_bf16), _state(v, state_bf16)
    du, dm1, dv1 = _f32(du), _f32(dm1), _f32(dv1)
    hp = _hp([lr, b1, b2, eps, eps_root])
    out = np.empty(6 * n)
    hs = np.zeros(4)
    he = np.empty(4 * n)
    _mag_lib().oracle_adam_mag(n, int(t), _p(hp), int(state_bf16), _p(g), _p(m), _p(v), _p(du),
                               _p(dm1), _p(dv1), _p(out), _p(hs), _p(he))
    o = out.reshape(6, n)
    return dict(u=o[0], m1=o[1], v1=o[2], dg=o[3], dm=o[4], dv=o[5], dhp=hs, h=he.reshape(4, n))


def rmsprop_mag(g, v, du, dv1, lr, alpha, eps, state_bf16=False):
    g = _f32(g)
    n = g.size
    v = _state(v, state_bf16)
    du, dv1 = _f32(du), _f32(dv1)
    hp = _hp([lr, alpha, eps])
    out = np.empty(4 * n)
    hs = np.zeros(3)
    he = np.empty(3 * n)
    _mag_lib().oracle_rmsprop_mag(n, _p(hp), int(state_bf16), _p(g), _p(v), _p(du), _p(dv1),
                                  _p(out), _p(hs), _p(he))
    o = out.reshape(4, n)
    return dict(u=o[0], v1=o[1], dg=o[2], dv=o[3], dhp=hs, h=he.reshape(3, n))


def sgd_mag(g, b, du, db1, lr, momentum, nesterov=False, state_bf16=False):
    g = _f32(g)
    n = g.size
    b = _state(b, state_bf16)
    du, db1 = _f32(du), _f32(db1)
    hp = _hp([lr, momentum, 1.0 if nesterov else 0.0])
    out = np.empty(4 * n)
    hs = np.zeros(2)
    he = np.empty(2 * n)
    _mag_lib().oracle_sgd_mag(n, _p(hp), int(state_bf16), _p(g), _p(b), _p(du), _p(db1), _p(out),
                              _p(hs), _p(he))
    o = out.reshape(4, n)
    return dict(u=o[0], b1=o[1], dg=o[2], db=o[3], dhp=hs, h=he.reshape(2, n))


# ------------------------------------------- optimizer variants (NEXT-1)
def _ex_lib():
    L = lib()
    if getattr(L, "_ex_ready", False):
        return L
    P, i64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.oracle_adam_fwd_ex.argtypes = [i64, i64, P, P, P, i64, P, I, I, P, P, P, P, P, P, P]
    L.oracle_adam_vjp_ex.argtypes = [i64, i64, P, P, P, i64, P, I, I] + [P] * 14
    L.oracle_rmsprop_fwd_ex.argtypes = [i64, P, P, P, i64, P, I, I, P, P, P, P, P]
    L.oracle_rmsprop_vjp_ex.argtypes = [i64, P, P, P, i64, P, I, I] + [P] * 11
    L.oracle_sgd_fwd_ex.argtypes = [i64, P, P, P, i64, P, I, I, P, P, P, P, P]
    L.oracle_sgd_vjp_ex.argtypes = [i64, P, P, P, i64, P, I, I] + [P] * 11
    L.oracle_adam_fwd_ex_cplx.argtypes = [i64, i64, P, P, D, D, I, I] + [P] * 16
    L.oracle_rmsprop_fwd_ex_cplx.argtypes = [i64, P, P, D, D, I] + [P] * 12
    L.oracle_sgd_fwd_ex_cplx.argtypes = [i64, P, P, I, D, D, I] + [P] * 12
    L._ex_ready = True
    return L


def _ext(weight_decay, decoupled, maximize):
    return _hp([weight_decay, 1.0 if decoupled else 0.0, 1.0 if maximize else 0.0])


def _leaf_args(lr_leaf, offsets):
    if lr_leaf is None and offsets is None:
        return None, 0, None
    nl, off = _offsets(offsets)
    lrl = None if lr_leaf is None else np.ascontiguousarray(lr_leaf, dtype=np.float64)
    return lrl, nl, off


def adam_fwd_ex(g, m, v, theta, t, lr, b1, b2, eps, eps_root=0.0, weight_decay=0.0,
                decoupled=False, maximize=False, lr_leaf=None, offsets=None, state_bf16=False,
                prec=0):
    """Adam step with weight decay (L2 or decoupled/AdamW), maximize and
    per-leaf learning rates (lr_leaf[l] replaces lr on leaf l)."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    m, v = _state(m, state_bf16), _state(v, state_bf16)
    hp = _hp([lr, b1, b2, eps, eps_root])
    ext = _ext(weight_decay, decoupled, maximize)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    u, m1, v1 = _out(n), _out(n), _out(n)
    _ex_lib().oracle_adam_fwd_ex(n, int(t), _p(hp), _p(ext), _p(lrl), nl, _p(off),
                                 int(state_bf16), int(prec), _p(g), _p(m), _p(v), _p(theta),
                                 _p(u), _p(m1), _p(v1))
    return u, m1, v1


def adam_vjp_ex(g, m, v, theta, du, dm1, dv1, t, lr, b1, b2, eps, eps_root=0.0,
                weight_decay=0.0, decoupled=False, maximize=False, lr_leaf=None, offsets=None,
                state_bf16=False, prec=0):
    """VJP of adam_fwd_ex: dg, dm, dv, dtheta (through the update only) and
    dhp = (lr, b1, b2, eps, wd) sums (+ dhp_leaf per leaf when offsets)."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    m, v = _state(m, state_bf16), _state(v, state_bf16)
    du, dm1, dv1 = _f32(du), _f32(dm1), _f32(dv1)
    hp = _hp([lr, b1, b2, eps, eps_root])
    ext = _ext(weight_decay, decoupled, maximize)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    dg, dm, dv, dth = _out(n), _out(n), _out(n), _out(n)
    dhp, dabs = np.zeros(5), np.zeros(5)
    leaf = np.zeros((nl, 5)) if off is not None else None
    _ex_lib().oracle_adam_vjp_ex(n, int(t), _p(hp), _p(ext), _p(lrl), nl, _p(off),
                                 int(state_bf16), int(prec), _p(g), _p(m), _p(v), _p(theta),
                                 _p(du), _p(dm1), _p(dv1), _p(dg), _p(dm), _p(dv), _p(dth),
                                 _p(dhp), _p(dabs), _p(leaf))
    return dict(dg=dg, dm=dm, dv=dv, dtheta=dth, dhp=dhp, dhp_abs=dabs, dhp_leaf=leaf)


def rmsprop_fwd_ex(g, v, theta, lr, alpha, eps, weight_decay=0.0, maximize=False, lr_leaf=None,
                   offsets=None, state_bf16=False, prec=0):
    g, theta = _f32(g), _f32(theta)
    n = g.size
    v = _state(v, state_bf16)
    hp = _hp([lr, alpha, eps])
    ext = _ext(weight_decay, False, maximize)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    u, v1 = _out(n), _out(n)
    _ex_lib().oracle_rmsprop_fwd_ex(n, _p(hp), _p(ext), _p(lrl), nl, _p(off), int(state_bf16),
                                    int(prec), _p(g), _p(v), _p(theta), _p(u), _p(v1))
    return u, v1


def rmsprop_vjp_ex(g, v, theta, du, dv1, lr, alpha, eps, weight_decay=0.0, maximize=False,
                   lr_leaf=None, offsets=None, state_bf16=False, prec=0):
    """dhp = (lr, alpha, eps, wd)."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    v = _state(v, state_bf16)
    du, dv1 = _f32(du), _f32(dv1)
    hp = _hp([lr, alpha, eps])
    ext = _ext(weight_decay, False, maximize)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    dg, dv, dth = _out(n), _out(n), _out(n)
    dhp, dabs = np.zeros(4), np.zeros(4)
    leaf = np.zeros((nl, 4)) if off is not None else None
    _ex_lib().oracle_rmsprop_vjp_ex(n, _p(hp), _p(ext), _p(lrl), nl, _p(off), int(state_bf16),
                                    int(prec), _p(g), _p(v), _p(theta), _p(du), _p(dv1), _p(dg),
                                    _p(dv), _p(dth), _p(dhp), _p(dabs), _p(leaf))
    return dict(dg=dg, dv=dv, dtheta=dth, dhp=dhp, dhp_abs=dabs, dhp_leaf=leaf)


def sgd_fwd_ex(g, b, theta, lr, momentum, nesterov=False, weight_decay=0.0, maximize=False,
               lr_leaf=None, offsets=None, state_bf16=False, prec=0):
    g, theta = _f32(g), _f32(theta)
    n = g.size
    b = _state(b, state_bf16)
    hp = _hp([lr, momentum, 1.0 if nesterov else 0.0])
    ext = _ext(weight_decay, False, maximize)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    u, b1 = _out(n), _out(n)
    _ex_lib().oracle_sgd_fwd_ex(n, _p(hp), _p(ext), _p(lrl), nl, _p(off), int(state_bf16),
                                int(prec), _p(g), _p(b), _p(theta), _p(u), _p(b1))
    return u, b1


def sgd_vjp_ex(g, b, theta, du, db1, lr, momentum, nesterov=False, weight_decay=0.0,
               maximize=False, lr_leaf=None, offsets=None, state_bf16=False, prec=0):
    """dhp = (lr, momentum, wd)."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    b = _state(b, state_bf16)
    du, db1 = _f32(du), _f32(db1)
    hp = _hp([lr, momentum, 1.0 if nesterov else 0.0])
    ext = _ext(weight_decay, False, maximize)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    dg, db, dth = _out(n), _out(n), _out(n)
    dhp, dabs = np.zeros(3), np.zeros(3)
    leaf = np.zeros((nl, 3)) if off is not None else None
    _ex_lib().oracle_sgd_vjp_ex(n, _p(hp), _p(ext), _p(lrl), nl, _p(off), int(state_bf16),
                                int(prec), _p(g), _p(b), _p(theta), _p(du), _p(db1), _p(dg),
                                _p(db), _p(dth), _p(dhp), _p(dabs), _p(leaf))
    return dict(dg=dg, db=db, dtheta=dth, dhp=dhp, dhp_abs=dabs, dhp_leaf=leaf)


def adam_fwd_ex_complex(g, m, v, theta, t, hp, lr_elem, weight_decay=0.0, decoupled=False,
                        maximize=False):
    """Complex forward of adam_fwd_ex; hp[0] unused, lr given per element."""
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 5)
    lr_r, lr_i = _cparts(lr_elem, n)
    gr, gi = _cparts(g, n)
    mr, mi = _cparts(m, n)
    vr, vi = _cparts(v, n)
    tr, ti = _cparts(theta, n)
    wd = complex(weight_decay)
    outs = [np.empty(n) for _ in range(6)]
    _ex_lib().oracle_adam_fwd_ex_cplx(n, int(t), _p(hr), _p(hi), wd.real, wd.imag, int(decoupled),
                                      int(maximize), _p(lr_r), _p(lr_i), _p(gr), _p(gi), _p(mr),
                                      _p(mi), _p(vr), _p(vi), _p(tr), _p(ti),
                                      *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(3))


def rmsprop_fwd_ex_complex(g, v, theta, hp, lr_elem, weight_decay=0.0, maximize=False):
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 3)
    lr_r, lr_i = _cparts(lr_elem, n)
    gr, gi = _cparts(g, n)
    vr, vi = _cparts(v, n)
    tr, ti = _cparts(theta, n)
    wd = complex(weight_decay)
    outs = [np.empty(n) for _ in range(4)]
    _ex_lib().oracle_rmsprop_fwd_ex_cplx(n, _p(hr), _p(hi), wd.real, wd.imag, int(maximize),
                                         _p(lr_r), _p(lr_i), _p(gr), _p(gi), _p(vr), _p(vi),
                                         _p(tr), _p(ti), *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(2))


def sgd_fwd_ex_complex(g, b, theta, hp, lr_elem, nesterov=False, weight_decay=0.0,
                       maximize=False):
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 2)
    lr_r, lr_i = _cparts(lr_elem, n)
    gr, gi = _cparts(g, n)
    br, bi = _cparts(b, n)
    tr, ti = _cparts(theta, n)
    wd = complex(weight_decay)
    outs = [np.empty(n) for _ in range(4)]
    _ex_lib().oracle_sgd_fwd_ex_cplx(n, _p(hr), _p(hi), int(nesterov), wd.real, wd.imag,
                                     int(maximize), _p(lr_r), _p(lr_i), _p(gr), _p(gi), _p(br),
                                     _p(bi), _p(tr), _p(ti), *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(2))


# ------------------------- RMSProp centred / momentum (NEXT-1, reading N4)
def _cm_lib():
    L = _ex_lib()
    if getattr(L, "_cm_ready", False):
        return L
    P, i64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.oracle_rmsprop_cm_fwd.argtypes = [i64, P, P, P, i64, P, I, I] + [P] * 9
    L.oracle_rmsprop_cm_vjp.argtypes = [i64, P, P, P, i64, P, I, I] + [P] * 17
    L.oracle_rmsprop_cm_mag.argtypes = [i64, P, P, P, i64, P, I] + [P] * 12
    L.oracle_rmsprop_cm_fwd_cplx.argtypes = [i64, P, P, I, D, D, I] + [P] * 20
    L._cm_ready = True
    return L


def _cm_hp(lr, alpha, eps, momentum, centered):
    return _hp([lr, alpha, eps, momentum, 1.0 if centered else 0.0])


def rmsprop_cm_fwd(g, v, a, b, theta, lr, alpha, eps, momentum=0.0, centered=False,
                   weight_decay=0.0, maximize=False, lr_leaf=None, offsets=None,
                   state_bf16=False, prec=0):
    """Centred and/or momentum RMSProp step (torch.optim.RMSprop semantics):
    (u, v', a', b'); v, a (gradient average), b (momentum buffer) None = 0."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    v, a, b = (_state(x, state_bf16) for x in (v, a, b))
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    u, v1, a1, b1 = _out(n), _out(n), _out(n), _out(n)
    _cm_lib().oracle_rmsprop_cm_fwd(n, _p(_cm_hp(lr, alpha, eps, momentum, centered)),
                                    _p(_ext(weight_decay, False, maximize)), _p(lrl), nl,
                                    _p(off), int(state_bf16), int(prec), _p(g), _p(v), _p(a),
                                    _p(b), _p(theta), _p(u), _p(v1), _p(a1), _p(b1))
    return u, v1, a1, b1


def rmsprop_cm_vjp(g, v, a, b, theta, du, dv1, da1, db1, lr, alpha, eps, momentum=0.0,
                   centered=False, weight_decay=0.0, maximize=False, lr_leaf=None, offsets=None,
                   state_bf16=False, prec=0):
    """VJP of rmsprop_cm_fwd: dg, dv, da, db, dtheta (through the update) and
    dhp = (lr, alpha, eps, momentum, wd) (+ dhp_abs, dhp_leaf)."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    v, a, b = (_state(x, state_bf16) for x in (v, a, b))
    du, dv1, da1, db1 = _f32(du), _f32(dv1), _f32(da1), _f32(db1)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    dg, dv, da, db, dth = (_out(n) for _ in range(5))
    dhp, dabs = np.zeros(5), np.zeros(5)
    leaf = np.zeros((nl, 5)) if off is not None else None
    _cm_lib().oracle_rmsprop_cm_vjp(n, _p(_cm_hp(lr, alpha, eps, momentum, centered)),
                                    _p(_ext(weight_decay, False, maximize)), _p(lrl), nl,
                                    _p(off), int(state_bf16), int(prec), _p(g), _p(v), _p(a),
                                    _p(b), _p(theta), _p(du), _p(dv1), _p(da1), _p(db1), _p(dg),
                                    _p(dv), _p(da), _p(db), _p(dth), _p(dhp), _p(dabs), _p(leaf))
    return dict(dg=dg, dv=dv, da=da, db=db, dtheta=dth, dhp=dhp, dhp_abs=dabs, dhp_leaf=leaf)


def rmsprop_cm_mag(g, v, a, b, theta, du, dv1, da1, db1, lr, alpha, eps, momentum=0.0,
                   centered=False, weight_decay=0.0, maximize=False, lr_leaf=None, offsets=None,
                   state_bf16=False):
    """Magnitude twins (Z10) of every output and of the 5 hyper sums."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    v, a, b = (_state(x, state_bf16) for x in (v, a, b))
    du, dv1, da1, db1 = _f32(du), _f32(dv1), _f32(da1), _f32(db1)
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    out = np.empty(9 * n)
    hs = np.zeros(5)
    he = np.empty(5 * n)
    _cm_lib().oracle_rmsprop_cm_mag(n, _p(_cm_hp(lr, alpha, eps, momentum, centered)),
                                    _p(_ext(weight_decay, False, maximize)), _p(lrl), nl,
                                    _p(off), int(state_bf16), _p(g), _p(v), _p(a), _p(b),
                                    _p(theta), _p(du), _p(dv1), _p(da1), _p(db1), _p(out),
                                    _p(hs), _p(he))
    o = out.reshape(9, n)
    keys = ("u", "v1", "a1", "b1", "dg", "dv", "da", "db", "dtheta")
    r = {k: o[i] for i, k in enumerate(keys)}
    r["dhp"] = hs
    r["h"] = he.reshape(5, n)
    return r


def rmsprop_cm_fwd_complex(g, v, a, b, theta, hp, lr_elem, centered=False, weight_decay=0.0,
                           maximize=False):
    """Complex forward of rmsprop_cm_fwd (complex-step pins): hp = (lr
    unused, alpha, eps, momentum), complex; lr given per element."""
    g = np.asarray(g, dtype=np.complex128)
    n = g.size
    hr, hi = _cparts(hp, 4)
    parts = [_cparts(x, n) for x in (lr_elem, g, v, a, b, theta)]
    flat = [q for pr in parts for q in pr]
    wd = complex(weight_decay)
    outs = [np.empty(n) for _ in range(8)]
    _cm_lib().oracle_rmsprop_cm_fwd_cplx(n, _p(hr), _p(hi), int(centered), wd.real, wd.imag,
                                         int(maximize), *[_p(q) for q in flat],
                                         *[_p(o) for o in outs])
    return tuple(outs[2 * k] + 1j * outs[2 * k + 1] for k in range(4))


def ex_mag(kind, g, state, theta, du, ds1, dv1=None, t=1, hp=(), weight_decay=0.0,
           decoupled=False, maximize=False, lr_leaf=None, offsets=None, state_bf16=False):
    """Magnitude twins (Z10) of the variant outputs (oracle.hpp ``ex_mag``):
    the base twins at the decayed gradient (its value in denominators, the
    magnitude |g| + wd |theta| in numerators) with each element's lr, plus
    the weight-decay terms. ``state`` is (m, v) for adam, the single state
    array otherwise; ``hp`` the base hyper-parameters. Returns the output
    twins keyed like the base twins plus 'dtheta', the hyper twins per
    element ('h', nh x n: adam lr, b1, b2, eps, wd; rmsprop lr, alpha, eps,
    wd; sgd lr, mu, wd) and their sums ('dhp')."""
    g, theta = _f32(g), _f32(theta)
    n = g.size
    k = {"adam": 0, "rmsprop": 1, "sgd": 2}[kind]
    s0, s1 = (state if kind == "adam" else (state, None))
    s0, s1 = _state(s0, state_bf16), _state(s1, state_bf16)
    du, ds1_, dv1_ = _f32(du), _f32(ds1), _f32(dv1)
    if kind == "adam":
        hv = _hp(list(hp) + [0.0] * (5 - len(hp)))
    else:
        hv = _hp([hp[0], hp[1], float(hp[2]) if len(hp) > 2 else 0.0, 0.0, 0.0])
    lrl, nl, off = _leaf_args(lr_leaf, offsets)
    nh = (5, 4, 3)[k]
    out = np.empty(7 * n)
    hs = np.zeros(5)
    he = np.empty(nh * n)
    _mag_lib().oracle_ex_mag(k, n, int(t), _p(hv), _p(_ext(weight_decay, decoupled, maximize)),
                             _p(lrl), nl, _p(off), int(state_bf16), _p(g), _p(s0), _p(s1),
                             _p(theta), _p(du), _p(ds1_), _p(dv1_), _p(out), _p(hs), _p(he))
    o = out.reshape(7, n)
    names = {"adam": ("u", "m1", "v1", "dg", "dm", "dv"), "rmsprop": ("u", "v1", None, "dg", "dv", None),
             "sgd": ("u", "b1", None, "dg", "db", None)}[kind]
    r = {nm: o[i] for i, nm in enumerate(names) if nm is not None}
    r["dtheta"] = o[6]
    r["h"] = he.reshape(nh, n)
    r["dhp"] = hs[:nh]
    return r


# ------------------------------------------------ zero-order ES (NEXT-3)
def _es_lib():
    L = lib()
    if not getattr(L, "_es_ready", False):
        P, i64, I, D, U = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                           ctypes.c_uint64)
        L.oracle_es_noise.argtypes = [i64, i64, U, P]
        L.oracle_es_perturb.argtypes = [i64, i64, I, D, U, P, P]
        L.oracle_es_grad.argtypes = [i64, i64, I, D, U, P, P, P]
        L._es_ready = True
    return L


def es_noise(numel, n_samples, seed):
    z = np.empty((n_samples, numel))
    _es_lib().oracle_es_noise(int(numel), int(n_samples), int(seed), _p(z))
    return z


def es_perturb(theta, n_samples, sigma, seed, antithetic=True):
    """Rows theta + sigma z_i (antithetic: +/- interleaved), float64."""
    theta = _f32(theta)
    reps = 2 if antithetic else 1
    out = np.empty((n_samples * reps, theta.size))
    _es_lib().oracle_es_perturb(theta.size, int(n_samples), int(antithetic), float(sigma),
                                int(seed), _p(theta), _p(out))
    return out


def es_grad(f_values, numel, n_samples, sigma, seed, antithetic=True):
    """ES gradient estimate from f at the perturbed rows; returns
    (g, g_abs) where g_abs = sum_i |term_ij| (tolerance scale)."""
    f = np.ascontiguousarray(f_values, dtype=np.float64)
    g, ga = np.empty(numel), np.empty(numel)
    _es_lib().oracle_es_grad(int(numel), int(n_samples), int(antithetic), float(sigma),
                             int(seed), _p(f), _p(g), _p(ga))
    return g, ga


# ---------------------------------------- implicit gradients (NEXT-4)
def _ig_lib():
    L = lib()
    if not getattr(L, "_ig_ready", False):
        P, i64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
        L.oracle_cg_iter.argtypes = [i64, P, P, P, P, D, P, P, P, P]
        L.oracle_cg_dense.argtypes = [i64, P, P, i64, P]
        L.oracle_neumann_dense.argtypes = [i64, P, P, i64, D, P]
        L._ig_ready = True
    return L


def cg_iter(x, r, p, Ap, rr):
    """One textbook CG iteration (iMAML); returns x', r', p' and
    dict(pAp, alpha, rr_new, beta)."""
    x, r, p, Ap = (_f32(a) for a in (x, r, p, Ap))
    n = x.size
    x1, r1, p1, s = _out(n), _out(n), _out(n), np.zeros(4)
    _ig_lib().oracle_cg_iter(n, _p(x), _p(r), _p(p), _p(Ap), float(rr), _p(x1), _p(r1), _p(p1),
                             _p(s))
    return x1, r1, p1, dict(pAp=s[0], alpha=s[1], rr_new=s[2], beta=s[3])


def cg_dense(A, b, iters):
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(b.size)
    _ig_lib().oracle_cg_dense(b.size, _p(A), _p(b), int(iters), _p(x))
    return x


def neumann_dense(A, b, K, alpha):
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(b.size)
    _ig_lib().oracle_neumann_dense(b.size, _p(A), _p(b), int(K), float(alpha), _p(x))
    return x
