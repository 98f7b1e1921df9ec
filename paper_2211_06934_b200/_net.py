"""Thin ctypes binding of include/mamlnet.h (argument marshalling only).

Each function has the name of the C entry point it calls and forwards device
pointers, sizes and the current CUDA stream; the arithmetic runs in
libmamlnet.so. There is no CPU fallback: importing this module without the
library raises.
"""
from __future__ import annotations

import ctypes
import os

from ._lib import _ptr, _stream

HERE = os.path.dirname(os.path.abspath(__file__))
# MAMLNET_LIB: load another build of the same ABI (A/B kernel experiments, tools/)
LIB_PATH = os.environ.get("MAMLNET_LIB") or os.path.join(HERE, "libmamlnet.so")
NET_OK = 0

EXPORTS = ["net_im2col3x3", "net_col2im3x3", "net_bnpool_fwd", "net_bnpool_bwd",
           "net_bnpool_bwd2", "net_gemm_nt_workspace_bytes", "net_gemm_nt",
           "net_gemm_nt2_workspace_bytes", "net_gemm_nt2",  "net_bnpool_jvp",
           "net_bnpool_bwd_jvp", "net_bnpool_fwd_cols", "net_bnpool_jvp_cols", "net_fc_xent", "net_fc_xent_jvp", "net_task_sum",
           "net_last_error",
           "net_abi_version", "net_launch_count"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python paper_2211_06934_b200/build.py` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
    L.net_im2col3x3.argtypes = [i64] * 4 + [P, P, P]
    L.net_col2im3x3.argtypes = [i64] * 4 + [P, P, P]
    L.net_bnpool_fwd.argtypes = [i64] * 4 + [P, P, P, D] + [P] * 4 + [P]
    L.net_bnpool_fwd_cols.argtypes = [i64] * 4 + [P, P, P, D] + [P] * 5 + [P]
    L.net_bnpool_jvp_cols.argtypes = [i64] * 4 + [P] * 12 + [P]
    L.net_bnpool_bwd.argtypes = [i64] * 4 + [P] * 9 + [P]
    L.net_bnpool_bwd2.argtypes = [i64] * 4 + [P] * 14 + [P]
    L.net_gemm_nt_workspace_bytes.argtypes = [i64] * 4
    L.net_gemm_nt_workspace_bytes.restype = ctypes.c_size_t
    L.net_gemm_nt.argtypes = [i64] * 4 + [P, P, P, P, ctypes.c_size_t, P]
    C, sz = ctypes.c_int, ctypes.c_size_t
    L.net_gemm_nt2_workspace_bytes.argtypes = [i64] * 4 + [C, C]
    L.net_gemm_nt2_workspace_bytes.restype = sz
    L.net_gemm_nt2.argtypes = [i64] * 4 + [P] * 5 + [C, P, sz, P]
    L.net_bnpool_jvp.argtypes = [i64] * 4 + [P] * 11 + [P]
    L.net_bnpool_bwd_jvp.argtypes = [i64] * 4 + [P] * 16 + [P]
    L.net_fc_xent.argtypes = [i64] * 4 + [P] * 9 + [P]
    L.net_fc_xent_jvp.argtypes = [i64] * 4 + [P] * 10 + [P]
    L.net_task_sum.argtypes = [i64, i64, P, P, P, P, P]
    for n in ("net_gemm_nt2", "net_bnpool_jvp", "net_bnpool_bwd_jvp", "net_bnpool_fwd_cols", "net_bnpool_jvp_cols", "net_fc_xent",
              "net_fc_xent_jvp", "net_task_sum", "net_gemm_nt", "net_im2col3x3", "net_col2im3x3", "net_bnpool_fwd", "net_bnpool_bwd",
              "net_bnpool_bwd2", "net_abi_version", "net_bnpool_fwd_cols", "net_bnpool_jvp_cols"):
        getattr(L, n).restype = ctypes.c_int
    L.net_last_error.restype = ctypes.c_char_p
    L.net_launch_count.restype = i64
    return L


lib = _load()


def _check(rc):
    if rc != NET_OK:
        raise RuntimeError(f"libmamlnet error {rc}: {lib.net_last_error().decode()}")


def net_im2col3x3(G, B, H, W, h, cols, stream=None):
    _check(lib.net_im2col3x3(G, B, H, W, _ptr(h), _ptr(cols), _stream(stream)))


def net_col2im3x3(G, B, H, W, cols, dh, stream=None):
    _check(lib.net_col2im3x3(G, B, H, W, _ptr(cols), _ptr(dh), _stream(stream)))


def net_bnpool_fwd(G, B, H, W, x, gamma, beta, eps, out, code, mean, rstd, stream=None):
    _check(lib.net_bnpool_fwd(G, B, H, W, _ptr(x), _ptr(gamma), _ptr(beta), float(eps), _ptr(out),
                              _ptr(code), _ptr(mean), _ptr(rstd), _stream(stream)))


def net_bnpool_fwd_cols(G, B, H, W, x, gamma, beta, eps, out, code, mean, rstd, cols,
                        stream=None):
    _check(lib.net_bnpool_fwd_cols(G, B, H, W, _ptr(x), _ptr(gamma), _ptr(beta), float(eps),
                                   _ptr(out), _ptr(code), _ptr(mean), _ptr(rstd), _ptr(cols),
                                   _stream(stream)))


def net_bnpool_bwd(G, B, H, W, dp, code, x, gamma, mean, rstd, dx, dgamma, dbeta, stream=None):
    _check(lib.net_bnpool_bwd(G, B, H, W, _ptr(dp), _ptr(code), _ptr(x), _ptr(gamma), _ptr(mean),
                              _ptr(rstd), _ptr(dx), _ptr(dgamma), _ptr(dbeta), _stream(stream)))


def net_bnpool_bwd2(G, B, H, W, gdx, gdgamma, gdbeta, dp, code, x, gamma, mean, rstd, dgamma,
                    dbeta, g_dp, g_x, g_gamma, stream=None):
    _check(lib.net_bnpool_bwd2(G, B, H, W, _ptr(gdx), _ptr(gdgamma), _ptr(gdbeta), _ptr(dp),
                               _ptr(code), _ptr(x), _ptr(gamma), _ptr(mean), _ptr(rstd),
                               _ptr(dgamma), _ptr(dbeta), _ptr(g_dp), _ptr(g_x), _ptr(g_gamma),
                               _stream(stream)))


def net_gemm_nt_workspace_bytes(T, M, P, N):
    return int(lib.net_gemm_nt_workspace_bytes(T, M, P, N))


def net_gemm_nt(T, M, P, N, A, B, C, workspace=None, stream=None):
    wb = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib.net_gemm_nt(T, M, P, N, _ptr(A), _ptr(B), _ptr(C), _ptr(workspace), wb,
                           _stream(stream)))


def net_gemm_nt2_workspace_bytes(T, M, P, N, npairs, accumulate):
    return int(lib.net_gemm_nt2_workspace_bytes(T, M, P, N, npairs, int(bool(accumulate))))


def net_gemm_nt2(T, M, P, N, A, B, A2, B2, C, accumulate, workspace=None, stream=None):
    wb = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib.net_gemm_nt2(T, M, P, N, _ptr(A), _ptr(B), _ptr(A2), _ptr(B2), _ptr(C),
                            int(bool(accumulate)), _ptr(workspace), wb, _stream(stream)))


def net_bnpool_jvp(G, B, H, W, x, xd, gamma, gd, bd, code, mean, rstd, outd, s1, s2, stream=None):
    _check(lib.net_bnpool_jvp(G, B, H, W, _ptr(x), _ptr(xd), _ptr(gamma), _ptr(gd), _ptr(bd),
                              _ptr(code), _ptr(mean), _ptr(rstd), _ptr(outd), _ptr(s1), _ptr(s2),
                              _stream(stream)))


def net_bnpool_jvp_cols(G, B, H, W, x, xd, gamma, gd, bd, code, mean, rstd, outd, s1, s2, cols,
                        stream=None):
    _check(lib.net_bnpool_jvp_cols(G, B, H, W, _ptr(x), _ptr(xd), _ptr(gamma), _ptr(gd),
                                   _ptr(bd), _ptr(code), _ptr(mean), _ptr(rstd), _ptr(outd),
                                   _ptr(s1), _ptr(s2), _ptr(cols), _stream(stream)))


def net_bnpool_bwd_jvp(G, B, H, W, dp, dpd, code, x, xd, gamma, gd, mean, rstd, dgamma, dbeta,
                       s1, s2, dxd, dgd_acc, dbd_acc, stream=None):
    _check(lib.net_bnpool_bwd_jvp(G, B, H, W, _ptr(dp), _ptr(dpd), _ptr(code), _ptr(x), _ptr(xd),
                                  _ptr(gamma), _ptr(gd), _ptr(mean), _ptr(rstd), _ptr(dgamma),
                                  _ptr(dbeta), _ptr(s1), _ptr(s2), _ptr(dxd), _ptr(dgd_acc),
                                  _ptr(dbd_acc), _stream(stream)))


def net_fc_xent(T, B, C, J, h4, Wfc, bfc, labels, loss, prob, dW, db, dh4, stream=None):
    _check(lib.net_fc_xent(T, B, C, J, _ptr(h4), _ptr(Wfc), _ptr(bfc), _ptr(labels), _ptr(loss),
                           _ptr(prob), _ptr(dW), _ptr(db), _ptr(dh4), _stream(stream)))


def net_fc_xent_jvp(T, B, C, J, h4, h4d, Wfc, Wd, bd, labels, prob, dWd_acc, dbd_acc, dh4d,
                    stream=None):
    _check(lib.net_fc_xent_jvp(T, B, C, J, _ptr(h4), _ptr(h4d), _ptr(Wfc), _ptr(Wd), _ptr(bd),
                               _ptr(labels), _ptr(prob), _ptr(dWd_acc), _ptr(dbd_acc), _ptr(dh4d),
                               _stream(stream)))


def net_task_sum(T, n_leaves, h_offsets, d_offsets, x, out, stream=None):
    """h_offsets: a host ctypes int64 array (or CPU int64 tensor); d_offsets: device int64."""
    _check(lib.net_task_sum(T, n_leaves, _ptr(h_offsets), _ptr(d_offsets), _ptr(x), _ptr(out),
                            _stream(stream)))


def net_abi_version():
    return int(lib.net_abi_version())


def net_launch_count():
    return int(lib.net_launch_count())
