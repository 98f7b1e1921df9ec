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
    L.net_bnpool_bwd.argtypes = [i64] * 4 + [P] * 9 + [P]
    L.net_bnpool_bwd2.argtypes = [i64] * 4 + [P] * 14 + [P]
    L.net_gemm_nt_workspace_bytes.argtypes = [i64] * 4
    L.net_gemm_nt_workspace_bytes.restype = ctypes.c_size_t
    L.net_gemm_nt.argtypes = [i64] * 4 + [P, P, P, P, ctypes.c_size_t, P]
    for n in ("net_gemm_nt", "net_im2col3x3", "net_col2im3x3", "net_bnpool_fwd", "net_bnpool_bwd",
              "net_bnpool_bwd2", "net_abi_version"):
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


def net_abi_version():
    return int(lib.net_abi_version())


def net_launch_count():
    return int(lib.net_launch_count())
