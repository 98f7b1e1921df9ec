"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/diffopt.h declares, and host-side validation rejects bad
arguments with the documented status codes before any CUDA call."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__

    __graft_entry__.build()  # (re)builds a stale libdiffopt.so before the package loads it
    from paper_2211_06934_b200 import _lib

    return _lib


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "diffopt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(opt_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_all_exported(L):
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L.lib, s), f"{s} declared in diffopt.h but not exported"
    assert set(syms) == set(L.EXPORTS)


def test_exports_are_extern_c():
    so = os.path.join(ROOT, "paper_2211_06934_b200", "libdiffopt.so")
    out = os.popen(f"nm -D --defined-only {so}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), f"{s} not an unmangled text symbol"


def test_so_contains_sm100a_cubin():
    so = os.path.join(ROOT, "paper_2211_06934_b200", "libdiffopt.so")
    out = os.popen(f"cuobjdump --list-elf {so}").read()
    assert "sm_100a" in out


def _call_adam_fwd(L, tree, step=1, hp=(1e-3, 0.9, 0.999, 1e-8, 0.0), sd=0, ct=0, ptrs=None):
    p = ptrs or [0x10000] * 3
    h = L.opt_adam_hp(*hp)
    return L.lib.opt_adam_fwd(ctypes.byref(tree.c), step, ctypes.byref(h), sd, ct, p[0], p[1],
                              p[2], p[0], p[1], p[2], None, None, 0)


def test_validation_codes(L):
    t = L.Tree(numel=1024)
    assert _call_adam_fwd(L, t, step=0) == L.OPT_EINVAL
    assert "step" in L.lib.opt_last_error().decode()
    assert _call_adam_fwd(L, t, hp=(1e-3, 1.0, 0.999, 1e-8, 0.0)) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, hp=(1e-3, 0.9, -0.1, 1e-8, 0.0)) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, hp=(float("nan"), 0.9, 0.999, 1e-8, 0.0)) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, hp=(1e-3, 0.9, 0.999, -1.0, 0.0)) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, hp=(1e-3, 0.9, 0.999, 1e-8, -1.0)) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, sd=7) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, ct=9) == L.OPT_EINVAL
    assert _call_adam_fwd(L, t, ptrs=[0x10000, 0x10004, 0x10000]) == L.OPT_EALIGN
    # a negative lr is allowed at the ABI (meta-learned lr may cross zero)
    rc = _call_adam_fwd(L, L.Tree(numel=0), hp=(-1e-3, 0.9, 0.999, 1e-8, 0.0))
    assert rc == L.OPT_OK  # numel = 0: nothing to launch


def test_tree_validation(L):
    bad = L.Tree(offsets=[0, 10, 20])
    bad.h_offsets[1] = 30  # non-monotone
    assert _call_adam_fwd(L, bad) == L.OPT_EINVAL
    t = L.Tree(offsets=[0, 10, 20])
    t.c.numel = 21  # offsets[n] != numel
    assert _call_adam_fwd(L, t) == L.OPT_EINVAL
    t = L.Tree(offsets=[1, 10, 20])
    assert _call_adam_fwd(L, t) == L.OPT_EINVAL


def test_workspace_sizes_and_error(L):
    t = L.Tree.from_sizes([5, 4096, 1, 9000])
    small = t.workspace_bytes(False)
    big = t.workspace_bytes(True)
    assert small >= 256 + 8 * 4 * 4096 and big >= small
    many = L.Tree.from_sizes([4096 * 3] * 2000)  # per-leaf: one slot per (chunk, leaf) piece
    n = 4096 * 3 * 2000
    assert many.workspace_bytes(True) >= 256 + 8 * 4 * (n // 256 + 2000 + n // 8192 + 2000)
    h = L.opt_adam_hp(1e-3, 0.9, 0.999, 1e-8, 0.0)
    P = 0x10000
    dhp = 0x20000
    rc = L.lib.opt_adam_bwd(ctypes.byref(t.c), 1, ctypes.byref(h), 0, 0, P, P, P, P, P, P, P, P,
                            P, dhp, None, 0x30000, small - 8, 0)
    assert rc == L.OPT_EWORKSPACE
    # per-leaf output without device offsets
    rc = L.lib.opt_adam_bwd(ctypes.byref(t.c), 1, ctypes.byref(h), 0, 0, P, P, P, P, P, P, P, P,
                            P, dhp, dhp, 0x30000, big, 0)
    assert rc == L.OPT_EINVAL and "d_offsets" in L.lib.opt_last_error().decode()


def test_rmsprop_sgd_validation(L):
    t = L.Tree(numel=16)
    h = L.opt_rmsprop_hp(1e-2, 1.0, 1e-8)
    assert L.lib.opt_rmsprop_fwd(ctypes.byref(t.c), ctypes.byref(h), 0, 0, 0x100, None, 0x100,
                                 None, None, None, 0) == L.OPT_EINVAL
    h = L.opt_sgd_hp(0.1, -0.5, 0)
    assert L.lib.opt_sgd_fwd(ctypes.byref(t.c), ctypes.byref(h), 0, 0, 0x100, None, 0x100, None,
                             None, None, 0) == L.OPT_EINVAL
    assert L.lib.opt_apply_updates(-1, None, None, None, 0) == L.OPT_EINVAL
    assert L.lib.opt_quadratic_grad(8, 0x104, 0x100, 0x100, 0x100, 0) == L.OPT_EALIGN
    # opt_copy_rows (ABI v6 plumbing): host-side validation, nothing enqueued
    assert L.lib.opt_copy_rows(None, 64, 0x100, 64, 32, 2, 0) == L.OPT_EINVAL
    assert L.lib.opt_copy_rows(0x100, 16, 0x200, 64, 32, 2, 0) == L.OPT_EINVAL  # width > dpitch
    assert L.lib.opt_copy_rows(None, 0, None, 0, 0, 5, 0) == L.OPT_OK  # empty rows
    assert L.lib.opt_copy_rows(None, 0, None, 0, 64, 0, 0) == L.OPT_OK  # no rows
    assert L.opt_abi_version() == 6


def test_status_strings(L):
    for c in range(5):
        assert L.lib.opt_status_string(c).decode().startswith("OPT_")


def test_python_api_validation():
    from paper_2211_06934_b200 import adam, rmsprop, sgd

    with pytest.raises(ValueError):
        adam(lr=-1.0)
    with pytest.raises(ValueError):
        adam(b1=1.0)
    with pytest.raises(ValueError):
        rmsprop(alpha=1.5)
    with pytest.raises(ValueError):
        sgd(lr=0.1, momentum=1.0)


def test_variant_validation(L):
    t = L.Tree(numel=64)
    h = L.opt_adam_hp(1e-3, 0.9, 0.999, 1e-8, 0.0)
    P = 0x10000

    def fwd(ext, params=P):
        return L.lib.opt_adam_fwd_ex(ctypes.byref(t.c), 1, ctypes.byref(h), ctypes.byref(ext), 0,
                                     0, P, None, None, params, P, P, P, None, 0)

    assert fwd(L._ext(weight_decay=-1.0)) == L.OPT_EINVAL
    assert fwd(L._ext(weight_decay=0.1), params=None) == L.OPT_EINVAL
    assert fwd(L._ext(lr_leaf=0x20004)) == L.OPT_EALIGN
    # per-leaf lr needs leaves and device offsets
    assert fwd(L._ext(lr_leaf=0x20000)) == L.OPT_EINVAL
    assert "n_leaves" in L.lib.opt_last_error().decode() or "d_offsets" in L.lib.opt_last_error().decode()
    t2 = L.Tree.from_sizes([32, 32])
    rc = L.lib.opt_sgd_bwd_ex(ctypes.byref(t2.c), ctypes.byref(L.opt_sgd_hp(0.1, 0.9, 0)),
                              ctypes.byref(L._ext(lr_leaf=0x20000)), 0, 0, P, P, P, P, P, P, P, P,
                              None, None, None, 0, 0)
    assert rc == L.OPT_EINVAL and "d_offsets" in L.lib.opt_last_error().decode()


def test_rmsprop_cm_validation(L):
    """Centred / momentum RMSProp: invalid hyper-parameters are rejected on
    the host before any launch (no GPU needed)."""
    t = L.Tree(numel=64)
    P = 0x10000
    ext = L._ext()
    for hp in ((1e-2, 1.0, 1e-8, 0.0, 0), (1e-2, 0.9, -1.0, 0.0, 0), (1e-2, 0.9, 1e-8, 1.0, 1),
               (float("nan"), 0.9, 1e-8, 0.5, 1)):
        h = L.opt_rmsprop_cm_hp(*hp)
        rc = L.lib.opt_rmsprop_cm_fwd(ctypes.byref(t.c), ctypes.byref(h), ctypes.byref(ext), 0, 0,
                                      P, P, P, P, P, P, P, P, P, P, 0)
        assert rc == L.OPT_EINVAL
    h = L.opt_rmsprop_cm_hp(1e-2, 0.9, 1e-8, 0.5, 1)
    rc = L.lib.opt_rmsprop_cm_fwd(ctypes.byref(t.c), ctypes.byref(h), ctypes.byref(ext), 0, 0,
                                  P + 4, P, P, P, P, P, P, P, P, P, 0)
    assert rc == L.OPT_EALIGN


def test_peer_sharded_step_validation(L):
    """opt_adam_fwd_peers rejects bad arguments before any CUDA call."""
    h = L.opt_adam_hp(1e-3, 0.9, 0.999, 1e-8, 0.0)
    P = 0x10000

    def call(world, lo=0, n=16, g_null=False, step=1, align_bad=False):
        pr = L.opt_peers()
        for w in range(min(world, L.OPT_MAX_PEERS)):
            pr.g[w] = None if g_null else P + (4 if align_bad else 0)
            pr.params[w] = P
        return L.lib.opt_adam_fwd_peers(world, ctypes.byref(pr), lo, n, step, ctypes.byref(h),
                                        1.0, P, P, P, 0)

    assert call(0) == L.OPT_EINVAL
    assert call(L.OPT_MAX_PEERS + 1) == L.OPT_EINVAL
    assert call(2, lo=2) == L.OPT_EALIGN
    assert call(2, g_null=True) == L.OPT_EINVAL
    assert call(2, align_bad=True) == L.OPT_EALIGN
    assert call(2, step=0) == L.OPT_EINVAL
    assert call(2, n=0) == L.OPT_OK  # empty shard: nothing launched
