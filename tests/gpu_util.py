"""Helpers for the GPU parity tests: run one op through the C ABI on seeded
inputs and compare with the oracle element by element."""
import numpy as np
import torch

import synth

DEV = "cuda:0"
HP_NAMES = {"adam": 4, "rmsprop": 3, "sgd": 2}


def dev_f32(x):
    return None if x is None else torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(DEV)


def dev_state(x, bf16):
    if x is None:
        return None
    if bf16:
        bits = synth.to_bf16_bits(x) if x.dtype != np.uint16 else x
        return torch.from_numpy(bits.view(np.int16)).to(DEV).view(torch.bfloat16)
    return dev_f32(x)


def host(t):
    if t is None:
        return None
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def state_host_bits(x, bf16):
    """The state values the oracle must see (bf16 bit patterns when bf16)."""
    if x is None:
        return None
    return synth.to_bf16_bits(x) if bf16 else x


def tol_fail(x, ref, rtol=1e-5, atol=1e-6, scale=None):
    """Boolean mask of elements outside |x - ref| <= atol + rtol * scale
    (scale defaults to |ref|)."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    sc = np.abs(ref) if scale is None else np.asarray(scale, np.float64)
    return ~(np.abs(x - ref) <= atol + rtol * sc)


def assert_close(name, x, ref, rtol=1e-5, atol=1e-6, scale=None):
    bad = tol_fail(x, ref, rtol, atol, scale)
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        raise AssertionError(f"{name}: {bad.sum()}/{bad.size} outside tol (rtol={rtol}, atol={atol});"
                             f" idx {i.tolist()} got {np.asarray(x)[i].tolist()} "
                             f"want {np.asarray(ref)[i].tolist()}")


def assert_sum_close(name, x, ref, ref_abs, rtol=1e-5, atol=1e-6):
    """Hyper-gradient sums: error scaled by Sigma |term| (reading Z10)."""
    x, ref, ref_abs = (np.asarray(a, np.float64) for a in (x, ref, ref_abs))
    ok = np.abs(x - ref) <= atol + rtol * ref_abs
    if not ok.all():
        raise AssertionError(f"{name}: got {x.tolist()} want {ref.tolist()} (Sigma|t| {ref_abs.tolist()})")


def leaf_scale(h, offsets):
    """Per-leaf error scale of per-leaf hyper-gradient sums: the per-element
    hyper twins h (nh x n, oracle *_mag()['h'], each >= |term| -- pinned in
    tests/test_oracle.py) summed over each leaf's elements -> (n_leaves, nh).
    A leaf is held to its OWN Sigma |term| scale (reading Z10), never the
    whole tree's."""
    h = np.asarray(h, np.float64)
    off = np.asarray(offsets, np.int64)
    return np.stack([h[:, lo:hi].sum(1) for lo, hi in zip(off[:-1], off[1:])])


def assert_leaf_sums_close(name, got, ref, scale, rtol=1e-5, atol=1e-6):
    """Per-leaf sums: |got - ref| <= atol + rtol * (that leaf's scale)."""
    got, ref, scale = (np.asarray(a, np.float64) for a in (got, ref, scale))
    bad = ~(np.abs(got - ref) <= atol + rtol * scale)
    if bad.any():
        i = np.argwhere(bad)[:5]
        raise AssertionError(f"{name}: {int(bad.sum())} per-leaf sums outside tol; (leaf, k) "
                             f"{i.tolist()} got {got[bad][:5].tolist()} want "
                             f"{ref[bad][:5].tolist()} scale {scale[bad][:5].tolist()}")
