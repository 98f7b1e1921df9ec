"""GPU parity of the optimizer variants (weight decay,
AdamW, maximize, per-leaf learning rates) through the *_ex C-ABI entry
points, against the oracle's variant step and VJP (pinned to torch.optim
and complex step in tests/test_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import (DEV, assert_close, assert_leaf_sums_close, assert_sum_close, dev_f32,
                      dev_state, host, leaf_scale, state_host_bits)

pytestmark = pytest.mark.gpu

LEAVES = [5, 4096, 1, 300, 9000, 3, 1027, 64]


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06934_b200 import _lib

    return _lib


def _scale(ct, ref, mag):
    return np.abs(ref) if ct == 2 else np.maximum(np.abs(ref), mag)


def _setup(per_leaf):
    x = synth.state_tree(0xE1, LEAVES)
    n = x["g"].size
    th = synth.normal(0xE1, synth.S_THETA0, n).astype(np.float32)
    off = synth.offsets_of(LEAVES)
    lr_leaf = None
    if per_leaf:
        lr_leaf = (10.0 ** np.linspace(-3, -1, len(LEAVES))).astype(np.float32)
    return x, th, off, lr_leaf


@pytest.mark.parametrize("per_leaf", [False, True])
@pytest.mark.parametrize("decoupled", [False, True])
@pytest.mark.parametrize("maximize", [False, True])
@pytest.mark.parametrize("ct", [1, 2])
def test_adam_variants(L, per_leaf, decoupled, maximize, ct):
    x, th, off, lr_leaf = _setup(per_leaf)
    n = th.size
    wd, t = 0.05, 7
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    tree = L.Tree(offsets=off, device=DEV)
    lrl_dev = None if lr_leaf is None else dev_f32(lr_leaf)
    ext = L._ext(wd, decoupled, maximize, lrl_dev)
    g, m, v, p = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"]), dev_f32(th)
    u, m1, v1, p1 = (torch.empty_like(g) for _ in range(4))
    L.opt_adam_fwd_ex(tree, t, hp, ext, 0, ct, g, m, v, p, u, m1, v1, p1)
    lr_o = None if lr_leaf is None else lr_leaf.astype(np.float64)
    kw = dict(weight_decay=wd, decoupled=decoupled, maximize=maximize, lr_leaf=lr_o, offsets=off)
    ru, rm1, rv1 = oracle.adam_fwd_ex(x["g"], x["m"], x["v"], th, t, *hp, prec=1, **kw)
    mag = oracle.ex_mag("adam", x["g"], (x["m"], x["v"]), th, x["du"], x["dm1"], x["dv1"], t, hp,
                        weight_decay=wd, decoupled=decoupled, maximize=maximize, lr_leaf=lr_o,
                        offsets=off)
    assert_close("u", host(u), ru, scale=_scale(ct, ru, mag["u"]))
    assert_close("m1", host(m1), rm1, scale=_scale(ct, rm1, mag["m1"]))
    assert_close("v1", host(v1), rv1, scale=_scale(ct, rv1, mag["v1"]))
    ref_p = th.astype(np.float64) + ru
    assert_close("params_out", host(p1), ref_p, scale=np.abs(th) + np.abs(ru) + mag["u"])
    du, dm1, dv1 = dev_f32(x["du"]), dev_f32(x["dm1"]), dev_f32(x["dv1"])
    dg, dm, dv, dth = (torch.empty_like(g) for _ in range(4))
    dhp = torch.empty(5, dtype=torch.float64, device=DEV)
    dhl = torch.empty(len(LEAVES) * 5, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd_ex(tree, t, hp, ext, 0, ct, g, m, v, p, du, dm1, dv1, dg, dm, dv, dth, dhp, dhl,
                      tree.workspace(DEV, per_leaf=True))
    r = oracle.adam_vjp_ex(x["g"], x["m"], x["v"], th, x["du"], x["dm1"], x["dv1"], t, *hp, prec=1,
                           **kw)
    for name, got, key in (("dg", dg, "dg"), ("dm", dm, "dm"), ("dv", dv, "dv"),
                           ("dtheta", dth, "dtheta")):
        assert_close(name, host(got), r[key], scale=_scale(ct, r[key], mag[key]))
    # error scales: the variant twins (oracle ex_mag, pinned >= |term| per
    # element in tests/test_oracle.py), summed globally and per leaf
    assert_sum_close("dhp", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
    assert_leaf_sums_close("dhp_leaf", host(dhl).reshape(-1, 5), r["dhp_leaf"],
                           leaf_scale(mag["h"], off))


@pytest.mark.parametrize("kind", ["rmsprop", "sgd", "sgd_nesterov"])
@pytest.mark.parametrize("per_leaf", [False, True])
@pytest.mark.parametrize("maximize", [False, True])
@pytest.mark.parametrize("ct", [1, 2])
def test_rmsprop_sgd_variants(L, kind, per_leaf, maximize, ct):
    x, th, off, lr_leaf = _setup(per_leaf)
    wd = 0.03
    tree = L.Tree(offsets=off, device=DEV)
    lrl_dev = None if lr_leaf is None else dev_f32(lr_leaf)
    ext = L._ext(wd, False, maximize, lrl_dev)
    lr_o = None if lr_leaf is None else lr_leaf.astype(np.float64)
    kw = dict(weight_decay=wd, maximize=maximize, lr_leaf=lr_o, offsets=off)
    st = x["v"] if kind == "rmsprop" else x["m"]
    g, s, p = dev_f32(x["g"]), dev_f32(st), dev_f32(th)
    u, s1, p1 = (torch.empty_like(g) for _ in range(3))
    du, ds1 = dev_f32(x["du"]), dev_f32(x["dm1"])
    dg, ds, dth = (torch.empty_like(g) for _ in range(3))
    if kind == "rmsprop":
        hp = (1e-2, 0.95, 1e-8)
        nh = 4
        L.opt_rmsprop_fwd_ex(tree, hp, ext, 0, ct, g, s, p, u, s1, p1)
        ru, rs1 = oracle.rmsprop_fwd_ex(x["g"], st, th, *hp, prec=1, **kw)
        dhp = torch.empty(nh, dtype=torch.float64, device=DEV)
        dhl = torch.empty(len(LEAVES) * nh, dtype=torch.float64, device=DEV)
        L.opt_rmsprop_bwd_ex(tree, hp, ext, 0, ct, g, s, p, du, ds1, dg, ds, dth, dhp, dhl,
                             tree.workspace(DEV, per_leaf=True))
        r = oracle.rmsprop_vjp_ex(x["g"], st, th, x["du"], x["dm1"], *hp, prec=1, **kw)
        mag = oracle.ex_mag("rmsprop", x["g"], st, th, x["du"], x["dm1"], hp=hp, **kw)
        sk, sref = "dv", "v1"
    else:
        hp = (0.1, 0.9, kind == "sgd_nesterov")
        nh = 3
        L.opt_sgd_fwd_ex(tree, hp, ext, 0, ct, g, s, p, u, s1, p1)
        ru, rs1 = oracle.sgd_fwd_ex(x["g"], st, th, *hp, prec=1, **kw)
        dhp = torch.empty(nh, dtype=torch.float64, device=DEV)
        dhl = torch.empty(len(LEAVES) * nh, dtype=torch.float64, device=DEV)
        L.opt_sgd_bwd_ex(tree, hp, ext, 0, ct, g, s, p, du, ds1, dg, ds, dth, dhp, dhl,
                         tree.workspace(DEV, per_leaf=True))
        r = oracle.sgd_vjp_ex(x["g"], st, th, x["du"], x["dm1"], *hp, prec=1, **kw)
        mag = oracle.ex_mag("sgd", x["g"], st, th, x["du"], x["dm1"], hp=hp, **kw)
        sk, sref = "db", "b1"
    assert_close("u", host(u), ru, scale=_scale(ct, ru, mag["u"]))
    assert_close("state'", host(s1), rs1, scale=_scale(ct, rs1, mag[sref]))
    for name, got in (("dg", dg), (sk, ds), ("dtheta", dth)):
        assert_close(name, host(got), r[name], scale=_scale(ct, r[name], mag[name]))
    assert_sum_close("dhp", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
    assert_leaf_sums_close("dhp_leaf", host(dhl).reshape(-1, nh), r["dhp_leaf"],
                           leaf_scale(mag["h"], off))


def test_variant_with_defaults_equals_base(L):
    """wd = 0, no maximize, lr_leaf = NULL: the *_ex entry points agree with
    the base kernels to within fp32 rounding of the same arithmetic (FMA
    contraction may differ between the two instantiations, so the scale is
    the magnitude twin), and dtheta = 0 exactly."""
    x, th, off, _ = _setup(False)
    tree = L.Tree(offsets=off, device=DEV)
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    g, m, v, p = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"]), dev_f32(th)
    mag = oracle.adam_mag(x["g"], x["m"], x["v"], x["du"], None, None, 3, *hp)
    a = [torch.empty_like(g) for _ in range(3)]
    b = [torch.empty_like(g) for _ in range(3)]
    L.opt_adam_fwd(tree, 3, hp, 0, 1, g, m, v, *a)
    L.opt_adam_fwd_ex(tree, 3, hp, L._ext(), 0, 1, g, m, v, p, *b)
    for x1, x2, k in zip(a, b, ("u", "m1", "v1")):
        assert np.all(np.abs(host(x1) - host(x2)) <= 1e-6 * mag[k] + 1e-30), k
    du = dev_f32(x["du"])
    a = [torch.empty_like(g) for _ in range(3)]
    b = [torch.empty_like(g) for _ in range(4)]
    L.opt_adam_bwd(tree, 3, hp, 0, 1, g, m, v, du, None, None, *a)
    L.opt_adam_bwd_ex(tree, 3, hp, L._ext(), 0, 1, g, m, v, p, du, None, None, *b)
    for x1, x2, k in zip(a, b[:3], ("dg", "dm", "dv")):
        assert np.all(np.abs(host(x1) - host(x2)) <= 1e-6 * mag[k] + 1e-30), k
    assert torch.all(b[3] == 0)
