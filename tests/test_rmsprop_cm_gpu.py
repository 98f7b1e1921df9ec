"""GPU parity of centred / momentum RMSProp (DESIGN.md
reading N4) through opt_rmsprop_cm_fwd / opt_rmsprop_cm_bwd, against the
oracle's step and VJP (pinned to torch.optim.RMSprop and complex step in
tests/test_oracle.py). Tolerance: 1e-5 of the magnitude twin for fp32
arithmetic, of |ref| for fp64 arithmetic (reading Z10)."""
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


CASES = [(c, m, pl, ct, bf) for c in (False, True) for m in (0.0, 0.9) for pl in (False, True)
         for ct in (1, 2) for bf in (False,)]
CASES += [(True, 0.9, False, 1, True), (False, 0.9, True, 1, True)]


@pytest.mark.parametrize("centered,momentum,per_leaf,ct,bf16", CASES)
def test_rmsprop_cm_fwd_bwd(L, centered, momentum, per_leaf, ct, bf16):
    x = synth.rms_cm_tree(0xE7, LEAVES)
    off = synth.offsets_of(LEAVES)
    n = x["g"].size
    lr_leaf = (10.0 ** np.linspace(-3, -1, len(LEAVES))).astype(np.float32) if per_leaf else None
    wd, maximize = 0.02, True
    hp = (1e-2, 0.95, 1e-6, momentum, centered)
    tree = L.Tree(offsets=off, device=DEV)
    lrl_dev = None if lr_leaf is None else dev_f32(lr_leaf)  # must outlive ext (raw pointer)
    ext = L._ext(wd, False, maximize, lrl_dev)
    sd = 1 if bf16 else 0
    sh = {k: state_host_bits(x[k], bf16) for k in ("v", "a", "b")}
    g, p = dev_f32(x["g"]), dev_f32(x["theta"])
    v, a, b = (dev_state(x[k], bf16) for k in ("v", "a", "b"))
    sdt = torch.bfloat16 if bf16 else torch.float32
    u, p1 = torch.empty_like(g), torch.empty_like(g)
    v1, a1, b1 = (torch.empty(n, dtype=sdt, device=DEV) for _ in range(3))
    L.opt_rmsprop_cm_fwd(tree, hp, ext, sd, ct, g, v, a, b, p, u, v1, a1, b1, p1)
    lr_o = None if lr_leaf is None else lr_leaf.astype(np.float64)
    kw = dict(momentum=momentum, centered=centered, weight_decay=wd, maximize=maximize,
              lr_leaf=lr_o, offsets=off, state_bf16=bf16)
    ru, rv1, ra1, rb1 = oracle.rmsprop_cm_fwd(x["g"], sh["v"], sh["a"], sh["b"], x["theta"],
                                              *hp[:3], prec=1, **kw)
    mag = oracle.rmsprop_cm_mag(x["g"], sh["v"], sh["a"], sh["b"], x["theta"], x["du"], x["dv1"],
                                x["da1"], x["db1"], *hp[:3], **kw)
    assert_close("u", host(u), ru, scale=_scale(ct, ru, mag["u"]))
    outs = [("v1", v1, rv1), ("b1", b1, rb1)] + ([("a1", a1, ra1)] if centered else [])
    for name, got, ref in outs:
        if bf16:
            assert_close(name, oracle.bf16_to_f64(host(got)), ref, rtol=1e-2, atol=0,
                         scale=np.maximum(np.abs(ref), 1e-2 * mag[name]))
        else:
            assert_close(name, host(got), ref, scale=_scale(ct, ref, mag[name]))
    assert_close("params_out", host(p1), x["theta"].astype(np.float64) + ru,
                 scale=np.abs(x["theta"]) + np.abs(ru) + mag["u"])

    du, dv1, da1, db1 = (dev_f32(x[k]) for k in ("du", "dv1", "da1", "db1"))
    dg, dv, da, db, dth = (torch.empty_like(g) for _ in range(5))
    dhp = torch.empty(5, dtype=torch.float64, device=DEV)
    dhl = torch.empty(len(LEAVES) * 5, dtype=torch.float64, device=DEV)
    L.opt_rmsprop_cm_bwd(tree, hp, ext, sd, ct, g, v, a, b, p, du, dv1, da1, db1, dg, dv, da, db,
                         dth, dhp, dhl, tree.workspace(DEV, per_leaf=True))
    r = oracle.rmsprop_cm_vjp(x["g"], sh["v"], sh["a"], sh["b"], x["theta"], x["du"], x["dv1"],
                              x["da1"], x["db1"], *hp[:3], prec=1, **kw)
    for name, got in (("dg", dg), ("dv", dv), ("da", da), ("db", db), ("dtheta", dth)):
        assert_close(name, host(got), r[name], scale=_scale(ct, r[name], mag[name]))
    assert_sum_close("dhp", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
    assert_leaf_sums_close("dhp_leaf", host(dhl).reshape(-1, 5), r["dhp_leaf"],
                           leaf_scale(mag["h"], off))


def test_rmsprop_cm_zero_state_and_null_outputs(L):
    """Step 1 (NULL = zero state in), some outputs not requested (NULL out),
    and the not-centred op never touches the gradient-average arrays."""
    x = synth.rms_cm_tree(0xE8, [777, 33])
    n = x["g"].size
    tree = L.Tree(numel=n, device=DEV)
    ext = L._ext()
    g = dev_f32(x["g"])
    u, b1 = torch.empty_like(g), torch.empty_like(g)
    poison = torch.full_like(g, float("nan"))
    hp = (1e-2, 0.99, 1e-8, 0.9, False)
    L.opt_rmsprop_cm_fwd(tree, hp, ext, 0, 1, g, None, poison, None, None, u, None, poison, b1)
    ru, _, _, rb1 = oracle.rmsprop_cm_fwd(x["g"], None, None, None, None, *hp[:3], momentum=0.9,
                                          prec=1)
    mag = oracle.rmsprop_cm_mag(x["g"], None, None, None, None, None, None, None, None, *hp[:3],
                                momentum=0.9)
    assert_close("u", host(u), ru, scale=np.maximum(np.abs(ru), mag["u"]))
    assert_close("b1", host(b1), rb1, scale=np.maximum(np.abs(rb1), mag["b1"]))
    assert torch.isnan(poison).all()  # untouched
    dg = torch.empty_like(g)
    dhp = torch.empty(5, dtype=torch.float64, device=DEV)
    du = dev_f32(x["du"])
    L.opt_rmsprop_cm_bwd(tree, hp, ext, 0, 1, g, None, poison, None, None, du, None, None, None,
                         dg, None, None, None, None, dhp, None, tree.workspace(DEV))
    r = oracle.rmsprop_cm_vjp(x["g"], None, None, None, None, x["du"], None, None, None, *hp[:3],
                              momentum=0.9, prec=1)
    mag = oracle.rmsprop_cm_mag(x["g"], None, None, None, None, x["du"], None, None, None, *hp[:3],
                                momentum=0.9)
    assert_close("dg", host(dg), r["dg"], scale=np.maximum(np.abs(r["dg"]), mag["dg"]))
    assert_sum_close("dhp", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
