"""GPU parity: every CUDA op, called through the C ABI, against the oracle on
the same seeded inputs (bar: |x - ref| <= 1e-6 + 1e-5 |ref| for fp32 outputs,
1e-2 relative for bf16-stored state, hyper-gradient sums scaled by
Sigma|term|)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import (DEV, assert_close, assert_leaf_sums_close, assert_sum_close, dev_f32,
                      dev_state, host, leaf_scale, state_host_bits)

pytestmark = pytest.mark.gpu

LEAVES_RAGGED = [5, 4096, 1, 300, 9000, 3, 1027, 64]   # 14,560 elements: tiles + ragged tails


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06934_b200 import _lib

    return _lib


def _inputs(case):
    if case == "c1":
        x = synth.c1_inputs()
        return x, None, 1
    x = synth.state_tree(0xA1, LEAVES_RAGGED)
    return x, synth.offsets_of(LEAVES_RAGGED), 10


COMPUTES = [1, 2]  # OPT_COMPUTE_F32, OPT_COMPUTE_F64


def _scale(ct, ref, mag):
    """Error scale of the 1e-5 relative bar: |ref| for fp64 arithmetic;
    the magnitude twin (reduced-form tree over |.|, reading Z10) for fp32
    arithmetic, whose rounding is charged only for input conditioning."""
    return np.abs(ref) if ct == 2 else np.maximum(np.abs(ref), mag)


def check(name, got, ref, mag, ct):
    assert_close(name, got, ref, scale=_scale(ct, ref, mag))


# ------------------------------------------------------------------ Adam
@pytest.mark.parametrize("case", ["c1", "ragged"])
@pytest.mark.parametrize("lr", [1e-3, 1.0])
@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("ct", COMPUTES)
def test_adam_fwd_bwd(L, case, lr, bf16, ct):
    x, off, t = _inputs(case)
    hp = (lr, 0.9, 0.999, 1e-8, 0.0)
    n = x["g"].size
    tree = L.Tree(offsets=off if off is not None else [0, n], device=DEV)
    m_h, v_h = state_host_bits(x["m"], bf16), state_host_bits(x["v"], bf16)
    g, m, v = dev_f32(x["g"]), dev_state(x["m"], bf16), dev_state(x["v"], bf16)
    sd = 1 if bf16 else 0
    u = torch.empty_like(g)
    sdt = torch.bfloat16 if bf16 else torch.float32
    m1, v1 = torch.empty(n, dtype=sdt, device=DEV), torch.empty(n, dtype=sdt, device=DEV)
    L.opt_adam_fwd(tree, t, hp, sd, ct, g, m, v, u, m1, v1)
    ru, rm1, rv1 = oracle.adam_fwd(x["g"], m_h, v_h, t, *hp, state_bf16=bf16, prec=1)
    mag = oracle.adam_mag(x["g"], m_h, v_h, x["du"], x["dm1"], x["dv1"], t, *hp, state_bf16=bf16)
    check("u", host(u), ru, mag["u"], ct)
    if bf16:
        assert_close("m1", oracle.bf16_to_f64(host(m1)), rm1, rtol=1e-2, atol=0)
        assert_close("v1", oracle.bf16_to_f64(host(v1)), rv1, rtol=1e-2, atol=0)
    else:
        check("m1", host(m1), rm1, mag["m1"], ct)
        check("v1", host(v1), rv1, mag["v1"], ct)
    # backward with all cotangents + global and per-leaf hyper-gradients
    du, dm1, dv1 = dev_f32(x["du"]), dev_f32(x["dm1"]), dev_f32(x["dv1"])
    dg, dm, dv = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    dhl = torch.empty(tree.n_leaves * 4, dtype=torch.float64, device=DEV)
    ws = tree.workspace(DEV, per_leaf=True)
    L.opt_adam_bwd(tree, t, hp, sd, ct, g, m, v, du, dm1, dv1, dg, dm, dv, dhp, dhl, ws)
    r = oracle.adam_vjp(x["g"], m_h, v_h, x["du"], x["dm1"], x["dv1"], t, *hp, state_bf16=bf16,
                        prec=1, offsets=tree.h_offsets)
    check("dg", host(dg), r["dg"], mag["dg"], ct)
    check("dm", host(dm), r["dm"], mag["dm"], ct)
    check("dv", host(dv), r["dv"], mag["dv"], ct)
    hs = np.maximum(r["dhp_abs"], mag["dhp"])
    assert_sum_close("dhp", host(dhp), r["dhp"], hs)
    assert np.allclose(host(dhl).reshape(-1, 4).sum(0), host(dhp), rtol=1e-12,
                       atol=1e-12 * hs.max())
    assert_leaf_sums_close("dhp_leaf", host(dhl).reshape(-1, 4), r["dhp_leaf"],
                           leaf_scale(mag["h"], tree.h_offsets))
    # global-only reduction path gives the same sums
    dhp2 = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, t, hp, sd, ct, g, m, v, du, dm1, dv1, None, None, None, dhp2, None, ws)
    assert_sum_close("dhp(uniform)", host(dhp2), r["dhp"], hs)


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("ct", COMPUTES)
def test_rmsprop_fwd_bwd(L, bf16, ct):
    x, off, t = _inputs("ragged")
    hp = (1e-2, 0.99, 1e-8)
    n = x["g"].size
    tree = L.Tree(offsets=off, device=DEV)
    v_h = state_host_bits(x["v"], bf16)
    g, v = dev_f32(x["g"]), dev_state(x["v"], bf16)
    sd = 1 if bf16 else 0
    u = torch.empty_like(g)
    v1 = torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device=DEV)
    L.opt_rmsprop_fwd(tree, hp, sd, ct, g, v, u, v1)
    ru, rv1 = oracle.rmsprop_fwd(x["g"], v_h, *hp, state_bf16=bf16, prec=1)
    mag = oracle.rmsprop_mag(x["g"], v_h, x["du"], x["dv1"], *hp, state_bf16=bf16)
    check("u", host(u), ru, mag["u"], ct)
    if bf16:
        assert_close("v1", oracle.bf16_to_f64(host(v1)), rv1, rtol=1e-2, atol=0)
    else:
        check("v1", host(v1), rv1, mag["v1"], ct)
    du, dv1 = dev_f32(x["du"]), dev_f32(x["dv1"])
    dg, dv = torch.empty_like(g), torch.empty_like(g)
    dhp = torch.empty(3, dtype=torch.float64, device=DEV)
    dhl = torch.empty(tree.n_leaves * 3, dtype=torch.float64, device=DEV)
    ws = tree.workspace(DEV, per_leaf=True)
    L.opt_rmsprop_bwd(tree, hp, sd, ct, g, v, du, dv1, dg, dv, dhp, dhl, ws)
    r = oracle.rmsprop_vjp(x["g"], v_h, x["du"], x["dv1"], *hp, state_bf16=bf16, prec=1,
                           offsets=tree.h_offsets)
    check("dg", host(dg), r["dg"], mag["dg"], ct)
    check("dv", host(dv), r["dv"], mag["dv"], ct)
    hs = np.maximum(r["dhp_abs"], mag["dhp"])
    assert_sum_close("dhp", host(dhp), r["dhp"], hs)
    assert_leaf_sums_close("dhp_leaf", host(dhl).reshape(-1, 3), r["dhp_leaf"],
                           leaf_scale(mag["h"], tree.h_offsets))


@pytest.mark.parametrize("nesterov", [False, True])
@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("ct", COMPUTES)
def test_sgd_fwd_bwd(L, nesterov, bf16, ct):
    x, off, t = _inputs("ragged")
    hp = (0.1, 0.9, nesterov)
    n = x["g"].size
    tree = L.Tree(offsets=off, device=DEV)
    b_h = state_host_bits(x["m"], bf16)
    g, b = dev_f32(x["g"]), dev_state(x["m"], bf16)
    sd = 1 if bf16 else 0
    u = torch.empty_like(g)
    b1 = torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device=DEV)
    L.opt_sgd_fwd(tree, hp, sd, ct, g, b, u, b1)
    ru, rb1 = oracle.sgd_fwd(x["g"], b_h, *hp, state_bf16=bf16, prec=1)
    mag = oracle.sgd_mag(x["g"], b_h, x["du"], x["dm1"], *hp, state_bf16=bf16)
    check("u", host(u), ru, mag["u"], ct)
    if bf16:
        assert_close("b1", oracle.bf16_to_f64(host(b1)), rb1, rtol=1e-2, atol=0)
    else:
        check("b1", host(b1), rb1, mag["b1"], ct)
    du, db1 = dev_f32(x["du"]), dev_f32(x["dm1"])
    dg, db = torch.empty_like(g), torch.empty_like(g)
    dhp = torch.empty(2, dtype=torch.float64, device=DEV)
    ws = tree.workspace(DEV)
    L.opt_sgd_bwd(tree, hp, sd, ct, g, b, du, db1, dg, db, dhp, None, ws)
    r = oracle.sgd_vjp(x["g"], b_h, x["du"], x["dm1"], *hp, state_bf16=bf16, prec=1)
    check("dg", host(dg), r["dg"], mag["dg"], ct)
    check("db", host(db), r["db"], mag["db"], ct)
    assert_sum_close("dhp", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))


# --------------------------------------------------- ABI conventions
def test_null_cotangent_is_zero_bitwise(L):
    x, off, t = _inputs("ragged")
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.0)
    tree = L.Tree(offsets=off, device=DEV)
    g, m, v, du = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"]), dev_f32(x["du"])
    z = torch.zeros_like(g)
    outs = []
    for dm1, dv1 in ((None, None), (z, z)):
        dg, dm, dv = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
        dhp = torch.empty(4, dtype=torch.float64, device=DEV)
        L.opt_adam_bwd(tree, t, hp, 0, 0, g, m, v, du, dm1, dv1, dg, dm, dv, dhp, None,
                       tree.workspace(DEV))
        outs.append([host(a) for a in (dg, dm, dv, dhp)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


def test_inplace_aliasing_matches_out_of_place(L):
    x, off, t = _inputs("ragged")
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.0)
    tree = L.Tree(offsets=off, device=DEV)
    g, m, v = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"])
    u, m1, v1 = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    L.opt_adam_fwd(tree, t, hp, 0, 0, g, m, v, u, m1, v1)
    g2, m2, v2 = g.clone(), m.clone(), v.clone()
    L.opt_adam_fwd(tree, t, hp, 0, 0, g2, m2, v2, g2, m2, v2)  # updates == g, mu_out == mu ...
    for a, b in ((u, g2), (m1, m2), (v1, v2)):
        assert torch.equal(a, b)


def test_fused_apply_equals_params_plus_update(L):
    x, off, t = _inputs("ragged")
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    tree = L.Tree(offsets=off, device=DEV)
    g, m, v = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"])
    p = dev_f32(x["du"])
    u, m1, v1 = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    p_out = torch.empty_like(g)
    L.opt_adam_fwd(tree, t, hp, 0, 2, g, m, v, u, m1, v1, p, p_out)
    ru, _, _ = oracle.adam_fwd(x["g"], x["m"], x["v"], t, *hp, prec=1)
    ref = x["du"].astype(np.float64) + ru
    assert_close("params_out", host(p_out), ref, scale=np.abs(x["du"]) + np.abs(ru))
    out2 = torch.empty_like(g)
    L.opt_apply_updates(g.numel(), p, u, out2)
    np.testing.assert_allclose(host(out2), x["du"].astype(np.float64) + host(u).astype(np.float64),
                               rtol=1e-7, atol=1e-7)


def test_hyper_gradients_deterministic(L):
    x = synth.state_tree(0xD, [1 << 20, 3333])
    tree = L.Tree(offsets=synth.offsets_of([1 << 20, 3333]), device=DEV)
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.0)
    args = [dev_f32(x[k]) for k in ("g", "m", "v", "du", "dm1", "dv1")]
    ws = tree.workspace(DEV, per_leaf=True)
    res = []
    for _ in range(3):
        dhp = torch.empty(4, dtype=torch.float64, device=DEV)
        dhl = torch.empty(8, dtype=torch.float64, device=DEV)
        L.opt_adam_bwd(tree, 7, hp, 0, 0, *args, None, None, None, dhp, dhl, ws)
        res.append((host(dhp), host(dhl)))
    for a, b in res[1:]:
        np.testing.assert_array_equal(a, res[0][0])
        np.testing.assert_array_equal(b, res[0][1])


def test_empty_tree_zeroes_hyper_gradients(L):
    tree = L.Tree(offsets=[0, 0, 0], device=DEV)
    dhp = torch.full((4,), 7.0, dtype=torch.float64, device=DEV)
    dhl = torch.full((8,), 7.0, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, 1, (1e-3, 0.9, 0.999, 1e-8, 0.0), 0, 0, None, None, None, None, None,
                   None, None, None, None, dhp, dhl, None)
    assert torch.all(dhp == 0) and torch.all(dhl == 0)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 255, 1023, 4097])
def test_tiny_and_ragged_sizes(L, n):
    x = synth.state_tree(n, None, n=n)
    tree = L.Tree(numel=n, device=DEV)
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    g, m, v = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"])
    u, m1, v1 = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    L.opt_adam_fwd(tree, 3, hp, 0, 0, g, m, v, u, m1, v1)
    ru, rm1, rv1 = oracle.adam_fwd(x["g"], x["m"], x["v"], 3, *hp, prec=1)
    mag = oracle.adam_mag(x["g"], x["m"], x["v"], x["du"], None, None, 3, *hp)
    check("u", host(u), ru, mag["u"], 1)
    dg = torch.empty_like(g)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, 3, hp, 0, 0, g, m, v, dev_f32(x["du"]), None, None, dg, None, None, dhp,
                   None, tree.workspace(DEV))
    r = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], None, None, 3, *hp, prec=1)
    check("dg", host(dg), r["dg"], mag["dg"], 1)
    assert_sum_close("dhp", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))


# ------------------------------------------ full-size C2, sampled check
@pytest.mark.slow
@pytest.mark.parametrize("ct", COMPUTES)
def test_c2_resnet18_full_size_sampled(L, ct):
    """Config C2 at full size (11,689,512 elements, 62 leaves) in the launch
    configuration bench.py times; 2^16 sampled elements against the oracle
    (elementwise independence makes the sample exact) and the hyper-gradient
    sums against the full oracle sum."""
    leaves = synth.RESNET18_LEAVES
    x = synth.state_tree(0xC2, leaves)
    tree = L.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.0)
    t = 10
    g, m, v, du, dm1, dv1 = (dev_f32(x[k]) for k in ("g", "m", "v", "du", "dm1", "dv1"))
    u, m1, v1 = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    L.opt_adam_fwd(tree, t, hp, 0, ct, g, m, v, u, m1, v1)
    dg, dm, dv = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, t, hp, 0, ct, g, m, v, du, dm1, dv1, dg, dm, dv, dhp, None,
                   tree.workspace(DEV))
    idx = np.sort(np.random.default_rng(0).choice(tree.numel, 1 << 16, replace=False))
    xs = {k: x[k][idx] for k in x}
    ru, rm1, rv1 = oracle.adam_fwd(xs["g"], xs["m"], xs["v"], t, *hp, prec=1)
    r = oracle.adam_vjp(xs["g"], xs["m"], xs["v"], xs["du"], xs["dm1"], xs["dv1"], t, *hp, prec=1)
    mag = oracle.adam_mag(xs["g"], xs["m"], xs["v"], xs["du"], xs["dm1"], xs["dv1"], t, *hp)
    for name, got, ref in (("u", u, ru), ("m1", m1, rm1), ("v1", v1, rv1), ("dg", dg, r["dg"]),
                           ("dm", dm, r["dm"]), ("dv", dv, r["dv"])):
        check(name, host(got)[idx], ref, mag[name], ct)
    oracle.set_num_threads(0)
    full = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], t, *hp)
    oracle.set_num_threads(1)
    fmag = oracle.adam_mag(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], t, *hp)
    assert_sum_close("dhp", host(dhp), full["dhp"], np.maximum(full["dhp_abs"], fmag["dhp"]))


# ----------------------------------------------- more structural cases
@pytest.mark.parametrize("n_leaves", [4096, 10000])
def test_many_leaves_per_leaf_sums(L, n_leaves):
    """Thousands of ragged leaves, empty ones included (4096: the offset table
    staged in shared memory; 10000: searched in global memory): per-leaf
    hyper-gradient sums and the total equal the oracle's."""
    rng = np.random.default_rng(5)
    leaves = rng.integers(0, 600, n_leaves).tolist()
    leaves[7] = 0  # an empty leaf
    leaves[-1] = 0  # empty last leaf
    x = synth.state_tree(0xB5, leaves)
    off = synth.offsets_of(leaves)
    tree = L.Tree(offsets=off, device=DEV)
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    g, m, v, du, dm1, dv1 = (dev_f32(x[k]) for k in ("g", "m", "v", "du", "dm1", "dv1"))
    dg = torch.empty_like(g)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    dhl = torch.empty(n_leaves * 4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, 4, hp, 0, 0, g, m, v, du, dm1, dv1, dg, None, None, dhp, dhl,
                   tree.workspace(DEV, per_leaf=True))
    r = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 4, *hp, prec=1,
                        offsets=off)
    mag = oracle.adam_mag(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 4, *hp)
    check("dg", host(dg), r["dg"], mag["dg"], 1)
    got = host(dhl).reshape(-1, 4)
    hs = np.maximum(r["dhp_abs"], mag["dhp"])
    assert_leaf_sums_close("dhp_leaf", got, r["dhp_leaf"], leaf_scale(mag["h"], off))
    assert np.all(got[7] == 0) and np.all(got[-1] == 0)
    assert_sum_close("dhp", host(dhp), r["dhp"], hs)


def test_per_leaf_sums_large_leaves(L):
    """Leaves spanning many 256-element chunks and 8192-element super-chunks,
    with boundaries inside chunks, an empty leaf and a 1-element leaf: the
    three-level piece/super-chunk/leaf folds give the oracle's per-leaf sums."""
    leaves = [1_000_003, 3, 8192 * 5 + 1, 0, 77_777, 1, 255, 257]
    x = synth.state_tree(0xB6, leaves)
    off = synth.offsets_of(leaves)
    tree = L.Tree(offsets=off, device=DEV)
    hp = (3e-3, 0.9, 0.999, 1e-8, 0.0)
    g, m, v, du, dm1, dv1 = (dev_f32(x[k]) for k in ("g", "m", "v", "du", "dm1", "dv1"))
    dg, dm, dv = (torch.empty_like(g) for _ in range(3))
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    dhl = torch.empty(len(leaves) * 4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, 7, hp, 0, 0, g, m, v, du, dm1, dv1, dg, dm, dv, dhp, dhl,
                   tree.workspace(DEV, per_leaf=True))
    r = oracle.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 7, *hp, prec=1,
                        offsets=off)
    mag = oracle.adam_mag(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 7, *hp)
    for k, out in (("dg", dg), ("dm", dm), ("dv", dv)):
        check(k, host(out), r[k], mag[k], 1)
    got = host(dhl).reshape(-1, 4)
    hs = np.maximum(r["dhp_abs"], mag["dhp"])
    assert_leaf_sums_close("dhp_leaf", got, r["dhp_leaf"], leaf_scale(mag["h"], off))
    assert np.all(got[3] == 0)
    assert_sum_close("dhp", host(dhp), r["dhp"], hs)


def test_misaligned_device_pointer_rejected(L):
    tree = L.Tree(numel=64, device=DEV)
    buf = torch.zeros(80, device=DEV)
    with pytest.raises(L.DiffoptError) as e:
        L.opt_sgd_fwd(tree, (0.1, 0.0, False), 0, 0, buf[1:], None, buf[:64], None)
    assert e.value.code == L.OPT_EALIGN


def test_nan_propagates_locally(L):
    """Device-side NaN inputs are not checked: they propagate to that
    element's outputs and to the hyper-gradient sums, nowhere else."""
    x = synth.state_tree(0xAA, [4096])
    x["g"][100] = np.nan
    tree = L.Tree(numel=4096, device=DEV)
    hp = (1e-3, 0.9, 0.999, 1e-8, 0.0)
    g, m, v, du = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"]), dev_f32(x["du"])
    u, m1, v1 = torch.empty_like(g), torch.empty_like(g), torch.empty_like(g)
    L.opt_adam_fwd(tree, 5, hp, 0, 0, g, m, v, u, m1, v1)
    uh = host(u)
    assert np.isnan(uh[100]) and np.isfinite(np.delete(uh, 100)).all()
    dg = torch.empty_like(g)
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, 5, hp, 0, 0, g, m, v, du, None, None, dg, None, None, dhp, None,
                   tree.workspace(DEV))
    dgh = host(dg)
    assert np.isnan(dgh[100]) and np.isfinite(np.delete(dgh, 100)).all()
    assert np.isnan(host(dhp)[0])


@pytest.mark.parametrize("kind", ["rmsprop", "sgd", "sgd_nesterov"])
@pytest.mark.parametrize("lr", [1e-3, 1.0])
def test_cold_start_null_state(L, kind, lr):
    """t = 1 style zero state passed as NULL (no HBM read) equals explicit
    zeros, and matches the oracle (C1 inputs, 1/64 exact zeros)."""
    x = synth.c1_inputs()
    n = x["g"].size
    tree = L.Tree(numel=n, device=DEV)
    g, du, ds1 = dev_f32(x["g"]), dev_f32(x["du"]), dev_f32(x["dm1"])
    z = torch.zeros_like(g)
    outs = []
    for state in (None, z):
        u, s1 = torch.empty_like(g), torch.empty_like(g)
        dg, ds = torch.empty_like(g), torch.empty_like(g)
        if kind == "rmsprop":
            hp = (lr, 0.99, 1e-8)
            L.opt_rmsprop_fwd(tree, hp, 0, 0, g, state, u, s1)
            dhp = torch.empty(3, dtype=torch.float64, device=DEV)
            L.opt_rmsprop_bwd(tree, hp, 0, 0, g, state, du, ds1, dg, ds, dhp, None,
                              tree.workspace(DEV))
        else:
            hp = (lr, 0.9, kind == "sgd_nesterov")
            L.opt_sgd_fwd(tree, hp, 0, 0, g, state, u, s1)
            dhp = torch.empty(2, dtype=torch.float64, device=DEV)
            L.opt_sgd_bwd(tree, hp, 0, 0, g, state, du, ds1, dg, ds, dhp, None,
                          tree.workspace(DEV))
        outs.append([host(t) for t in (u, s1, dg, ds, dhp)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    u, s1, dg, ds, dhp = outs[0]
    if kind == "rmsprop":
        ru, rs1 = oracle.rmsprop_fwd(x["g"], None, *hp, prec=1)
        r = oracle.rmsprop_vjp(x["g"], None, x["du"], x["dm1"], *hp, prec=1)
        mag = oracle.rmsprop_mag(x["g"], None, x["du"], x["dm1"], *hp)
        names = (("u", u, ru), ("v1", s1, rs1), ("dg", dg, r["dg"]), ("dv", ds, r["dv"]))
    else:
        ru, rs1 = oracle.sgd_fwd(x["g"], None, *hp, prec=1)
        r = oracle.sgd_vjp(x["g"], None, x["du"], x["dm1"], *hp, prec=1)
        mag = oracle.sgd_mag(x["g"], None, x["du"], x["dm1"], *hp)
        names = (("u", u, ru), ("b1", s1, rs1), ("dg", dg, r["dg"]), ("db", ds, r["db"]))
    for name, got, ref in names:
        check(name, got, ref, mag[name], 1)
    assert_sum_close("dhp", dhp, r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["rmsprop", "sgd"])
@pytest.mark.parametrize("bf16", [False, True])
def test_c2_full_size_sampled_rmsprop_sgd(L, kind, bf16):
    leaves = synth.RESNET18_LEAVES
    x = synth.state_tree(0xC2, leaves)
    n = int(sum(leaves))
    tree = L.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    st_h = state_host_bits(x["v"] if kind == "rmsprop" else x["m"], bf16)
    g, st = dev_f32(x["g"]), dev_state(x["v"] if kind == "rmsprop" else x["m"], bf16)
    du, ds1 = dev_f32(x["du"]), dev_f32(x["dv1"] if kind == "rmsprop" else x["dm1"])
    u = torch.empty_like(g)
    s1 = torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device=DEV)
    dg, ds = torch.empty_like(g), torch.empty_like(g)
    sd = 1 if bf16 else 0
    ws = tree.workspace(DEV)
    if kind == "rmsprop":
        hp = (1e-2, 0.99, 1e-8)
        dhp = torch.empty(3, dtype=torch.float64, device=DEV)
        L.opt_rmsprop_fwd(tree, hp, sd, 0, g, st, u, s1)
        L.opt_rmsprop_bwd(tree, hp, sd, 0, g, st, du, ds1, dg, ds, dhp, None, ws)
    else:
        hp = (0.1, 0.9, True)
        dhp = torch.empty(2, dtype=torch.float64, device=DEV)
        L.opt_sgd_fwd(tree, hp, sd, 0, g, st, u, s1)
        L.opt_sgd_bwd(tree, hp, sd, 0, g, st, du, ds1, dg, ds, dhp, None, ws)
    idx = np.sort(np.random.default_rng(1).choice(n, 1 << 16, replace=False))
    sg, sst = x["g"][idx], st_h[idx]
    sdu = x["du"][idx]
    sds1 = (x["dv1"] if kind == "rmsprop" else x["dm1"])[idx]
    if kind == "rmsprop":
        ru, rs1 = oracle.rmsprop_fwd(sg, sst, *hp, state_bf16=bf16, prec=1)
        r = oracle.rmsprop_vjp(sg, sst, sdu, sds1, *hp, state_bf16=bf16, prec=1)
        mag = oracle.rmsprop_mag(sg, sst, sdu, sds1, *hp, state_bf16=bf16)
        pairs = (("u", u, ru), ("dg", dg, r["dg"]), ("dv", ds, r["dv"]))
    else:
        ru, rs1 = oracle.sgd_fwd(sg, sst, *hp, state_bf16=bf16, prec=1)
        r = oracle.sgd_vjp(sg, sst, sdu, sds1, *hp, state_bf16=bf16, prec=1)
        mag = oracle.sgd_mag(sg, sst, sdu, sds1, *hp, state_bf16=bf16)
        pairs = (("u", u, ru), ("dg", dg, r["dg"]), ("db", ds, r["db"]))
    for name, got, ref in pairs:
        check(name, host(got)[idx], ref, mag[name], 1)
    s1h = host(s1)[idx]
    if bf16:
        assert_close("state'", oracle.bf16_to_f64(s1h), rs1, rtol=1e-2, atol=0)
    else:
        check("state'", s1h, rs1, mag["v1" if kind == "rmsprop" else "b1"], 1)
    # global hyper-gradient sums over all 11.7M elements vs the full oracle
    # sum (bar: the oracle's per-element magnitude twin summed, as for Adam)
    oracle.set_num_threads(0)
    if kind == "rmsprop":
        full = oracle.rmsprop_vjp(x["g"], st_h, x["du"], x["dv1"], *hp, state_bf16=bf16)
        fmag = oracle.rmsprop_mag(x["g"], st_h, x["du"], x["dv1"], *hp, state_bf16=bf16)
    else:
        full = oracle.sgd_vjp(x["g"], st_h, x["du"], x["dm1"], *hp, state_bf16=bf16)
        fmag = oracle.sgd_mag(x["g"], st_h, x["du"], x["dm1"], *hp, state_bf16=bf16)
    oracle.set_num_threads(1)
    assert_sum_close("dhp", host(dhp), full["dhp"], np.maximum(full["dhp_abs"], fmag["dhp"]))


# ------------------------------------------------- beyond 32-bit indexing
def test_adam_beyond_int32_elements_sampled(L):
    """Maximum-size edge case: one flat leaf of 2^31 + 3 elements (past every
    32-bit index), C5 recipe generated in device memory
    (synth.device_state_flat), Adam fwd + bwd in the bench launch
    configuration. 2^16 sampled elements (incl. the last 64 and the ones
    straddling 2^31) against the oracle on the inputs read back at those
    indices; the global hyper-gradient sums against the sum of 129 separate
    launches over 2^24-element pieces (the last straddling 2^31) (different grids, same arithmetic;
    fp64 partials: agree to ~1e-12 of the sum's magnitude), and the last
    piece's sums (which lie beyond 2^31) against the oracle."""
    n = (1 << 31) + 3
    if torch.cuda.mem_get_info()[0] < 100e9:
        pytest.skip("needs ~80 GB of free device memory")
    hp, t = (1e-3, 0.9, 0.999, 1e-8, 0.0), 10
    x = synth.device_state_flat(0xB16, n, DEV)
    tree = L.Tree(numel=n, device=DEV)
    u, m1, v1 = (torch.empty(n, device=DEV) for _ in range(3))
    L.opt_adam_fwd(tree, t, hp, 0, 1, x["g"], x["m"], x["v"], u, m1, v1)
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([rng.choice(n, 1 << 16, replace=False),
                                    np.arange(n - 64, n), np.arange((1 << 31) - 32, (1 << 31) + 3)]))
    di = torch.from_numpy(idx).to(DEV)
    xs = {k: host(x[k][di]) for k in x}
    ru, rm1, rv1 = oracle.adam_fwd(xs["g"], xs["m"], xs["v"], t, *hp, prec=1)
    mag = oracle.adam_mag(xs["g"], xs["m"], xs["v"], xs["du"], xs["dm1"], xs["dv1"], t, *hp)
    for name, got, ref in (("u", u, ru), ("m1", m1, rm1), ("v1", v1, rv1)):
        check(name, host(got[di]), ref, mag[name], 1)
    del u, m1, v1
    dg, dm, dv = (torch.empty(n, device=DEV) for _ in range(3))
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, t, hp, 0, 1, x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], dg,
                   dm, dv, dhp, None, tree.workspace(DEV))
    r = oracle.adam_vjp(xs["g"], xs["m"], xs["v"], xs["du"], xs["dm1"], xs["dv1"], t, *hp, prec=1)
    for name, got in (("dg", dg), ("dm", dm), ("dv", dv)):
        check(name, host(got[di]), r[name], mag[name], 1)
    # global sums: one launch over 2^31+3 vs the sum of 2^24-element pieces
    piece = 1 << 24
    starts = list(range(0, n, piece))
    if n - starts[-1] < piece:
        starts.pop()  # the last piece takes the remainder: it straddles 2^31
    parts = []
    for s, e in zip(starts, starts[1:] + [n]):
        tr = L.Tree(numel=e - s, device=DEV)
        hp_s = torch.empty(4, dtype=torch.float64, device=DEV)
        sl = lambda a: a[s:e]
        L.opt_adam_bwd(tr, t, hp, 0, 1, sl(x["g"]), sl(x["m"]), sl(x["v"]), sl(x["du"]),
                       sl(x["dm1"]), sl(x["dv1"]), None, None, None, hp_s, None, tr.workspace(DEV))
        parts.append(hp_s)
    total = torch.stack(parts).sum(0)
    got, want = host(dhp), host(total)
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12 * float(np.abs(want).max()))
    last = {k: host(x[k][starts[-1]:]) for k in x}
    oracle.set_num_threads(0)
    full = oracle.adam_vjp(last["g"], last["m"], last["v"], last["du"], last["dm1"], last["dv1"],
                           t, *hp)
    oracle.set_num_threads(1)
    fmag = oracle.adam_mag(last["g"], last["m"], last["v"], last["du"], last["dm1"], last["dv1"],
                           t, *hp)
    assert_sum_close("dhp(last piece)", host(parts[-1]), full["dhp"],
                     np.maximum(full["dhp_abs"], fmag["dhp"]))


def test_prepared_calls_equal_marshalled_calls(L):
    """_lib.prepare_adam_fwd/bwd (arguments marshalled once, step per call)
    give bitwise the outputs of the per-call wrappers, at two step counts
    and with state and hyper-gradients."""
    leaves = [5, 4096, 300, 3]
    x = synth.state_tree(0x7E, leaves)
    tree = L.Tree(offsets=synth.offsets_of(leaves), device=DEV)
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    up = lambda a: torch.from_numpy(a).to(DEV)
    g, m, v, du, dm1, dv1 = (up(x[k]) for k in ("g", "m", "v", "du", "dm1", "dv1"))
    outs = {k: [torch.empty_like(g) for _ in range(2)] for k in ("u", "m1", "v1", "dg", "dm", "dv")}
    dhp = [torch.empty(4, dtype=torch.float64, device=DEV) for _ in range(2)]
    ws = tree.workspace(DEV)
    pf = L.prepare_adam_fwd(tree, hp, 0, 0, g, m, v, outs["u"][1], outs["m1"][1], outs["v1"][1])
    pb = L.prepare_adam_bwd(tree, hp, 0, 0, g, m, v, du, dm1, dv1, outs["dg"][1], outs["dm"][1],
                            outs["dv"][1], dhp[1], None, ws)
    for t in (1, 7):
        L.opt_adam_fwd(tree, t, hp, 0, 0, g, m, v, outs["u"][0], outs["m1"][0], outs["v1"][0])
        L.opt_adam_bwd(tree, t, hp, 0, 0, g, m, v, du, dm1, dv1, outs["dg"][0], outs["dm"][0],
                       outs["dv"][0], dhp[0], None, ws)
        pf(t)
        pb(t)
        torch.cuda.synchronize()
        for k, (a, b) in outs.items():
            assert torch.equal(a, b), (t, k)
        assert torch.equal(dhp[0], dhp[1])
    with pytest.raises(L.DiffoptError):
        pf(0)  # step >= 1 is still validated per call
