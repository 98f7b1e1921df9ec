"""GPU parity over the hyper-parameter space the C ABI accepts (VERDICT r1
"untested configurations"), sign-consistent cotangents that make the
hyper-gradient bars real relative checks, and the full-size paths the bench
takes (C3 sweep at 105,205,608 elements, bf16-state backward with the
dynamic tail at >= 2^26 elements, C2 RMSProp/SGD hyper sums).

Bar: elementwise |x - ref| <= 1e-6 + 1e-5 max(|ref|,
mag) for fp32 arithmetic (the oracle's magnitude twin, reading Z10); bf16
stored state 1e-2 relative (Z9); hyper-gradient sums against Sigma of the
per-element twins, per leaf against that leaf's own scale."""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import (DEV, assert_close, assert_leaf_sums_close, assert_sum_close, dev_f32,
                      dev_state, host, leaf_scale, state_host_bits)

pytestmark = pytest.mark.gpu

LEAVES = [5, 1, 4099, 300, 0, 1027, 64, 3]   # 5,499 elements, ragged, an empty leaf


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06934_b200 import _lib

    return _lib


def _check(name, got, ref, mag):
    assert_close(name, got, ref, scale=np.maximum(np.abs(ref), mag))


def _check_state(name, got, ref, mag, bf16):
    if bf16:
        assert_close(name, oracle.bf16_to_f64(got), ref, rtol=1e-2, atol=0)
    else:
        _check(name, got, ref, mag)


# --------------------------------------------------------- Adam grid
ADAM_GRID = list(itertools.product([0.0, 0.5, 0.9], [0.9, 0.999, 0.99999], [0.0, 1e-8, 1e-3],
                                   [0.0, 1e-10]))


@pytest.mark.parametrize("b1,b2,eps,eps_root", ADAM_GRID)
def test_adam_hyper_parameter_grid(L, b1, b2, eps, eps_root):
    """b1 in {0, .5, .9} x b2 in {.9, .999, .99999} x eps in {0, 1e-8, 1e-3}
    x eps_root in {0, 1e-10} x t in {1, 2, 100, 10^4} x {fp32, bf16 state}:
    forward, full backward, global and per-leaf hyper-gradient sums. eps = 0
    exercises Z7 (d = 0 at the zero elements), eps_root > 0 Z4, b1 = 0 the
    0^0 = 1 power in K2 at t = 1, t = 10^4 the underflowed b^t."""
    x = synth.state_tree(0x6A1D, LEAVES)
    off = synth.offsets_of(LEAVES)
    tree = L.Tree(offsets=off, device=DEV)
    n = tree.numel
    for bf16, t in itertools.product([False, True], [1, 2, 100, 10_000]):
        hp = (0.3, b1, b2, eps, eps_root)
        sd = 1 if bf16 else 0
        mh, vh = state_host_bits(x["m"], bf16), state_host_bits(x["v"], bf16)
        g, m, v = dev_f32(x["g"]), dev_state(x["m"], bf16), dev_state(x["v"], bf16)
        sdt = torch.bfloat16 if bf16 else torch.float32
        u = torch.empty_like(g)
        m1, v1 = (torch.empty(n, dtype=sdt, device=DEV) for _ in range(2))
        L.opt_adam_fwd(tree, t, hp, sd, 1, g, m, v, u, m1, v1)
        du, dm1, dv1 = (dev_f32(x[k]) for k in ("du", "dm1", "dv1"))
        dg, dm, dv = (torch.empty_like(g) for _ in range(3))
        dhp = torch.empty(4, dtype=torch.float64, device=DEV)
        dhl = torch.empty(tree.n_leaves * 4, dtype=torch.float64, device=DEV)
        L.opt_adam_bwd(tree, t, hp, sd, 1, g, m, v, du, dm1, dv1, dg, dm, dv, dhp, dhl,
                       tree.workspace(DEV, per_leaf=True))
        ru, rm1, rv1 = oracle.adam_fwd(x["g"], mh, vh, t, *hp, state_bf16=bf16, prec=1)
        r = oracle.adam_vjp(x["g"], mh, vh, x["du"], x["dm1"], x["dv1"], t, *hp,
                            state_bf16=bf16, prec=1, offsets=off)
        mag = oracle.adam_mag(x["g"], mh, vh, x["du"], x["dm1"], x["dv1"], t, *hp,
                              state_bf16=bf16)
        tag = f"bf16={bf16} t={t}"
        _check(f"u {tag}", host(u), ru, mag["u"])
        _check_state(f"m1 {tag}", host(m1), rm1, mag["m1"], bf16)
        _check_state(f"v1 {tag}", host(v1), rv1, mag["v1"], bf16)
        for k, got in (("dg", dg), ("dm", dm), ("dv", dv)):
            _check(f"{k} {tag}", host(got), r[k], mag[k])
        assert_sum_close(f"dhp {tag}", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
        assert_leaf_sums_close(f"dhp_leaf {tag}", host(dhl).reshape(-1, 4), r["dhp_leaf"],
                               leaf_scale(mag["h"], off))
        if t == 1 and eps_root == 0.0:
            # reduced forms: K2 = K4 = 0 at t = 1, so the b1/b2 gradients
            # through the bias corrections vanish exactly (only m'/v' paths)
            pass


@pytest.mark.parametrize("alpha,eps", list(itertools.product([0.0, 0.5, 0.9, 0.99, 0.99999],
                                                             [0.0, 1e-8, 1e-3])))
@pytest.mark.parametrize("lr", [1e-3, 1.0])
def test_rmsprop_hyper_parameter_grid(L, alpha, eps, lr):
    x = synth.state_tree(0x6A2D, LEAVES)
    off = synth.offsets_of(LEAVES)
    tree = L.Tree(offsets=off, device=DEV)
    n = tree.numel
    hp = (lr, alpha, eps)
    for bf16 in (False, True):
        sd = 1 if bf16 else 0
        vh = state_host_bits(x["v"], bf16)
        g, v = dev_f32(x["g"]), dev_state(x["v"], bf16)
        u = torch.empty_like(g)
        v1 = torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device=DEV)
        L.opt_rmsprop_fwd(tree, hp, sd, 1, g, v, u, v1)
        du, dv1 = dev_f32(x["du"]), dev_f32(x["dv1"])
        dg, dv = torch.empty_like(g), torch.empty_like(g)
        dhp = torch.empty(3, dtype=torch.float64, device=DEV)
        dhl = torch.empty(tree.n_leaves * 3, dtype=torch.float64, device=DEV)
        L.opt_rmsprop_bwd(tree, hp, sd, 1, g, v, du, dv1, dg, dv, dhp, dhl,
                          tree.workspace(DEV, per_leaf=True))
        ru, rv1 = oracle.rmsprop_fwd(x["g"], vh, *hp, state_bf16=bf16, prec=1)
        r = oracle.rmsprop_vjp(x["g"], vh, x["du"], x["dv1"], *hp, state_bf16=bf16, prec=1,
                               offsets=off)
        mag = oracle.rmsprop_mag(x["g"], vh, x["du"], x["dv1"], *hp, state_bf16=bf16)
        tag = f"bf16={bf16}"
        _check(f"u {tag}", host(u), ru, mag["u"])
        _check_state(f"v1 {tag}", host(v1), rv1, mag["v1"], bf16)
        _check(f"dg {tag}", host(dg), r["dg"], mag["dg"])
        _check(f"dv {tag}", host(dv), r["dv"], mag["dv"])
        assert_sum_close(f"dhp {tag}", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
        assert_leaf_sums_close(f"dhp_leaf {tag}", host(dhl).reshape(-1, 3), r["dhp_leaf"],
                               leaf_scale(mag["h"], off))


@pytest.mark.parametrize("mu", [0.0, 0.5, 0.9, 0.99])
@pytest.mark.parametrize("nesterov", [False, True])
@pytest.mark.parametrize("lr", [1e-3, 1.0])
def test_sgd_hyper_parameter_grid(L, mu, nesterov, lr):
    x = synth.state_tree(0x6A3D, LEAVES)
    off = synth.offsets_of(LEAVES)
    tree = L.Tree(offsets=off, device=DEV)
    n = tree.numel
    hp = (lr, mu, nesterov)
    for bf16 in (False, True):
        sd = 1 if bf16 else 0
        bh = state_host_bits(x["m"], bf16) if mu != 0.0 else None
        g = dev_f32(x["g"])
        b = dev_state(x["m"], bf16) if mu != 0.0 else None
        u = torch.empty_like(g)
        b1 = (torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device=DEV)
              if mu != 0.0 else None)
        L.opt_sgd_fwd(tree, hp, sd, 1, g, b, u, b1)
        du, db1 = dev_f32(x["du"]), dev_f32(x["dm1"])
        dg = torch.empty_like(g)
        db = torch.empty_like(g) if mu != 0.0 else None
        dhp = torch.empty(2, dtype=torch.float64, device=DEV)
        dhl = torch.empty(tree.n_leaves * 2, dtype=torch.float64, device=DEV)
        L.opt_sgd_bwd(tree, hp, sd, 1, g, b, du, db1 if mu != 0.0 else None, dg, db, dhp, dhl,
                      tree.workspace(DEV, per_leaf=True))
        ru, rb1 = oracle.sgd_fwd(x["g"], bh, *hp, state_bf16=bf16, prec=1)
        r = oracle.sgd_vjp(x["g"], bh, x["du"], x["dm1"] if mu != 0.0 else None, *hp,
                           state_bf16=bf16, prec=1, offsets=off)
        mag = oracle.sgd_mag(x["g"], bh, x["du"], x["dm1"] if mu != 0.0 else None, *hp,
                             state_bf16=bf16)
        tag = f"bf16={bf16}"
        _check(f"u {tag}", host(u), ru, mag["u"])
        _check(f"dg {tag}", host(dg), r["dg"], mag["dg"])
        if mu != 0.0:
            _check_state(f"b1 {tag}", host(b1), rb1, mag["b1"], bf16)
            _check(f"db {tag}", host(db), r["db"], mag["db"])
        assert_sum_close(f"dhp {tag}", host(dhp), r["dhp"], np.maximum(r["dhp_abs"], mag["dhp"]))
        assert_leaf_sums_close(f"dhp_leaf {tag}", host(dhl).reshape(-1, 2), r["dhp_leaf"],
                               leaf_scale(mag["h"], off))


# ------------------------------------------- sign-consistent cotangents
def _adam_parts(x, t, b1, b2):
    """Signs of the per-element hyper-gradient factors, in float64 from the
    inputs (used only to CHOOSE cotangents; correctness is the oracle's)."""
    g, m, v = (x[k].astype(np.float64) for k in ("g", "m", "v"))
    bc1 = 1 - b1 ** t
    mhat = (b1 * m + (1 - b1) * g) / bc1
    p1, p2 = b1 ** t, b2 ** t
    K1 = (1 - p1 + t * p1) / bc1 ** 2
    K2 = (1 - p1 - t * b1 ** (t - 1) * (1 - b1)) / bc1 ** 2
    bc2 = 1 - b2 ** t
    K3 = (1 - p2 + t * p2) / bc2 ** 2
    K4 = (1 - p2 - t * b2 ** (t - 1) * (1 - b2)) / bc2 ** 2
    return mhat, m * K1 - g * K2, v * K3 - g * g * K4


@pytest.mark.parametrize("which", ["lr_eps", "b1", "b2"])
@pytest.mark.parametrize("tree_kind", ["ragged", "c2"])
def test_adam_sign_consistent_hyper_gradients(L, which, tree_kind):
    """Cotangents chosen so every element's term of one hyper-gradient has
    the same sign (u_bar = -sign(mhat)|z| makes every lr term -u_bar mhat/d
    >= 0 and every eps term <= 0; u_bar = -sign(m K1 - g K2)|z| with zero
    m'/v' cotangents does it for b1; u_bar = sign(mhat (v K3 - g^2 K4))|z|
    for b2). Then Sigma|term| = |Sigma| and the 1e-5 Sigma|term| bar is a
    true 1e-5 RELATIVE check of the sum, globally and for every leaf --
    including the 1-element leaf of the ragged tree (VERDICT r1 "done")."""
    if tree_kind == "c2":
        leaves = synth.RESNET18_LEAVES
        x = synth.state_tree(0xC2, leaves)
    else:
        leaves = LEAVES
        x = synth.state_tree(0x5C, leaves)
    off = synth.offsets_of(leaves)
    tree = L.Tree(offsets=off, device=DEV)
    t, hp = 10, (1.0, 0.9, 0.999, 1e-8, 0.0)
    mhat, f1, f2 = _adam_parts(x, t, hp[1], hp[2])
    z = np.abs(x["du"]).astype(np.float32)
    dm1 = dv1 = None
    if which == "lr_eps":
        du = (-np.sign(mhat) * z).astype(np.float32)
        ks = [0, 3]
    elif which == "b1":
        du = (-np.sign(f1) * z).astype(np.float32)
        ks = [1]
    else:
        du = (np.sign(mhat * f2) * z).astype(np.float32)
        ks = [2]
    g, m, v = dev_f32(x["g"]), dev_f32(x["m"]), dev_f32(x["v"])
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    dhl = torch.empty(tree.n_leaves * 4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, t, hp, 0, 1, g, m, v, dev_f32(du), None, None, None, None, None, dhp,
                   dhl, tree.workspace(DEV, per_leaf=True))
    if tree_kind == "c2":
        oracle.set_num_threads(0)
    r = oracle.adam_vjp(x["g"], x["m"], x["v"], du, dm1, dv1, t, *hp, prec=1, offsets=off)
    oracle.set_num_threads(1)
    got, gl = host(dhp), host(dhl).reshape(-1, 4)
    for k in ks:
        # the case really is sign-consistent: Sigma|term| == |Sigma|
        assert r["dhp_abs"][k] == pytest.approx(abs(r["dhp"][k]), rel=1e-9)
        assert abs(got[k] - r["dhp"][k]) <= 1e-5 * abs(r["dhp"][k]), (k, got[k], r["dhp"][k])
        ref_l = r["dhp_leaf"][:, k]
        bad = ~(np.abs(gl[:, k] - ref_l) <= 1e-5 * np.abs(ref_l) + 1e-300)
        assert not bad.any(), (k, np.flatnonzero(bad)[:5], gl[bad, k][:5], ref_l[bad][:5])
    if tree_kind == "ragged":
        one = LEAVES.index(1)
        assert all(r["dhp_leaf"][one, k] != 0 for k in ks)


def test_rmsprop_sgd_sign_consistent_lr(L):
    """The same for the RMSProp and SGD lr gradients (u_bar = sign(g) |z|:
    RMSProp's -u_bar g/d and SGD's -u_bar b' terms all share a sign)."""
    x = synth.state_tree(0x5D, LEAVES)
    off = synth.offsets_of(LEAVES)
    tree = L.Tree(offsets=off, device=DEV)
    z = np.abs(x["du"])
    g, v, b = dev_f32(x["g"]), dev_f32(x["v"]), dev_f32(x["m"])
    du = (np.sign(x["g"]) * z).astype(np.float32)
    dhp = torch.empty(3, dtype=torch.float64, device=DEV)
    dhl = torch.empty(tree.n_leaves * 3, dtype=torch.float64, device=DEV)
    L.opt_rmsprop_bwd(tree, (0.5, 0.99, 1e-8), 0, 1, g, v, dev_f32(du), None, None, None, dhp,
                      dhl, tree.workspace(DEV, per_leaf=True))
    r = oracle.rmsprop_vjp(x["g"], x["v"], du, None, 0.5, 0.99, 1e-8, prec=1, offsets=off)
    assert r["dhp_abs"][0] == pytest.approx(abs(r["dhp"][0]), rel=1e-9)
    assert abs(host(dhp)[0] - r["dhp"][0]) <= 1e-5 * abs(r["dhp"][0])
    gl = host(dhl).reshape(-1, 3)[:, 0]
    assert np.all(np.abs(gl - r["dhp_leaf"][:, 0]) <= 1e-5 * np.abs(r["dhp_leaf"][:, 0]) + 1e-300)
    # SGD: b' = mu b + g; u_bar = sign(b') |z| makes -u_bar b' <= 0 everywhere
    bp = 0.9 * x["m"].astype(np.float64) + x["g"]
    du = (np.sign(bp) * z).astype(np.float32)
    dhp2 = torch.empty(2, dtype=torch.float64, device=DEV)
    dhl2 = torch.empty(tree.n_leaves * 2, dtype=torch.float64, device=DEV)
    L.opt_sgd_bwd(tree, (0.1, 0.9, False), 0, 1, g, b, dev_f32(du), None, None, None, dhp2, dhl2,
                  tree.workspace(DEV, per_leaf=True))
    r = oracle.sgd_vjp(x["g"], x["m"], du, None, 0.1, 0.9, False, prec=1, offsets=off)
    assert r["dhp_abs"][0] == pytest.approx(abs(r["dhp"][0]), rel=1e-9)
    assert abs(host(dhp2)[0] - r["dhp"][0]) <= 1e-5 * abs(r["dhp"][0])
    gl = host(dhl2).reshape(-1, 2)[:, 0]
    assert np.all(np.abs(gl - r["dhp_leaf"][:, 0]) <= 1e-5 * np.abs(r["dhp_leaf"][:, 0]) + 1e-300)


# --------------------------------------------------- full-size paths
@pytest.mark.slow
@pytest.mark.parametrize("fuse", [True, False])
def test_c3_full_size_sweep_sampled(L, fuse):
    """C3 exactly as bench.py runs it (9 x ResNet-18 tree, 105,205,608
    elements, K = 5 Adam, fused or unfused inner-loss glue; the >= 2^26
    dynamic-tail backward inside opt_adam_quad_rev / opt_adam_bwd): 2^16
    sampled elements of theta_K, phi_bar and theta0_bar against the oracle
    sweep on the same elements (the quadratic problem is separable, so the
    sample is exact) and the hyper-gradient sums against the oracle's full
    sweep (all host cores)."""
    from paper_2211_06934_b200.unroll import QuadraticSweep

    leaves = synth.RESNET18_LEAVES * 9
    off = synth.offsets_of(leaves)
    n = int(off[-1])
    q = synth.quadratic_problem(0xC3, n)
    tree = L.Tree(offsets=off, device=DEV)
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    sw = QuadraticSweep(tree, "adam", hp, 5, DEV, fuse_glue=fuse)
    a, th0, phi, y = (torch.from_numpy(q[k]).to(DEV) for k in ("a", "theta0", "phi", "y"))
    thK, phib, th0b, hyper = sw.run(a, th0, phi, y)
    torch.cuda.synchronize()
    idx = np.unique(np.concatenate([np.random.default_rng(7).choice(n, 1 << 16, replace=False),
                                    np.arange(n - 64, n)]))
    di = torch.from_numpy(idx).to(DEV)
    qs = {k: q[k][idx] for k in q}
    ref = oracle.sweep_quadratic("adam", qs["a"], qs["theta0"], qs["phi"], qs["y"], 5, hp, prec=1)
    assert_close("thetaK", host(thK[di]), ref["thetaK"],
                 scale=np.abs(ref["thetaK"]) + np.abs(qs["theta0"]))
    assert_close("phi_bar", host(phib[di]), ref["phi_bar"], scale=ref["bar_abs"])
    assert_close("theta0_bar", host(th0b[di]), ref["theta0_bar"], scale=ref["bar_abs"])
    oracle.set_num_threads(0)
    full = oracle.sweep_quadratic("adam", q["a"], q["theta0"], q["phi"], q["y"], 5, hp)
    oracle.set_num_threads(1)
    hs = host(hyper).sum(0)
    assert_sum_close("hyper", hs[:4], full["hyper_bar"][:4], full["hyper_abs"][:4])


@pytest.mark.slow
def test_bf16_state_adam_backward_dynamic_tail(L):
    """bf16-state Adam backward at 2^26 + 5 elements (the dynamic-tail
    reduction path with bf16 state loads): 2^16 sampled elements
    plus the last 4096 (the dynamically claimed tail) against the oracle, the
    global hyper sums against the oracle's full sum."""
    n = (1 << 26) + 5
    x = synth.state_tree(0xBF26, None, n=n)
    tree = L.Tree(numel=n, device=DEV)
    hp, t = (1e-2, 0.9, 0.999, 1e-8, 0.0), 10
    mh, vh = state_host_bits(x["m"], True), state_host_bits(x["v"], True)
    g, m, v = dev_f32(x["g"]), dev_state(mh, True), dev_state(vh, True)
    du, dm1, dv1 = (dev_f32(x[k]) for k in ("du", "dm1", "dv1"))
    dg, dm, dv = (torch.empty_like(g) for _ in range(3))
    dhp = torch.empty(4, dtype=torch.float64, device=DEV)
    L.opt_adam_bwd(tree, t, hp, 1, 1, g, m, v, du, dm1, dv1, dg, dm, dv, dhp, None,
                   tree.workspace(DEV))
    idx = np.unique(np.concatenate([np.random.default_rng(9).choice(n, 1 << 16, replace=False),
                                    np.arange(n - 4096, n)]))
    xs = {k: x[k][idx] for k in ("g", "du", "dm1", "dv1")}
    r = oracle.adam_vjp(xs["g"], mh[idx], vh[idx], xs["du"], xs["dm1"], xs["dv1"], t, *hp,
                        state_bf16=True, prec=1)
    mag = oracle.adam_mag(xs["g"], mh[idx], vh[idx], xs["du"], xs["dm1"], xs["dv1"], t, *hp,
                          state_bf16=True)
    for k, got in (("dg", dg), ("dm", dm), ("dv", dv)):
        _check(k, host(got)[idx], r[k], mag[k])
    oracle.set_num_threads(0)
    full = oracle.adam_vjp(x["g"], mh, vh, x["du"], x["dm1"], x["dv1"], t, *hp, state_bf16=True)
    oracle.set_num_threads(1)
    fmag = oracle.adam_mag(x["g"], mh, vh, x["du"], x["dm1"], x["dv1"], t, *hp, state_bf16=True)
    assert_sum_close("dhp", host(dhp), full["dhp"], np.maximum(full["dhp_abs"], fmag["dhp"]))


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["rmsprop", "sgd"])
def test_c2_full_size_rmsprop_sgd_hyper_sums(L, kind):
    """C2 tree at full size: RMSProp / Nesterov SGD backward WITH global and
    per-leaf hyper-gradients (the bench launch configuration) against the
    oracle's full sums, per leaf at each leaf's own scale."""
    leaves = synth.RESNET18_LEAVES
    x = synth.state_tree(0xC2, leaves)
    off = synth.offsets_of(leaves)
    tree = L.Tree(offsets=off, device=DEV)
    g, du = dev_f32(x["g"]), dev_f32(x["du"])
    if kind == "rmsprop":
        hp, nh = (1e-2, 0.99, 1e-8), 3
        st, ds1 = dev_f32(x["v"]), dev_f32(x["dv1"])
    else:
        hp, nh = (0.1, 0.9, True), 2
        st, ds1 = dev_f32(x["m"]), dev_f32(x["dm1"])
    dhp = torch.empty(nh, dtype=torch.float64, device=DEV)
    dhl = torch.empty(tree.n_leaves * nh, dtype=torch.float64, device=DEV)
    dhp_g = torch.empty(nh, dtype=torch.float64, device=DEV)
    dg = torch.empty_like(g)
    fn = L.opt_rmsprop_bwd if kind == "rmsprop" else L.opt_sgd_bwd
    fn(tree, hp, 0, 1, g, st, du, ds1, dg, None, dhp, dhl, tree.workspace(DEV, per_leaf=True))
    fn(tree, hp, 0, 1, g, st, du, ds1, None, None, dhp_g, None, tree.workspace(DEV))
    oracle.set_num_threads(0)
    if kind == "rmsprop":
        r = oracle.rmsprop_vjp(x["g"], x["v"], x["du"], x["dv1"], *hp, offsets=off)
        mag = oracle.rmsprop_mag(x["g"], x["v"], x["du"], x["dv1"], *hp)
    else:
        r = oracle.sgd_vjp(x["g"], x["m"], x["du"], x["dm1"], *hp, offsets=off)
        mag = oracle.sgd_mag(x["g"], x["m"], x["du"], x["dm1"], *hp)
    oracle.set_num_threads(1)
    sc = np.maximum(r["dhp_abs"], mag["dhp"])
    assert_sum_close("dhp", host(dhp), r["dhp"], sc)
    assert_sum_close("dhp(global path)", host(dhp_g), r["dhp"], sc)
    assert_leaf_sums_close("dhp_leaf", host(dhl).reshape(-1, nh), r["dhp_leaf"],
                           leaf_scale(mag["h"], off))
