"""Pins of the CPU oracle against things other than itself (no GPU).

Each test names what fixes the expected value: a worked example printed in
SPEC.md (tests/golden/spec_examples.json), a closed form derived by hand, a
library routine (torch.optim in float64), the complex-step derivative of the
oracle's own *forward* (which is pinned separately), central finite
differences, or an algebraic property of a VJP. A plausible slip in the
oracle's VJP (dropped term, wrong sign, wrong power of bc, transposed
operand) changes at least one of these.
"""
import json
import os

import numpy as np
import pytest
import torch

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
H = 1e-30  # complex-step size


def rel_err(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    return np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1e-300))


# ------------------------------------------------ worked examples (SPEC)
def test_spec_adam_first_step(orc):
    e = GOLD["adam_first_step"]
    u, m1, v1 = orc.adam_fwd([e["g"]], None, None, e["t"], e["lr"], e["b1"], e["b2"], e["eps"])
    assert m1[0] == pytest.approx(e["m1"], rel=1e-15)
    assert v1[0] == pytest.approx(e["v1"], rel=1e-12)
    assert u[0] == pytest.approx(e["delta"], rel=1e-15)
    assert e["theta"] + u[0] == pytest.approx(e["theta1"], rel=1e-7)


def test_spec_adam_zero_grad_exact(orc):
    e = GOLD["adam_zero_grad"]
    u, m1, v1 = orc.adam_fwd([e["g"]], None, None, 1, e["lr"], e["b1"], e["b2"], e["eps"])
    assert u[0] == 0.0 and m1[0] == 0.0 and v1[0] == 0.0


def test_spec_sgd_examples(orc):
    e = GOLD["sgd_plain"]
    u, _ = orc.sgd_fwd([e["g"]], None, e["lr"], e["momentum"])
    assert u[0] == e["delta"]
    e = GOLD["sgd_momentum_two_steps"]
    b = None
    for k in range(2):
        u, b1 = orc.sgd_fwd([e["g"][k]], b, e["lr"], e["momentum"])
        assert b1[0] == pytest.approx(e["buffers"][k], rel=1e-15)
        assert u[0] == pytest.approx(e["deltas"][k], rel=1e-15)
        b = b1.astype(np.float32)
    e = GOLD["sgd_zero_grad"]
    u, _ = orc.sgd_fwd([e["g"]], np.zeros(1, np.float32), e["lr"], e["momentum"])
    assert u[0] == 0.0


def test_spec_rmsprop_first_step(orc):
    e = GOLD["rmsprop_first_step"]
    u, v1 = orc.rmsprop_fwd([e["g"]], None, e["lr"], e["alpha"], e["eps"])
    assert v1[0] == pytest.approx(e["nu"], rel=1e-14)
    assert u[0] == pytest.approx(e["delta"], rel=1e-13)


# ------------------------------------------------------- closed forms
def test_adam_t1_closed_form_forward_and_vjp(orc):
    """SURVEY P1 / north star: at t=1 from zero state, u = -lr g/(|g|+eps),
    du/dg = -lr eps/(|g|+eps)^2, du/dlr = -g/(|g|+eps),
    du/deps = lr g/(|g|+eps)^2, du/db1 = du/db2 = 0; with zero m', v'
    cotangents dm = -b1 lr/((1-b1)(|g|+eps)), dv = b2 lr sgn(g)/(2(1-b2)(|g|+eps)^2)."""
    rng = np.random.default_rng(1)
    g = (rng.standard_normal(64) * 10.0 ** rng.uniform(-3, 0, 64)).astype(np.float32)
    lr, b1, b2, eps = 0.3, 0.9, 0.999, 1e-8
    gd = g.astype(np.float64)
    a = np.abs(gd) + eps
    u, m1, v1 = orc.adam_fwd(g, None, None, 1, lr, b1, b2, eps)
    assert rel_err(u, -lr * gd / a) < 1e-14
    assert rel_err(m1, (1 - b1) * gd) < 1e-15
    assert rel_err(v1, (1 - b2) * gd * gd) < 1e-14
    for prec, tol in ((0, 1e-6), (1, 1e-10)):
        for i in range(g.size):  # per element: hyper-gradients of one element
            r = orc.adam_vjp(g[i:i + 1], None, None, np.ones(1), None, None, 1, lr, b1, b2, eps,
                             prec=prec)
            ai = a[i]
            assert r["dg"][0] == pytest.approx(-lr * eps / ai ** 2, rel=tol)
            assert r["dhp"][0] == pytest.approx(-gd[i] / ai, rel=1e-13)
            assert r["dhp"][3] == pytest.approx(lr * gd[i] / ai ** 2, rel=1e-13)
            assert abs(r["dhp"][1]) <= 1e-12 * lr / ai
            assert abs(r["dhp"][2]) <= 1e-12 * lr / ai
            assert r["dm"][0] == pytest.approx(-b1 * lr / ((1 - b1) * ai), rel=1e-13)
            assert r["dv"][0] == pytest.approx(b2 * lr * np.sign(gd[i]) / (2 * (1 - b2) * ai ** 2),
                                               rel=1e-12)


def test_adam_zero_point_conventions(orc):
    """SURVEY P3 / readings Z6, Z7: g = m = v = 0 gives u = 0 exactly and finite
    cotangents; dg = (1-b1) dm1 - lr A du/eps with A = (1-b1)/bc1,
    dm = b1 (dm1 - du lr/(bc1 eps)), dv = b2 dv1."""
    lr, b1, b2, eps = 0.5, 0.9, 0.999, 1e-8
    du = np.array([1.0, -2.0, 0.5], np.float32)
    dm1 = np.array([0.3, 0.0, -1.0], np.float32)
    dv1 = np.array([2.0, 1.0, 0.0], np.float32)
    z = np.zeros(3, np.float32)
    dud, dm1d = du.astype(np.float64), dm1.astype(np.float64)
    for t in (1, 3, 50):
        u, m1, v1 = orc.adam_fwd(z, z, z, t, lr, b1, b2, eps)
        assert np.all(u == 0) and np.all(m1 == 0) and np.all(v1 == 0)
        r = orc.adam_vjp(z, z, z, du, dm1, dv1, t, lr, b1, b2, eps)
        bc1 = 1 - b1 ** t
        A = (1 - b1) / bc1
        for k in ("dg", "dm", "dv"):
            assert np.all(np.isfinite(r[k]))
        np.testing.assert_allclose(r["dg"], (1 - b1) * dm1d - lr * A * dud / eps, rtol=1e-12)
        np.testing.assert_allclose(r["dm"], b1 * (dm1d - dud * lr / (bc1 * eps)), rtol=1e-12)
        np.testing.assert_allclose(r["dv"], b2 * dv1.astype(np.float64), rtol=1e-15)


def test_adam_constant_gradient_invariant(orc):
    """a constant g from zero state keeps mhat = g, vhat = g^2, so
    u_t = -lr g/(|g|+eps) at every step t (bias correction exactness)."""
    g = np.array([0.7, -1e-3, 2.5, 1e-6], np.float32)
    lr, b1, b2, eps = 1e-2, 0.9, 0.999, 1e-8
    gd = g.astype(np.float64)
    m = v = None
    for t in range(1, 31):
        u, m1, v1 = orc.adam_fwd(g, m, v, t, lr, b1, b2, eps)
        assert rel_err(u, -lr * gd / (np.abs(gd) + eps)) < 1e-6  # fp32 state storage
        m, v = m1.astype(np.float32), v1.astype(np.float32)


def test_rmsprop_zero_point(orc):
    """Reading Z6 for RMSProp: g = v = 0 gives dg = -lr du/eps, dv = alpha dv1."""
    du = np.array([1.0, -3.0], np.float32)
    dv1 = np.array([0.5, 2.0], np.float32)
    z = np.zeros(2, np.float32)
    r = orc.rmsprop_vjp(z, z, du, dv1, 0.1, 0.99, 1e-8)
    np.testing.assert_allclose(r["dg"], -0.1 * du.astype(np.float64) / 1e-8, rtol=1e-12)
    np.testing.assert_allclose(r["dv"], 0.99 * dv1.astype(np.float64), rtol=1e-15)


def test_eps_zero_convention(orc):
    """Reading Z7: eps = 0 and g = v = 0 -> u := 0 and finite backward."""
    z = np.zeros(1, np.float32)
    u, v1 = orc.rmsprop_fwd(z, z, 1.0, 0.99, 0.0)
    assert u[0] == 0.0
    r = orc.rmsprop_vjp(z, z, np.ones(1), np.ones(1), 1.0, 0.99, 0.0)
    assert np.all(np.isfinite(r["dg"])) and r["dg"][0] == 0.0


# ----------------------------------------- library routine: torch.optim
def _torch_steps(opt_cls, kwargs, grads):
    p = torch.zeros(grads[0].shape, dtype=torch.float64, requires_grad=True)
    opt = opt_cls([p], **kwargs)
    ups = []
    for g in grads:
        before = p.detach().clone()
        p.grad = torch.as_tensor(g, dtype=torch.float64)
        opt.step()
        ups.append((p.detach() - before).numpy())
    return ups, opt.state[p]


def test_forward_matches_torch_optim_float64(orc):
    """torch.optim.Adam / RMSprop / SGD (float64, CPU) are an
    independent implementation of the same recurrences (eps outside the
    sqrt, bias correction, dampening 0). Compared over 12 steps; the oracle
    state is kept in float64 by exact float32 grads and fp64 chaining via
    prec=0 outputs fed back through float32 only where exact."""
    rng = np.random.default_rng(7)
    grads = [(rng.standard_normal(257) * 10.0 ** rng.uniform(-4, 0, 257)).astype(np.float32)
             for _ in range(12)]
    # Adam: chain the oracle with float64 state by calling the complex forward
    # (real inputs) which accepts float64 state exactly.
    ups, _ = _torch_steps(torch.optim.Adam, dict(lr=1e-2, betas=(0.9, 0.999), eps=1e-8), grads)
    m = v = np.zeros(257)
    for t, g in enumerate(grads, 1):
        u, m, v = (x.real for x in orc.adam_fwd_complex(g.astype(np.float64), m, v, t,
                                                         [1e-2, 0.9, 0.999, 1e-8, 0.0]))
        np.testing.assert_allclose(u, ups[t - 1], rtol=1e-9, atol=1e-300)
    ups, _ = _torch_steps(torch.optim.RMSprop, dict(lr=1e-2, alpha=0.99, eps=1e-8), grads)
    v = np.zeros(257)
    for t, g in enumerate(grads, 1):
        u, v = (x.real for x in orc.rmsprop_fwd_complex(g.astype(np.float64), v, [1e-2, 0.99, 1e-8]))
        np.testing.assert_allclose(u, ups[t - 1], rtol=1e-9, atol=1e-300)
    for nest in (False, True):
        ups, _ = _torch_steps(torch.optim.SGD, dict(lr=0.1, momentum=0.9, nesterov=nest), grads)
        b = np.zeros(257)
        for t, g in enumerate(grads, 1):
            u, b = (x.real for x in orc.sgd_fwd_complex(g.astype(np.float64), b, [0.1, 0.9], nest))
            np.testing.assert_allclose(u, ups[t - 1], rtol=1e-9, atol=1e-300)


def test_real_and_complex_forward_agree(orc):
    """The float64 entry points and the complex128 entry points evaluate the
    same template; on real inputs they must agree to rounding."""
    x = synth.state_tree(3, [1000, 24])
    u, m1, v1 = orc.adam_fwd(x["g"], x["m"], x["v"], 4, 1e-3, 0.9, 0.999, 1e-8)
    uc, mc, vc = orc.adam_fwd_complex(x["g"], x["m"], x["v"], 4, [1e-3, 0.9, 0.999, 1e-8, 0])
    np.testing.assert_array_equal(u, uc.real)
    np.testing.assert_array_equal(m1, mc.real)


# ---------------------------------------------- complex-step VJP pins
def _state_inputs(seed, n, t_warm=True):
    x = synth.state_tree(seed, [n // 2, n - n // 2], warm=t_warm, zero_frac=0.0)
    return x


@pytest.mark.parametrize("t", [1, 2, 7, 100])
@pytest.mark.parametrize("eps_root", [0.0, 1e-10])
def test_adam_vjp_vs_complex_step(orc, t, eps_root):
    """every VJP output, including the four hyper-gradient sums,
    equals the complex-step Jacobian of the (separately pinned) forward
    contracted with the cotangents."""
    x = _state_inputs(11 + t, 200, t_warm=(t > 1))
    g, m, v, du, dm1, dv1 = (x[k] for k in ("g", "m", "v", "du", "dm1", "dv1"))
    hp = np.array([0.05, 0.9, 0.999, 1e-8, eps_root])
    gd = g.astype(np.float64)
    md = np.zeros_like(gd) if m is None else m.astype(np.float64)
    vd = np.zeros_like(gd) if v is None else v.astype(np.float64)
    cot = (du.astype(np.float64), dm1.astype(np.float64), dv1.astype(np.float64))

    def contract(outs):
        return sum(c * o.imag / H for c, o in zip(cot, outs))

    r = orc.adam_vjp(g, m, v, du, dm1, dv1, t, *hp, prec=1)
    cs_g = contract(orc.adam_fwd_complex(gd + 1j * H, md, vd, t, hp))
    cs_m = contract(orc.adam_fwd_complex(gd, md + 1j * H, vd, t, hp))
    cs_v = contract(orc.adam_fwd_complex(gd, md, vd + 1j * H, t, hp))
    scale = lambda a: np.abs(a) + 1e-12 * np.max(np.abs(a))
    assert np.max(np.abs(r["dg"] - cs_g) / scale(cs_g)) < 1e-8
    assert np.max(np.abs(r["dm"] - cs_m) / scale(cs_m)) < 1e-8
    assert np.max(np.abs(r["dv"] - cs_v) / scale(cs_v)) < 1e-8
    for k in range(4):  # lr, b1, b2, eps
        hpc = hp.astype(np.complex128)
        hpc[k] += 1j * H
        cs = contract(orc.adam_fwd_complex(gd, md, vd, t, hpc)).sum()
        assert r["dhp"][k] == pytest.approx(cs, rel=1e-8, abs=1e-10 * r["dhp_abs"][k] + 1e-300)


def test_rmsprop_vjp_vs_complex_step(orc):
    x = _state_inputs(5, 300)
    g, v, du, dv1 = x["g"], x["v"], x["du"], x["dv1"]
    hp = np.array([0.01, 0.95, 1e-8])
    gd, vd = g.astype(np.float64), v.astype(np.float64)
    cot = (du.astype(np.float64), dv1.astype(np.float64))
    contract = lambda outs: sum(c * o.imag / H for c, o in zip(cot, outs))
    r = orc.rmsprop_vjp(g, v, du, dv1, *hp, prec=1)
    np.testing.assert_allclose(r["dg"], contract(orc.rmsprop_fwd_complex(gd + 1j * H, vd, hp)),
                               rtol=1e-8)
    np.testing.assert_allclose(r["dv"], contract(orc.rmsprop_fwd_complex(gd, vd + 1j * H, hp)),
                               rtol=1e-8)
    for k in range(3):
        hpc = hp.astype(np.complex128)
        hpc[k] += 1j * H
        cs = contract(orc.rmsprop_fwd_complex(gd, vd, hpc)).sum()
        assert r["dhp"][k] == pytest.approx(cs, rel=1e-8)


@pytest.mark.parametrize("nesterov", [False, True])
def test_sgd_vjp_vs_complex_step(orc, nesterov):
    x = _state_inputs(9, 300)
    g, b, du, db1 = x["g"], x["m"], x["du"], x["dm1"]
    hp = np.array([0.1, 0.9])
    gd, bd = g.astype(np.float64), b.astype(np.float64)
    cot = (du.astype(np.float64), db1.astype(np.float64))
    contract = lambda outs: sum(c * o.imag / H for c, o in zip(cot, outs))
    r = orc.sgd_vjp(g, b, du, db1, *hp, nesterov=nesterov, prec=1)
    np.testing.assert_allclose(r["dg"], contract(orc.sgd_fwd_complex(gd + 1j * H, bd, hp, nesterov)),
                               rtol=1e-12)
    np.testing.assert_allclose(r["db"], contract(orc.sgd_fwd_complex(gd, bd + 1j * H, hp, nesterov)),
                               rtol=1e-12)
    for k in range(2):
        hpc = hp.astype(np.complex128)
        hpc[k] += 1j * H
        cs = contract(orc.sgd_fwd_complex(gd, bd, hpc, nesterov)).sum()
        assert r["dhp"][k] == pytest.approx(cs, rel=1e-10)


# ------------------------------------------------ finite differences
def test_adam_vjp_vs_central_fd(orc):
    """central differences in double on a few elements (an
    independent numerical derivative, not reusing complex arithmetic)."""
    x = _state_inputs(21, 8)
    g, m, v = (x[k].astype(np.float64) for k in ("g", "m", "v"))
    du = x["du"].astype(np.float64)
    hp = [0.05, 0.9, 0.999, 1e-8, 0.0]
    t = 5

    def U(gg, mm, vv, h=hp):
        return orc.adam_fwd_complex(gg, mm, vv, t, h)[0].real

    r = orc.adam_vjp(x["g"], x["m"], x["v"], x["du"], None, None, t, *hp, prec=1)
    for i in range(8):
        e = np.zeros(8)
        hstep = 1e-6 * max(abs(g[i]), 1e-6)
        e[i] = hstep
        fd = (U(g + e, m, v) - U(g - e, m, v))[i] / (2 * hstep) * du[i]
        assert r["dg"][i] == pytest.approx(fd, rel=2e-5, abs=1e-9 * abs(du[i]))
    hstep = 1e-7
    for k, hk in ((0, 1e-7), (1, 1e-7), (2, 1e-7)):
        hpp, hpm = list(hp), list(hp)
        hpp[k] += hk
        hpm[k] -= hk
        fd = np.sum((U(g, m, v, hpp) - U(g, m, v, hpm)) / (2 * hk) * du)
        assert r["dhp"][k] == pytest.approx(fd, rel=1e-5, abs=1e-6 * r["dhp_abs"][k])


# ------------------------------------------------ algebraic properties
def test_vjp_linear_in_cotangents_and_null_is_zero(orc):
    """the VJP is linear in (du, dm1, dv1); a NULL cotangent is
    bitwise the zero cotangent."""
    x = synth.state_tree(31, [500, 12])
    g, m, v, du, dm1, dv1 = (x[k] for k in ("g", "m", "v", "du", "dm1", "dv1"))
    hp = (1e-3, 0.9, 0.999, 1e-8)
    r_all = orc.adam_vjp(g, m, v, du, dm1, dv1, 10, *hp)
    r_u = orc.adam_vjp(g, m, v, du, None, None, 10, *hp)
    r_u0 = orc.adam_vjp(g, m, v, du, np.zeros_like(du), np.zeros_like(du), 10, *hp)
    r_m = orc.adam_vjp(g, m, v, None, dm1, None, 10, *hp)
    r_v = orc.adam_vjp(g, m, v, None, None, dv1, 10, *hp)
    for k in ("dg", "dm", "dv"):
        np.testing.assert_array_equal(r_u[k], r_u0[k])
        s = r_u[k] + r_m[k] + r_v[k]
        np.testing.assert_allclose(r_all[k], s, rtol=1e-9, atol=1e-9 * np.max(np.abs(s)))
    np.testing.assert_allclose(r_all["dhp"], r_u["dhp"] + r_m["dhp"] + r_v["dhp"], rtol=1e-9,
                               atol=1e-12 * np.max(r_all["dhp_abs"]))


def test_per_leaf_sums_add_to_global(orc):
    leaves = [5, 4096, 1, 300, 9000]
    x = synth.state_tree(41, leaves)
    off = synth.offsets_of(leaves)
    r = orc.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 3, 1e-3, 0.9, 0.999,
                     1e-8, offsets=off)
    np.testing.assert_allclose(r["dhp_leaf"].sum(0), r["dhp"], rtol=1e-12,
                               atol=1e-14 * r["dhp_abs"].max())
    # each leaf's sum equals the global sum over that leaf alone
    l = 3
    sl = slice(off[l], off[l + 1])
    r3 = orc.adam_vjp(x["g"][sl], x["m"][sl], x["v"][sl], x["du"][sl], x["dm1"][sl],
                      x["dv1"][sl], 3, 1e-3, 0.9, 0.999, 1e-8)
    np.testing.assert_allclose(r["dhp_leaf"][l], r3["dhp"], rtol=1e-13)


def test_thread_count_independent(orc):
    x = synth.state_tree(51, [70000])
    args = (x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 4, 1e-3, 0.9, 0.999, 1e-8)
    orc.set_num_threads(1)
    r1 = orc.adam_vjp(*args)
    orc.set_num_threads(0)
    r2 = orc.adam_vjp(*args)
    orc.set_num_threads(1)
    np.testing.assert_array_equal(r1["dhp"], r2["dhp"])
    np.testing.assert_array_equal(r1["dg"], r2["dg"])


# ---------------------------------------------------------- bf16 state
def test_bf16_rne_against_hand_cases_and_torch(orc):
    """Reading Z9: RNE to bf16. Hand cases: exact ties go to even; values
    just above a tie go up. Float32-representable values must match torch's
    float32 -> bfloat16 conversion (RNE)."""
    one = 1.0
    cases = {one + 2 ** -8: 0x3F80, one + 3 * 2 ** -8: 0x3F82, one + 2 ** -8 + 2 ** -30: 0x3F81,
             -(one + 2 ** -8): 0xBF80, 0.0: 0x0000}
    bits = orc.bf16_rne(np.array(list(cases.keys())))
    assert [int(b) for b in bits] == list(cases.values())
    rng = np.random.default_rng(0)
    f = (rng.standard_normal(10000) * 10.0 ** rng.uniform(-20, 20, 10000)).astype(np.float32)
    tb = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(orc.bf16_rne(f.astype(np.float64)), tb)


def test_bf16_state_inputs_are_promoted_exactly(orc):
    x = synth.state_tree(61, [1000])
    mb, vb = synth.to_bf16_bits(x["m"]), synth.to_bf16_bits(x["v"])
    u_b, m_b, v_b = orc.adam_fwd(x["g"], mb, vb, 10, 1e-3, 0.9, 0.999, 1e-8, state_bf16=True)
    mf = orc.bf16_to_f64(mb).astype(np.float32)
    vf = orc.bf16_to_f64(vb).astype(np.float32)
    u_f, m_f, v_f = orc.adam_fwd(x["g"], mf, vf, 10, 1e-3, 0.9, 0.999, 1e-8)
    np.testing.assert_array_equal(u_b, u_f)
    np.testing.assert_array_equal(m_b, m_f)


# ----------------------------------------------- K-step sweep (row a9)
def _quad(seed, n):
    return synth.quadratic_problem(seed, n)


@pytest.mark.parametrize("K", [1, 3, 5, 10])
def test_sweep_sgd_closed_form(orc, K):
    """SURVEY P6 / S:281: plain SGD on 1/2 a (theta-phi)^2 gives
    theta_K = phi + (1 - lr a)^K (theta0 - phi); so
    phi_bar = (theta_K - y)(1 - (1-lr a)^K), theta0_bar = (theta_K - y)(1-lr a)^K,
    lr_bar = sum (theta_K - y) * (-K a (1-lr a)^(K-1) (theta0 - phi))."""
    q = _quad(3, 64)
    a, th0, phi, y = (q[k].astype(np.float64) for k in ("a", "theta0", "phi", "y"))
    for lr in (0.1, 0.5):
        r = orc.sweep_quadratic("sgd", q["a"], q["theta0"], q["phi"], q["y"], K, [lr, 0.0, 0.0])
        c = (1 - lr * a) ** K
        thK = phi + c * (th0 - phi)
        np.testing.assert_allclose(r["thetaK"], thK, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(r["phi_bar"], (thK - y) * (1 - c), rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(r["theta0_bar"], (thK - y) * c, rtol=1e-10, atol=1e-13)
        lr_bar = np.sum((thK - y) * (-K * a * (1 - lr * a) ** (K - 1) * (th0 - phi)))
        assert r["hyper_bar"][0] == pytest.approx(lr_bar, rel=1e-10)
        assert r["loss"] == pytest.approx(0.5 * np.sum((thK - y) ** 2), rel=1e-12)


@pytest.mark.parametrize("nesterov", [False, True])
def test_sweep_momentum_closed_form(orc, nesterov):
    """with momentum, [theta-phi; b] evolves by T = [[1-lr a, -lr mu],
    [a, mu]] (Nesterov: [[1-lr a(1+mu), -lr mu^2], [a, mu]]); b_0 = 0 so
    dtheta_K/dtheta0 = (T^K)_00 and dtheta_K/dphi = 1 - (T^K)_00."""
    q = _quad(4, 32)
    a, th0, phi, y = (q[k].astype(np.float64) for k in ("a", "theta0", "phi", "y"))
    lr, mu, K = 0.2, 0.9, 5
    r = orc.sweep_quadratic("sgd", q["a"], q["theta0"], q["phi"], q["y"], K,
                            [lr, mu, 1.0 if nesterov else 0.0])
    for i in range(32):
        if nesterov:
            T = np.array([[1 - lr * a[i] * (1 + mu), -lr * mu * mu], [a[i], mu]])
        else:
            T = np.array([[1 - lr * a[i], -lr * mu], [a[i], mu]])
        c = np.linalg.matrix_power(T, K)[0, 0]
        thK = phi[i] + c * (th0[i] - phi[i])
        assert r["thetaK"][i] == pytest.approx(thK, rel=1e-12, abs=1e-14)
        assert r["theta0_bar"][i] == pytest.approx((thK - y[i]) * c, rel=1e-10, abs=1e-13)
        assert r["phi_bar"][i] == pytest.approx((thK - y[i]) * (1 - c), rel=1e-10, abs=1e-13)


@pytest.mark.parametrize("kind,hp", [("adam", [1e-2, 0.9, 0.999, 1e-8, 0.0]),
                                     ("rmsprop", [1e-2, 0.99, 1e-8]),
                                     ("sgd", [0.1, 0.9, 0.0]), ("sgd", [0.1, 0.9, 1.0])])
def test_sweep_vs_complex_step(orc, kind, hp):
    """The reverse sweep (VJP of every step, in reverse, plus the quadratic's
    Hessian) equals the complex-step derivative of the K-step forward map."""
    K = 5
    q = _quad(5, 40)
    a, th0, phi, y = (q[k].astype(np.float64) for k in ("a", "theta0", "phi", "y"))
    r = orc.sweep_quadratic(kind, q["a"], q["theta0"], q["phi"], q["y"], K, hp, prec=1)
    nest = bool(hp[2]) if kind == "sgd" else False
    hpf = hp[:2] if kind == "sgd" else hp
    thK = orc.sweep_forward_complex(kind, a, th0, phi, K, hpf, nest).real
    res = thK - y
    d_phi = orc.sweep_forward_complex(kind, a, th0, phi + 1j * H, K, hpf, nest).imag / H
    d_th0 = orc.sweep_forward_complex(kind, a, th0 + 1j * H, phi, K, hpf, nest).imag / H
    np.testing.assert_allclose(r["phi_bar"], res * d_phi, rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(r["theta0_bar"], res * d_th0, rtol=1e-7, atol=1e-12)
    nh = {"adam": 4, "rmsprop": 3, "sgd": 2}[kind]
    for k in range(nh):
        hpc = np.array(hpf, dtype=np.complex128)
        hpc[k] += 1j * H
        cs = np.sum(res * orc.sweep_forward_complex(kind, a, th0, phi, K, hpc, nest).imag / H)
        assert r["hyper_bar"][k] == pytest.approx(cs, rel=1e-7, abs=1e-9)


def test_sweep_adam_vs_central_fd(orc):
    """meta-gradient of a 5-step Adam inner loop matches central
    finite differences over phi (rel <= 1e-4)."""
    q = _quad(6, 6)
    a, th0, phi, y = (q[k].astype(np.float64) for k in ("a", "theta0", "phi", "y"))
    hp = [1e-2, 0.9, 0.999, 1e-8, 0.0]
    r = orc.sweep_quadratic("adam", q["a"], q["theta0"], q["phi"], q["y"], 5, hp, prec=1)

    def L(ph):
        thK = orc.sweep_forward_complex("adam", a, th0, ph, 5, hp).real
        return 0.5 * (thK - y) ** 2

    h = 1e-6
    fd = (L(phi + h) - L(phi - h)) / (2 * h)
    np.testing.assert_allclose(r["phi_bar"], fd, rtol=1e-4, atol=1e-9)


# ------------------------------------ magnitude twins (tolerance, Z10)
def test_mag_twins_bound_the_values(orc):
    """Every magnitude twin is the same expression tree over |.|, so it
    bounds the absolute value of the exact result (a property any slip in
    the twin -- a missing term -- would eventually break)."""
    x = synth.state_tree(71, [3000, 97])
    g, m, v, du, dm1, dv1 = (x[k] for k in ("g", "m", "v", "du", "dm1", "dv1"))
    for t in (1, 10):
        hp = (0.5, 0.9, 0.999, 1e-8)
        mag = orc.adam_mag(g, m, v, du, dm1, dv1, t, *hp)
        u, m1, v1 = orc.adam_fwd(g, m, v, t, *hp, prec=1)
        r = orc.adam_vjp(g, m, v, du, dm1, dv1, t, *hp, prec=1)
        for k, val in (("u", u), ("m1", m1), ("v1", v1), ("dg", r["dg"]), ("dm", r["dm"]),
                       ("dv", r["dv"])):
            assert np.all(np.abs(val) <= mag[k] * (1 + 1e-9) + 1e-300), k
        assert np.all(np.abs(r["dhp"]) <= mag["dhp"] * (1 + 1e-9))
    magr = orc.rmsprop_mag(g, v, du, dv1, 0.3, 0.99, 1e-8)
    rr = orc.rmsprop_vjp(g, v, du, dv1, 0.3, 0.99, 1e-8, prec=1)
    ur, vr = orc.rmsprop_fwd(g, v, 0.3, 0.99, 1e-8, prec=1)
    for k, val in (("u", ur), ("v1", vr), ("dg", rr["dg"]), ("dv", rr["dv"])):
        assert np.all(np.abs(val) <= magr[k] * (1 + 1e-9) + 1e-300), k
    for nest in (False, True):
        mags = orc.sgd_mag(g, m, du, dm1, 0.1, 0.9, nest)
        rs = orc.sgd_vjp(g, m, du, dm1, 0.1, 0.9, nest, prec=1)
        us, bs = orc.sgd_fwd(g, m, 0.1, 0.9, nest, prec=1)
        for k, val in (("u", us), ("b1", bs), ("dg", rs["dg"]), ("db", rs["db"])):
            assert np.all(np.abs(val) <= mags[k] * (1 + 1e-9) + 1e-300), k


def _f32_adam_dg(g, du, lr, b1, b2, eps, reduced):
    """numpy float32 emulation of an fp32 kernel's dg at t=1 from zero state
    with zero m'/v' cotangents: the textbook chain rule vs the reduced form."""
    f = np.float32
    g, du = g.astype(f), du.astype(f)
    b1, b2, lr, eps = f(b1), f(b2), f(lr), f(eps)
    bc1, bc2 = f(1) - b1, f(1) - b2
    A, C = (f(1) - b1) / bc1, (f(1) - b2) / bc2
    mhat = A * g
    s = np.sqrt(C * g * g)
    d = s + eps
    if reduced:
        rs = np.where(s == 0, f(0), f(1) / np.where(s == 0, f(1), s))
        return -du * lr * (A * eps + (f(0) - f(0) * C * g) * rs) / (d * d)
    dmhat = du * (-lr / d)
    dd = du * (lr * mhat / (d * d))
    dvhat = np.where(s == 0, f(0), dd / (f(2) * np.where(s == 0, f(1), s)))
    return dmhat / bc1 * (f(1) - b1) + dvhat / bc2 * (f(1) - b2) * f(2) * g


def test_mag_criterion_has_teeth(orc):
    """The fp32 criterion |x-ref| <= 1e-6 + 1e-5 mag is passed by an fp32
    evaluation of the reduced form and failed by an fp32 evaluation of the
    textbook chain rule (100% vs ~7% at lr=1, t=1)."""
    rng = np.random.default_rng(3)
    n = 1 << 16
    g = (1e-2 * rng.standard_normal(n)).astype(np.float32)
    du = rng.standard_normal(n).astype(np.float32)
    hp = (1.0, 0.9, 0.999, 1e-8)
    r = orc.adam_vjp(g, None, None, du, None, None, 1, *hp, prec=1)
    mag = orc.adam_mag(g, None, None, du, None, None, 1, *hp)
    ok = lambda x: np.abs(x.astype(np.float64) - r["dg"]) <= 1e-6 + 1e-5 * np.maximum(
        mag["dg"], np.abs(r["dg"]))
    assert ok(_f32_adam_dg(g, du, *hp, reduced=True)).mean() == 1.0
    assert ok(_f32_adam_dg(g, du, *hp, reduced=False)).mean() < 0.5


# ------------------------------------ optimizer variants (NEXT-1 pins)
def _torch_steps_p(opt_cls, kwargs, grads, p0):
    p = torch.tensor(p0, dtype=torch.float64, requires_grad=True)
    opt = opt_cls([p], **kwargs)
    ups, ps = [], []
    for g in grads:
        before = p.detach().clone()
        ps.append(before.numpy().copy())
        p.grad = torch.as_tensor(g, dtype=torch.float64)
        opt.step()
        ups.append((p.detach() - before).numpy())
    return ups, ps


@pytest.mark.parametrize("maximize", [False, True])
@pytest.mark.parametrize("decoupled", [False, True])
def test_adam_variants_match_torch_optim(orc, maximize, decoupled):
    """Weight decay (torch.optim.Adam L2 / torch.optim.AdamW decoupled) and
    maximize: the oracle's variant forward reproduces torch.optim in float64
    over 8 steps (reading N1)."""
    rng = np.random.default_rng(11)
    n = 129
    grads = [(rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 0, n)) for _ in range(8)]
    p0 = rng.standard_normal(n)
    wd, lr = 0.05, 1e-2
    cls = torch.optim.AdamW if decoupled else torch.optim.Adam
    ups, ps = _torch_steps_p(cls, dict(lr=lr, weight_decay=wd, maximize=maximize), grads, p0)
    m = v = np.zeros(n)
    for t, (g, th) in enumerate(zip(grads, ps), 1):
        u, m, v = (x.real for x in orc.adam_fwd_ex_complex(
            g, m, v, th, t, [lr, 0.9, 0.999, 1e-8, 0.0], np.full(n, lr), wd, decoupled, maximize))
        np.testing.assert_allclose(u, ups[t - 1], rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("maximize", [False, True])
def test_rmsprop_sgd_variants_match_torch_optim(orc, maximize):
    rng = np.random.default_rng(12)
    n = 77
    grads = [rng.standard_normal(n) for _ in range(6)]
    p0 = rng.standard_normal(n)
    ups, ps = _torch_steps_p(torch.optim.RMSprop, dict(lr=1e-2, alpha=0.9, weight_decay=0.1,
                                                       maximize=maximize), grads, p0)
    v = np.zeros(n)
    for t, (g, th) in enumerate(zip(grads, ps), 1):
        u, v = (x.real for x in orc.rmsprop_fwd_ex_complex(g, v, th, [1e-2, 0.9, 1e-8],
                                                            np.full(n, 1e-2), 0.1, maximize))
        np.testing.assert_allclose(u, ups[t - 1], rtol=1e-9, atol=1e-14)
    for nest in (False, True):
        ups, ps = _torch_steps_p(torch.optim.SGD, dict(lr=0.1, momentum=0.9, nesterov=nest,
                                                       weight_decay=0.1, maximize=maximize),
                                 grads, p0)
        b = np.zeros(n)
        for t, (g, th) in enumerate(zip(grads, ps), 1):
            u, b = (x.real for x in orc.sgd_fwd_ex_complex(g, b, th, [0.1, 0.9], np.full(n, 0.1),
                                                            nest, 0.1, maximize))
            np.testing.assert_allclose(u, ups[t - 1], rtol=1e-9, atol=1e-14)


def test_variants_reduce_to_base(orc):
    """wd = 0, maximize off, one lr for every leaf: the variant equals the
    plain step bitwise (dtheta = 0)."""
    x = synth.state_tree(81, [300, 200])
    th = x["du"]
    off = synth.offsets_of([300, 200])
    hp = (1e-3, 0.9, 0.999, 1e-8)
    a = orc.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], 4, *hp)
    b = orc.adam_vjp_ex(x["g"], x["m"], x["v"], th, x["du"], x["dm1"], x["dv1"], 4, *hp,
                        lr_leaf=[1e-3, 1e-3], offsets=off)
    for k in ("dg", "dm", "dv"):
        np.testing.assert_array_equal(a[k], b[k])
    assert np.all(b["dtheta"] == 0)
    # d/dwd at wd = 0 (L2): sum of dg~ * theta
    assert b["dhp"][4] == pytest.approx(np.sum(a["dg"] * th.astype(np.float64)), rel=1e-12)
    np.testing.assert_allclose(a["dhp"], b["dhp"][:4], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("decoupled", [False, True])
@pytest.mark.parametrize("maximize", [False, True])
def test_adam_variant_vjp_vs_complex_step(orc, decoupled, maximize):
    """Every VJP output of the variant (dg, dm, dv, dtheta, the five global
    hyper-gradients and the per-leaf lr gradients) equals the complex-step
    derivative of the (torch-pinned) variant forward."""
    leaves = [60, 90, 50]
    off = synth.offsets_of(leaves)
    x = synth.state_tree(91, leaves, zero_frac=0.0)
    th = synth.normal(91, synth.S_THETA0, 200).astype(np.float32)
    lr_leaf = np.array([1e-2, 3e-2, 5e-3])
    lr_e = np.repeat(lr_leaf, leaves)
    hp = np.array([0.0, 0.9, 0.999, 1e-8, 0.0])
    wd, t = 0.07, 6
    gd, md, vd, td = (a.astype(np.float64) for a in (x["g"], x["m"], x["v"], th))
    cot = (x["du"].astype(np.float64), x["dm1"].astype(np.float64), x["dv1"].astype(np.float64))
    contract = lambda outs: sum(c * o.imag / H for c, o in zip(cot, outs))
    F = lambda g=gd, m=md, v=vd, th_=td, hp_=hp, lr=lr_e, w=wd: orc.adam_fwd_ex_complex(
        g, m, v, th_, t, hp_, lr, w, decoupled, maximize)
    r = orc.adam_vjp_ex(x["g"], x["m"], x["v"], th, x["du"], x["dm1"], x["dv1"], t, 0.0, 0.9,
                        0.999, 1e-8, weight_decay=wd, decoupled=decoupled, maximize=maximize,
                        lr_leaf=lr_leaf, offsets=off, prec=1)
    for name, kw in (("dg", dict(g=gd + 1j * H)), ("dm", dict(m=md + 1j * H)),
                     ("dv", dict(v=vd + 1j * H)), ("dtheta", dict(th_=td + 1j * H))):
        cs = contract(F(**kw))
        np.testing.assert_allclose(r[name], cs, rtol=1e-8, atol=1e-12 * np.abs(cs).max())
    for k in (1, 2, 3):  # b1, b2, eps
        hpc = hp.astype(np.complex128)
        hpc[k] += 1j * H
        assert r["dhp"][k] == pytest.approx(contract(F(hp_=hpc)).sum(), rel=1e-8, abs=1e-12)
    assert r["dhp"][4] == pytest.approx(contract(F(w=wd + 1j * H)).sum(), rel=1e-8)
    for l in range(3):  # per-leaf lr gradients
        lrc = lr_e.astype(np.complex128)
        lrc[off[l]:off[l + 1]] += 1j * H
        assert r["dhp_leaf"][l, 0] == pytest.approx(contract(F(lr=lrc)).sum(), rel=1e-8)
    assert r["dhp"][0] == pytest.approx(r["dhp_leaf"][:, 0].sum(), rel=1e-12)


@pytest.mark.parametrize("kind", ["rmsprop", "sgd", "sgd_nesterov"])
def test_rms_sgd_variant_vjp_vs_complex_step(orc, kind):
    leaves = [70, 80]
    off = synth.offsets_of(leaves)
    x = synth.state_tree(92, leaves, zero_frac=0.0)
    th = synth.normal(92, synth.S_THETA0, 150).astype(np.float32)
    lr_leaf = np.array([2e-2, 7e-3])
    lr_e = np.repeat(lr_leaf, leaves)
    wd = 0.03
    s = x["v"] if kind == "rmsprop" else x["m"]
    gd, sd, td = (a.astype(np.float64) for a in (x["g"], s, th))
    cot = (x["du"].astype(np.float64), x["dm1"].astype(np.float64))
    contract = lambda outs: sum(c * o.imag / H for c, o in zip(cot, outs))
    nest = kind == "sgd_nesterov"
    if kind == "rmsprop":
        hp = np.array([0.0, 0.95, 1e-8])
        F = lambda g=gd, st=sd, th_=td, hp_=hp, lr=lr_e, w=wd: orc.rmsprop_fwd_ex_complex(
            g, st, th_, hp_, lr, w, True)
        r = orc.rmsprop_vjp_ex(x["g"], s, th, x["du"], x["dm1"], 0.0, 0.95, 1e-8, weight_decay=wd,
                               maximize=True, lr_leaf=lr_leaf, offsets=off, prec=1)
        sname, hps = "dv", (1, 2)
    else:
        hp = np.array([0.0, 0.9])
        F = lambda g=gd, st=sd, th_=td, hp_=hp, lr=lr_e, w=wd: orc.sgd_fwd_ex_complex(
            g, st, th_, hp_, lr, nest, w, True)
        r = orc.sgd_vjp_ex(x["g"], s, th, x["du"], x["dm1"], 0.0, 0.9, nest, weight_decay=wd,
                           maximize=True, lr_leaf=lr_leaf, offsets=off, prec=1)
        sname, hps = "db", (1,)
    for name, kw in (("dg", dict(g=gd + 1j * H)), (sname, dict(st=sd + 1j * H)),
                     ("dtheta", dict(th_=td + 1j * H))):
        np.testing.assert_allclose(r[name], contract(F(**kw)), rtol=1e-8, atol=1e-14)
    for k in hps:
        hpc = hp.astype(np.complex128)
        hpc[k] += 1j * H
        assert r["dhp"][k] == pytest.approx(contract(F(hp_=hpc)).sum(), rel=1e-8)
    assert r["dhp"][-1] == pytest.approx(contract(F(w=wd + 1j * H)).sum(), rel=1e-8)
    for l in range(2):
        lrc = lr_e.astype(np.complex128)
        lrc[off[l]:off[l + 1]] += 1j * H
        assert r["dhp_leaf"][l, 0] == pytest.approx(contract(F(lr=lrc)).sum(), rel=1e-8)


# ------------------------- centred / momentum RMSProp (NEXT-1 pins, N4)
def _torch_rmsprop_one_step(g, v, a, b, th, lr, alpha, eps, momentum, centered, wd, maximize):
    """torch.optim.RMSprop (float64), one step from the given state."""
    p = torch.tensor(th, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.RMSprop([p], lr=lr, alpha=alpha, eps=eps, momentum=momentum,
                              centered=centered, weight_decay=wd, maximize=maximize)
    p.grad = torch.zeros_like(p)
    opt.step()  # creates the state tensors
    st = opt.state[p]
    with torch.no_grad():
        p.copy_(torch.as_tensor(th, dtype=torch.float64))
        st["square_avg"].copy_(torch.as_tensor(v, dtype=torch.float64))
        if centered:
            st["grad_avg"].copy_(torch.as_tensor(a, dtype=torch.float64))
        if momentum > 0:
            st["momentum_buffer"].copy_(torch.as_tensor(b, dtype=torch.float64))
    p.grad = torch.as_tensor(g, dtype=torch.float64)
    opt.step()
    out = dict(u=(p.detach() - torch.as_tensor(th, dtype=torch.float64)).numpy(),
               v1=st["square_avg"].numpy())
    if centered:
        out["a1"] = st["grad_avg"].numpy()
    if momentum > 0:
        out["b1"] = st["momentum_buffer"].numpy()
    return out


@pytest.mark.parametrize("centered", [False, True])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
@pytest.mark.parametrize("maximize", [False, True])
def test_rmsprop_cm_matches_torch_optim(orc, centered, momentum, maximize):
    """The centred / momentum RMSProp forward (reading N4) reproduces one
    torch.optim.RMSprop step in float64 from a warm state: update, square
    average, gradient average and momentum buffer."""
    x = synth.rms_cm_tree(0xC7, [200, 57], zero_frac=0.02)
    kw = dict(lr=1e-2, alpha=0.95, eps=1e-6, momentum=momentum, centered=centered)
    wd = 0.05
    ref = _torch_rmsprop_one_step(x["g"], x["v"], x["a"], x["b"], x["theta"], wd=wd,
                                  maximize=maximize, **kw)
    u, v1, a1, b1 = orc.rmsprop_cm_fwd(x["g"], x["v"], x["a"], x["b"], x["theta"],
                                       weight_decay=wd, maximize=maximize, **kw)
    np.testing.assert_allclose(u, ref["u"], rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(v1, ref["v1"], rtol=1e-12, atol=1e-300)
    if centered:
        np.testing.assert_allclose(a1, ref["a1"], rtol=1e-12, atol=1e-300)
    if momentum > 0:
        np.testing.assert_allclose(b1, ref["b1"], rtol=1e-10, atol=1e-15)


def test_rmsprop_cm_reduces_to_plain_rmsprop(orc):
    """Not centred, momentum 0: update, v' and every VJP output equal the
    plain RMSProp variant's; the momentum gradient is Sigma (db1 - lr du) b."""
    x = synth.rms_cm_tree(0xC8, [300])
    kw = dict(weight_decay=0.02, maximize=True)
    u, v1, _, _ = orc.rmsprop_cm_fwd(x["g"], x["v"], None, None, x["theta"], 1e-2, 0.9, 1e-8, **kw)
    u0, v0 = orc.rmsprop_fwd_ex(x["g"], x["v"], x["theta"], 1e-2, 0.9, 1e-8, **kw)
    np.testing.assert_allclose(u, u0, rtol=1e-15, atol=0)
    np.testing.assert_array_equal(v1, v0)
    r = orc.rmsprop_cm_vjp(x["g"], x["v"], None, x["b"], x["theta"], x["du"], x["dv1"], None,
                           None, 1e-2, 0.9, 1e-8, **kw)
    r0 = orc.rmsprop_vjp_ex(x["g"], x["v"], x["theta"], x["du"], x["dv1"], 1e-2, 0.9, 1e-8, **kw)
    for k in ("dg", "dv", "dtheta"):
        np.testing.assert_allclose(r[k], r0[k], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(r["dhp"][[0, 1, 2, 4]], r0["dhp"], rtol=1e-12)
    assert r["dhp"][3] == pytest.approx(
        np.sum(-1e-2 * x["du"].astype(np.float64) * x["b"].astype(np.float64)), rel=1e-12)


@pytest.mark.parametrize("centered", [False, True])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_rmsprop_cm_vjp_vs_complex_step(orc, centered, momentum):
    """Every VJP output of the centred / momentum RMSProp step (dg, dv, da,
    db, dtheta, the five global hyper-gradients and the per-leaf lr
    gradients) equals the complex-step derivative of the torch-pinned
    forward, contracted with the four cotangents."""
    leaves = [90, 60]
    off = synth.offsets_of(leaves)
    x = synth.rms_cm_tree(0xC9, leaves, zero_frac=0.0)
    lr_leaf = np.array([2e-2, 6e-3])
    lr_e = np.repeat(lr_leaf, leaves)
    hp = np.array([0.0, 0.93, 1e-7, momentum])
    wd = 0.04
    d = {k: x[k].astype(np.float64) for k in x}
    cot = (d["du"], d["dv1"], d["da1"], d["db1"])
    contract = lambda outs: sum(c * o.imag / H for c, o in zip(cot, outs))

    def F(g=d["g"], v=d["v"], a=d["a"], b=d["b"], th=d["theta"], hp_=hp, lr=lr_e, w=wd):
        return orc.rmsprop_cm_fwd_complex(g, v, a, b, th, hp_, lr, centered, w, True)

    r = orc.rmsprop_cm_vjp(x["g"], x["v"], x["a"], x["b"], x["theta"], x["du"], x["dv1"],
                           x["da1"], x["db1"], 0.0, 0.93, 1e-7, momentum=momentum,
                           centered=centered, weight_decay=wd, maximize=True, lr_leaf=lr_leaf,
                           offsets=off, prec=1)
    for name, kw in (("dg", dict(g=d["g"] + 1j * H)), ("dv", dict(v=d["v"] + 1j * H)),
                     ("da", dict(a=d["a"] + 1j * H)), ("db", dict(b=d["b"] + 1j * H)),
                     ("dtheta", dict(th=d["theta"] + 1j * H))):
        cs = contract(F(**kw))
        np.testing.assert_allclose(r[name], cs, rtol=1e-8, atol=1e-12 * np.abs(cs).max())
    for k in (1, 2, 3):  # alpha, eps, momentum
        hpc = hp.astype(np.complex128)
        hpc[k] += 1j * H
        assert r["dhp"][k] == pytest.approx(contract(F(hp_=hpc)).sum(), rel=1e-8, abs=1e-12)
    assert r["dhp"][4] == pytest.approx(contract(F(w=wd + 1j * H)).sum(), rel=1e-8)
    for l in range(2):
        lrc = lr_e.astype(np.complex128)
        lrc[off[l]:off[l + 1]] += 1j * H
        assert r["dhp_leaf"][l, 0] == pytest.approx(contract(F(lr=lrc)).sum(), rel=1e-8)


def test_rmsprop_cm_zero_point_conventions(orc):
    """g = a = v = 0 with eps = 0: q = 0, d = 0, so w := 0 (u = -lr mu b),
    and the q-adjoint is 0 (no inf/nan anywhere)."""
    z = np.zeros(4, np.float32)
    b = np.array([1.0, -2.0, 0.5, 0.0], np.float32)
    u, v1, a1, b1 = orc.rmsprop_cm_fwd(z, z, z, b, z, 0.1, 0.9, 0.0, momentum=0.5, centered=True)
    np.testing.assert_array_equal(u, -0.1 * 0.5 * b.astype(np.float64))
    r = orc.rmsprop_cm_vjp(z, z, z, b, z, np.ones(4, np.float32), np.ones(4, np.float32),
                           np.ones(4, np.float32), np.ones(4, np.float32), 0.1, 0.9, 0.0,
                           momentum=0.5, centered=True)
    for k in ("dg", "dv", "da", "db"):
        assert np.all(np.isfinite(r[k]))
    np.testing.assert_allclose(r["dg"], 0.1 * 1.0, rtol=1e-15)  # (1-alpha) da1
    np.testing.assert_allclose(r["dv"], 0.9, rtol=1e-15)  # alpha dv1


# --------------------------------------------- zero-order ES (NEXT-3 pins)
def test_es_noise_is_standard_normal_and_independent(orc):
    """The counter-based noise (reading N3) has the moments of N(0,1), matches
    the normal CDF at a few quantiles, and is uncorrelated across samples
    and elements; the same seed reproduces it, another seed does not."""
    z = orc.es_noise(4096, 64, seed=11)
    flat = z.ravel()
    N = flat.size
    assert abs(flat.mean()) < 5 / np.sqrt(N)
    assert abs(flat.var() - 1) < 5 * np.sqrt(2 / N)
    assert abs(np.mean(flat ** 4) - 3) < 5 * np.sqrt(96 / N)
    from math import erf
    for q in (-2.0, -1.0, 0.0, 0.5, 1.5):
        p = 0.5 * (1 + erf(q / np.sqrt(2)))
        assert abs(np.mean(flat < q) - p) < 5 * np.sqrt(p * (1 - p) / N)
    c = np.corrcoef(z[:8])  # across samples
    assert np.max(np.abs(c - np.eye(8))) < 5 / np.sqrt(4096)
    assert abs(np.corrcoef(z[:, :-1].ravel(), z[:, 1:].ravel())[0, 1]) < 5 / np.sqrt(N)
    np.testing.assert_array_equal(z, orc.es_noise(4096, 64, seed=11))
    assert not np.array_equal(z, orc.es_noise(4096, 64, seed=12))


def test_es_constant_f_antithetic_is_exactly_zero(orc):
    g, _ = orc.es_grad(np.full(2 * 50, 3.25), 100, 50, 0.1, seed=3, antithetic=True)
    assert np.all(g == 0)


@pytest.mark.parametrize("antithetic", [True, False])
def test_es_linear_f_estimates_c(orc, antithetic):
    """SPEC zero-order-diff example: f(theta) = c.theta; E[g] = c (E[zz^T] = I);
    each antithetic sample contributes exactly (c.z) z. Checked at 5 standard
    errors with n = 20000."""
    d, n, sigma = 6, 20000, 0.05
    c = np.array([1.0, -2.0, 0.5, 0.0, 3.0, -1.0])
    theta = np.linspace(-1, 1, d).astype(np.float32)
    pts = orc.es_perturb(theta, n, sigma, seed=5, antithetic=antithetic)
    f = pts @ c
    g, _ = orc.es_grad(f, d, n, sigma, seed=5, antithetic=antithetic)
    if antithetic:
        se = np.sqrt((c @ c + c ** 2) / n)
    else:  # naive carries f(theta)/sigma noise too
        f0 = float(theta.astype(np.float64) @ c)
        se = np.sqrt((c @ c + c ** 2 + (f0 / sigma) ** 2) / n)
    assert np.all(np.abs(g - c) < 5 * se)
    # antithetic: the per-sample contributions are exactly (c.z) z
    if antithetic:
        z = orc.es_noise(d, 4, seed=5)
        g4, _ = orc.es_grad(f[:8], d, 4, sigma, seed=5)
        np.testing.assert_allclose(g4, np.mean([(c @ zi) * zi for zi in z], axis=0), rtol=1e-9,
                                   atol=1e-12)


def test_es_quadratic_smoothing_identity(orc):
    """f = 1/2 ||theta||^2: f~_sigma = f + sigma^2 d/2, so E[g] = theta exactly
    for any sigma (Gaussian-moment identity); 5 standard errors, n = 20000."""
    d, n, sigma = 5, 20000, 0.1
    theta = np.array([0.3, -1.2, 2.0, 0.0, 0.7], np.float32)
    pts = orc.es_perturb(theta, n, sigma, seed=9, antithetic=True)
    f = 0.5 * np.sum(pts ** 2, axis=1)
    g, _ = orc.es_grad(f, d, n, sigma, seed=9)
    th = theta.astype(np.float64)
    se = np.sqrt((th @ th + th ** 2) / n)
    assert np.all(np.abs(g - th) < 5 * se + 1e-12)


# ------------------------------------ implicit-gradient solvers (NEXT-4 pins)
def _spd(n, seed, shift=1.0):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    return M.T @ M / n + shift * np.eye(n)


def test_cg_dense_hand_cases_and_library_solve(orc):
    """SPEC implicit-diff examples: A = I -> x = b in one iteration;
    A = diag(1, 2), b = (1, 2) -> x = (1, 1); random SPD 8x8 matches the
    dense LU solve of numpy.linalg.solve (a different method) to 1e-8."""
    b = np.array([0.3, -1.0, 2.0])
    np.testing.assert_allclose(orc.cg_dense(np.eye(3), b, 1), b, rtol=1e-15)
    np.testing.assert_allclose(orc.cg_dense(np.diag([1.0, 2.0]), [1.0, 2.0], 2), [1.0, 1.0],
                               rtol=1e-14)
    A = _spd(8, 1)
    b = np.random.default_rng(2).standard_normal(8)
    np.testing.assert_allclose(orc.cg_dense(A, b, 30), np.linalg.solve(A, b), rtol=1e-8)


def test_cg_iteration_terminates_in_n_steps(orc):
    """n textbook CG iterations solve an n x n SPD system (finite termination
    in exact arithmetic): cg_iter chained n times reaches the dense solve."""
    n = 6
    A = _spd(n, 3, shift=2.0)
    b = np.random.default_rng(4).standard_normal(n)
    x, r, p = np.zeros(n), b.copy(), b.copy()
    rr = float(b @ b)
    for _ in range(n):
        Ap = A @ p
        # cg_iter takes fp32 inputs: use float32-exact values via a scaled grid
        x, r, p, s = orc.cg_iter(x.astype(np.float32), r.astype(np.float32),
                                 p.astype(np.float32), Ap.astype(np.float32), rr)
        rr = s["rr_new"]
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=2e-3, atol=2e-3)


def test_cg_iteration_scalars(orc):
    rng = np.random.default_rng(5)
    x, r, p, Ap = (rng.standard_normal(50).astype(np.float32) for _ in range(4))
    rr = float(r.astype(np.float64) @ r.astype(np.float64))
    x1, r1, p1, s = orc.cg_iter(x, r, p, Ap, rr)
    pap = float(p.astype(np.float64) @ Ap.astype(np.float64))
    assert s["pAp"] == pytest.approx(pap, rel=1e-14)
    assert s["alpha"] == pytest.approx(rr / pap, rel=1e-14)
    assert s["rr_new"] == pytest.approx(float(r1 @ r1), rel=1e-12)
    np.testing.assert_allclose(p1, r1 + s["beta"] * p.astype(np.float64), rtol=1e-14)


def test_neumann_series_closed_forms(orc):
    """SPEC: A = I, alpha = 1 -> x = b for any K; A = 2I, alpha = 0.25:
    x_K = (b/2)(1 - (1/2)^(K+1)) (geometric series) -> b/2, K = 20 within 1e-5."""
    b = np.array([1.0, -4.0, 0.5])
    for K in (0, 3, 10):
        np.testing.assert_allclose(orc.neumann_dense(np.eye(3), b, K, 1.0), b, rtol=1e-15)
    for K in (0, 5, 20):
        x = orc.neumann_dense(2 * np.eye(3), b, K, 0.25)
        np.testing.assert_allclose(x, b / 2 * (1 - 0.5 ** (K + 1)), rtol=1e-14)
    assert np.max(np.abs(orc.neumann_dense(2 * np.eye(3), b, 20, 0.25) - b / 2)) < 1e-5


# ------------------- tolerance twins: bounds, teeth, looseness (Z10, r2)
def _per_elem_terms(fn, n):
    """Per-element hyper-gradient terms from an oracle VJP: every element its
    own leaf (offsets 0..n), so dhp_leaf[i] is element i's term."""
    return fn(np.arange(n + 1, dtype=np.int64))["dhp_leaf"].T


def _assert_bounds(name, val, mag):
    val, mag = np.abs(np.asarray(val, np.float64)), np.asarray(mag, np.float64)
    bad = ~(val <= mag * (1 + 1e-9) + 1e-300)
    assert not bad.any(), (name, np.flatnonzero(bad)[:5], val[bad][:5], mag[bad][:5])


def test_base_hyper_twins_bound_each_term(orc):
    """Per-element hyper twins (the 'h' arrays the per-leaf bars sum) bound
    every element's hyper-gradient term, not only the sums."""
    x = synth.state_tree(72, [2000, 33])
    g, m, v, du, dm1, dv1 = (x[k] for k in ("g", "m", "v", "du", "dm1", "dv1"))
    n = g.size
    for t in (1, 10):
        hp = (0.5, 0.9, 0.999, 1e-8)
        mag = orc.adam_mag(g, m, v, du, dm1, dv1, t, *hp)
        terms = _per_elem_terms(lambda o: orc.adam_vjp(g, m, v, du, dm1, dv1, t, *hp, prec=1,
                                                       offsets=o), n)
        _assert_bounds("adam h", terms, mag["h"])
        np.testing.assert_allclose(mag["h"].sum(1), mag["dhp"], rtol=1e-12)
    mr = orc.rmsprop_mag(g, v, du, dv1, 0.3, 0.99, 1e-8)
    tr = _per_elem_terms(lambda o: orc.rmsprop_vjp(g, v, du, dv1, 0.3, 0.99, 1e-8, prec=1,
                                                   offsets=o), n)
    _assert_bounds("rmsprop h", tr, mr["h"])
    for nest in (False, True):
        ms = orc.sgd_mag(g, m, du, dm1, 0.1, 0.9, nest)
        ts = _per_elem_terms(lambda o: orc.sgd_vjp(g, m, du, dm1, 0.1, 0.9, nest, prec=1,
                                                   offsets=o), n)
        _assert_bounds("sgd h", ts, ms["h"])


def _ex_case(seed=73):
    leaves = [1500, 1, 400, 7]
    x = synth.state_tree(seed, leaves)
    th = synth.normal(seed, synth.S_THETA0, sum(leaves)).astype(np.float32)
    off = synth.offsets_of(leaves)
    lr_leaf = np.array([0.5, 2e-2, 1.0, 3e-3])
    return x, th, off, lr_leaf


@pytest.mark.parametrize("kind", ["adam", "adamw", "rmsprop", "sgd", "sgd_nesterov"])
@pytest.mark.parametrize("maximize", [False, True])
def test_ex_twins_bound_the_values(orc, kind, maximize):
    """ex_mag (the NEXT-1 variants' tolerance) bounds |value| of every output
    and of every element's hyper-gradient term (weight decay, maximize,
    per-leaf lr), at t = 1 and t = 10."""
    x, th, off, lrl = _ex_case()
    n = x["g"].size
    wd = 0.05
    kw = dict(weight_decay=wd, maximize=maximize, lr_leaf=lrl, offsets=off)
    for t in (1, 10):
        if kind in ("adam", "adamw"):
            hp = (0.5, 0.9, 0.999, 1e-8, 0.0)
            dec = kind == "adamw"
            u, m1, v1 = orc.adam_fwd_ex(x["g"], x["m"], x["v"], th, t, *hp, decoupled=dec,
                                        prec=1, **kw)
            r = orc.adam_vjp_ex(x["g"], x["m"], x["v"], th, x["du"], x["dm1"], x["dv1"], t, *hp,
                                decoupled=dec, prec=1, **kw)
            mag = orc.ex_mag("adam", x["g"], (x["m"], x["v"]), th, x["du"], x["dm1"], x["dv1"],
                             t, hp, decoupled=dec, **kw)
            vals = dict(u=u, m1=m1, v1=v1, dg=r["dg"], dm=r["dm"], dv=r["dv"],
                        dtheta=r["dtheta"])
            terms = _per_elem_terms(lambda o: orc.adam_vjp_ex(
                x["g"], x["m"], x["v"], th, x["du"], x["dm1"], x["dv1"], t, *hp, decoupled=dec,
                prec=1, weight_decay=wd, maximize=maximize,
                lr_leaf=np.repeat(lrl, np.diff(off)), offsets=o), n)
        elif kind == "rmsprop":
            hp = (0.3, 0.95, 1e-8)
            u, v1 = orc.rmsprop_fwd_ex(x["g"], x["v"], th, *hp, prec=1, **kw)
            r = orc.rmsprop_vjp_ex(x["g"], x["v"], th, x["du"], x["dv1"], *hp, prec=1, **kw)
            mag = orc.ex_mag("rmsprop", x["g"], x["v"], th, x["du"], x["dv1"], hp=hp, **kw)
            vals = dict(u=u, v1=v1, dg=r["dg"], dv=r["dv"], dtheta=r["dtheta"])
            terms = _per_elem_terms(lambda o: orc.rmsprop_vjp_ex(
                x["g"], x["v"], th, x["du"], x["dv1"], *hp, prec=1, weight_decay=wd,
                maximize=maximize, lr_leaf=np.repeat(lrl, np.diff(off)), offsets=o), n)
        else:
            hp = (0.1, 0.9, kind == "sgd_nesterov")
            u, b1 = orc.sgd_fwd_ex(x["g"], x["m"], th, *hp, prec=1, **kw)
            r = orc.sgd_vjp_ex(x["g"], x["m"], th, x["du"], x["dm1"], *hp, prec=1, **kw)
            mag = orc.ex_mag("sgd", x["g"], x["m"], th, x["du"], x["dm1"], hp=hp, **kw)
            vals = dict(u=u, b1=b1, dg=r["dg"], db=r["db"], dtheta=r["dtheta"])
            terms = _per_elem_terms(lambda o: orc.sgd_vjp_ex(
                x["g"], x["m"], th, x["du"], x["dm1"], *hp, prec=1, weight_decay=wd,
                maximize=maximize, lr_leaf=np.repeat(lrl, np.diff(off)), offsets=o), n)
        for k, val in vals.items():
            _assert_bounds(f"{kind} {k} t={t}", val, mag[k])
        _assert_bounds(f"{kind} h t={t}", terms, mag["h"])
        _assert_bounds(f"{kind} dhp t={t}", r["dhp"], mag["dhp"])


@pytest.mark.parametrize("centered", [False, True])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_rmsprop_cm_twins_bound_the_values(orc, centered, momentum):
    """rmsprop_cm_mag bounds |value| of every output and element term."""
    leaves = [900, 1, 300]
    x = synth.rms_cm_tree(74, leaves)
    off = synth.offsets_of(leaves)
    lrl = np.array([0.3, 1e-2, 1.0])
    n = x["g"].size
    hp = (0.3, 0.9, 1e-6, momentum, centered)
    kw = dict(weight_decay=0.05, maximize=False)
    args = (x["g"], x["v"], x["a"], x["b"], x["theta"])
    cots = (x["du"], x["dv1"], x["da1"], x["db1"])
    u, v1, a1, b1 = orc.rmsprop_cm_fwd(*args, *hp[:4], centered=centered, prec=1, lr_leaf=lrl,
                                       offsets=off, **kw)
    r = orc.rmsprop_cm_vjp(*args, *cots, *hp[:4], centered=centered, prec=1, lr_leaf=lrl,
                           offsets=off, **kw)
    mag = orc.rmsprop_cm_mag(*args, *cots, *hp[:4], centered=centered, lr_leaf=lrl, offsets=off,
                             **kw)
    vals = dict(u=u, v1=v1, b1=b1, dg=r["dg"], dv=r["dv"], db=r["db"], dtheta=r["dtheta"])
    if centered:
        vals.update(a1=a1, da=r["da"])
    for k, val in vals.items():
        _assert_bounds(f"cm {k}", val, mag[k])
    terms = _per_elem_terms(lambda o: orc.rmsprop_cm_vjp(
        *args, *cots, *hp[:4], centered=centered, prec=1, lr_leaf=np.repeat(lrl, np.diff(off)),
        offsets=o, **kw), n)
    _assert_bounds("cm h", terms, mag["h"])


def test_ex_mag_has_teeth(orc):
    """The variants' fp32 bar is passed by an fp32 evaluation of the reduced
    form and failed by an fp32 evaluation of the textbook chain rule, with
    L2 weight decay folded into the gradient (Adam, t = 1, zero state)."""
    rng = np.random.default_rng(5)
    n = 1 << 15
    g = (1e-2 * rng.standard_normal(n)).astype(np.float32)
    th = rng.standard_normal(n).astype(np.float32)
    du = rng.standard_normal(n).astype(np.float32)
    wd = 1e-3
    hp = (1.0, 0.9, 0.999, 1e-8, 0.0)
    r = orc.adam_vjp_ex(g, None, None, th, du, None, None, 1, *hp, weight_decay=wd, prec=1)
    mag = orc.ex_mag("adam", g, (None, None), th, du, None, None, 1, hp, weight_decay=wd)
    gt = (g + np.float32(wd) * th).astype(np.float32)
    ok = lambda y: np.abs(y.astype(np.float64) - r["dg"]) <= 1e-6 + 1e-5 * np.maximum(
        mag["dg"], np.abs(r["dg"]))
    assert ok(_f32_adam_dg(gt, du, *hp[:4], reduced=True)).mean() == 1.0
    assert ok(_f32_adam_dg(gt, du, *hp[:4], reduced=False)).mean() < 0.5


def test_rmsprop_cm_mag_has_teeth(orc):
    """Centred RMSProp (zero state, no momentum): the fp32 reduced form
    dg = -du lr eps / d^2 passes the bar, the fp32 textbook chain rule
    (-lr/d + lr g/d^2 * dq/dg / (2r), which cancels down to it) fails."""
    rng = np.random.default_rng(6)
    n = 1 << 15
    f = np.float32
    g = (1e-2 * rng.standard_normal(n)).astype(f)
    du = rng.standard_normal(n).astype(f)
    z = np.zeros(n, f)
    lr, al, eps = 1.0, 0.9, 1e-8
    r = orc.rmsprop_cm_vjp(g, None, None, None, z, du, None, None, None, lr, al, eps,
                           centered=True, prec=1)
    mag = orc.rmsprop_cm_mag(g, None, None, None, z, du, None, None, None, lr, al, eps,
                             centered=True)
    om = f(1) - f(al)
    v1, a1 = om * g * g, om * g
    q = v1 - a1 * a1
    rr = np.sqrt(q)
    d = rr + f(eps)
    reduced = -du * f(lr) * f(eps) / (d * d)
    dd = du * f(lr) * g / (d * d)
    dq = np.where(rr == 0, f(0), dd / (f(2) * np.where(rr == 0, f(1), rr)))
    textbook = du * (-f(lr) / d) + dq * (f(2) * om * g) + (-f(2) * a1 * dq) * om
    ok = lambda y: np.abs(y.astype(np.float64) - r["dg"]) <= 1e-6 + 1e-5 * np.maximum(
        mag["dg"], np.abs(r["dg"]))
    assert ok(reduced).mean() == 1.0
    assert ok(textbook).mean() < 0.5


def _rho(s, a):
    """Cancellation ratio |sum| / sum|terms| of a sum node (1 where 0/0)."""
    s, a = np.abs(s), np.asarray(a)
    return np.where(a > 0, s / np.where(a > 0, a, 1.0), 1.0)


def _check_loose(name, mag, ref, bound):
    """mag / |ref| <= bound wherever ref != 0 and the bound is finite."""
    ref = np.abs(ref)
    sel = (ref > 0) & np.isfinite(bound)
    ratio = mag[sel] / ref[sel]
    bad = ratio > bound[sel] * (1 + 1e-6) + 1e-9
    assert not bad.any(), (name, ratio[bad][:5], bound[sel][bad][:5])
    return float(np.mean(ratio > 10)), float(np.mean(bound[sel] > 10))


def test_adam_twin_looseness_is_input_cancellation(orc):
    """Looseness pin: on the C2 recipe at lr = 1, t = 10 the twin
    may exceed |ref| only by the cancellation of the sums of the REDUCED
    form. With rho = |sum| / sum|terms| of each sum node (m' = b1 m + (1-b1)
    g, the reduced dg bracket A eps + (A Q - P C g)/s, dg's top-level three
    terms, dm's and dv's two terms), mag / |ref| <= prod 1/rho exactly
    (mag is the tree over |.|), so every element with mag > 10 |ref| shows a
    cancellation in one of those sums; no other looseness is allowed."""
    idx = synth.uniform(0x1005E, 1, 1 << 16) * sum(synth.RESNET18_LEAVES)
    x = synth.state_tree(0xC2, synth.RESNET18_LEAVES, index=idx.astype(np.int64))
    t, lr, b1, b2, eps = 10, 1.0, 0.9, 0.999, 1e-8
    g, m, v, du, dm1, dv1 = (x[k].astype(np.float64) for k in ("g", "m", "v", "du", "dm1", "dv1"))
    u, m1, v1 = orc.adam_fwd(x["g"], x["m"], x["v"], t, lr, b1, b2, eps, prec=1)
    r = orc.adam_vjp(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], t, lr, b1, b2, eps,
                     prec=1)
    mag = orc.adam_mag(x["g"], x["m"], x["v"], x["du"], x["dm1"], x["dv1"], t, lr, b1, b2, eps)
    bc1, bc2 = 1 - b1 ** t, 1 - b2 ** t
    A, C = (1 - b1) / bc1, (1 - b2) / bc2
    P, Q = b1 * m / bc1, b2 * v / bc2
    mh = A * g + P
    s = np.sqrt(C * g * g + Q)
    d = s + eps
    rs = np.where(s > 0, 1 / np.where(s > 0, s, 1), 0)
    rho_m = _rho(mh, A * np.abs(g) + np.abs(P))
    br = A * eps + (A * Q - P * C * g) * rs
    rho_in = _rho(br, A * eps + (A * Q + np.abs(P * C * g)) * rs)
    T = [(1 - b1) * dm1, 2 * (1 - b2) * g * dv1, -du * lr * br / d ** 2]
    rho_top = _rho(sum(T), sum(np.abs(x) for x in T))
    y = du * lr / (bc1 * d)
    rho_dm = _rho(dm1 - y, np.abs(dm1) + np.abs(y))
    w = du * lr * mh * rs / (2 * bc2 * d ** 2)
    rho_dv = _rho(dv1 + w, np.abs(dv1) + np.abs(w))
    inv = lambda *rh: 1.0 / np.prod(rh, axis=0)
    stats = {}
    stats["u"] = _check_loose("u", mag["u"], u, inv(rho_m))
    stats["m1"] = _check_loose("m1", mag["m1"], m1, inv(rho_m))
    stats["v1"] = _check_loose("v1", mag["v1"], v1, np.ones_like(v1))
    stats["dg"] = _check_loose("dg", mag["dg"], r["dg"], inv(rho_in, rho_top))
    stats["dm"] = _check_loose("dm", mag["dm"], r["dm"], inv(rho_dm))
    stats["dv"] = _check_loose("dv", mag["dv"], r["dv"], inv(rho_dv, rho_m))
    # the reading's premise on this recipe: looseness happens, and is rare
    assert stats["dv"][0] > 0 and all(f < 0.2 for f, _ in stats.values())


def test_rmsprop_twin_looseness_is_input_cancellation(orc):
    """The same pin for RMSProp: u and v' are cancellation-free (ratio 1);
    dg and dv only by their top-level sums."""
    x = synth.state_tree(0xC2, None, n=1 << 16)
    lr, al, eps = 1.0, 0.99, 1e-8
    g, v, du, dv1 = (x[k].astype(np.float64) for k in ("g", "v", "du", "dv1"))
    u, v1 = orc.rmsprop_fwd(x["g"], x["v"], lr, al, eps, prec=1)
    r = orc.rmsprop_vjp(x["g"], x["v"], x["du"], x["dv1"], lr, al, eps, prec=1)
    mag = orc.rmsprop_mag(x["g"], x["v"], x["du"], x["dv1"], lr, al, eps)
    s = np.sqrt(al * v + (1 - al) * g * g)
    d = s + eps
    rs = np.where(s > 0, 1 / np.where(s > 0, s, 1), 0)
    T = [2 * (1 - al) * g * dv1, -du * lr * (eps + al * v * rs) / d ** 2]
    rho_top = _rho(sum(T), sum(np.abs(t) for t in T))
    w = du * lr * g * rs / (2 * d ** 2)
    rho_dv = _rho(dv1 + w, np.abs(dv1) + np.abs(w))
    _check_loose("u", mag["u"], u, np.ones_like(u))
    _check_loose("v1", mag["v1"], v1, np.ones_like(v1))
    _check_loose("dg", mag["dg"], r["dg"], 1 / rho_top)
    _check_loose("dv", mag["dv"], r["dv"], 1 / rho_dv)


def test_ex_twin_looseness_adds_only_the_decay_sum(orc):
    """Adam with L2 decay: beyond the base step's sums, the twin may exceed
    |ref| only through gt = g + wd theta: rho_gt in the numerators (squared
    in v') and the Lipschitz factor f_d = 1 + sqrt(C) (|g| + wd |theta| -
    |gt|) / d on 1/d (oracle.hpp adam_mag2)."""
    x, th, off, _ = _ex_case(75)
    t, hp, wd = 10, (1.0, 0.9, 0.999, 1e-8, 0.0), 0.05
    u, m1, v1 = orc.adam_fwd_ex(x["g"], x["m"], x["v"], th, t, *hp, weight_decay=wd, prec=1)
    mag = orc.ex_mag("adam", x["g"], (x["m"], x["v"]), th, x["du"], x["dm1"], x["dv1"], t, hp,
                     weight_decay=wd)
    g, m, thd = x["g"].astype(np.float64), x["m"].astype(np.float64), th.astype(np.float64)
    gt = g + wd * thd
    rho_gt = _rho(gt, np.abs(g) + wd * np.abs(thd))
    b1 = hp[1]
    rho_m = _rho(b1 * m + (1 - b1) * gt, b1 * np.abs(m) + (1 - b1) * np.abs(gt))
    bc1, bc2 = 1 - b1 ** t, 1 - hp[2] ** t
    C = (1 - hp[2]) / bc2
    s = np.sqrt(C * gt * gt + hp[2] * x["v"].astype(np.float64) / bc2)
    f_d = 1 + np.sqrt(C) * (np.abs(g) + wd * np.abs(thd) - np.abs(gt)) / (s + hp[3])
    _check_loose("u", mag["u"], u, f_d / (rho_m * rho_gt))
    _check_loose("m1", mag["m1"], m1, 1 / (rho_m * rho_gt))
    _check_loose("v1", mag["v1"], v1, 1 / rho_gt ** 2)
