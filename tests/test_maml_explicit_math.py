"""CPU pin (float64, no GPU) of the hand-scheduled second-order MAML step's
ALGORITHM (paper_2211_06934_b200/maml_explicit.py), independent
of its kernels: the same schedule -- K SGD-momentum inner steps with saved
intermediates, the reverse sweep (v = b̄' − lr·θ̄, b̄ = μ·v, θ̄ += H_k v) and
each H_k v as forward-over-reverse through the saved forward and backward
passes, layer by layer (conv tangents as sums of two products, norm/pool
and head tangents by the include/mamlnet.h formulas restated in
tests/test_mamlnet_math.py) -- written here with torch float64 ops, against
PyTorch autograd's create_graph MAML of the same network. A wrong sign, a
dropped tangent term (e.g. W·Rcols or dy·Rcolsᵀ), a wrong momentum adjoint
or a misplaced accumulation fails it. Small geometry (16×16 images, 4
channels, 3 ways) so it runs in seconds."""
import os
import sys

import pytest
import torch
import torch.nn.functional as F
from torch.nn.grad import conv2d_input, conv2d_weight

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_mamlnet_math import (EPS, header_bwd, header_bwd_jvp, header_fc_xent,  # noqa: E402
                               header_fc_xent_jvp, header_jvp)

C, WAYS, HW, BLOCKS = 4, 3, 16, 4


def make_params(gen):
    r = lambda *s: torch.randn(*s, generator=gen, dtype=torch.float64)
    p = []
    for blk in range(BLOCKS):
        cin = 1 if blk == 0 else C
        p += [r(C, cin, 3, 3) * (2.0 / (cin * 9)) ** 0.5, r(C) * 0.1,
              1.0 + 0.2 * r(C), 0.1 * r(C)]
    p += [r(WAYS, C) * 0.5, 0.1 * r(WAYS)]
    return p


def ref_net(params, x):
    """The network with PyTorch ops (conv biases included: inert, N5)."""
    h = x
    for blk in range(BLOCKS):
        w, b, g, be = params[4 * blk: 4 * blk + 4]
        h = F.conv2d(h, w, b, padding=1)
        h = F.batch_norm(h, None, None, g, be, training=True, eps=EPS)
        h = F.max_pool2d(F.relu(h), 2)
    return F.linear(h.flatten(1), params[16], params[17])


def ref_meta_grad(phi, xs, ys, xq, yq, K, lr, mom, nesterov=False):
    """Autograd (create_graph) second-order MAML meta-gradient."""
    phi = [p.clone().requires_grad_(True) for p in phi]
    theta, buf = phi, None
    for _ in range(K):
        grads = torch.autograd.grad(F.cross_entropy(ref_net(theta, xs), ys), theta,
                                    create_graph=True)
        buf = list(grads) if buf is None else [mom * b + g for b, g in zip(buf, grads)]
        step = [g + mom * b for g, b in zip(grads, buf)] if nesterov else buf
        theta = [t - lr * st for t, st in zip(theta, step)]
    return [g.detach() for g in torch.autograd.grad(F.cross_entropy(ref_net(theta, xq), yq), phi)]


# ------------------------------------------------- the explicit schedule
def cgrp(t):  # [B, C, H, W] <-> [C, B, H, W] (the kernels' per-channel group layout)
    return t.permute(1, 0, 2, 3).contiguous()


def grad_pass(theta, x, y):
    """Forward + backward with every intermediate saved (as _grad)."""
    S = {"h": [x], "y": [], "dh": [None] * BLOCKS, "dy": [None] * BLOCKS}
    for l in range(BLOCKS):
        w, _, g, be = theta[4 * l: 4 * l + 4]
        yl = F.conv2d(S["h"][-1], w, None, padding=1)       # bias left out (inert)
        S["y"].append(yl)
        z = F.batch_norm(yl, None, None, g, be, training=True, eps=EPS)
        S["h"].append(F.max_pool2d(F.relu(z), 2))
    B = x.shape[0]
    h4 = S["h"][-1].reshape(B, C).t().unsqueeze(0)          # [1, C, B]
    loss, prob, dW, db, dh4 = header_fc_xent(h4, theta[16].unsqueeze(0), theta[17].unsqueeze(0),
                                            y.unsqueeze(0))
    grad = [torch.zeros_like(t) for t in theta]
    grad[16], grad[17] = dW[0], db[0]
    S["h4"], S["prob"] = h4, prob
    dh = dh4[0].t().reshape(B, C, 1, 1)
    for l in range(BLOCKS - 1, -1, -1):
        w, _, g, be = theta[4 * l: 4 * l + 4]
        S["dh"][l] = dh
        dx, dg, dbe = header_bwd(cgrp(S["y"][l]), g, be, cgrp(dh))
        dy = cgrp(dx)
        S["dy"][l] = dy
        grad[4 * l + 2], grad[4 * l + 3] = dg, dbe
        grad[4 * l] = conv2d_weight(S["h"][l], w.shape, dy, padding=1)
        if l > 0:
            dh = conv2d_input(S["h"][l].shape, w, dy, padding=1)
    return grad, S, float(loss[0])


def hvp(theta, S, grad, v, labels, drop=()):
    """H(theta) v by forward-over-reverse through the saved passes (as _hvp).
    drop: names of terms to leave out (mutation checks only)."""
    Rh, Ry = [torch.zeros_like(S["h"][0])], []
    for l in range(BLOCKS):
        w, _, g, be = theta[4 * l: 4 * l + 4]
        ry = F.conv2d(S["h"][l], v[4 * l], None, padding=1)            # RW·cols
        if l > 0 and "W.Rcols" not in drop:
            ry = ry + F.conv2d(Rh[l], w, None, padding=1)             # + W·Rcols
        Ry.append(ry)
        outd, _, _ = header_jvp(cgrp(S["y"][l]), g, be, cgrp(ry), v[4 * l + 2], v[4 * l + 3])
        Rh.append(cgrp(outd))
    B = S["h"][0].shape[0]
    rh4 = Rh[-1].reshape(B, C).t().unsqueeze(0)
    dWd, dbd, dh4d = header_fc_xent_jvp(S["h4"], theta[16].unsqueeze(0), theta[17].unsqueeze(0),
                                        labels.unsqueeze(0), rh4, v[16].unsqueeze(0),
                                        v[17].unsqueeze(0))
    out = [torch.zeros_like(t) for t in theta]
    out[16], out[17] = dWd[0], dbd[0]
    rdh = dh4d[0].t().reshape(B, C, 1, 1)
    for l in range(BLOCKS - 1, -1, -1):
        w, _, g, be = theta[4 * l: 4 * l + 4]
        dxd, dgd, dbd_ = header_bwd_jvp(cgrp(S["y"][l]), g, be, cgrp(S["dh"][l]), cgrp(Ry[l]),
                                        v[4 * l + 2], cgrp(rdh))
        rdy = cgrp(dxd)
        out[4 * l + 2], out[4 * l + 3] = dgd, dbd_
        rdw = conv2d_weight(S["h"][l], w.shape, rdy, padding=1)          # Rdy·colsᵀ
        if l > 0:
            if "dy.Rcols" not in drop:
                rdw = rdw + conv2d_weight(Rh[l], w.shape, S["dy"][l], padding=1)  # + dy·Rcolsᵀ
            rdh = conv2d_input(S["h"][l].shape, w, rdy, padding=1)             # Wᵀ·Rdy
            if "RW.dy" not in drop:
                rdh = rdh + conv2d_input(S["h"][l].shape, v[4 * l], S["dy"][l], padding=1)
        out[4 * l] = rdw
    return out


def explicit_meta_grad(phi, xs, ys, xq, yq, K, lr, mom, drop=(), nesterov=False):
    thetas, grads, saved, bufs = [list(phi)], [], [], [None]
    for _ in range(K):
        g, S, _ = grad_pass(thetas[-1], xs, ys)
        grads.append(g)
        saved.append(S)
        b = g if bufs[-1] is None else [mom * bb + gg for bb, gg in zip(bufs[-1], g)]
        bufs.append(b)
        step = [gg + mom * bb for gg, bb in zip(g, b)] if nesterov else b
        thetas.append([t - lr * st for t, st in zip(thetas[-1], step)])
    theta_bar, _, _ = grad_pass(thetas[-1], xq, yq)
    b_bar = None
    for k in range(K - 1, -1, -1):
        if nesterov:  # opt_sgd_bwd, Nesterov: B = b̄' − lr μ ū, ḡ = −lr ū + B, b̄ = μ B
            Bv = [(0 if b_bar is None else bb) - lr * mom * tb for bb, tb in
                  zip(b_bar or theta_bar, theta_bar)]
            v = [-lr * tb + bv for tb, bv in zip(theta_bar, Bv)]
            b_bar = [mom * bv for bv in Bv]
        else:
            v = [(0 if b_bar is None else bb) - lr * tb for bb, tb in
                 zip(b_bar or theta_bar, theta_bar)]              # opt_sgd_bwd: ḡ = b̄' − lr ū
            b_bar = [(0.0 if "momentum" in drop else mom) * vv for vv in v]   # b̄ = μ ḡ
        hv = hvp(thetas[k], saved[k], grads[k], v, ys, drop)
        theta_bar = [tb + h for tb, h in zip(theta_bar, hv)]
    return theta_bar


@pytest.mark.parametrize("K,mom,seed,nesterov", [(1, 0.9, 0, False), (3, 0.9, 1, False),
                                                 (3, 0.0, 2, False), (5, 0.5, 3, False),
                                                 (3, 0.9, 4, True), (2, 0.5, 5, True)])
def test_explicit_schedule_equals_autograd_maml(K, mom, seed, nesterov):
    gen = torch.Generator().manual_seed(seed)
    phi = make_params(gen)
    Bs, Bq = 2 * WAYS, 3 * WAYS
    xs = torch.randn(Bs, 1, HW, HW, generator=gen, dtype=torch.float64)
    xq = torch.randn(Bq, 1, HW, HW, generator=gen, dtype=torch.float64)
    ys = torch.arange(WAYS).repeat_interleave(2)
    yq = torch.arange(WAYS).repeat_interleave(3)
    lr = 0.1
    ref = ref_meta_grad(phi, xs, ys, xq, yq, K, lr, mom, nesterov)
    got = explicit_meta_grad(phi, xs, ys, xq, yq, K, lr, mom, nesterov=nesterov)
    scale = max(float(r.abs().max()) for r in ref)
    for i, (a, r) in enumerate(zip(got, ref)):
        if i < 16 and i % 4 == 1:  # conv bias: inert (N5), exactly 0 in the schedule
            assert float(a.abs().max()) == 0.0 and float(r.abs().max()) <= 1e-10 * scale
            continue
        torch.testing.assert_close(a, r, rtol=1e-8, atol=1e-11 * scale, msg=f"leaf {i}")


@pytest.mark.parametrize("term", ["W.Rcols", "dy.Rcols", "RW.dy", "momentum"])
def test_dropping_a_term_is_detected(term):
    """Teeth: the schedule with one term left out (a plausible slip: a
    tangent product of the conv, or the momentum adjoint) misses the
    autograd meta-gradient by far more than the bar above."""
    gen = torch.Generator().manual_seed(9)
    phi = make_params(gen)
    xs = torch.randn(6, 1, HW, HW, generator=gen, dtype=torch.float64)
    xq = torch.randn(9, 1, HW, HW, generator=gen, dtype=torch.float64)
    ys = torch.arange(WAYS).repeat_interleave(2)
    yq = torch.arange(WAYS).repeat_interleave(3)
    ref = ref_meta_grad(phi, xs, ys, xq, yq, 2, 0.1, 0.9)
    got = explicit_meta_grad(phi, xs, ys, xq, yq, 2, 0.1, 0.9, drop=(term,))
    err = max(float((a - r).abs().max()) for a, r in zip(got, ref))
    scale = max(float(r.abs().max()) for r in ref)
    assert err > 1e-5 * scale, (term, err, scale)


# ------------------------------------------------ Adam inner loop (inner_opt="adam")
B1, B2, AEPS = 0.9, 0.999, 1e-8


def adam_step(g, m, v, t, lr):
    """One Adam step (bias-corrected, eps outside the sqrt: reading Z1)."""
    m1 = B1 * m + (1 - B1) * g
    v1 = B2 * v + (1 - B2) * g * g
    u = -lr * (m1 / (1 - B1 ** t)) / (torch.sqrt(v1 / (1 - B2 ** t)) + AEPS)
    return u, m1, v1


BIAS = [4 * b + 1 for b in range(BLOCKS)]  # conv biases: inert (N5), held constant here


def ref_net_nb(params, x):
    """ref_net without the (inert) conv biases: with an Adam inner loop their
    exactly-zero gradients would put sqrt(0)'s infinite slope (times 0) into
    autograd's second derivative -- the 0/0 the library resolves by reading Z6."""
    return ref_net([None if i in BIAS else p for i, p in enumerate(params)], x)


def ref_meta_grad_adam(phi, xs, ys, xq, yq, K, lr):
    phi = [p.clone().requires_grad_(i not in BIAS) for i, p in enumerate(phi)]
    theta = phi
    m = [torch.zeros_like(p) for p in phi]
    v = [torch.zeros_like(p) for p in phi]
    live = [i for i in range(len(phi)) if i not in BIAS]
    for k in range(K):
        gl = torch.autograd.grad(F.cross_entropy(ref_net_nb(theta, xs), ys),
                                 [theta[i] for i in live], create_graph=True)
        grads = [torch.zeros_like(p) for p in phi]
        for i, g in zip(live, gl):
            grads[i] = g
        outs = [adam_step(g, mm, vv, k + 1, lr) if i in live else (torch.zeros_like(g), mm, vv)
                for i, (g, mm, vv) in enumerate(zip(grads, m, v))]
        theta = [t + o[0] for t, o in zip(theta, outs)]
        m, v = [o[1] for o in outs], [o[2] for o in outs]
    gq = torch.autograd.grad(F.cross_entropy(ref_net_nb(theta, xq), yq), [phi[i] for i in live])
    out = [torch.zeros_like(p) for p in phi]
    for i, g in zip(live, gq):
        out[i] = g.detach()
    return out


def explicit_meta_grad_adam(phi, xs, ys, xq, yq, K, lr):
    """The explicit schedule with an Adam inner loop: forward steps with saved
    (g, m, v); reverse: the Adam VJP (here torch.func.vjp of adam_step, an
    independent derivation from the kernels) then θ̄ += H_k ḡ."""
    from torch.func import vjp

    thetas, grads, saved = [list(phi)], [], []
    ms, vs = [[torch.zeros_like(p) for p in phi]], [[torch.zeros_like(p) for p in phi]]
    for k in range(K):
        g, S, _ = grad_pass(thetas[-1], xs, ys)
        grads.append(g)
        saved.append(S)
        outs = [adam_step(gg, mm, vv, k + 1, lr) for gg, mm, vv in zip(g, ms[-1], vs[-1])]
        thetas.append([t + o[0] for t, o in zip(thetas[-1], outs)])
        ms.append([o[1] for o in outs])
        vs.append([o[2] for o in outs])
    theta_bar, _, _ = grad_pass(thetas[-1], xq, yq)
    m_bar = [torch.zeros_like(p) for p in phi]
    v_bar = [torch.zeros_like(p) for p in phi]
    for k in range(K - 1, -1, -1):
        gb, mb, vb = [], [], []
        for i in range(len(phi)):
            if i in BIAS:  # exact-zero gradient and state: the Z6 convention gives 0
                gb.append(torch.zeros_like(phi[i]))
                mb.append(torch.zeros_like(phi[i]))
                vb.append(torch.zeros_like(phi[i]))
                continue
            _, f = vjp(lambda g_, m_, v_: adam_step(g_, m_, v_, k + 1, lr),
                       grads[k][i], ms[k][i], vs[k][i])
            a, b, c = f((theta_bar[i], m_bar[i], v_bar[i]))
            gb.append(a)
            mb.append(b)
            vb.append(c)
        m_bar, v_bar = mb, vb
        hv = hvp(thetas[k], saved[k], grads[k], gb, ys)
        theta_bar = [tb + h for tb, h in zip(theta_bar, hv)]
    return theta_bar


@pytest.mark.parametrize("K,seed", [(1, 10), (3, 11)])
def test_explicit_schedule_adam_inner_equals_autograd_maml(K, seed):
    gen = torch.Generator().manual_seed(seed)
    phi = make_params(gen)
    xs = torch.randn(2 * WAYS, 1, HW, HW, generator=gen, dtype=torch.float64)
    xq = torch.randn(3 * WAYS, 1, HW, HW, generator=gen, dtype=torch.float64)
    ys = torch.arange(WAYS).repeat_interleave(2)
    yq = torch.arange(WAYS).repeat_interleave(3)
    ref = ref_meta_grad_adam(phi, xs, ys, xq, yq, K, 0.01)
    got = explicit_meta_grad_adam(phi, xs, ys, xq, yq, K, 0.01)
    scale = max(float(r.abs().max()) for r in ref)
    for i, (a, r) in enumerate(zip(got, ref)):
        if i < 16 and i % 4 == 1:  # conv bias: inert
            continue
        torch.testing.assert_close(a, r, rtol=1e-7, atol=1e-10 * scale, msg=f"leaf {i}")
