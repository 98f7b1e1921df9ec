"""GPU parity of the zero-order ES kernels
against the oracle: perturbed points elementwise, and the gradient estimate
from the same f values."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import DEV, assert_close, dev_f32, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_06934_b200 import _lib

    return _lib


@pytest.mark.parametrize("numel", [1, 5, 1001, 4096, 70001])
@pytest.mark.parametrize("antithetic", [True, False])
def test_es_perturb_matches_oracle(L, numel, antithetic):
    theta = synth.normal(0xE5, synth.S_THETA0, numel).astype(np.float32)
    n, sigma, seed, s0 = 7, 0.05, 1234, 3
    ld = L.es_row_stride(numel)
    reps = 2 if antithetic else 1
    out = torch.full((n * reps, ld), float("nan"), device=DEV)
    L.opt_es_perturb(numel, n, s0, antithetic, sigma, seed, dev_f32(theta), out)
    got = host(out)[:, :numel]
    # oracle rows for samples s0 .. s0+n-1
    ref = oracle.es_perturb(theta, s0 + n, sigma, seed, antithetic)[s0 * reps:]
    z = oracle.es_noise(numel, s0 + n, seed)[s0:]
    scale = np.abs(theta.astype(np.float64))[None, :] + sigma * np.abs(np.repeat(z, reps, axis=0))
    assert_close("perturb", got.ravel(), ref.ravel(), scale=scale.ravel())


@pytest.mark.parametrize("numel", [3, 4096, 70001])
@pytest.mark.parametrize("antithetic", [True, False])
def test_es_grad_matches_oracle(L, numel, antithetic):
    n, sigma, seed = 37, 0.1, 99
    rows = n * (2 if antithetic else 1)
    f = synth.normal(0xE6, synth.S_G, rows).astype(np.float32)
    grad = torch.empty(numel, device=DEV)
    L.opt_es_grad(numel, n, antithetic, sigma, seed, dev_f32(f), grad)
    ref, ref_abs = oracle.es_grad(f.astype(np.float64), numel, n, sigma, seed, antithetic)
    assert_close("es_grad", host(grad), ref, scale=ref_abs)


def test_es_linear_objective_end_to_end(L):
    """Black-box f(theta) = c.theta evaluated (by torch, as the caller's f)
    on the GPU-generated points: the estimate is within 5 standard errors of
    c (SPEC linear example); generating the points in two sample0 chunks
    equals one call; > 4096 samples per call is rejected."""
    d, n, sigma, seed = 8, 4096, 0.05, 7
    c = torch.tensor([1.0, -2.0, 0.5, 0.0, 3.0, -1.0, 0.25, 2.0], device=DEV)
    theta = torch.linspace(-1, 1, d, device=DEV)
    ld = L.es_row_stride(d)
    pts = torch.empty(2 * n, ld, device=DEV)
    L.opt_es_perturb(d, n, 0, True, sigma, seed, theta, pts)
    half = torch.empty(n, ld, device=DEV)
    L.opt_es_perturb(d, n // 2, n // 2, True, sigma, seed, theta, half)
    assert torch.equal(half, pts[n:])
    f = (pts[:, :d] @ c).contiguous()
    g = torch.empty(d, device=DEV)
    L.opt_es_grad(d, n, True, sigma, seed, f, g)
    cc = c.double().cpu().numpy()
    se = np.sqrt((cc @ cc + cc ** 2) / n)
    assert np.all(np.abs(g.double().cpu().numpy() - cc) < 5 * se)
    with pytest.raises(L.DiffoptError):
        L.opt_es_grad(d, 4097, True, sigma, seed, torch.zeros(2 * 4097, device=DEV), g)
