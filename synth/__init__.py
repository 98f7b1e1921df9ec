"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py. Holds none of the method's arithmetic: only counter-based random
numbers and the workload recipes of SURVEY.md §8(d) / DESIGN.md "Input recipe".

Generator: SplitMix64 keyed on (seed, stream, index) -> 53-bit uniforms ->
Box-Muller normals, computed in float64 and rounded once to float32. Because
it is counter based, any index subset (``index=``) reproduces exactly the
values of the full array, which is how full-size parity tests sample outputs.
"""
from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 22

# stream ids: one per input role
S_G, S_M, S_V, S_DU, S_DM1, S_DV1, S_ZERO, S_SCALE = 1, 2, 3, 4, 5, 6, 7, 8
S_A, S_THETA0, S_PHI, S_Y = 9, 10, 11, 12
S_GAVG, S_BUF, S_DA1, S_DB1 = 13, 14, 15, 16

RESNET18_LEAVES = [
    9408, 64, 64, 36864, 64, 64, 36864, 64, 64, 36864, 64, 64, 36864, 64, 64, 73728, 128, 128,
    147456, 128, 128, 8192, 128, 128, 147456, 128, 128, 147456, 128, 128, 294912, 256, 256,
    589824, 256, 256, 32768, 256, 256, 589824, 256, 256, 589824, 256, 256, 1179648, 512, 512,
    2359296, 512, 512, 131072, 512, 512, 2359296, 512, 512, 2359296, 512, 512, 512000, 1000,
]  # torchvision resnet18 parameter order (62 leaves, 11,689,512 elements)

# 4-conv64 + BN + fc(5) for 28x28x1 inputs: 18 leaves, 112,261 elements
CONV4_LEAVES = [576, 64, 64, 64] + [36864, 64, 64, 64] * 3 + [320, 5]


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def _bits(seed, stream, idx):
    with np.errstate(over="ignore"):
        key = _mix(np.uint64(seed) * _GOLD + np.uint64(stream) + _GOLD)
        return _mix(idx.astype(np.uint64) * _GOLD + key)


def _u01(b):
    return ((b >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def _indices(n, index):
    if index is not None:
        return [np.asarray(index, dtype=np.int64)]
    return [np.arange(s, min(s + _CHUNK, n), dtype=np.int64) for s in range(0, n, _CHUNK)]


def uniform(seed, stream, n=0, index=None):
    """U(0,1) float64, element i keyed on (seed, stream, i)."""
    parts = [_u01(_bits(seed, stream, 2 * i)) for i in _indices(n, index)]
    return np.concatenate(parts) if parts else np.zeros(0)


def normal(seed, stream, n=0, index=None):
    """N(0,1) float64 (Box-Muller on counters 2i, 2i+1)."""
    out = []
    for i in _indices(n, index):
        u1 = _u01(_bits(seed, stream, 2 * i))
        u2 = _u01(_bits(seed, stream, 2 * i + 1))
        out.append(np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2))
    return np.concatenate(out) if out else np.zeros(0)


def offsets_of(leaves):
    off = np.zeros(len(leaves) + 1, dtype=np.int64)
    off[1:] = np.cumsum(np.asarray(leaves, dtype=np.int64))
    return off


def leaf_ids(offsets, index):
    """Leaf of each flat index."""
    return np.searchsorted(offsets, np.asarray(index), side="right") - 1


# ----------------------------------------------------------------- recipes
ADAM_HP = dict(lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, eps_root=0.0)  # S:187 defaults


def state_tree(seed, leaves, index=None, warm=True, zero_frac=1.0 / 256, n=None):
    """Per-leaf-scaled gradient / state / cotangent inputs.

    Leaf l has scale s_l = 10^(-4 U_l); g = s_l N; warm state m = 0.3 s_l N,
    v = (s_l (|N| + 0.1))^2; a fraction ``zero_frac`` of elements have
    g = m = v = 0 exactly (the 0/0 points of P:246); cotangents N(0,1).
    Returns float32 arrays g, m, v, du, dm1, dv1 (m, v None if not warm).
    ``leaves`` may be None for a single flat leaf of n elements whose scale is
    drawn per 4096-element block (C5)."""
    if leaves is None:
        total = n
    else:
        total = int(sum(leaves))
    idx = np.arange(total, dtype=np.int64) if index is None else np.asarray(index, np.int64)
    if leaves is None:
        grp = idx // 4096
    else:
        grp = leaf_ids(offsets_of(leaves), idx)
    scale = 10.0 ** (-4.0 * uniform(seed, S_SCALE, index=grp))
    zero = uniform(seed, S_ZERO, index=idx) < zero_frac
    g = scale * normal(seed, S_G, index=idx)
    g[zero] = 0.0
    m = v = None
    if warm:
        m = 0.3 * scale * normal(seed, S_M, index=idx)
        v = (scale * (np.abs(normal(seed, S_V, index=idx)) + 0.1)) ** 2
        m[zero] = 0.0
        v[zero] = 0.0
        m = m.astype(np.float32)
        v = v.astype(np.float32)
    du = normal(seed, S_DU, index=idx).astype(np.float32)
    dm1 = normal(seed, S_DM1, index=idx).astype(np.float32)
    dv1 = normal(seed, S_DV1, index=idx).astype(np.float32)
    return dict(g=g.astype(np.float32), m=m, v=v, du=du, dm1=dm1, dv1=dv1)


def rms_cm_tree(seed, leaves, index=None, zero_frac=1.0 / 256):
    """Inputs of the centred / momentum RMSProp step (NEXT-1, reading N4):
    per-leaf scale s as in state_tree; g = s N; gradient average a = 0.5 s N;
    v = a^2 + (s (|N| + 0.1))^2 (a consistent centred state: v >= a^2, so
    q = v' - a'^2 > 0); momentum buffer b ~ N(0,1) (it accumulates g/d);
    theta ~ N(0,1); cotangents du, dv1, da1, db1 ~ N(0,1); a fraction
    ``zero_frac`` of elements have g = a = v = 0 exactly."""
    total = int(sum(leaves))
    idx = np.arange(total, dtype=np.int64) if index is None else np.asarray(index, np.int64)
    scale = 10.0 ** (-4.0 * uniform(seed, S_SCALE, index=leaf_ids(offsets_of(leaves), idx)))
    zero = uniform(seed, S_ZERO, index=idx) < zero_frac
    g = scale * normal(seed, S_G, index=idx)
    a = 0.5 * scale * normal(seed, S_GAVG, index=idx)
    v = a * a + (scale * (np.abs(normal(seed, S_V, index=idx)) + 0.1)) ** 2
    for x in (g, a, v):
        x[zero] = 0.0
    f = lambda x: x.astype(np.float32)
    return dict(g=f(g), v=f(v), a=f(a), b=f(normal(seed, S_BUF, index=idx)),
                theta=f(normal(seed, S_THETA0, index=idx)),
                du=f(normal(seed, S_DU, index=idx)), dv1=f(normal(seed, S_DV1, index=idx)),
                da1=f(normal(seed, S_DA1, index=idx)), db1=f(normal(seed, S_DB1, index=idx)))


def c1_inputs(seed=0xC1, n=4096):
    """Config 1: one flat leaf, g ~ N(0,1) with 1/64 exact zeros, zero state,
    t = 1, cotangents N(0,1)."""
    idx = np.arange(n, dtype=np.int64)
    g = normal(seed, S_G, index=idx)
    g[uniform(seed, S_ZERO, index=idx) < 1.0 / 64] = 0.0
    return dict(g=g.astype(np.float32), m=None, v=None,
                du=normal(seed, S_DU, index=idx).astype(np.float32),
                dm1=normal(seed, S_DM1, index=idx).astype(np.float32),
                dv1=normal(seed, S_DV1, index=idx).astype(np.float32))


def quadratic_problem(seed, n, index=None):
    """Config 3 inner/outer problem (reading Z17): a ~ U[0.5, 1.5];
    theta0, phi, y ~ N(0,1)."""
    idx = np.arange(n, dtype=np.int64) if index is None else np.asarray(index, np.int64)
    return dict(a=(0.5 + uniform(seed, S_A, index=idx)).astype(np.float32),
                theta0=normal(seed, S_THETA0, index=idx).astype(np.float32),
                phi=normal(seed, S_PHI, index=idx).astype(np.float32),
                y=normal(seed, S_Y, index=idx).astype(np.float32))


def to_bf16_bits(x):
    """float32 -> bf16 bit patterns by round-to-nearest-even (input recipe
    for bf16 state: the state the caller holds is already bf16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def device_state_flat(seed, n, device, chunk=1 << 26):
    """The C5 recipe (one flat leaf, per-4096-block scale 10^(-4U), 1/256
    exact zeros in g, m, v, warm state m = 0.3 s N, v = (s(|N| + 0.1))^2,
    cotangents N(0,1)) generated directly in device memory with torch's
    seeded CUDA generator, chunk by chunk, for sizes too large to build on
    the host (> 2^31 elements). Not counter based: tests read the sampled
    inputs back from the device arrays. Returns float32 device tensors
    g, m, v, du, dm1, dv1."""
    import torch

    gen = torch.Generator(device=device).manual_seed(int(seed))
    out = {k: torch.empty(n, dtype=torch.float32, device=device)
           for k in ("g", "m", "v", "du", "dm1", "dv1")}
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        k = e - s
        blocks = (e - 1) // 4096 - s // 4096 + 1
        bscale = 10.0 ** (-4.0 * torch.rand(blocks, generator=gen, device=device,
                                            dtype=torch.float64))
        b0 = s // 4096
        scale = bscale[torch.arange(s, e, device=device) // 4096 - b0]
        zero = torch.rand(k, generator=gen, device=device) < 1.0 / 256
        nrm = lambda: torch.randn(k, generator=gen, device=device, dtype=torch.float64)
        g = scale * nrm()
        m = 0.3 * scale * nrm()
        v = (scale * (nrm().abs() + 0.1)) ** 2
        for name, x in (("g", g), ("m", m), ("v", v)):
            x[zero] = 0.0
            out[name][s:e] = x.float()
        for name in ("du", "dm1", "dv1"):
            out[name][s:e] = nrm().float()
    return out
