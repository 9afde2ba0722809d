"""Shared test fixtures: seeded cases (data, Q, samples) for both the oracle and GPU tests.

Samples are produced by the ORACLE's fp32 sampler (z = fmaf(sqrtf(v), eps, m))
from host eps, so the GPU E-step consumes exactly the oracle's inputs.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc
from paper_2503_08264_b200 import synth


def make_case(m, q_seed=11, eps_seed=12, data_seed=None, q_spread=1.0, q=None):
    data = synth.make_data(m, data_seed)
    if q is None:
        q = synth.random_q(m, q_seed, q_spread)
    eps = [synth.eps_normal((n * dd, m.K), eps_seed * 31 + lvl) for lvl, (n, dd) in enumerate(synth.latent_shapes(m))]
    z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
    return data, q, eps, z


def posterior_like_q(m, data, seed=5, shrink=1.0):
    """A Q centred near the data-generating truth with roughly posterior widths:
    the converged regime of QEM, where the root weights are spread (H1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    t = data.truth
    if m.family == synth.FAMILY_TWO_LEVEL:
        rm = list(t["mu"]) + ([t["s"]] if m.scale_kind != synth.SCALE_FIXED else [])
        rsd = shrink * 1.0 / np.sqrt(max(m.n, 1))
        root_m = np.asarray(rm) + rsd * rng.standard_normal(m.R)
        root_v = np.full(m.R, rsd ** 2)
        z = np.asarray(t["z"]).reshape(-1)
        gsd = shrink * 1.0 / np.sqrt(max(m.J, 1) * 0.25 + 1.0)
        gm = z + gsd * rng.standard_normal(z.size)
        gv = np.full(z.size, gsd ** 2)
        return [(root_m.astype(np.float32), root_v.astype(np.float32)),
                (gm.astype(np.float32), gv.astype(np.float32))]
    rm = [t["g"]] + list(t["beta"])
    rsd = shrink * 0.01
    root_m = np.asarray(rm) + rsd * rng.standard_normal(m.R)
    u, v = np.asarray(t["u"]), np.asarray(t["v"])
    return [(root_m.astype(np.float32), np.full(m.R, rsd ** 2, np.float32)),
            ((u + 0.3 * rng.standard_normal(u.size)).astype(np.float32), np.full(u.size, 0.09, np.float32)),
            ((v + 0.01 * rng.standard_normal(v.size)).astype(np.float32), np.full(v.size, 1e-4, np.float32))]
