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


from paper_2503_08264_b200.synth import posterior_like_q  # noqa: E402,F401  (input generator)
