"""Invariants of the device E-step at sizes the oracle is not needed for (SURVEY.md §8(c)
"Invariants"): App. E's reparameterisation invariance (rescaling a location-scale
latent by alpha leaves the importance weights unchanged), permutation equivariance of the K
samples, and the weights' normalisation -- on a config-1-shaped model with 2000 groups."""
import dataclasses

import numpy as np
import pytest

from paper_2503_08264_b200 import synth

pytestmark = pytest.mark.gpu


def _estep(m, data, q, eps):
    from paper_2503_08264_b200.qem import QEM
    g = QEM(m)
    g.set_data(data)
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    out = g.result()
    g.close()
    return out


def _case(n=2000, K=256):
    m = synth.config(1, n=n, K=K)
    data = synth.make_data(m)
    q = synth.random_q(m, 3, 0.5)
    eps = [synth.eps_normal((nn * dd, m.K), 40 + lvl) for lvl, (nn, dd) in enumerate(synth.latent_shapes(m))]
    return m, data, q, eps


@pytest.mark.parametrize("alpha", [0.25, 4.0])
def test_rescaled_model_has_the_same_weights(alpha):
    """z' = alpha z for every latent, x' = alpha x, all variances times alpha^2 (a power of two:
    the fp32 samples scale exactly): the weights are unchanged and log Pe shifts by the
    observations' Jacobian, -(#obs) ln alpha (App. E)."""
    m, data, q, eps = _case()
    a2 = alpha * alpha
    ms = dataclasses.replace(m, prior_var=m.prior_var * a2, fixed_var=m.fixed_var * a2, obs_var=m.obs_var * a2)
    ds = dataclasses.replace(data, xg=(data.xg * alpha).astype(np.float32))
    qs = [((qm * alpha).astype(np.float32), (qv * a2).astype(np.float32)) for qm, qv in q]
    a = _estep(m, data, q, eps)
    b = _estep(ms, ds, qs, eps)
    for lvl in range(2):
        np.testing.assert_allclose(b["w"][lvl], a["w"][lvl], atol=2e-6)
        np.testing.assert_allclose(b["m1"][lvl], a["m1"][lvl] * alpha, rtol=1e-5, atol=1e-6 * alpha)
    n_obs = m.n * m.J
    assert abs((b["log_pe"] - a["log_pe"]) + n_obs * np.log(alpha)) <= 1e-6 * abs(a["log_pe"])


def test_permuting_group_samples_permutes_their_weights():
    """Reordering one group's K samples (its eps columns) reorders its weights and leaves log Pe,
    the root weights and every moment unchanged (Eq. 7 sums over all index tuples)."""
    m, data, q, eps = _case(n=500, K=128)
    a = _estep(m, data, q, eps)
    perm = np.random.default_rng(1).permutation(m.K)
    eps2 = [eps[0], eps[1].copy()]
    eps2[1][7] = eps[1][7][perm]  # group 7 (d = 1: row 7)
    b = _estep(m, data, q, eps2)
    assert abs(b["log_pe"] - a["log_pe"]) <= 1e-6 * abs(a["log_pe"])
    np.testing.assert_allclose(b["w"][0], a["w"][0], atol=1e-6)
    np.testing.assert_allclose(b["w"][1][7], a["w"][1][7][perm], atol=1e-6)
    np.testing.assert_allclose(b["m1"][1], a["m1"][1], rtol=1e-5, atol=1e-6)
    for lvl in range(2):
        np.testing.assert_allclose(b["w"][lvl].reshape(-1, m.K).sum(axis=1), 1.0, atol=1e-5)


def test_tensor_core_path_permutation_equivariance():
    """The same on the tcgen05 path (config 5's shape, d = 16, K = 1024, 2000 groups): permuting
    one group's K samples (all 16 dims alike) permutes its weights and leaves log Pe, the root
    weights and the other groups unchanged up to the fp32 tile rounding."""
    from paper_2503_08264_b200.qem import QEM
    m = synth.config(5, n=2000, K=1024)
    data = synth.make_data(m)
    q = synth.random_q(m, 5, 0.3)
    eps = [synth.eps_normal((nn * dd, m.K), 70 + lvl) for lvl, (nn, dd) in enumerate(synth.latent_shapes(m))]
    g = QEM(m)
    assert g.pair_path() == 1
    g.close()
    a = _estep(m, data, q, eps)
    perm = np.random.default_rng(2).permutation(m.K)
    eps2 = [eps[0], eps[1].copy()]
    rows = slice(11 * m.d, 12 * m.d)  # group 11's 16 dims
    eps2[1][rows] = eps[1][rows][:, perm]
    b = _estep(m, data, q, eps2)
    assert abs(b["log_pe"] - a["log_pe"]) <= 1e-5 * abs(a["log_pe"])
    np.testing.assert_allclose(b["w"][0], a["w"][0], atol=1e-5)
    np.testing.assert_allclose(b["w"][1][11], a["w"][1][11][perm], atol=1e-5)
    others = np.ones(m.n, bool)
    others[11] = False
    np.testing.assert_allclose(b["w"][1][others], a["w"][1][others], atol=1e-5)
