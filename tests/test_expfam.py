"""Exponential-family M-steps from mean parameters (NEXT row f1; PAPER.md:218, 247;
SPEC.md:92-115): the oracle pinned against the closed-form forward maps and SPEC.md's worked
examples, and (GPU) the device kernel qem_mstep_family against the oracle."""
import math

import numpy as np
import pytest
from scipy.special import digamma

from oracle import expfam


# ------------------------------------------------------------------ oracle pins (CPU)


def test_spec_examples():
    # SPEC.md:99 Beta m = (-1, -1) -> (1, 1): E[ln z] = psi(1) - psi(2) = -1 for Beta(1, 1)
    np.testing.assert_allclose(expfam.beta_params([-1.0, -1.0]), [1.0, 1.0], rtol=1e-10)
    # SPEC.md:100 Gamma (k=3, th=2): m = (1.5, psi(3) - ln 2) -> (3, 2)
    np.testing.assert_allclose(expfam.gamma_params([1.5, digamma(3.0) - math.log(2.0)]), [3.0, 2.0], rtol=1e-9)
    # Bernoulli p = 0.3
    np.testing.assert_allclose(expfam.params_from_mean(expfam.BERNOULLI, [[0.3]]), [[0.3]])


def test_forward_maps_match_monte_carlo():
    """The closed-form mean parameters are the expected sufficient statistics:
    Monte Carlo over 1e6 numpy draws, 4 standard errors."""
    rng = np.random.default_rng(3)
    for k, th in [(0.7, 1.3), (3.0, 2.0)]:
        z = rng.gamma(k, 1.0 / th, 1_000_000)
        t = np.stack([z, np.log(z)])
        se = t.std(axis=1) / 1000
        assert np.all(np.abs(t.mean(axis=1) - expfam.gamma_mean(k, th)) < 4 * se)
    for a, b in [(2.0, 5.0), (0.6, 0.9)]:
        z = rng.beta(a, b, 1_000_000)
        t = np.stack([np.log(z), np.log1p(-z)])
        se = t.std(axis=1) / 1000
        assert np.all(np.abs(t.mean(axis=1) - expfam.beta_mean(a, b)) < 4 * se)


@pytest.mark.parametrize("family", [expfam.GAMMA, expfam.BETA])
def test_round_trip(family):
    """mean -> conventional -> mean is the identity to 1e-9 over a parameter grid."""
    rng = np.random.default_rng(family)
    for _ in range(200):
        p = np.exp(rng.uniform(-2.5, 3.5, 2))
        m = expfam.gamma_mean(*p) if family == expfam.GAMMA else expfam.beta_mean(*p)
        q = expfam.params_from_mean(family, m[None])[0]
        np.testing.assert_allclose(q, p, rtol=1e-7)
        m2 = expfam.gamma_mean(*q) if family == expfam.GAMMA else expfam.beta_mean(*q)
        np.testing.assert_allclose(m2, m, rtol=1e-9, atol=1e-12)


def test_dirichlet_round_trip_and_beta_special_case():
    """Dirichlet: mean -> conventional -> mean over random a (C = 2..6); C = 2 is the Beta."""
    rng = np.random.default_rng(21)
    for C in (2, 3, 6):
        for _ in range(40):
            a = np.exp(rng.uniform(-1.5, 2.5, C))
            q = expfam.dirichlet_params(expfam.dirichlet_mean(a))
            np.testing.assert_allclose(q, a, rtol=1e-7)
    a = np.array([2.5, 0.7])
    np.testing.assert_allclose(expfam.dirichlet_mean(a), expfam.beta_mean(*a), rtol=1e-14)
    np.testing.assert_allclose(expfam.dirichlet_params(expfam.beta_mean(*a)), expfam.beta_params(expfam.beta_mean(*a)),
                               rtol=1e-8)


def test_binomial_and_multinomial_mean_maps():
    """E z = N p for Binomial(N, p) and Multinomial(N, p) (textbook means), so p = m / N."""
    np.testing.assert_allclose(expfam.params_from_mean(expfam.BINOMIAL, [[6.0]], C=20), [[0.3]])
    m = 12 * np.array([[0.2, 0.5, 0.3]])
    np.testing.assert_allclose(expfam.params_from_mean(expfam.MULTINOMIAL, m), [[0.2, 0.5, 0.3]])


def test_infeasible_moments_rejected():
    with pytest.raises(ValueError):
        expfam.gamma_params([1.0, 0.5])  # E[ln z] >= ln E[z] violates Jensen
    with pytest.raises(ValueError):
        expfam.beta_params([-0.1, -0.1])  # e^-0.1 + e^-0.1 > 1


def test_ema_fixed_point():
    """The EMA over mean parameters with a constant input converges to it (App. D law)."""
    m = np.array([[1.5, digamma(3.0) - math.log(2.0)]])
    s = np.array([[1.0, -0.6]])
    for _ in range(200):
        s, p = expfam.ema_mstep(expfam.GAMMA, 0.7, s, m)
    np.testing.assert_allclose(p, [[3.0, 2.0]], rtol=1e-8)


# ------------------------------------------------------------------ device kernel (GPU)


@pytest.mark.gpu
@pytest.mark.parametrize("family", [expfam.GAMMA, expfam.BETA, expfam.BERNOULLI, expfam.CATEGORICAL,
                                    expfam.DIRICHLET, expfam.BINOMIAL, expfam.MULTINOMIAL])
def test_device_mstep_family_matches_oracle(family):
    import torch
    from paper_2503_08264_b200.qem import mstep_family
    rng = np.random.default_rng(10 + family)
    n, C = 2000, 5
    if family in (expfam.GAMMA, expfam.BETA):
        fwd = expfam.gamma_mean if family == expfam.GAMMA else expfam.beta_mean
        pa = np.exp(rng.uniform(-2.0, 3.0, (n, 2)))
        pb = np.exp(rng.uniform(-2.0, 3.0, (n, 2)))
        m_ema = np.array([fwd(*p) for p in pa])
        m_new = np.array([fwd(*p) for p in pb])
    elif family == expfam.BERNOULLI:
        m_ema, m_new = rng.uniform(0, 1, (n, 1)), rng.uniform(0, 1, (n, 1))
    elif family == expfam.DIRICHLET:
        n = 400  # the oracle's scipy root per instance is slow
        m_ema = np.array([expfam.dirichlet_mean(a) for a in np.exp(rng.uniform(-1.0, 2.0, (n, C)))])
        m_new = np.array([expfam.dirichlet_mean(a) for a in np.exp(rng.uniform(-1.0, 2.0, (n, C)))])
    elif family == expfam.BINOMIAL:
        C = 20  # trials
        m_ema, m_new = rng.uniform(0, C, (n, 1)), rng.uniform(0, C, (n, 1))
    elif family == expfam.MULTINOMIAL:
        m_ema, m_new = 9 * rng.dirichlet(np.ones(C), n), 9 * rng.dirichlet(np.ones(C), n)
    else:
        m_ema, m_new = rng.dirichlet(np.ones(C), n), rng.dirichlet(np.ones(C), n)
    lam = 0.7
    s_ref, p_ref = expfam.ema_mstep(family, lam, m_ema, m_new, C=C)
    dev = torch.device("cuda")
    te, tn = torch.tensor(m_ema, device=dev), torch.tensor(m_new, device=dev)
    params, status = mstep_family(family, lam, tn, te, C=C)
    np.testing.assert_allclose(te.cpu().numpy(), s_ref, rtol=1e-14, atol=1e-15)
    assert int(status.max().item()) == 0
    np.testing.assert_allclose(params.cpu().numpy(), p_ref, rtol=1e-8)


@pytest.mark.gpu
def test_device_mstep_family_flags_infeasible():
    import torch
    from paper_2503_08264_b200.qem import mstep_family
    dev = torch.device("cuda")
    m = torch.tensor([[1.0, 0.5], [1.5, digamma(3.0) - math.log(2.0)]], dtype=torch.float64, device=dev)
    params, status = mstep_family(expfam.GAMMA, 0.0, m.clone(), m.clone())
    assert status.cpu().tolist() == [1, 0]
    np.testing.assert_allclose(params[1].cpu().numpy(), [3.0, 2.0], rtol=1e-12)
