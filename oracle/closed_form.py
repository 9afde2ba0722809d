"""Closed-form conjugate Gaussian posterior and evidence -- TEST INFRASTRUCTURE ONLY.

For the config-1 model (mu ~ N(0, pv), z_i | mu ~ N(mu, V), x_ij | z_i ~ N(z_i, s2))
the joint over theta = (mu, z_1..z_M) and x is Gaussian, so Bayes' theorem
(Sec. 3.1: P(z'|x) = P(x|z')P(z')/P(x)) has a closed form.
Two independent routes are provided:
  posterior()   joint precision  Lambda = Lambda_prior + Lambda_lik,
                mean = Lambda^{-1} b, cov = Lambda^{-1}          (textbook update)
  log_evidence() marginal x ~ N(0, s2 I + V blockdiag(11^T) + pv 11^T)
                evaluated with scipy's multivariate normal log-pdf.
These pin the oracle's K -> infinity limit (App. C) and the
unbiasedness of Pe.
"""
from __future__ import annotations

import numpy as np
from scipy.stats import multivariate_normal


def posterior(x, prior_var=1.0, group_var=1.0, obs_var=1.0):
    """x: [M][J] observations. Returns (mean [1+M], cov [1+M][1+M]) over (mu, z_1..z_M)."""
    x = np.asarray(x, np.float64)
    M, J = x.shape
    Lam = np.zeros((M + 1, M + 1))
    b = np.zeros(M + 1)
    # prior: -mu^2/(2 pv) - sum_i (z_i - mu)^2 / (2 V)
    Lam[0, 0] = 1.0 / prior_var + M / group_var
    for i in range(M):
        Lam[0, 1 + i] = Lam[1 + i, 0] = -1.0 / group_var
        Lam[1 + i, 1 + i] = 1.0 / group_var + J / obs_var
        b[1 + i] = x[i].sum() / obs_var
    cov = np.linalg.inv(Lam)
    return cov @ b, cov


def log_evidence(x, prior_var=1.0, group_var=1.0, obs_var=1.0):
    """log p(x) from the marginal covariance of the flattened observations."""
    x = np.asarray(x, np.float64)
    M, J = x.shape
    n = M * J
    S = obs_var * np.eye(n) + prior_var * np.ones((n, n))
    for i in range(M):
        S[i * J:(i + 1) * J, i * J:(i + 1) * J] += group_var
    return float(multivariate_normal(mean=np.zeros(n), cov=S).logpdf(x.reshape(-1)))


def single_latent(x, prior_var=1.0, obs_var=1.0):
    """z ~ N(0, pv), x_j | z ~ N(z, s2): posterior (mean, var) and log p(x) (SPEC.md:514 example)."""
    x = np.atleast_1d(np.asarray(x, np.float64))
    prec = 1.0 / prior_var + x.size / obs_var
    var = 1.0 / prec
    mean = var * x.sum() / obs_var
    n = x.size
    S = obs_var * np.eye(n) + prior_var * np.ones((n, n))
    return mean, var, float(multivariate_normal(mean=np.zeros(n), cov=S).logpdf(x))
