"""Non-factorised massively parallel proposal Q_MP with its parent-copy schemes (App. A,
PAPER.md:470-479, second half) -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Conjugate two-level Gaussian hierarchy (the config-1 / config-4 family): mu ~ N(0, pv),
z_i | mu ~ N(mu, gv), x_ij | z_i ~ N(z_i, ov), with the single-sample proposal
Q(mu) = N(m, v), Q(z_i | mu) = N(alpha_i + beta_i mu, s_i)   (a child that depends on its parent).
Plain numpy / scipy fp64, written from the definitions:

  Q_MP     PAPER.md:470-476: every latent has K copies; "a scheme for choosing which of the K copies of
           a parent latent gets used in the sampling of each K copy of the child":
             permutation  copy[i] a uniformly random permutation of 0..K-1 ("the permutation strategy
                          was used"): z_i^k' ~ Q(. | mu^copy[i][k']), so
                          q_MP,i(k') = N(z_i^k'; alpha_i + beta_i mu^copy[i][k'], s_i)
             mixture      "a uniform mixture over the K parent samples": the copy index
                          is drawn uniformly per child copy and marginalised in the density,
                          q_MP,i(k') = (1/K) sum_k N(z_i^k'; alpha_i + beta_i mu^k, s_i)
           The copy indices and the standard normals eps are inputs (drawn by the caller).
  tables   Eq. 7c's ratio r_k(z) = P(x, z^k) / prod_i Q_MP(z_i^k_i | parents) as
           log-factor tables: f_root(k) = log N(mu^k; 0, pv) - log N(mu^k; m, v),
           f_i(k, k') = log N(z_i^k'; mu^k, gv) + sum_j log N(x_ij; z_i^k', ov) - log q_MP,i(k')
  E-step   oracle/tables.py (Eq. 7, pinned by enumeration)
  moments  (E z_i, E z_i^2) per group and (E mu, E mu^2) under the marginal weights (Eq. 7a)

DESIGN.md R43.  Pinned by tests/test_qmp.py: beta = 0 reduces to the factorised Q of qem_oracle.c
(independent C code, same samples); exp(log Pe) is unbiased for the closed-form evidence under both
schemes (oracle/closed_form.py); K = 1 makes the two schemes the same density; the mixture density
integrates to 1 (quadrature).
"""
from __future__ import annotations

import numpy as np
from scipy.special import logsumexp
from scipy.stats import norm

from . import tables

PERMUTATION, MIXTURE = 0, 1


def draw_copies(rng, n, K, scheme):
    """Parent-copy indices [n][K]: a random permutation per group, or iid uniform indices."""
    if scheme == PERMUTATION:
        return np.array([rng.permutation(K) for _ in range(n)], np.int32).reshape(n, K)
    return rng.integers(0, K, size=(n, K)).astype(np.int32)


def sample_children(mu, q, copy, eps):
    """z[i][k'] = alpha_i + beta_i mu^copy[i][k'] + sqrt(s_i) eps[i][k'] (fp64)."""
    mu = np.asarray(mu, np.float64)
    q = np.asarray(q, np.float64)
    return q[:, 0:1] + q[:, 1:2] * mu[copy] + np.sqrt(q[:, 2:3]) * np.asarray(eps, np.float64)


def log_qmp(z, mu, q, copy, scheme):
    """log q_MP,i(k') [n][K] under the scheme."""
    mu = np.asarray(mu, np.float64)
    q = np.asarray(q, np.float64)
    sd = np.sqrt(q[:, 2:3])
    if scheme == PERMUTATION:
        return norm.logpdf(z, loc=q[:, 0:1] + q[:, 1:2] * mu[copy], scale=sd)
    K = mu.shape[0]
    loc = q[:, 0, None, None] + q[:, 1, None, None] * mu[None, None, :]  # [n][1][K parents]
    return logsumexp(norm.logpdf(z[:, :, None], loc=loc, scale=sd[:, :, None]), axis=2) - np.log(K)


def make_tables(mu, root_mean, root_var, q, copy, z, x, scheme, prior_var=1.0, group_var=1.0, obs_var=1.0):
    mu = np.asarray(mu, np.float64)
    x = np.asarray(x, np.float64)
    f_root = norm.logpdf(mu, 0.0, np.sqrt(prior_var)) - norm.logpdf(mu, float(root_mean), np.sqrt(float(root_var)))
    ll = norm.logpdf(x[:, None, :], loc=z[:, :, None], scale=np.sqrt(obs_var)).sum(axis=2)  # [n][K']
    lq = log_qmp(z, mu, q, copy, scheme)
    f = norm.logpdf(z[:, None, :], loc=mu[None, :, None], scale=np.sqrt(group_var)) + (ll - lq)[:, None, :]
    return f_root, f


def estep(mu, root_mean, root_var, q, copy, eps, x, scheme, **var):
    z = sample_children(mu, q, copy, eps)
    f_root, f = make_tables(mu, root_mean, root_var, q, copy, z, x, scheme, **var)
    out = tables.estep_tables(f_root, f)
    mu = np.asarray(mu, np.float64)
    out["z"] = z
    out["root_m"] = np.array([out["w_root"] @ mu, out["w_root"] @ (mu * mu)])
    out["gm"] = np.stack([(out["w"] * z).sum(axis=1), (out["w"] * z * z).sum(axis=1)], axis=1)
    return out
