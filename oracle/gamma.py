"""Gamma and Beta approximate posteriors on the E-step side: the Gamma-Poisson and Beta-Binomial
hierarchies of row f1 (R32) -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).
Beta draws are X / (X + Y) of two Marsaglia-Tsang Gammas (Philox streams 7<<24, 8<<24); the
Beta-Binomial tables use scipy.stats beta / binom log-densities; the rest mirrors the Gamma
model below.  numpy/scipy fp64, following
Algorithm 1 step by step:

  sample   root mu^k = fmaf(sqrtf(v), eps, m) (fp32, R22; oracle.sample); lambda_i^k by
           Marsaglia-Tsang: attempt a of (i, k) from Philox4x32-10 at (k, a, i, 6<<24 | t):
           x = sqrt(-2 ln u0) cos(2 pi u1), accept if ln u2 < x^2/2 + d - d v + d ln v,
           v = (1 + c x)^3, d = shape' - 1/3, c = 1/sqrt(9 d) (shape' = shape, or shape + 1 with the
           boost u3^(1/shape) when shape < 1); u_j = (word_j + 1/2) 2^-32
  tables   f_root(k) = log N(mu^k; 0, 1) - log N(mu^k; m, v)
           f_i(k,k') = log Gamma(l; alpha, rate alpha e^-mu^k) + sum_j log Pois(y_ij; l)
                       - log Gamma(l; shape_i, rate_i)      (scipy.stats log-densities)
  E-step   oracle/tables.py (Eq. 7)
  moments  (E l, E ln l) per group, (E mu, E mu^2) for the root
  M-step   EMA (history weight lam) + oracle/expfam.py's Gamma inverse (brentq), root Gaussian
Pinned by tests/test_gamma.py: sampler moments, exp(log Pe) unbiased for p(y) from 1-D quadrature
over mu with the rates integrated out in closed form (negative binomial), and the M-step round trip.
"""
from __future__ import annotations

import numpy as np
from scipy import stats

from . import expfam, oracle, tables

TAG = 6 << 24


def _u(w):
    return (w + 0.5) * 2.0 ** -32


def _mt_gamma(a, k, i, word, key):
    """Gamma(a, rate 1) by Marsaglia-Tsang, attempt att from Philox at (k, att, i, word)."""
    d = (a + 1.0 if a < 1.0 else a) - 1.0 / 3.0
    c = 1.0 / np.sqrt(9.0 * d)
    for att in range(64):
        w = oracle.philox((k, att, i, word), key)
        x = np.sqrt(-2.0 * np.log(_u(w[0]))) * np.cos(2.0 * np.pi * _u(w[1]))
        v1 = 1.0 + c * x
        if v1 <= 0.0:
            continue
        v = v1 ** 3
        if np.log(_u(w[2])) < 0.5 * x * x + d - d * v + d * np.log(v):
            g = d * v
            if a < 1.0:
                g *= _u(w[3]) ** (1.0 / a)
            return g
    return np.nan


def sample_gamma(q, K, seed, t):
    q = np.asarray(q, np.float64)
    key = (seed & 0xffffffff, (seed >> 32) & 0xffffffff)
    z = np.full((q.shape[0], K), np.nan)
    for i in range(q.shape[0]):
        for k in range(K):
            z[i, k] = _mt_gamma(q[i, 0], k, i, TAG | (t & 0xffffff), key) / q[i, 1]
    return z


def sample_beta(q, K, seed, t):
    """Beta(a, b) = X / (X + Y), X ~ Gamma(a) on stream 7 << 24, Y ~ Gamma(b) on 8 << 24."""
    q = np.asarray(q, np.float64)
    key = (seed & 0xffffffff, (seed >> 32) & 0xffffffff)
    z = np.full((q.shape[0], K), np.nan)
    for i in range(q.shape[0]):
        for k in range(K):
            x = _mt_gamma(q[i, 0], k, i, (7 << 24) | (t & 0xffffff), key)
            y = _mt_gamma(q[i, 1], k, i, (8 << 24) | (t & 0xffffff), key)
            z[i, k] = x / (x + y)
    return z


def make_tables(gp, mu, root_mean, root_var, q, z):
    mu = np.asarray(mu, np.float64)
    m = float(np.float32(root_mean))
    v = float(np.float32(root_var))
    f_root = stats.norm.logpdf(mu, 0.0, 1.0) - stats.norm.logpdf(mu, m, np.sqrt(v))
    q = np.asarray(q, np.float64)
    lam = np.asarray(z, np.float64)                                    # [n][K']
    prior = stats.gamma.logpdf(lam[:, None, :], gp.alpha, scale=(np.exp(mu) / gp.alpha)[None, :, None])
    lik = stats.poisson.logpmf(np.asarray(gp.y)[:, None, :], lam[:, :, None]).sum(axis=2)  # [n][K']
    lq = stats.gamma.logpdf(lam, q[:, 0:1], scale=1.0 / q[:, 1:2])
    return f_root, prior + (lik - lq)[:, None, :]


def moments(mu, z, w_root, w):
    mu = np.asarray(mu, np.float64)
    root_m = np.array([(w_root * mu).sum(), (w_root * mu * mu).sum()])
    lam = np.asarray(z, np.float64)
    gm = np.stack([(w * lam).sum(axis=1), (w * np.log(lam)).sum(axis=1)], axis=1)
    return root_m, gm


def initial_state(gp):
    q = np.tile([1.0, 1.0], (gp.n, 1))                           # Gamma(1, 1)
    g_ema = np.array([expfam.gamma_mean(1.0, 1.0)] * gp.n)
    return dict(root_mean=np.float32(0.0), root_var=np.float32(1.0), root_ema=np.array([0.0, 1.0]), q=q,
                g_ema=g_ema)


def qem_step(gp, state, t, seed, eps_root, new_weight=0.3, floor=1e-8):
    mu = oracle.sample(np.array([state["root_mean"]]), np.array([state["root_var"]]), eps_root[None, :])[0]
    z = sample_gamma(state["q"], gp.K, seed, t)
    f_root, f = make_tables(gp, mu, state["root_mean"], state["root_var"], state["q"], z)
    est = tables.estep_tables(f_root, f)
    root_m, gm = moments(mu, z, est["w_root"], est["w"])
    lam = oracle.lam(t, new_weight, 0.0)
    root_ema = lam * state["root_ema"] + (1 - lam) * root_m
    var = root_ema[1] - root_ema[0] ** 2
    g_ema, q = expfam.ema_mstep(expfam.GAMMA, lam, state["g_ema"], gm)
    nxt = dict(root_ema=root_ema, root_mean=np.float32(root_ema[0]), root_var=np.float32(max(var, floor)),
               g_ema=g_ema, q=q)
    return dict(mu=mu, z=z, f_root=f_root, f=f, est=est, root_m=root_m, gm=gm, next=nxt)


# ---------------------------------------------------------------- Beta-Binomial (Beta Q)


def make_tables_beta(bb, mu, root_mean, root_var, q, z):
    mu = np.asarray(mu, np.float64)
    m = float(np.float32(root_mean))
    v = float(np.float32(root_var))
    f_root = stats.norm.logpdf(mu, 0.0, 1.0) - stats.norm.logpdf(mu, m, np.sqrt(v))
    q = np.asarray(q, np.float64)
    p = np.asarray(z, np.float64)                                      # [n][K']
    s = 1.0 / (1.0 + np.exp(-mu))                                      # [K]
    prior = stats.beta.logpdf(p[:, None, :], (bb.kappa * s)[None, :, None], (bb.kappa * (1 - s))[None, :, None])
    lik = stats.binom.logpmf(np.asarray(bb.y)[:, None], np.asarray(bb.N)[:, None], p)
    lq = stats.beta.logpdf(p, q[:, 0:1], q[:, 1:2])
    return f_root, prior + (lik - lq)[:, None, :]


def moments_beta(mu, z, w_root, w):
    mu = np.asarray(mu, np.float64)
    root_m = np.array([(w_root * mu).sum(), (w_root * mu * mu).sum()])
    p = np.asarray(z, np.float64)
    gm = np.stack([(w * np.log(p)).sum(axis=1), (w * np.log1p(-p)).sum(axis=1)], axis=1)
    return root_m, gm


def initial_state_beta(bb):
    q = np.tile([1.0, 1.0], (bb.n, 1))                           # Beta(1, 1)
    g_ema = np.array([expfam.beta_mean(1.0, 1.0)] * bb.n)
    return dict(root_mean=np.float32(0.0), root_var=np.float32(1.0), root_ema=np.array([0.0, 1.0]), q=q,
                g_ema=g_ema)


def qem_step_beta(bb, state, t, seed, eps_root, new_weight=0.3, floor=1e-8):
    mu = oracle.sample(np.array([state["root_mean"]]), np.array([state["root_var"]]), eps_root[None, :])[0]
    z = sample_beta(state["q"], bb.K, seed, t)
    f_root, f = make_tables_beta(bb, mu, state["root_mean"], state["root_var"], state["q"], z)
    est = tables.estep_tables(f_root, f)
    root_m, gm = moments_beta(mu, z, est["w_root"], est["w"])
    lam = oracle.lam(t, new_weight, 0.0)
    root_ema = lam * state["root_ema"] + (1 - lam) * root_m
    var = root_ema[1] - root_ema[0] ** 2
    g_ema, q = expfam.ema_mstep(expfam.BETA, lam, state["g_ema"], gm)
    nxt = dict(root_ema=root_ema, root_mean=np.float32(root_ema[0]), root_var=np.float32(max(var, floor)),
               g_ema=g_ema, q=q)
    return dict(mu=mu, z=z, f_root=f_root, f=f, est=est, root_m=root_m, gm=gm, next=nxt)
