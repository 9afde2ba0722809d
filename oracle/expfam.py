"""Exponential-family M-steps from mean parameters -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

QEM's M-step sets Q_t from the EMA of its mean parameters (Alg. 1 line 3, PAPER.md:175;
"exponential family distributions are completely determined by their mean parameters",
PAPER.md:247; "a Beta's parameters are recovered from expectations of log transformations",
PAPER.md:218).  Plain scipy, fp64, following the definitions:

  Gamma(k shape, th rate)  T(z) = (z, ln z)          m = (k/th, psi(k) - ln th)
  Beta(a, b)               T(z) = (ln z, ln(1-z))    m = (psi(a) - psi(a+b), psi(b) - psi(a+b))
  Dirichlet(a_1..a_C)      T(z) = ln z               m = psi(a) - psi(sum a)
  Binomial(N, p)           T(z) = z                  m = N p
  Multinomial(N, p)        T(z) = z                  m = N p
  Bernoulli(p)             T(z) = z                  m = p
  Categorical(p_1..p_C)    T(z) = onehot(z)          m = p

The inverse maps are solved with scipy root finders (brentq for the Gamma shape on
psi(k) - ln k = m2 - ln m1, a 2-d hybrid root for Beta in log-parameter space) -- a different
algorithm from the device Newton iterations; they are pinned against the closed-form forward maps
above and against SPEC.md's worked examples.
"""
from __future__ import annotations

import numpy as np
from scipy import optimize
from scipy.special import digamma

GAMMA, BETA, BERNOULLI, CATEGORICAL, DIRICHLET, BINOMIAL, MULTINOMIAL = 1, 2, 3, 4, 5, 6, 7


def gamma_mean(k, th):
    return np.array([k / th, digamma(k) - np.log(th)])


def beta_mean(a, b):
    s = digamma(a + b)
    return np.array([digamma(a) - s, digamma(b) - s])


def gamma_params(m):
    """(k, th) with gamma_mean(k, th) = m; requires ln m1 > m2 (Jensen)."""
    m1, m2 = float(m[0]), float(m[1])
    s = m2 - np.log(m1)  # psi(k) - ln k, < 0, increasing in k
    if not s < 0:
        raise ValueError("infeasible Gamma moments: need ln E[z] > E[ln z]")
    f = lambda lk: digamma(np.exp(lk)) - lk - s  # noqa: E731
    lo, hi = -40.0, 40.0
    lk = optimize.brentq(f, lo, hi, xtol=1e-15, rtol=1e-15, maxiter=500)
    k = np.exp(lk)
    return np.array([k, k / m1])


def beta_params(m):
    """(a, b) with beta_mean(a, b) = m; requires both components < 0 and exp(m1) + exp(m2) < 1."""
    m = np.asarray(m, np.float64)
    if not (m[0] < 0 and m[1] < 0 and np.exp(m[0]) + np.exp(m[1]) < 1):
        raise ValueError("infeasible Beta moments")
    f = lambda x: beta_mean(np.exp(x[0]), np.exp(x[1])) - m  # noqa: E731
    # moment-matching start (mean e^m1 share, precision 1)
    r = optimize.root(f, x0=np.log([1.0, 1.0]), method="hybr", tol=1e-15)
    if not r.success or np.max(np.abs(f(r.x))) > 1e-10:
        r = optimize.root(f, x0=np.log([0.5, 0.5]), method="lm", tol=1e-15)
    return np.exp(r.x)


def dirichlet_mean(a):
    a = np.asarray(a, np.float64)
    return digamma(a) - digamma(a.sum())


def dirichlet_params(m):
    """a with dirichlet_mean(a) = m; requires every m_c < 0 and sum exp(m) < 1."""
    m = np.asarray(m, np.float64)
    if not (np.all(m < 0) and np.exp(m).sum() < 1):
        raise ValueError("infeasible Dirichlet moments")
    f = lambda x: dirichlet_mean(np.exp(x)) - m  # noqa: E731
    r = optimize.root(f, x0=np.zeros_like(m), method="hybr", tol=1e-15)
    if not r.success or np.max(np.abs(f(r.x))) > 1e-10:
        r = optimize.root(f, x0=np.full_like(m, -0.5), method="lm", tol=1e-15)
    return np.exp(r.x)


def params_from_mean(family, m, C=None):
    """Conventional parameters from mean parameters, row by row (m: [n][S])."""
    m = np.atleast_2d(np.asarray(m, np.float64))
    if family == GAMMA:
        return np.array([gamma_params(r) for r in m])
    if family == BETA:
        return np.array([beta_params(r) for r in m])
    if family == BERNOULLI:
        return m.copy()
    if family in (CATEGORICAL, MULTINOMIAL):
        return m / m.sum(axis=1, keepdims=True)
    if family == DIRICHLET:
        return np.array([dirichlet_params(r) for r in m])
    if family == BINOMIAL:
        return m / C
    raise ValueError(family)


def ema_mstep(family, lam, m_ema, m_new, C=None):
    """EMA over mean parameters (Eq. 9, history weight lam, R5), then the M-step."""
    m = lam * np.asarray(m_ema, np.float64) + (1.0 - lam) * np.asarray(m_new, np.float64)
    return m, params_from_mean(family, m, C)
