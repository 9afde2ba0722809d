"""Backward ancestral index resampling and the predictive log-likelihood -- TEST INFRASTRUCTURE
ONLY (oracle/__init__.py).  NEXT row f3 (R31): "we draw latent samples conditioned on
'training' data ... and use these to predict a separate 'test' set",
"averaged over 100 predictive samples", for the two-level family.

Given the oracle's E-step (oracle.estep: w_root, messages g_i(k)), the posterior over index
tuples (Eq. 7a-c) factorises in reverse elimination order:
  k_root ~ w_root,   k_i | k_root ~ P_i(k'|k) = exp(B_i(k,k') + A_i(k') - ln K - g_i(k))
with B_i(k,k') = log N(z_i^k'; mu_k, V_k I) and A_i(k') = sum_j log p(x_ij | z_i^k') -
log q_i(z_i^k'), written here in numpy from the model's densities (independent of qem_oracle.c,
whose g must make every P_i(.|k) sum to 1 -- pinned in tests/test_predict.py).  Draws: inverse
CDF with a sequential fp64 prefix (np.cumsum) on u = ((w >> 8) + 1/2) 2^-24, w = word 0 of
Philox4x32-10 at (s, 0, 0, 5<<24) (root) and (s, 1 + i, 0, 5<<24) (instance i).
PLL = log (1/S) sum_s exp(sum_i sum_j log p(x_test_ij | z_i^{k_i,s})).
"""
from __future__ import annotations

import numpy as np
from scipy.special import logsumexp

from . import oracle

TAG = 5 << 24


def _lnN(x, m, v):
    return -0.5 * np.log(2 * np.pi * v) - (x - m) ** 2 / (2 * v)


def _uniform(s, slot, seed):
    w = oracle.philox((s, slot, 0, TAG), (seed & 0xffffffff, (seed >> 32) & 0xffffffff))[0]
    return ((w >> 8) + 0.5) * 2.0 ** -24


def _inverse_cdf(p, u):
    """First index whose sequential prefix exceeds u * sum; also the distance of u * sum to the
    nearest prefix boundary (relative to the sum), for tie-tolerant comparisons."""
    c = np.cumsum(p)
    t = u * c[-1]
    k = int(min(np.searchsorted(c, t, side="right"), len(p) - 1))
    margin = float(np.min(np.abs(c - t)) / c[-1])
    return k, margin


def log_conditionals(m, z, q, data, g, i):
    """log P_i(k'|k) [K(k)][K(k')] for group i (two-level)."""
    K, d, R = m.K, m.d, m.R
    zr = np.asarray(z[0], np.float64).reshape(R, K)
    zi = np.asarray(z[1], np.float64).reshape(m.n, d, K)[i]
    qm = np.asarray(q[1][0], np.float64).reshape(m.n, d)[i]
    qv = np.asarray(q[1][1], np.float64).reshape(m.n, d)[i]
    if m.scale_kind == 0:
        V = np.full(K, m.fixed_var)
    elif m.scale_kind == 1:
        V = np.exp(2 * zr[d])
    else:
        V = np.exp(zr[d])
    B = sum(_lnN(zi[r][None, :], zr[r][:, None], V[:, None]) for r in range(d))
    A = -sum(_lnN(zi[r], qm[r], qv[r]) for r in range(d))
    if m.obs_kind == 1:
        A = A + sum(_lnN(float(data.xg[i, j]), zi[0], m.obs_var) for j in range(m.J))
    else:
        for j in range(m.J):
            eta = data.xb[i, j].astype(np.float64) @ zi
            A = A + float(data.yb[i, j]) * eta - np.logaddexp(0.0, eta)
    return B + A[None, :] - np.log(K) - np.asarray(g)[i][:, None]


def resample(m, z, q, data, est, S, seed, g_begin=0):
    """S index tuples: idx_root [S], idx [S][n], and the CDF margins of every draw.  g_begin: the
    global index of local instance 0 (the uniforms are keyed by the global instance)."""
    w_root = np.asarray(est["w"][0]).reshape(-1)
    idx_root, mr = np.zeros(S, np.int32), np.zeros(S)
    idx, mg = np.zeros((S, m.n), np.int32), np.zeros((S, m.n))
    logp = [log_conditionals(m, z, q, data, est["g"], i) for i in range(m.n)]
    for s in range(S):
        idx_root[s], mr[s] = _inverse_cdf(w_root, _uniform(s, 0, seed))
        for i in range(m.n):
            row = logp[i][idx_root[s]]
            idx[s, i], mg[s, i] = _inverse_cdf(np.exp(row - row.max()), _uniform(s, 1 + g_begin + i, seed))
    return dict(idx_root=idx_root, idx=idx, margin_root=mr, margin=mg)


def test_loglik(m, z, test, idx):
    """ll_part [S][n]: sum_j log p(x_test_ij | z_i^{idx[s][i]})."""
    K, d = m.K, m.d
    zi = np.asarray(z[1], np.float64).reshape(m.n, d, K)
    S = idx.shape[0]
    out = np.zeros((S, m.n))
    for s in range(S):
        zs = zi[np.arange(m.n), :, idx[s]]                     # [n][d]
        if m.obs_kind == 1:
            out[s] = _lnN(np.asarray(test.xg, np.float64), zs[:, 0:1], m.obs_var).sum(axis=1)
        else:
            eta = np.einsum("njd,nd->nj", np.asarray(test.xb, np.float64), zs)
            out[s] = (np.asarray(test.yb, np.float64) * eta - np.logaddexp(0.0, eta)).sum(axis=1)
    return out


def predictive_loglik(ll_part):
    ll_s = np.asarray(ll_part).sum(axis=1)
    return float(logsumexp(ll_s) - np.log(len(ll_s))), ll_s


def global_iw(m, z, q, data, est):
    """Global importance weighting (App. A, Eq. glob_iw): K joint draws with every
    latent at index k.  log r_k = f_root(k) + sum_i [B_i(k, z_i^k) + A_i(z_i^k)] with B + A recovered
    from the conditionals (log P + ln K + g); returns log_pe, weights w [K], group means m1 [n][d]."""
    K, d, R = m.K, m.d, m.R
    lk = np.log(K)
    diag = np.zeros((m.n, K))
    for i in range(m.n):
        lp = log_conditionals(m, z, q, data, est["g"], i)
        diag[i] = np.diag(lp) + lk + np.asarray(est["g"])[i]
    zr = np.asarray(z[0], np.float64).reshape(R, K)
    qrm, qrv = (np.asarray(a, np.float64) for a in q[0])
    f_root = sum(_lnN(zr[r], m.prior_mean, m.prior_var) - _lnN(zr[r], qrm[r], qrv[r]) for r in range(R))
    a = f_root + diag.sum(axis=0)
    lse = logsumexp(a)
    w = np.exp(a - lse)
    zg = np.asarray(z[1], np.float64).reshape(m.n, d, K)
    return dict(log_pe=lse - lk, w=w, m1=(zg * w[None, None, :]).sum(axis=2), diag=diag)
