"""Literal K^n enumeration of Eq. 7a-c -- TEST INFRASTRUCTURE ONLY.

Independent of qem_oracle.c (different language, no elimination): it
materialises log r_k for EVERY index tuple k in K^n (PAPER.md:143-149,
Sec. 3.2, Eq. 7b: r_k = P(x, z^k) / prod_i Q(z_i^{k_i})), then
  Pe   = (1/K^n) sum_k r_k                                   (Eq. 7c)
  w_i  = sum_{k: k_i = c} r_k / sum_k r_k                    (Eq. 7a, m = 1[k_i = c])
  E[T] = sum_k r_k T(z_i^{k_i}) / sum_k r_k                  (Eq. 7a, T = (z, z^2))
Densities are written from their textbook formulas with numpy/scipy special
functions.  Guarded to K^n <= 2e6.
"""
from __future__ import annotations

import numpy as np
from scipy.special import gammaln, logsumexp


def _lnN(x, m, v):
    return -0.5 * np.log(2 * np.pi * v) - (x - m) ** 2 / (2 * v)


def _axis(a, ax, n):
    """Reshape 1-D/2-D table so its axes land on tuple axes ``ax`` of an n-axis grid."""
    shape = [1] * n
    if np.ndim(a) == 1:
        shape[ax[0]] = a.shape[0]
        return a.reshape(shape)
    if ax[0] < ax[1]:
        shape[ax[0]], shape[ax[1]] = a.shape
        return a.reshape(shape)
    shape[ax[1]], shape[ax[0]] = a.shape[1], a.shape[0]
    return a.T.reshape(shape)


def _finish(logr, zs_per_axis):
    n = logr.ndim
    K = logr.shape[0]
    log_pe = logsumexp(logr) - n * np.log(K)
    wfull = np.exp(logr - logsumexp(logr))
    ws, m1s, m2s = [], [], []
    for ax, zax in enumerate(zs_per_axis):
        w = wfull.sum(axis=tuple(a for a in range(n) if a != ax))
        ws.append(w)
        m1s.append(zax @ w)           # zax: [dims][K]
        m2s.append((zax ** 2) @ w)
    return log_pe, ws, m1s, m2s


def estep2(m, z, q, data, joint=False):
    """Enumerate a two-level model (axes: root, group 0..n-1). Same I/O as oracle.estep; with
    joint=True also the normalised weight of every index tuple, [K]*(n+1) (root axis first)."""
    K, n, d, R = m.K, m.n, m.d, m.R
    assert K ** (n + 1) <= 2_000_000, "enumeration guard"
    zr = np.asarray(z[0], np.float64).reshape(R, K)
    zg = np.asarray(z[1], np.float64).reshape(n, d, K)
    qrm, qrv = (np.asarray(a, np.float64) for a in q[0])
    qgm, qgv = (np.asarray(a, np.float64).reshape(n, d) for a in q[1])
    N = n + 1
    logr = np.zeros([K] * N)
    # log p(root^k) - log q(root^k)
    f = sum(_lnN(zr[r], m.prior_mean, m.prior_var) - _lnN(zr[r], qrm[r], qrv[r]) for r in range(R))
    logr = logr + _axis(f, [0], N)
    if m.scale_kind == 0:
        V = np.full(K, m.fixed_var)
    elif m.scale_kind == 1:
        V = np.exp(2 * zr[d])
    else:
        V = np.exp(zr[d])
    for i in range(n):
        # log p(z_i^{k_i} | root^{k_0}) : table [k0][ki]
        t = np.zeros((K, K))
        for r in range(d):
            t += _lnN(zg[i, r][None, :], zr[r][:, None], V[:, None])
        logr = logr + _axis(t, [0, i + 1], N)
        # log p(x_i | z_i^{k_i}) - log q(z_i^{k_i}) : [ki]
        u = np.zeros(K)
        for r in range(d):
            u -= _lnN(zg[i, r], qgm[i, r], qgv[i, r])
        if m.obs_kind == 1:
            for j in range(m.J):
                u += _lnN(float(data.xg[i, j]), zg[i, 0], m.obs_var)
        else:
            for j in range(m.J):
                eta = data.xb[i, j].astype(np.float64) @ zg[i]
                y = float(data.yb[i, j])
                u += y * eta - np.logaddexp(0.0, eta)
        logr = logr + _axis(u, [i + 1], N)
    zs = [zr] + [zg[i] for i in range(n)]
    log_pe, ws, m1s, m2s = _finish(logr, zs)
    out = dict(log_pe=log_pe, w=[ws[0][None, :], np.stack(ws[1:])],
               m1=[m1s[0], np.concatenate(m1s[1:])], m2=[m2s[0], np.concatenate(m2s[1:])])
    if joint:
        out["joint"] = np.exp(logr - logsumexp(logr))
    return out


def estep3(m, z, q, data):
    """Enumerate the three-level model (axes: root, tops a, subs ab)."""
    K, A, B, P, R = m.K, m.n, m.B, m.P, m.R
    N = 1 + A + A * B
    assert K ** N <= 2_000_000, "enumeration guard"
    zr = np.asarray(z[0], np.float64).reshape(R, K)
    zt = np.asarray(z[1], np.float64).reshape(A, K)
    zs = np.asarray(z[2], np.float64).reshape(A * B, K)
    (qrm, qrv), (qtm, qtv), (qsm, qsv) = [(np.asarray(a, np.float64), np.asarray(b, np.float64)) for a, b in q]
    logr = np.zeros([K] * N)
    f = sum(_lnN(zr[r], m.prior_mean, m.prior_var) - _lnN(zr[r], qrm[r], qrv[r]) for r in range(R))
    logr = logr + _axis(f, [0], N)
    for a in range(A):
        ax_a = 1 + a
        t = _lnN(zt[a][None, :], zr[0][:, None], m.top_var)            # [kr][ka]
        logr = logr + _axis(t, [0, ax_a], N)
        logr = logr + _axis(-_lnN(zt[a], qtm[a], qtv[a]), [ax_a], N)
        for b in range(B):
            ab = a * B + b
            ax_ab = 1 + A + ab
            t = _lnN(zs[ab][None, :], zt[a][:, None], m.sub_var)         # [ka][kab]
            logr = logr + _axis(t, [ax_a, ax_ab], N)
            logr = logr + _axis(-_lnN(zs[ab], qsm[ab], qsv[ab]), [ax_ab], N)
            ll = np.zeros((K, K))                                        # [kr][kab]
            for j in range(m.J):
                eta = zs[ab][None, :] + (np.asarray(data.xp[ab, j], np.float64) @ zr[1:])[:, None]
                y = float(data.yp[ab, j])
                ll += y * eta - np.exp(eta) - gammaln(y + 1.0)
            logr = logr + _axis(ll, [0, ax_ab], N)
    zlist = [zr] + [zt[a][None, :] for a in range(A)] + [zs[ab][None, :] for ab in range(A * B)]
    log_pe, ws, m1s, m2s = _finish(logr, zlist)
    return dict(log_pe=log_pe, w=[ws[0][None, :], np.stack(ws[1:1 + A]), np.stack(ws[1 + A:])],
                m1=[m1s[0], np.concatenate(m1s[1:1 + A]), np.concatenate(m1s[1 + A:])],
                m2=[m2s[0], np.concatenate(m2s[1:1 + A]), np.concatenate(m2s[1 + A:])])


def estep(m, z, q, data):
    return estep2(m, z, q, data) if m.family == 2 else estep3(m, z, q, data)
