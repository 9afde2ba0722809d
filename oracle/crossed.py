"""Crossed effects (row f4, R33) -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Bus-Breakdown-shaped model: root (mu, company weights cw_c, journey-type
weights jw_t) ~ N(0, I) sharing one sample index; groups w_i ~ N(mu, 1); delays y_ij ~
Bernoulli(sigmoid(w_i + cw_{comp_ij} + jw_{jtype_ij})).  numpy/scipy fp64, Algorithm 1 step by step:
  tables   f_root(k) = sum_r log N(r^k; 0, 1) - log q(r^k)
           f_i(k,k') = log N(w_i^k'; mu^k, 1) + sum_j log Bernoulli(y_ij; sigmoid(eta))
                       - log q_i(w_i^k'),  eta = w_i^k' + cw^k_{comp_ij} + jw^k_{jtype_ij}
  E-step   oracle/tables.py (Eq. 7)
  moments  (E x, E x^2) for every root dim and group latent; EMA + Gaussian M-step (floor).
Pinned by tests/test_crossed.py: exp(log Pe) unbiased for p(y) from 4-D Gauss-Hermite quadrature on
a one-company / one-journey-type / one-group model.
"""
from __future__ import annotations

import numpy as np
from scipy import stats
from scipy.special import log_expit

from . import oracle, tables


def make_tables(cm, rz, root_mean, root_var, z, q_mean, q_var):
    rz = np.asarray(rz, np.float64)                                    # [R][K]
    rm = np.asarray(root_mean, np.float32).astype(np.float64)
    rv = np.asarray(root_var, np.float32).astype(np.float64)
    f_root = (stats.norm.logpdf(rz) - stats.norm.logpdf(rz, rm[:, None], np.sqrt(rv)[:, None])).sum(axis=0)
    z = np.asarray(z, np.float64)                                      # [n][K']
    qm = np.asarray(q_mean, np.float32).astype(np.float64)
    qv = np.asarray(q_var, np.float32).astype(np.float64)
    prior = stats.norm.logpdf(z[:, None, :], rz[0][None, :, None], 1.0)            # [n][K][K']
    off = rz[1 + cm.comp] + rz[1 + cm.C + cm.jtype]                                  # [n][J][K]
    eta = z[:, None, None, :] + off.transpose(0, 2, 1)[:, :, :, None]                # [n][K][J][K']
    y = np.asarray(cm.y, np.float64)[:, None, :, None]
    lik = (y * log_expit(eta) + (1 - y) * log_expit(-eta)).sum(axis=2)              # [n][K][K']
    lq = stats.norm.logpdf(z, qm[:, None], np.sqrt(qv)[:, None])
    return f_root, prior + lik - lq[:, None, :]


def moments(rz, z, w_root, w):
    rz = np.asarray(rz, np.float64)
    z = np.asarray(z, np.float64)
    root_m = np.stack([(w_root * rz).sum(axis=1), (w_root * rz * rz).sum(axis=1)], axis=1)
    gm = np.stack([(w * z).sum(axis=1), (w * z * z).sum(axis=1)], axis=1)
    return root_m, gm


def gaussian_mstep(lam, m_new, ema, floor=1e-8):
    ema = lam * np.asarray(ema) + (1 - lam) * np.asarray(m_new)
    var = ema[:, 1] - ema[:, 0] ** 2
    var = np.where(var >= floor, var, floor)
    return ema, ema[:, 0].astype(np.float32), var.astype(np.float32)


def initial_state(cm):
    R, n = cm.R, cm.n
    return dict(root_mean=np.zeros(R, np.float32), root_var=np.ones(R, np.float32),
                root_ema=np.tile([0.0, 1.0], (R, 1)), q_mean=np.zeros(n, np.float32),
                q_var=np.ones(n, np.float32), g_ema=np.tile([0.0, 1.0], (n, 1)))


def qem_step(cm, state, t, eps_root, eps_g, new_weight=0.3, floor=1e-8):
    rz = oracle.sample(state["root_mean"], state["root_var"], eps_root)       # [R][K] fp32
    z = oracle.sample(state["q_mean"], state["q_var"], eps_g)                 # [n][K] fp32
    f_root, f = make_tables(cm, rz, state["root_mean"], state["root_var"], z, state["q_mean"], state["q_var"])
    est = tables.estep_tables(f_root, f)
    root_m, gm = moments(rz, z, est["w_root"], est["w"])
    lam = oracle.lam(t, new_weight, 0.0)
    root_ema, rmean, rvar = gaussian_mstep(lam, root_m, state["root_ema"], floor)
    g_ema, qm, qv = gaussian_mstep(lam, gm, state["g_ema"], floor)
    nxt = dict(root_mean=rmean, root_var=rvar, root_ema=root_ema, q_mean=qm, q_var=qv, g_ema=g_ema)
    return dict(rz=rz, z=z, f_root=f_root, f=f, est=est, root_m=root_m, gm=gm, next=nxt)
