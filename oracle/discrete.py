"""Discrete (categorical) latents under a Gaussian root -- TEST INFRASTRUCTURE ONLY
(oracle/__init__.py).  The E-step side of NEXT row f1 (R30), plain numpy fp64,
following the model's definitions step by step (Algorithm 1):

  sample   root r^k = fmaf(sqrtf(v), eps, m) (fp32, R22; oracle.sample);
           z_i^k = min{c : u < p_i(0) + ... + p_i(c)} (fp64 sequential prefix, C-1 if none),
           u = ((w >> 8) + 1/2) 2^-24, w = word k%4 of Philox4x32-10 at (k/4, 0, i, 3<<24 | t)
  loglik   L_i(c) = sum_r y_ir l_irc - softplus(l_irc)                       (data only)
  tables   f_root(k) = log N(r^k; 0, I) - log N(r^k; m, diag v)
           f_i(k,k') = log softmax_c(x_i . r^k)[z_i^k'] + L_i(z_i^k') - log p_i(z_i^k')
  E-step   oracle/tables.py (Eq. 7; elimination pinned against enumeration)
  moments  (E r, E r^2) under w_root; E onehot(z_i) under w_i                   (Eq. 7a)
  M-step   EMA with history weight lam (Eq. 9, R5), Q_root = N(E r, max(Var r, floor)) rounded
           to fp32, p_i = normalised EMA of E onehot(z_i).
Pinned by tests/test_discrete.py: sampler frequencies, Bernoulli normalisation of L, and the
unbiasedness of exp(log Pe) for the evidence p(y) computed by Gauss-Hermite quadrature over the
root with the discrete latents summed exactly.
"""
from __future__ import annotations

import numpy as np
from scipy.special import log_softmax

from . import oracle, tables


def sample_categorical(p, K, seed, t):
    p = np.asarray(p, np.float64)
    n, C = p.shape
    key = (seed & 0xffffffff, (seed >> 32) & 0xffffffff)
    z = np.zeros((n, K), np.int32)
    for i in range(n):
        for q in range((K + 3) // 4):
            w = oracle.philox((q, 0, i, (3 << 24) | (t & 0xffffff)), key)
            for j in range(4):
                k = 4 * q + j
                if k >= K:
                    break
                u = ((w[j] >> 8) + 0.5) * 2.0 ** -24
                c, cum = 0, p[i, 0]
                while c < C - 1 and u >= cum:
                    c += 1
                    cum += p[i, c]
                z[i, k] = c
    return z


def loglik(y, logit):
    y = np.asarray(y, np.float64)[:, :, None]
    l = np.asarray(logit, np.float64)
    return (y * l - (np.maximum(l, 0.0) + np.log1p(np.exp(-np.abs(l))))).sum(axis=1)


def make_tables(root_z, root_mean, root_var, x, L, p, z):
    r = np.asarray(root_z, np.float64)                   # [d][K]
    m = np.asarray(root_mean, np.float32).astype(np.float64)[:, None]
    v = np.asarray(root_var, np.float32).astype(np.float64)[:, None]
    log_prior = (-0.5 * np.log(2 * np.pi) - 0.5 * r ** 2).sum(axis=0)
    log_q = (-0.5 * np.log(2 * np.pi * v) - 0.5 * (r - m) ** 2 / v).sum(axis=0)
    f_root = log_prior - log_q
    eta = np.einsum("icd,dk->ikc", np.asarray(x, np.float64), r)  # [n][K][C]
    ls = log_softmax(eta, axis=2)
    n, K = np.asarray(z).shape
    h = ls + (np.asarray(L) - np.log(np.asarray(p)))[:, None, :]   # [n][K][C]
    f = np.take_along_axis(h, np.broadcast_to(np.asarray(z)[:, None, :], (n, K, K)), axis=2)
    return f_root, f


def moments(root_z, w_root, w, z, C):
    r = np.asarray(root_z, np.float64)
    root_m = np.stack([(w_root * r).sum(axis=1), (w_root * r * r).sum(axis=1)], axis=1)  # [d][2]
    onehot = np.asarray(z)[:, :, None] == np.arange(C)[None, None, :]
    pm = (np.asarray(w)[:, :, None] * onehot).sum(axis=1)
    return root_m, pm


def mstep(lam, root_m, root_ema, pm, p_ema, floor=1e-8):
    root_ema = lam * np.asarray(root_ema) + (1 - lam) * np.asarray(root_m)
    var = root_ema[:, 1] - root_ema[:, 0] ** 2
    clamps = int((~(var >= floor)).sum())
    var = np.where(var >= floor, var, floor)
    p_ema = lam * np.asarray(p_ema) + (1 - lam) * np.asarray(pm)
    p = p_ema / p_ema.sum(axis=1, keepdims=True)
    return dict(root_ema=root_ema, root_mean=root_ema[:, 0].astype(np.float32), root_var=var.astype(np.float32),
                p_ema=p_ema, p=p, clamps=clamps)


def initial_state(om):
    return dict(root_ema=np.tile([0.0, 1.0], (om.d, 1)), root_mean=np.zeros(om.d, np.float32),
                root_var=np.ones(om.d, np.float32), p_ema=np.full((om.n, om.C), 1.0 / om.C),
                p=np.full((om.n, om.C), 1.0 / om.C))


def qem_step(om, state, t, seed, eps_root, L=None, new_weight=0.3, p_sched=0.0, floor=1e-8):
    """One QEM iteration (Alg. 1) from `state` with host root eps [d][K]; returns the step's values."""
    if L is None:
        L = loglik(om.y, om.logit)
    root_z = oracle.sample(state["root_mean"], state["root_var"], eps_root)   # [d][K] fp32
    z = sample_categorical(state["p"], om.K, seed, t)
    f_root, f = make_tables(root_z, state["root_mean"], state["root_var"], om.x, L, state["p"], z)
    est = tables.estep_tables(f_root, f)
    root_m, pm = moments(root_z, est["w_root"], est["w"], z, om.C)
    nxt = mstep(oracle.lam(t, new_weight, p_sched), root_m, state["root_ema"], pm, state["p_ema"], floor)
    return dict(root_z=root_z, z=z, f_root=f_root, f=f, est=est, root_m=root_m, pm=pm, next=nxt)
