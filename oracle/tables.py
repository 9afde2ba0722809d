"""MPIW E-step on explicit log-factor tables -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Eq. 7 for a root latent with K samples and n plate instances below it, the
log-factors given as tables (f_root[k] = log p(root^k) - log q(root^k); f[i][k][k'] =
log p(z_i^k', x_i | root^k) - log q(z_i^k')).  Two routes, fp64:

  estep_tables_brute   the literal sum over all K^(n+1) index tuples (Eq. 7c), marginal weights
                       by direct accumulation (Eq. 7a) -- tiny tables only;
  estep_tables         plate elimination: g_i(k) = lse_k' f_i(k,k') - ln K,
                       log Pe = lse_k (f_root(k) + sum_i g_i(k)) - ln K, w_root = softmax,
                       w_i(k') = sum_k w_root(k) exp(f_i(k,k') - ln K - g_i(k)).

The elimination is pinned against the enumeration (tests/test_tables.py).
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy.special import logsumexp


def estep_tables(f_root, f):
    f_root = np.asarray(f_root, np.float64)
    K = f_root.shape[0]
    f = np.asarray(f, np.float64).reshape(-1, K, K)
    lk = np.log(K)
    g = logsumexp(f, axis=2) - lk                     # [n][K]
    a = f_root + g.sum(axis=0)
    lse = logsumexp(a)
    w_root = np.exp(a - lse)
    live = w_root > 0  # root samples with zero weight carry no tuples (their g may be -inf)
    w = np.einsum("k,ikj->ij", w_root[live], np.exp(f[:, live, :] - lk - g[:, live, None]))
    return dict(log_pe=lse - lk, w_root=w_root, w=w, g=g)


def estep_tables_brute(f_root, f):
    f_root = np.asarray(f_root, np.float64)
    K = f_root.shape[0]
    f = np.asarray(f, np.float64).reshape(-1, K, K)
    n = f.shape[0]
    logr = []
    tuples = list(itertools.product(range(K), repeat=n + 1))
    for t in tuples:  # t = (k_root, k_1, ..., k_n)
        logr.append(f_root[t[0]] + sum(f[i, t[0], t[i + 1]] for i in range(n)))
    logr = np.array(logr)
    lse = logsumexp(logr)
    r = np.exp(logr - lse)
    w_root = np.zeros(K)
    w = np.zeros((n, K))
    for t, rt in zip(tuples, r):
        w_root[t[0]] += rt
        for i in range(n):
            w[i, t[i + 1]] += rt
    return dict(log_pe=lse - (n + 1) * np.log(K), w_root=w_root, w=w)
