"""ctypes wrapper around qem_oracle.c plus the QEM step of Algorithm 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Builds
``oracle/liboracle.so`` with plain gcc on first use (``__graft_entry__.build``
also builds it).  Arrays go in and come out as float64 numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile qem_oracle.c (fp64, -O2, OpenMP over groups, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _M2(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("scale_kind", ctypes.c_int), ("fixed_var", ctypes.c_double),
                ("obs_kind", ctypes.c_int), ("obs_var", ctypes.c_double), ("n", ctypes.c_long),
                ("J", ctypes.c_int), ("prior_mean", ctypes.c_double), ("prior_var", ctypes.c_double)]


class _M3(ctypes.Structure):
    _fields_ = [("A", ctypes.c_int), ("B", ctypes.c_int), ("J", ctypes.c_int), ("P", ctypes.c_int),
                ("top_var", ctypes.c_double), ("sub_var", ctypes.c_double),
                ("prior_mean", ctypes.c_double), ("prior_var", ctypes.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
            _lib.orc_lambda.restype = ctypes.c_double
            _lib.orc_lambda.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
            _lib.orc_mstep.restype = ctypes.c_long
            _lib.orc_num_threads.restype = ctypes.c_int
        return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _m2(m) -> _M2:
    return _M2(m.d, m.scale_kind, m.fixed_var, m.obs_kind, m.obs_var, m.n, m.J, m.prior_mean, m.prior_var)


def _m3(m) -> _M3:
    return _M3(m.n, m.B, m.J, m.P, m.top_var, m.sub_var, m.prior_mean, m.prior_var)


def estep(m, z, q, data):
    """One MPIW E-step (Eq. 7a-c) on host arrays.

    z: list of per-level sample arrays [instances*dims][K] (root first);
    q: list of per-level (mean, var) arrays [instances*dims];
    data: synth.Data.  Returns a dict of float64 arrays:
    log_pe, w (list per level, [instances][K]), m1 / m2 (list per level,
    [instances*dims]) and, for two-level models, g ([n][K] messages)."""
    L = lib()
    K = m.K
    zs = [_f64(a) for a in z]
    qs = [(_f64(a), _f64(b)) for a, b in q]
    log_pe = ctypes.c_double()
    if m.family == 2:
        n, d, R = m.n, m.d, m.R
        w_root, w = np.zeros(K), np.zeros((n, K))
        g = np.zeros((n, K))
        m1r, m2r, m1, m2 = np.zeros(R), np.zeros(R), np.zeros(n * d), np.zeros(n * d)
        xg = _f64(data.xg) if data.xg is not None else None
        xb = np.ascontiguousarray(data.xb, np.uint8) if data.xb is not None else None
        yb = np.ascontiguousarray(data.yb, np.uint8) if data.yb is not None else None
        mm = _m2(m)
        rc = L.orc2_estep(ctypes.byref(mm), K, _p(zs[0]), _p(zs[1]), _p(qs[0][0]), _p(qs[0][1]),
                          _p(qs[1][0]), _p(qs[1][1]), _p(xg), _p(xb), _p(yb), ctypes.byref(log_pe),
                          _p(w_root), _p(w), _p(g), _p(m1r), _p(m2r), _p(m1), _p(m2))
        return dict(rc=rc, log_pe=log_pe.value, w=[w_root[None, :], w], m1=[m1r, m1], m2=[m2r, m2], g=g)
    A, B, R = m.n, m.B, m.R
    w_root, w_top, w_sub = np.zeros(K), np.zeros((A, K)), np.zeros((A * B, K))
    m1r, m2r, m1t, m2t, m1s, m2s = (np.zeros(R), np.zeros(R), np.zeros(A), np.zeros(A),
                                    np.zeros(A * B), np.zeros(A * B))
    mm = _m3(m)
    x = _f64(data.xp)
    y = _f64(data.yp)
    rc = L.orc3_estep(ctypes.byref(mm), K, _p(zs[0]), _p(zs[1]), _p(zs[2]), _p(qs[0][0]), _p(qs[0][1]),
                      _p(qs[1][0]), _p(qs[1][1]), _p(qs[2][0]), _p(qs[2][1]), _p(x), _p(y),
                      ctypes.byref(log_pe), _p(w_root), _p(w_top), _p(w_sub), _p(m1r), _p(m2r), _p(m1t),
                      _p(m2t), _p(m1s), _p(m2s))
    return dict(rc=rc, log_pe=log_pe.value, w=[w_root[None, :], w_top, w_sub], m1=[m1r, m1t, m1s],
                m2=[m2r, m2t, m2s])


def _data2(data):
    xg = _f64(data.xg) if data.xg is not None else None
    xb = np.ascontiguousarray(data.xb, np.uint8) if data.xb is not None else None
    yb = np.ascontiguousarray(data.yb, np.uint8) if data.yb is not None else None
    return xg, xb, yb


def forward2(m, z, q, data):
    """Two-level forward half: (f_root [K], g [n][K]) (plate messages g_i(k))."""
    zs = [_f64(a) for a in z]
    qs = [(_f64(a), _f64(b)) for a, b in q]
    xg, xb, yb = _data2(data)
    f_root, g = np.zeros(m.K), np.zeros((m.n, m.K))
    mm = _m2(m)
    lib().orc2_forward(ctypes.byref(mm), m.K, _p(zs[0]), _p(zs[1]), _p(qs[0][0]), _p(qs[0][1]), _p(qs[1][0]),
                       _p(qs[1][1]), _p(xg), _p(xb), _p(yb), _p(f_root), _p(g))
    return f_root, g


def backward2(m, z, q, data, w_root, g):
    """Two-level backward half given root weights: (w [n][K], m1 [n*d], m2 [n*d])."""
    zs = [_f64(a) for a in z]
    qs = [(_f64(a), _f64(b)) for a, b in q]
    xg, xb, yb = _data2(data)
    w, m1, m2 = np.zeros((m.n, m.K)), np.zeros(m.n * m.d), np.zeros(m.n * m.d)
    mm = _m2(m)
    wr, gg = _f64(w_root), _f64(g)
    lib().orc2_backward(ctypes.byref(mm), m.K, _p(zs[0]), _p(zs[1]), _p(qs[1][0]), _p(qs[1][1]), _p(xg), _p(xb),
                        _p(yb), _p(wr), _p(gg), _p(w), _p(m1), _p(m2))
    return w, m1, m2


def sample(q_mean, q_var, eps):
    """z = fmaf(sqrtf(v), eps, m) in fp32 (R22); eps [n][K] fp32 -> z [n][K] fp32."""
    L = lib()
    qm = np.ascontiguousarray(q_mean, np.float32)
    qv = np.ascontiguousarray(q_var, np.float32)
    e = np.ascontiguousarray(eps, np.float32)
    n, K = e.shape
    z = np.empty((n, K), np.float32)
    L.orc_sample(ctypes.c_long(n), K, _p(qm), _p(qv), _p(e), _p(z))
    return z


def lam(t, new_weight=0.3, p=0.0):
    """History weight lambda_t (R5; Theorem 1 schedule when p > 0)."""
    return lib().orc_lambda(int(t), float(new_weight), float(p))


def ema(lmb, m1, m2, m1_new, m2_new):
    """EMA over mean parameters (Eq. 9); returns new (m1, m2) copies."""
    a, b = _f64(m1).copy(), _f64(m2).copy()
    lib().orc_ema(ctypes.c_long(a.size), ctypes.c_double(lmb), _p(a), _p(b), _p(_f64(m1_new)), _p(_f64(m2_new)))
    return a, b


def mstep(m1, m2, floor=1e-8):
    """Gaussian M-step from mean parameters; returns (mean f32, var f32, clamps)."""
    a, b = _f64(m1), _f64(m2)
    qm, qv = np.empty(a.size, np.float32), np.empty(a.size, np.float32)
    c = lib().orc_mstep(ctypes.c_long(a.size), _p(a), _p(b), ctypes.c_double(floor), _p(qm), _p(qv))
    return qm, qv, int(c)


def philox(ctr, key):
    L = lib()
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xffffffff for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xffffffff for v in key])
    o = (ctypes.c_uint32 * 4)()
    L.orc_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def normal_eps(seed, it, level, instance, ndim, K):
    """Philox + Box-Muller standard normals eps[dim][k] for one latent instance (fp64)."""
    out = np.zeros((ndim, K))
    lib().orc_normal_eps(ctypes.c_uint64(seed), ctypes.c_uint32(it), ctypes.c_uint32(level),
                         ctypes.c_uint32(instance), ndim, K, _p(out))
    return out


def num_threads():
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    """OpenMP threads of the group loops (timing only; results are thread-count independent)."""
    lib().orc_set_num_threads(int(n))


# ------------------------------------------------------------------ QEM loop


def initial_state(m):
    """m_0: mean parameters of N(0,1) per latent dim, i.e. (E z, E z^2) = (0, 1)."""
    from paper_2503_08264_b200 import synth  # input shapes only
    return [(np.zeros(n * dd), np.ones(n * dd)) for n, dd in synth.latent_shapes(m)]


def qem_step(m, state, q_t, eps_t, t, new_weight=0.3, p=0.0, floor=1e-8, data=None, eps_new=None):
    """One iteration t of Algorithm 1 after its M-step.

    state: per level (m1, m2) = m_{t-1}; q_t: per level (mean f32, var f32) =
    set_exp_family_params(m_{t-1}); eps_t: per level [instances*dims][K] fp32.
    eps_new (optional): a second, independent draw for the fresh-sample denominator
    (PAPER.md:274-275): the one-step moments become sum_k r_k(z) m(z^k) / Pe(z_new), i.e.
    the self-normalised moments times Pe(z) / Pe(z_new) (R28).
    Returns dict(z, est (E-step dict), state (m_t), q_next (Q_{t+1}), clamps, ratio)."""
    z = [sample(qm, qv, e) for (qm, qv), e in zip(q_t, eps_t)]
    est = estep(m, z, q_t, data)
    ratio, lp_new = 1.0, None
    if eps_new is not None:
        z_new = [sample(qm, qv, e) for (qm, qv), e in zip(q_t, eps_new)]
        lp_new = estep(m, z_new, q_t, data)["log_pe"]
        ratio = float(np.exp(est["log_pe"] - lp_new))
    lm = lam(t, new_weight, p)
    new_state, q_next, clamps = [], [], 0
    for (m1, m2), a, b in zip(state, est["m1"], est["m2"]):
        s = ema(lm, m1, m2, ratio * a, ratio * b)
        new_state.append(s)
        qm, qv, c = mstep(s[0], s[1], floor)
        q_next.append((qm, qv))
        clamps += c
    return dict(z=z, est=est, state=new_state, q_next=q_next, clamps=clamps, lam=lm, ratio=ratio,
                log_pe_new=lp_new)


# Offset of the seed of the fresh-sample (denominator) draw in host-eps mode.
FRESH_SEED_OFFSET = 7919


def eps_for_iteration(m, t, seed):
    """Host fp32 standard normals for iteration t (parity mode): one array per level."""
    from paper_2503_08264_b200 import synth
    return [synth.eps_normal((n * dd, m.K), seed * 1000003 + t * 7 + lvl)
            for lvl, (n, dd) in enumerate(synth.latent_shapes(m))]


def run_qem(m, data, T, seed, new_weight=0.3, p=0.0, floor=1e-8, fresh=False):
    """Free-running QEM for T iterations from m_0 (Algorithm 1). Returns the per-step dicts.
    fresh: use the fresh-sample denominator with eps from seed + FRESH_SEED_OFFSET."""
    state = initial_state(m)
    q = [mstep(a, b, floor)[:2] for a, b in state]
    out = []
    for t in range(1, T + 1):
        eps_new = eps_for_iteration(m, t, seed + FRESH_SEED_OFFSET) if fresh else None
        r = qem_step(m, state, q, eps_for_iteration(m, t, seed), t, new_weight, p, floor, data, eps_new=eps_new)
        out.append(r)
        state, q = r["state"], r["q_next"]
    return out
