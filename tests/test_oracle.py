"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/qem_oracle.c) is checked against things other than itself:
literal K^n enumeration (oracle/brute.py), closed-form conjugate posteriors
(oracle/closed_form.py), worked examples (tests/golden/), the App. E scaling
invariance, permutation invariance, the K=1 special case, the App. D EMA law,
and published Philox known-answer vectors.
"""
import math

import numpy as np
import pytest

from conftest import golden
from helpers import make_case, posterior_like_q
from oracle import brute, closed_form
from oracle import oracle as orc
from paper_2503_08264_b200 import synth

MINI = {
    "c1_full": dict(cid=1),
    "c2_mini": dict(cid=2, n=2, K=4, d=2),
    "c3_mini": dict(cid=3, n=1, B=2, K=3, J=3),
    "c4_mini": dict(cid=4, n=3, K=5),
    "c5_mini": dict(cid=5, n=2, K=6, d=3),
}


def _model(spec):
    spec = dict(spec)
    return synth.config(spec.pop("cid"), **spec)


def _cmp(a, b, name, rtol=1e-10, atol=1e-12):
    np.testing.assert_allclose(np.asarray(a), np.asarray(b), rtol=rtol, atol=atol, err_msg=name)


@pytest.mark.parametrize("case", sorted(MINI))
@pytest.mark.parametrize("qseed", [11, 12])
def test_oracle_equals_enumeration(case, qseed):
    """Elimination (O2) == literal K^n enumeration (O1) of Eq. 7a-c."""
    m = _model(MINI[case])
    data, q, eps, z = make_case(m, q_seed=qseed)
    if m.family == 3:
        q = posterior_like_q(m, data, seed=qseed, shrink=30.0)
        z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
    a = orc.estep(m, z, q, data)
    b = brute.estep(m, z, q, data)
    assert a["rc"] == 0
    _cmp(a["log_pe"], b["log_pe"], "log_pe")
    for lvl in range(len(b["w"])):
        _cmp(a["w"][lvl], b["w"][lvl], f"w[{lvl}]", rtol=0, atol=1e-12)
        _cmp(a["m1"][lvl], b["m1"][lvl], f"m1[{lvl}]", rtol=1e-9, atol=1e-12)
        _cmp(a["m2"][lvl], b["m2"][lvl], f"m2[{lvl}]", rtol=1e-9, atol=1e-12)


def test_weights_sum_to_one_and_messages():
    m = synth.config(4, n=50, K=16)
    data, q, eps, z = make_case(m)
    r = orc.estep(m, z, q, data)
    for w in r["w"]:
        np.testing.assert_allclose(w.sum(axis=1), 1.0, atol=1e-12)
    # log Pe = lse_k (f_root(k) + sum_i g_i(k)) - log K: recompute the root step from g
    zr = np.asarray(z[0], np.float64).reshape(m.R, m.K)
    qrm, qrv = q[0]
    ln = lambda x, mu, v: -0.5 * np.log(2 * np.pi * v) - (x - mu) ** 2 / (2 * v)
    f = sum(ln(zr[r], 0.0, 1.0) - ln(zr[r], float(qrm[r]), float(qrv[r])) for r in range(m.R))
    a = f + r["g"].sum(axis=0)
    from scipy.special import logsumexp
    assert abs(logsumexp(a) - math.log(m.K) - r["log_pe"]) < 1e-9 * abs(r["log_pe"])


@pytest.mark.parametrize("cid", [2, 4])
def test_permuting_samples_permutes_weights(cid):
    """Permuting one latent's K samples permutes its weights; log Pe and moments unchanged."""
    m = synth.config(cid, n=6, K=12, d=3 if cid == 2 else None)
    data, q, eps, z = make_case(m)
    r0 = orc.estep(m, z, q, data)
    rng = np.random.default_rng(0)
    perm_root = rng.permutation(m.K)
    perm_g = rng.permutation(m.K)
    z2 = [z[0][:, perm_root].copy(), z[1].copy()]
    # permute group 2's samples (all dims of that group)
    zz = z2[1].reshape(m.n, m.d, m.K)
    zz[2] = zz[2][:, perm_g]
    z2[1] = zz.reshape(m.n * m.d, m.K)
    r1 = orc.estep(m, z2, q, data)
    assert abs(r1["log_pe"] - r0["log_pe"]) < 1e-10 * abs(r0["log_pe"])
    np.testing.assert_allclose(r1["w"][0][0], r0["w"][0][0][perm_root], atol=1e-13)
    np.testing.assert_allclose(r1["w"][1][2], r0["w"][1][2][perm_g], atol=1e-13)
    for lvl in range(2):
        np.testing.assert_allclose(r1["m1"][lvl], r0["m1"][lvl], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(r1["m2"][lvl], r0["m2"][lvl], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("alpha", [1e-2, 1e-3, 10.0])
def test_scaling_invariance(alpha):
    """App. E: rescale every latent and observation by alpha with the
    same eps -> weights unchanged, moments map by f((m1,m2);alpha) = (a m1, a^2 m2),
    and log Pe shifts by -(#obs) log alpha (the Jacobian of x)."""
    m = synth.config(1, K=8)
    data, q, eps, z = make_case(m)
    r0 = orc.estep(m, z, q, data)
    ms = synth.config(1, K=8)
    ms.prior_var, ms.fixed_var, ms.obs_var = alpha ** 2, alpha ** 2, alpha ** 2
    qs = [(qm * np.float32(alpha), qv * np.float32(alpha) ** 2) for qm, qv in q]
    zs = [orc.sample(qm, qv, e) for (qm, qv), e in zip(qs, eps)]
    ds = synth.Data(xg=(data.xg.astype(np.float64) * alpha))
    # compare against z scaled exactly: use the same scaled samples on both sides
    r1 = orc.estep(ms, zs, qs, ds)
    # unscaled run on zs/alpha (exactly the scaled samples mapped back)
    zb = [np.asarray(a, np.float64) / alpha for a in zs]
    db = synth.Data(xg=ds.xg / alpha)
    r0 = orc.estep(m, zb, [(np.asarray(a, np.float64) / alpha, np.asarray(b, np.float64) / alpha ** 2) for a, b in qs], db)
    nobs = m.n * m.J
    assert abs(r1["log_pe"] - (r0["log_pe"] - nobs * math.log(alpha))) < 1e-9 * max(1, abs(r0["log_pe"]))
    for lvl in range(2):
        np.testing.assert_allclose(r1["w"][lvl], r0["w"][lvl], atol=1e-11)
        np.testing.assert_allclose(r1["m1"][lvl], alpha * r0["m1"][lvl], rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(r1["m2"][lvl], alpha ** 2 * r0["m2"][lvl], rtol=1e-9, atol=1e-18)


def test_K1_is_single_importance_ratio():
    """K=1: log Pe = log p(x,z) - log q(z), moments = T(z)."""
    m = synth.config(4, n=5, K=1, J=3)
    data, q, eps, z = make_case(m)
    r = orc.estep(m, z, q, data)
    mu, s = float(z[0][0, 0]), float(z[0][1, 0])
    zg = z[1][:, 0].astype(np.float64)
    from scipy.stats import norm
    lp = norm.logpdf(mu) + norm.logpdf(s) + norm.logpdf(zg, mu, math.exp(s)).sum()
    lp += norm.logpdf(data.xg.astype(np.float64), zg[:, None], 1.0).sum()
    lq = norm.logpdf(mu, q[0][0][0], math.sqrt(q[0][1][0])) + norm.logpdf(s, q[0][0][1], math.sqrt(q[0][1][1]))
    lq += norm.logpdf(zg, q[1][0].astype(np.float64), np.sqrt(q[1][1].astype(np.float64))).sum()
    assert abs(r["log_pe"] - (lp - lq)) < 1e-10 * abs(lp - lq)
    np.testing.assert_allclose(r["m1"][1], zg, rtol=1e-15)
    np.testing.assert_allclose(r["m2"][1], zg ** 2, rtol=1e-15)


def test_closed_form_textbook_example():
    g = golden("spec_examples.txt")
    mean, var, lpx = closed_form.single_latent([2.0])
    assert abs(mean - float(g["conj_post_mean"])) < 1e-15
    assert abs(var - float(g["conj_post_var"])) < 1e-15
    assert abs(lpx - float(g["conj_log_px"])) < 1e-12


def test_closed_form_routes_agree():
    """Precision-matrix posterior == Gaussian conditioning from the joint covariance."""
    m = synth.config(1)
    data = synth.make_data(m)
    x = data.xg.astype(np.float64)
    mean, cov = closed_form.posterior(x)
    M, J = x.shape
    # joint covariance of theta=(mu,z) and x
    n = M * J
    St = np.eye(M + 1)
    St[0, :] = 1.0
    St[:, 0] = 1.0
    St[1:, 1:] = np.ones((M, M)) + np.eye(M)
    Stx = np.zeros((M + 1, n))
    Stx[0, :] = 1.0
    for i in range(M):
        Stx[1:, i * J:(i + 1) * J] = 1.0
        Stx[1 + i, i * J:(i + 1) * J] = 2.0
    Sxx = np.eye(n) + np.ones((n, n))
    for i in range(M):
        Sxx[i * J:(i + 1) * J, i * J:(i + 1) * J] += 1.0
    cm = Stx @ np.linalg.solve(Sxx, x.reshape(-1))
    cc = St - Stx @ np.linalg.solve(Sxx, Stx.T)
    np.testing.assert_allclose(mean, cm, atol=1e-12)
    np.testing.assert_allclose(cov, cc, atol=1e-12)


def test_evidence_unbiased_conjugate():
    """E[Pe] = p(x): mean of Pe over many independent sample banks at K=8,
    under a non-posterior Q, vs the closed-form marginal (3.5 standard errors)."""
    m = synth.config(1)
    data = synth.make_data(m)
    truth = closed_form.log_evidence(data.xg)
    q = synth.initial_q(m)
    vals = []
    for s in range(3000):
        eps = [synth.eps_normal((n * dd, m.K), 100_000 + 3 * s + lvl) for lvl, (n, dd) in enumerate(synth.latent_shapes(m))]
        # widen Q a bit around the truth so Pe has finite variance
        qq = [(np.full_like(qm, 0.0), np.full_like(qv, 2.0)) for qm, qv in q]
        z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(qq, eps)]
        vals.append(orc.estep(m, z, qq, data)["log_pe"])
    vals = np.asarray(vals)
    c = vals.max()
    pe = np.exp(vals - c)
    mean, se = pe.mean(), pe.std(ddof=1) / math.sqrt(pe.size)
    assert abs(mean - math.exp(truth - c)) < 3.5 * se, (np.log(mean) + c, truth)


def test_large_K_moments_approach_closed_form():
    """K -> infinity consistency (App. C): MPIW moments with Q at the exact posterior marginals
    approach the closed-form posterior moments."""
    m = synth.config(1, K=2048)
    data = synth.make_data(m)
    mean, cov = closed_form.posterior(data.xg)
    sd = np.sqrt(np.diag(cov))
    q = [(np.float32([mean[0]]), np.float32([cov[0, 0]])),
         (mean[1:].astype(np.float32), np.diag(cov)[1:].astype(np.float32))]
    eps = [synth.eps_normal((n * dd, m.K), 77 + lvl) for lvl, (n, dd) in enumerate(synth.latent_shapes(m))]
    z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
    r = orc.estep(m, z, q, data)
    m1 = np.concatenate([r["m1"][0], r["m1"][1]])
    var = np.concatenate([r["m2"][0], r["m2"][1]]) - m1 ** 2
    assert np.all(np.abs(m1 - mean) < 0.08 * sd), (m1, mean)
    assert np.all(np.abs(var / np.diag(cov) - 1) < 0.15)
    assert abs(r["log_pe"] - closed_form.log_evidence(data.xg)) < 0.02


def test_qem_converges_to_closed_form():
    """QEM (Alg. 1) on config 1, K=64, w=0.3, 20 iterations: posterior means within MC error
    of the closed form, averaged over seeds (bias 4e-3, seed-sd 0.027)."""
    m = synth.config(1, K=64)
    data = synth.make_data(m)
    mean, cov = closed_form.posterior(data.xg)
    finals = []
    for seed in range(24):
        out = orc.run_qem(m, data, 20, seed)
        st = out[-1]["state"]
        finals.append(np.concatenate([st[0][0], st[1][0]]))
    finals = np.asarray(finals)
    err = finals.mean(axis=0) - mean
    se = finals.std(axis=0, ddof=1) / math.sqrt(len(finals))
    assert np.all(np.abs(err) < 4 * se + 0.01), (err, se)


def test_ema_mstep_examples():
    g = golden("spec_examples.txt")
    assert orc.lam(1, p=0.5) == float(g["lambda_p05_t1"])
    assert abs(orc.lam(4, p=0.5) - float(g["lambda_p05_t4"])) < 1e-15
    assert abs(orc.lam(7, new_weight=0.3) - float(g["lambda_w03"])) < 1e-15
    a, b = orc.ema(0.5, [0.0], [1.0], [2.0], [5.0])
    assert a[0] == float(g["ema_m1"]) and b[0] == float(g["ema_m2"])
    qm, qv, c = orc.mstep([2.0], [5.0])
    assert qm[0] == float(g["mstep_mean"]) and qv[0] == float(g["mstep_var"]) and c == 0
    qm, qv, c = orc.mstep([1.0], [1.0000001], floor=1e-6)
    assert qv[0] == np.float32(float(g["mstep_clamp_var"])) and c == 1


def test_ema_constant_input_law():
    """App. D: constant input c from m_0: m_t = (1 - lam^t) c + lam^t m_0."""
    lmb = orc.lam(1, new_weight=0.3)
    m1, m2 = np.array([0.5]), np.array([2.0])
    c1, c2 = np.array([3.0]), np.array([11.0])
    for t in range(1, 21):
        m1, m2 = orc.ema(lmb, m1, m2, c1, c2)
        exp1 = (1 - lmb ** t) * 3.0 + lmb ** t * 0.5
        exp2 = (1 - lmb ** t) * 11.0 + lmb ** t * 2.0
        assert abs(m1[0] - exp1) < 1e-12 and abs(m2[0] - exp2) < 1e-12


def test_ema_variance_decay_schedule():
    """Theorem 1: with lambda_t = 1 - t^-p and an i.i.d. noisy unbiased input, Var[m_t] decreases."""
    rng = np.random.default_rng(3)
    reps = 4000
    m1 = np.zeros(reps)
    m2 = np.zeros(reps)
    var_at = {}
    for t in range(1, 1001):
        x = 1.0 + rng.standard_normal(reps)
        m1, m2 = orc.ema(orc.lam(t, p=0.5), m1, m2, x, x * x)
        if t in (10, 100, 1000):
            var_at[t] = m1.var()
            assert abs(m1.mean() - 1.0) < 5 * math.sqrt(var_at[t] / reps) + 1e-3
    assert var_at[10] > var_at[100] > var_at[1000]


def test_philox_known_answers():
    rows = []
    with open("tests/golden/philox4x32_10_kat.txt") as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([int(v, 16) for v in line.split()])
    for r in rows:
        assert orc.philox(r[0:4], r[4:6]) == r[6:10]


def test_philox_normals_are_standard():
    eps = np.concatenate([orc.normal_eps(7, 3, 1, i, 4, 1024).ravel() for i in range(40)])
    assert abs(eps.mean()) < 0.01 and abs(eps.var() - 1) < 0.015
    from scipy.stats import kstest
    assert kstest(eps, "norm").pvalue > 1e-3


def test_box_muller_pairs_invert_to_the_philox_words():
    """Deterministic pin of the oracle's normal generator (R42; the paper fixes no sampler):
    samples k = 4c + {0, 1} are the Box-Muller pair of words (0, 1) of the Philox block at counter
    (c, dim, instance, level << 24 | iter), samples 4c + {2, 3} that of words (2, 3).  The pair's polar
    decomposition must give back the words' uniforms u = (top 23 bits + 1/2) / 2^23: radius^2 =
    -2 ln u_a and angle = 2 pi u_b (cos to the even sample, sin to the odd one).  The words come from
    orc.philox, itself pinned to the Random123 known answers above; a swapped word, a swapped sin / cos,
    a sign or another uniform mapping fails."""
    seed, it, level, inst, ndim, K = (0x9E3779B97F4A7C15, 37, 1, 1234, 3, 16)
    eps = orc.normal_eps(seed, it, level, inst, ndim, K)
    key = [seed & 0xffffffff, seed >> 32]
    for r in range(ndim):
        for c in range(K // 4):
            w = orc.philox([c, r, inst, (level << 24) | it], key)
            for half in range(2):
                e0, e1 = eps[r, 4 * c + 2 * half], eps[r, 4 * c + 2 * half + 1]
                ua = ((w[2 * half] >> 9) + 0.5) / 2.0 ** 23
                ub = ((w[2 * half + 1] >> 9) + 0.5) / 2.0 ** 23
                assert abs(math.exp(-0.5 * (e0 * e0 + e1 * e1)) - ua) < 1e-12
                ang = math.atan2(e1, e0) / (2 * math.pi) % 1.0
                assert min(abs(ang - ub), 1 - abs(ang - ub)) < 1e-9


def test_sampler_location_scale():
    """z = m + sqrt(v) eps (App. E inverse-transform / location-scale sampling), fp32 fmaf."""
    qm = np.array([0.25, -3.0], np.float32)
    qv = np.array([4.0, 1e-4], np.float32)
    eps = np.array([[0.0, 1.0, -2.0], [0.5, 0.0, 1.0]], np.float32)
    z = orc.sample(qm, qv, eps)
    np.testing.assert_array_equal(z[0], np.float32([0.25, 2.25, -3.75]))
    np.testing.assert_allclose(z[1], [-2.995, -3.0, -2.99], rtol=1e-6)


# ---------------------------------------------------------------- fresh-sample denominator
# "use a second, distinct sample z_new ~ Q_MP to calculate Pe(z_new) instead
# (with r_k(z) and m(z^k) unchanged)" -> m_one = sum_k r_k(z) m(z^k) / Pe(z_new)
# (R28).


def test_fresh_denominator_same_sample_is_self_normalised():
    """With z_new = z the fresh-sample step is exactly the self-normalised one (ratio 1)."""
    m = synth.config(2, n=7, K=16, d=3)
    data = synth.make_data(m)
    state = orc.initial_state(m)
    q = synth.random_q(m, 4)
    eps = orc.eps_for_iteration(m, 3, 21)
    a = orc.qem_step(m, state, q, eps, 3, data=data)
    b = orc.qem_step(m, state, q, eps, 3, data=data, eps_new=eps)
    assert b["ratio"] == 1.0
    for (x1, x2), (y1, y2) in zip(a["state"], b["state"]):
        np.testing.assert_array_equal(x1, y1)
        np.testing.assert_array_equal(x2, y2)


def test_fresh_denominator_scales_by_evidence_ratio():
    """The fresh-sample one-step mean parameters are the self-normalised ones times
    Pe(z) / Pe(z_new), with Pe(z_new) an independent E-step (checked through the EMA with w = 1)."""
    m = synth.config(1)
    data = synth.make_data(m)
    state = orc.initial_state(m)
    q = synth.random_q(m, 6)
    eps, eps_new = orc.eps_for_iteration(m, 2, 31), orc.eps_for_iteration(m, 2, 31 + orc.FRESH_SEED_OFFSET)
    r = orc.qem_step(m, state, q, eps, 2, new_weight=1.0, data=data, eps_new=eps_new)
    z_new = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps_new)]
    ratio = math.exp(r["est"]["log_pe"] - orc.estep(m, z_new, q, data)["log_pe"])
    assert abs(r["ratio"] / ratio - 1) < 1e-12
    for (s1, s2), a, b in zip(r["state"], r["est"]["m1"], r["est"]["m2"]):
        np.testing.assert_allclose(s1, ratio * a, rtol=1e-12)
        np.testing.assert_allclose(s2, ratio * b, rtol=1e-12)


def test_fresh_numerator_unbiased_conjugate():
    """The estimator's numerator sum_k r_k(z) m(z^k) = Pe(z) E_w[z] is unbiased for
    p(x) E_post[z] (importance sampling identity behind PAPER.md:274-275): Monte Carlo mean over
    independent banks vs the closed form, within 4 standard errors, for mu and every z_i."""
    m = synth.config(1)
    data = synth.make_data(m)
    lpx = closed_form.log_evidence(data.xg)
    mean, _ = closed_form.posterior(data.xg)
    qq = [(np.zeros(1, np.float32), np.full(1, 2.0, np.float32)),
          (np.zeros(m.n, np.float32), np.full(m.n, 2.0, np.float32))]
    num = []
    for s in range(3000):
        eps = [synth.eps_normal((n * dd, m.K), 500_000 + 3 * s + lvl) for lvl, (n, dd) in enumerate(synth.latent_shapes(m))]
        z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(qq, eps)]
        r = orc.estep(m, z, qq, data)
        num.append(math.exp(r["log_pe"] - lpx) * np.concatenate([r["m1"][0], r["m1"][1]]))
    num = np.asarray(num)
    est, se = num.mean(axis=0), num.std(axis=0, ddof=1) / math.sqrt(len(num))
    assert np.all(np.abs(est - mean) < 4 * se + 1e-3), (est, mean, se)
