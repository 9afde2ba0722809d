"""Backward index resampling + predictive log-likelihood (NEXT row f3; PAPER.md:326-327, 794;
DESIGN.md R31).  CPU: the oracle's conditionals normalise against the C oracle's messages,
its draws match brute-force enumeration (joint and marginals), and its predictive
log-likelihood matches the closed-form conjugate posterior predictive (config 1).  GPU: the
device draws and test log-likelihoods against the oracle's."""
import numpy as np
import pytest

from helpers import make_case, posterior_like_q
from oracle import brute, closed_form
from oracle import oracle as orc
from oracle import predict as op
from paper_2503_08264_b200 import synth


def _case(cid, n, K, seed=3, **kw):
    m = synth.config(cid, n=n, K=K, **kw)
    data, q, eps, z = make_case(m, q_seed=seed)
    return m, data, q, eps, z


# ------------------------------------------------------------------ oracle pins (CPU)


@pytest.mark.parametrize("cid", [1, 4, 2])
def test_conditionals_normalise_against_the_c_oracle(cid):
    """sum_k' P_i(k'|k) = 1 for every (i, k): the numpy B + A here and the C oracle's messages g
    are independent codes for the same Eq. 7 quantities."""
    m, data, q, eps, z = _case(cid, n=5, K=16, J=4, **({"d": 3} if cid == 2 else {}))
    est = orc.estep(m, z, q, data)
    for i in range(m.n):
        lp = op.log_conditionals(m, z, q, data, est["g"], i)
        np.testing.assert_allclose(np.exp(lp).sum(axis=1), 1.0, atol=1e-10)


def test_resampled_tuples_follow_the_enumerated_posterior():
    """Joint frequencies of (k_root, k_1, k_2) over S draws against the normalised weights of all
    K^3 tuples from brute-force enumeration (SPEC.md:340-342's chi-square example)."""
    m, data, q, eps, z = _case(1, n=2, K=3)
    est = orc.estep(m, z, q, data)
    joint = brute.estep2(m, z, q, data, joint=True)["joint"]
    S = 20000
    r = op.resample(m, z, q, data, est, S, seed=77)
    counts = np.zeros_like(joint)
    np.add.at(counts, (r["idx_root"], r["idx"][:, 0], r["idx"][:, 1]), 1)
    expct = joint * S
    live = expct > 5
    chi2 = (((counts - expct) ** 2)[live] / expct[live]).sum()
    dof = live.sum() - 1
    assert chi2 < dof + 6 * np.sqrt(2 * dof), (chi2, dof)
    assert counts[~live].sum() <= max(10, 3 * expct[~live].sum())


def test_predictive_loglik_matches_the_conjugate_posterior_predictive():
    """Config 1: log p(x_test | x) = log p(x, x_test) - log p(x) from the marginal Gaussians
    (closed_form.log_evidence) against the oracle's PLL at K = 256, S = 4000."""
    m = synth.config(1, K=256)
    data = synth.make_data(m)
    test = synth.make_test_data(m, data, J_test=3)
    mean, cov = closed_form.posterior(data.xg, m.prior_var, m.fixed_var, m.obs_var)
    sd = np.sqrt(np.diag(cov))
    q = [(np.array([mean[0]], np.float32), np.array([sd[0] ** 2], np.float32)),
         (mean[1:].astype(np.float32), (sd[1:] ** 2).astype(np.float32))]
    eps = [synth.eps_normal((nn * dd, m.K), 5 + lvl) for lvl, (nn, dd) in enumerate(synth.latent_shapes(m))]
    z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
    est = orc.estep(m, z, q, data)
    r = op.resample(m, z, q, data, est, 4000, seed=9)
    pll, _ = op.predictive_loglik(op.test_loglik(m, z, test, r["idx"]))
    x_all = np.concatenate([data.xg, test.xg], axis=1)
    exact = (closed_form.log_evidence(x_all, m.prior_var, m.fixed_var, m.obs_var)
             - closed_form.log_evidence(data.xg, m.prior_var, m.fixed_var, m.obs_var))
    assert abs(pll - exact) < 0.05, (pll, exact)


def test_single_predictive_sample():
    """S = 1: the PLL is the test log-likelihood at that one tuple."""
    m, data, q, eps, z = _case(4, n=6, K=8, J=3)
    test = synth.make_test_data(m, data)
    idx = np.array([[3, 1, 4, 1, 5, 2]], np.int32)
    ll = op.test_loglik(m, z, test, idx)
    pll, ll_s = op.predictive_loglik(ll)
    assert pll == pytest.approx(ll_s[0], abs=1e-12)


# ------------------------------------------------------------------ device path (GPU)


def _device_draws(m, data, q, eps, S, seed, test=None):
    import torch
    from paper_2503_08264_b200.qem import QEM
    g = QEM(m)
    g.set_data(data)
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    ir, ix = g.backward_resample(S, seed)
    out = dict(idx_root=ir.cpu().numpy(), idx=ix.cpu().numpy())
    if test is not None:
        pll, ll_s, ll_part = g.predictive_loglik(ix, test)
        torch.cuda.synchronize()
        out.update(pll=float(pll.item()), ll_s=ll_s.cpu().numpy(), ll_part=ll_part.cpu().numpy())
    g.close()
    return out


def _check_draws(dev, ref, tag):
    """Identical draws except where the oracle's u sits within a rounding distance of a CDF boundary
    (fp32 root weights / the column prep's fp32 softplus shift boundaries by <= ~1e-5)."""
    bad_root = dev["idx_root"] != ref["idx_root"]
    assert np.all(ref["margin_root"][bad_root] < 1e-5), (tag, ref["margin_root"][bad_root])
    same = ~bad_root
    bad = (dev["idx"] != ref["idx"]) & same[:, None]
    assert np.all(ref["margin"][bad] < 1e-4), (tag, ref["margin"][bad])
    assert bad.mean() < 1e-3 and bad_root.mean() < 0.05, (tag, bad.mean(), bad_root.mean())
    return same


@pytest.mark.gpu
@pytest.mark.parametrize("cid,n,K,extra", [(1, 4, 8, {}), (4, 300, 96, {"J": 8}), (2, 60, 30, {}),
                                           (5, 40, 256, {})])
def test_device_resample_and_predictive_match_oracle(cid, n, K, extra):
    m = synth.config(cid, n=n, K=K, **extra)
    data = synth.make_data(m)
    q = posterior_like_q(m, data, seed=4, shrink=1.0)
    _, _, eps, z = make_case(m, q=q)
    test = synth.make_test_data(m, data)
    S, seed = 100, 31
    est = orc.estep(m, z, q, data)
    ref = op.resample(m, z, q, data, est, S, seed)
    dev = _device_draws(m, data, q, eps, S, seed, test)
    same = _check_draws(dev, ref, f"c{cid}")
    ll_ref = op.test_loglik(m, z, test, ref["idx"])
    rows = same & np.all(dev["idx"] == ref["idx"], axis=1)
    np.testing.assert_allclose(dev["ll_part"][rows], ll_ref[rows], rtol=1e-12, atol=1e-10)
    if rows.all():
        pll_ref, _ = op.predictive_loglik(ll_ref)
        assert abs(dev["pll"] - pll_ref) <= 1e-10 * max(1.0, abs(pll_ref))


@pytest.mark.gpu
def test_device_resample_kernels_agree(monkeypatch):
    """The shared-memory tile kernel and the per-draw kernel (forced by QEM_RESAMPLE_NO_TILE) draw
    the same indices (same fp64 rows up to summation order)."""
    m = synth.config(5, n=30, K=256)
    data, q, eps, z = make_case(m)
    a = _device_draws(m, data, q, eps, 64, 5)
    monkeypatch.setenv("QEM_RESAMPLE_NO_TILE", "1")
    b = _device_draws(m, data, q, eps, 64, 5)
    np.testing.assert_array_equal(a["idx_root"], b["idx_root"])
    assert (a["idx"] != b["idx"]).mean() < 1e-3


@pytest.mark.gpu
def test_device_resample_is_deterministic_and_seeded():
    m = synth.config(5, n=20, K=256)
    data, q, eps, z = make_case(m)
    a = _device_draws(m, data, q, eps, 50, 1)
    b = _device_draws(m, data, q, eps, 50, 1)
    c = _device_draws(m, data, q, eps, 50, 2)
    np.testing.assert_array_equal(a["idx"], b["idx"])
    assert np.any(a["idx"] != c["idx"])
    assert a["idx"].min() >= 0 and a["idx"].max() < m.K


# ------------------------------------------------------------------ global IW (App. A)


def test_global_iw_is_unbiased_on_the_conjugate_model():
    """E[exp(log Pe_glob)] = p(x) (an importance-sampling estimate with joint proposals, App. A;
    p(x) from the marginal Gaussian, closed_form.log_evidence) on config 1."""
    m = synth.config(1, K=64)
    data = synth.make_data(m)
    mean, cov = closed_form.posterior(data.xg, m.prior_var, m.fixed_var, m.obs_var)
    sd = np.sqrt(np.diag(cov)) * 1.3
    q = [(np.array([mean[0]], np.float32), np.array([sd[0] ** 2], np.float32)),
         (mean[1:].astype(np.float32), (sd[1:] ** 2).astype(np.float32))]
    exact = closed_form.log_evidence(data.xg, m.prior_var, m.fixed_var, m.obs_var)
    vals = []
    for s in range(1500):
        eps = [synth.eps_normal((nn * dd, m.K), 10_000 + 7 * s + lvl) for lvl, (nn, dd) in enumerate(synth.latent_shapes(m))]
        z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
        est = orc.estep(m, z, q, data)
        vals.append(np.exp(op.global_iw(m, z, q, data, est)["log_pe"] - exact))
    vals = np.array(vals)
    se = vals.std() / np.sqrt(len(vals))
    assert abs(vals.mean() - 1.0) <= 4.5 * se, (vals.mean(), se)


@pytest.mark.gpu
@pytest.mark.parametrize("cid,n,K", [(1, 4, 8), (4, 200, 64), (5, 30, 256)])
def test_device_global_iw_matches_oracle(cid, n, K):
    import torch
    from paper_2503_08264_b200.qem import QEM
    m = synth.config(cid, n=n, K=K)
    data = synth.make_data(m)
    q = posterior_like_q(m, data, seed=2, shrink=1.5)
    _, _, eps, z = make_case(m, q=q)
    est = orc.estep(m, z, q, data)
    ref = op.global_iw(m, z, q, data, est)
    g = QEM(m)
    g.set_data(data)
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    out = g.global_iw()
    torch.cuda.synchronize()
    g.close()
    # north-star tolerances: the column prep's t_ref carries fp32 softplus sums on the Bernoulli
    # configs (R26), so the diagonal log-factors agree to ~1e-5 there, to ~1e-12 on the Gaussian ones
    np.testing.assert_allclose(out["diag"].cpu().numpy(), ref["diag"], rtol=1e-7, atol=5e-5)
    assert abs(float(out["log_pe"].item()) - ref["log_pe"]) <= 1e-5 * abs(ref["log_pe"])
    np.testing.assert_allclose(out["w"].cpu().numpy(), ref["w"], atol=1e-5)
    scale = np.maximum(np.abs(ref["m1"]), 1e-2)
    assert np.max(np.abs(out["m1"].cpu().numpy() - ref["m1"]) / scale) <= 1e-4
