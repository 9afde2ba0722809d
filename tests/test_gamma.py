"""Gamma and Beta approximate posteriors, E-step side (NEXT row f1; R32) on the
Gamma-Poisson and Beta-Binomial hierarchies: the oracle pinned on CPU (Marsaglia-Tsang draws against the Gamma law, evidence
unbiasedness against quadrature with the rates integrated out exactly), then the device calls
against it on GPU."""
import numpy as np
import pytest
from numpy.polynomial.hermite_e import hermegauss
from scipy import stats
from scipy.special import gammaln

from oracle import gamma as og
from oracle import tables
from paper_2503_08264_b200 import synth


# ------------------------------------------------------------------ oracle pins (CPU)


@pytest.mark.parametrize("shape,rate", [(0.4, 2.0), (1.0, 1.0), (3.5, 0.7), (40.0, 10.0)])
def test_gamma_sampler_follows_the_gamma_law(shape, rate):
    z = og.sample_gamma(np.array([[shape, rate]]), 4000, seed=3, t=2)[0]
    assert np.all(np.isfinite(z)) and np.all(z > 0)
    ks = stats.kstest(z, stats.gamma(shape, scale=1.0 / rate).cdf)
    assert ks.pvalue > 1e-3, ks
    assert abs(z.mean() - shape / rate) < 5 * np.sqrt(shape) / rate / np.sqrt(len(z))


def _evidence(gp):
    """p(y) = int N(mu; 0, 1) prod_i NegBin(y_i | alpha, alpha e^-mu) dmu (Gauss-Hermite): the
    Gamma rates integrate out in closed form (Gamma-Poisson conjugacy)."""
    t, wt = hermegauss(120)
    wt = wt / np.sqrt(2 * np.pi)
    y = np.asarray(gp.y, np.float64)
    S, J = y.sum(axis=1), y.shape[1]
    a = gp.alpha
    tot = np.zeros_like(t)
    for g, mu in enumerate(t):
        b = a * np.exp(-mu)
        lp = (a * np.log(b) - gammaln(a) + gammaln(a + S) - (a + S) * np.log(b + J) - gammaln(y + 1).sum(axis=1))
        tot[g] = lp.sum()
    return float((wt * np.exp(tot)).sum())


def test_evidence_estimate_is_unbiased():
    """E[exp(log Pe)] = p(y) for Gamma proposals."""
    gp = synth.gamma_poisson(n=3, J=4, K=4, seed=2)
    exact = _evidence(gp)
    rng = np.random.default_rng(4)
    q = np.array([[2.0, 1.5], [0.8, 0.5], [4.0, 2.0]])
    vals = []
    for s in range(2500):
        mu = np.float32(0.2) + np.sqrt(np.float32(0.9)) * rng.normal(size=gp.K).astype(np.float32)
        z = og.sample_gamma(q, gp.K, seed=500 + s, t=1)
        fr, f = og.make_tables(gp, mu, 0.2, 0.9, q, z)
        vals.append(np.exp(tables.estep_tables(fr, f)["log_pe"]))
    vals = np.array(vals)
    se = vals.std() / np.sqrt(len(vals))
    assert abs(vals.mean() - exact) <= 4.5 * se, (vals.mean(), exact, se)


@pytest.mark.parametrize("a,b", [(0.5, 0.7), (2.0, 5.0), (30.0, 3.0)])
def test_beta_sampler_follows_the_beta_law(a, b):
    z = og.sample_beta(np.array([[a, b]]), 3000, seed=5, t=1)[0]
    assert np.all((z > 0) & (z < 1))
    assert stats.kstest(z, stats.beta(a, b).cdf).pvalue > 1e-3


def _evidence_bb(bb):
    """p(y) = int N(mu; 0, 1) prod_i BetaBinomial(y_i; N_i, kappa s, kappa (1 - s)) dmu."""
    t, wt = hermegauss(120)
    wt = wt / np.sqrt(2 * np.pi)
    tot = np.array([stats.betabinom.logpmf(bb.y, bb.N, bb.kappa / (1 + np.exp(-mu)),
                                           bb.kappa * (1 - 1 / (1 + np.exp(-mu)))).sum() for mu in t])
    return float((wt * np.exp(tot)).sum())


def test_beta_evidence_estimate_is_unbiased():
    bb = synth.beta_binomial(n=3, K=4, seed=3, n_max=6)
    exact = _evidence_bb(bb)
    rng = np.random.default_rng(6)
    q = np.array([[2.0, 1.5], [0.9, 0.6], [3.0, 4.0]])
    vals = []
    for s in range(2500):
        mu = np.float32(-0.1) + np.sqrt(np.float32(1.2)) * rng.normal(size=bb.K).astype(np.float32)
        z = og.sample_beta(q, bb.K, seed=900 + s, t=1)
        fr, f = og.make_tables_beta(bb, mu, -0.1, 1.2, q, z)
        vals.append(np.exp(tables.estep_tables(fr, f)["log_pe"]))
    vals = np.array(vals)
    se = vals.std() / np.sqrt(len(vals))
    assert abs(vals.mean() - exact) <= 4.5 * se, (vals.mean(), exact, se)


# ------------------------------------------------------------------ device path (GPU)


def _factors(g):
    """The device's log-factor table: stored (tables path) or rebuilt from the separable rows and
    columns, f[i][k][k'] = a_k + sum_r b_k[r] phi_i(k')[r] + psi_i(k') (qem_estep_separable)."""
    if g.tables:
        return g.f.cpu().numpy()
    rows, cols = g.rows.cpu().numpy(), g.cols.cpu().numpy()
    R = rows.shape[1] - 1
    f = rows[None, :, 0, None] + cols[:, None, :, R]
    for r in range(R):
        f = f + rows[None, :, 1 + r, None] * cols[:, None, :, r]
    return f


@pytest.mark.gpu
@pytest.mark.parametrize("use_tables", [False, True], ids=["separable", "tables"])
@pytest.mark.parametrize("n,K,T", [(150, 64, 3), (29, 17, 2)])
def test_device_beta_qem_teacher_forced(n, K, T, use_tables):
    import torch
    from paper_2503_08264_b200.qem import BetaBinomialQEM
    bb = synth.beta_binomial(n=n, K=K, seed=4)
    g = BetaBinomialQEM(bb, tables=use_tables)
    state = og.initial_state_beta(bb)
    seed = 19
    for t in range(1, T + 1):
        g.set_state(state)
        eps = np.random.default_rng(10 + t).normal(size=K).astype(np.float32)
        ref = og.qem_step_beta(bb, state, t, seed, eps)
        g.step(t, seed, root_eps=torch.from_numpy(eps).cuda())
        torch.cuda.synchronize()
        tag = f"beta n{n} K{K} t={t}"
        np.testing.assert_allclose(g.z.cpu().numpy(), ref["z"], rtol=1e-12, err_msg=tag)
        np.testing.assert_allclose(_factors(g), ref["f"], rtol=1e-11, atol=1e-10, err_msg=tag)
        assert abs(float(g.log_pe.item()) - ref["est"]["log_pe"]) <= 1e-10 * abs(ref["est"]["log_pe"]), tag
        np.testing.assert_allclose(g.w.cpu().numpy(), ref["est"]["w"], rtol=1e-9, atol=1e-13, err_msg=tag)
        np.testing.assert_allclose(g.gm.cpu().numpy(), ref["gm"], rtol=1e-10, atol=1e-12, err_msg=tag)
        nxt = ref["next"]
        assert np.all(g.status.cpu().numpy() == 0), tag
        np.testing.assert_allclose(g.q.cpu().numpy(), nxt["q"], rtol=1e-8, err_msg=tag)
        state = nxt



@pytest.mark.gpu
@pytest.mark.parametrize("use_tables", [False, True], ids=["separable", "tables"])
@pytest.mark.parametrize("n,K,T", [(200, 64, 3), (37, 33, 2)])
def test_device_gamma_qem_teacher_forced(n, K, T, use_tables):
    import torch
    from paper_2503_08264_b200.qem import GammaPoissonQEM
    gp = synth.gamma_poisson(n=n, K=K, seed=3)
    g = GammaPoissonQEM(gp, tables=use_tables)
    state = og.initial_state(gp)
    seed = 17
    for t in range(1, T + 1):
        g.set_state(state)
        eps = np.random.default_rng(t).normal(size=K).astype(np.float32)
        ref = og.qem_step(gp, state, t, seed, eps)
        g.step(t, seed, root_eps=torch.from_numpy(eps).cuda())
        torch.cuda.synchronize()
        tag = f"n{n} K{K} t={t}"
        np.testing.assert_array_equal(g.mu.cpu().numpy()[0], ref["mu"], err_msg=tag)
        np.testing.assert_allclose(g.z.cpu().numpy(), ref["z"], rtol=1e-13, err_msg=tag)
        np.testing.assert_allclose(_factors(g), ref["f"], rtol=1e-11, atol=1e-10, err_msg=tag)
        assert abs(float(g.log_pe.item()) - ref["est"]["log_pe"]) <= 1e-10 * abs(ref["est"]["log_pe"]), tag
        np.testing.assert_allclose(g.w.cpu().numpy(), ref["est"]["w"], rtol=1e-9, atol=1e-13, err_msg=tag)
        np.testing.assert_allclose(g.gm.cpu().numpy(), ref["gm"], rtol=1e-10, atol=1e-12, err_msg=tag)
        nxt = ref["next"]
        assert np.all(g.status.cpu().numpy() == 0), tag
        np.testing.assert_allclose(g.q.cpu().numpy(), nxt["q"], rtol=1e-9, err_msg=tag)
        np.testing.assert_allclose(g.root_mean.cpu().numpy()[0], nxt["root_mean"], rtol=1e-6, atol=1e-7)
        state = nxt


@pytest.mark.gpu
def test_device_gamma_qem_learns_the_rates():
    """Free-running with device Philox draws: the Gamma posteriors' means approach the
    conjugate per-group posterior means (alpha + S) / (alpha e^-mu + J) at the true mu."""
    from paper_2503_08264_b200.qem import GammaPoissonQEM
    gp = synth.gamma_poisson(n=500, J=8, K=128)
    g = GammaPoissonQEM(gp)
    for t in range(1, 41):
        g.step(t, 23)
    q = g.q.cpu().numpy()
    assert np.all(np.isfinite(q)) and np.all(g.status.cpu().numpy() == 0)
    S = gp.y.sum(axis=1)
    target = (gp.alpha + S) / (gp.alpha * np.exp(-gp.mu_true) + gp.J)
    rel = np.abs(q[:, 0] / q[:, 1] - target) / target
    assert np.median(rel) < 0.1, np.median(rel)
