"""Discrete (categorical) latents under a Gaussian root (NEXT row f1, E-step side; R30):
the oracle pinned on CPU (sampler frequencies, likelihood normalisation, evidence unbiasedness
against Gauss-Hermite quadrature with the discrete latents summed exactly), then every device
call against it on GPU."""
import numpy as np
import pytest
from numpy.polynomial.hermite_e import hermegauss
from scipy.special import log_softmax, logsumexp

from oracle import discrete as od
from oracle import tables
from paper_2503_08264_b200 import synth


# ------------------------------------------------------------------ oracle pins (CPU)


def test_categorical_sampler_frequencies():
    p = np.array([[0.1, 0.6, 0.3], [0.5, 0.0, 0.5], [0.0, 0.0, 1.0]])
    K = 6000
    z = od.sample_categorical(p, K, seed=11, t=3)
    for i in range(3):
        freq = np.bincount(z[i], minlength=3) / K
        se = np.sqrt(p[i] * (1 - p[i]) / K)
        assert np.all(np.abs(freq - p[i]) <= 4.5 * se + 1e-12), (i, freq)
    # different iterations draw different streams
    assert np.any(od.sample_categorical(p, 64, 11, 4) != od.sample_categorical(p, 64, 11, 5))


def test_loglik_is_a_normalised_bernoulli_pmf():
    """sum over all y in {0,1}^R of exp(L(c)) = 1 for every state (catches a sign / term slip)."""
    rng = np.random.default_rng(2)
    R, C = 4, 3
    logit = rng.normal(0, 4, (1, R, C))
    ys = np.array([[(b >> r) & 1 for r in range(R)] for b in range(2 ** R)], np.uint8)
    tot = np.zeros(C)
    for y in ys:
        tot += np.exp(od.loglik(y[None, :], logit)[0])
    np.testing.assert_allclose(tot, 1.0, atol=1e-13)


def _small_model(n=3, C=2, R=3, K=4, seed=5):
    om = synth.occupancy(n=n, R=R, K=K, C=C, seed=seed)
    return om


def _exact_evidence(om, L):
    """p(y) = int N(r; 0, I) prod_i sum_c softmax(x_i . r)_c exp(L_i(c)) dr (2-D Gauss-Hermite)."""
    t, wt = hermegauss(80)
    wt = wt / np.sqrt(2 * np.pi)
    R0, R1 = np.meshgrid(t, t, indexing="ij")
    W = np.outer(wt, wt)
    r = np.stack([R0.ravel(), R1.ravel()])                          # [2][G]
    eta = np.einsum("icd,dg->igc", om.x, r)
    lik = logsumexp(log_softmax(eta, axis=2) + L[:, None, :], axis=2).sum(axis=0)  # [G]
    return float((W.ravel() * np.exp(lik)).sum())


@pytest.mark.parametrize("C", [2, 3])
def test_evidence_estimate_is_unbiased(C):
    """E[exp(log Pe)] = p(y) for any Q with full support."""
    om = _small_model(C=C)
    L = od.loglik(om.y, om.logit)
    exact = _exact_evidence(om, L)
    rng = np.random.default_rng(7)
    st = dict(root_mean=np.array([0.3, -0.2], np.float32), root_var=np.array([0.8, 1.4], np.float32),
              p=rng.dirichlet(np.ones(C), om.n))
    vals = []
    for s in range(2500):
        eps = rng.normal(0, 1, (om.d, om.K)).astype(np.float32)
        rz = od.oracle.sample(st["root_mean"], st["root_var"], eps)
        z = od.sample_categorical(st["p"], om.K, seed=1000 + s, t=1)
        fr, f = od.make_tables(rz, st["root_mean"], st["root_var"], om.x, L, st["p"], z)
        vals.append(np.exp(tables.estep_tables(fr, f)["log_pe"]))
    vals = np.array(vals)
    se = vals.std() / np.sqrt(len(vals))
    assert abs(vals.mean() - exact) <= 4.5 * se, (vals.mean(), exact, se)


def test_mstep_constant_input_reaches_its_fixed_point():
    """EMA of a constant mean-parameter input converges to it (PAPER.md:583 closed form)."""
    st = dict(root_ema=np.array([[0.0, 1.0]]), p_ema=np.array([[0.5, 0.5]]))
    rm, pm = np.array([[0.4, 0.41]]), np.array([[0.2, 0.8]])
    for _ in range(200):
        nxt = od.mstep(0.7, rm, st["root_ema"], pm, st["p_ema"])
        st = dict(root_ema=nxt["root_ema"], p_ema=nxt["p_ema"])
    np.testing.assert_allclose(nxt["p"], pm, atol=1e-12)
    np.testing.assert_allclose(nxt["root_mean"], [0.4], rtol=1e-6)
    np.testing.assert_allclose(nxt["root_var"], [0.41 - 0.16], rtol=1e-6)


# ------------------------------------------------------------------ device path (GPU)


def _eps(om, t, seed):
    return np.random.default_rng(seed * 7919 + t).normal(0, 1, (om.d, om.K)).astype(np.float32)


def _check_step(g, ref, tag):
    import torch
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g.root_z.cpu().numpy(), ref["root_z"], err_msg=tag)
    np.testing.assert_array_equal(g.z.cpu().numpy(), ref["z"], err_msg=tag)
    np.testing.assert_allclose(g.f_root.cpu().numpy(), ref["f_root"], rtol=1e-12, atol=1e-12, err_msg=tag)
    if g.tables:
        np.testing.assert_allclose(g.f.cpu().numpy(), ref["f"], rtol=1e-12, atol=1e-12, err_msg=tag)
    np.testing.assert_allclose(g.g.cpu().numpy(), ref["est"]["g"], rtol=1e-11, atol=1e-11, err_msg=tag)
    lp = float(g.log_pe.item())
    assert abs(lp - ref["est"]["log_pe"]) <= 1e-11 * max(1.0, abs(ref["est"]["log_pe"])), (tag, lp)
    np.testing.assert_allclose(g.w_root.cpu().numpy(), ref["est"]["w_root"], rtol=1e-10, atol=1e-14, err_msg=tag)
    np.testing.assert_allclose(g.w.cpu().numpy(), ref["est"]["w"], rtol=1e-10, atol=1e-14, err_msg=tag)
    np.testing.assert_allclose(g.root_m.cpu().numpy(), ref["root_m"], rtol=1e-10, atol=1e-13, err_msg=tag)
    np.testing.assert_allclose(g.pm.cpu().numpy(), ref["pm"], rtol=1e-10, atol=1e-13, err_msg=tag)


@pytest.mark.gpu
@pytest.mark.parametrize("tables", [False, True])
@pytest.mark.parametrize("n,C,K,T", [(300, 2, 64, 4), (97, 3, 37, 3), (1, 8, 5, 2)])
def test_device_discrete_qem_teacher_forced(n, C, K, T, tables):
    from paper_2503_08264_b200.qem import CategoricalQEM
    om = synth.occupancy(n=n, K=K, C=C, seed=3)
    L = od.loglik(om.y, om.logit)
    g = CategoricalQEM(om, tables=tables)
    np.testing.assert_allclose(g.L.cpu().numpy(), L, rtol=1e-13, atol=1e-13)
    import torch
    state = od.initial_state(om)
    seed = 21
    for t in range(1, T + 1):
        g.set_state(state)
        eps = _eps(om, t, seed)
        ref = od.qem_step(om, state, t, seed, eps, L=L)
        g.step(t, seed, root_eps=torch.from_numpy(eps).cuda())
        _check_step(g, ref, f"n{n} C{C} K{K} t={t}")
        nxt = ref["next"]
        np.testing.assert_allclose(g.p.cpu().numpy(), nxt["p"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(g.root_mean.cpu().numpy(), nxt["root_mean"], rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(g.root_var.cpu().numpy(), nxt["root_var"], rtol=1e-6)
        state = {k: nxt[k] for k in ("root_ema", "root_mean", "root_var", "p_ema", "p")}


@pytest.mark.gpu
@pytest.mark.parametrize("tables", [False, True])
def test_device_discrete_full_size_iteration(tables):
    """The Occupancy-shaped default (14400 sites, K = 64): one iteration against the oracle."""
    import torch
    from paper_2503_08264_b200.qem import CategoricalQEM
    om = synth.occupancy()
    L = od.loglik(om.y, om.logit)
    g = CategoricalQEM(om, tables=tables)
    state = od.initial_state(om)
    eps = _eps(om, 1, 5)
    ref = od.qem_step(om, state, 1, 5, eps, L=L)
    g.step(1, 5, root_eps=torch.from_numpy(eps).cuda())
    _check_step(g, ref, "occupancy full size")


@pytest.mark.gpu
def test_device_discrete_philox_run_is_finite_and_learns():
    """Free-running with device Philox root samples: finite, and the occupancy probabilities move
    toward the sites' detections (a site with a detection is occupied: p(present) -> 1)."""
    from paper_2503_08264_b200.qem import CategoricalQEM
    om = synth.occupancy(n=2000, K=64)
    g = CategoricalQEM(om)
    for t in range(1, 31):
        g.step(t, 99)
    p = g.p.cpu().numpy()
    assert np.all(np.isfinite(p)) and np.isfinite(float(g.log_pe.item()))
    detected = om.y.max(axis=1) == 1
    # posterior P(present | a detection) ~ 1 - 1e-4 (false-positive logit -10); the importance
    # weights of the rare absent samples (1/q large) keep single sites' estimates noisy
    assert p[detected, 1].mean() > 0.995 and p[detected, 1].min() > 0.9, p[detected, 1].min()
