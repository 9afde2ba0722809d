"""Non-factorised Q_MP with the permutation / mixture parent-copy schemes (App. A, PAPER.md:470-479;
NEXT row f4, R43): the oracle (oracle/qmp.py) pinned on CPU, then the device path
(qem_cols_qmp_gaussian -> qem_estep_separable -> qem_moments_qmp) against it on GPU."""
import numpy as np
import pytest
from scipy.stats import norm

from oracle import closed_form
from oracle import oracle as orc
from oracle import qmp as oq
from paper_2503_08264_b200 import synth

SCHEMES = [oq.PERMUTATION, oq.MIXTURE]


def _case(n, K, J, seed, scheme, beta=0.8, root=(0.3, 1.2), gv=1.0, ov=1.0):
    rng = np.random.default_rng(seed)
    mu_t = rng.standard_normal()
    zt = mu_t + np.sqrt(gv) * rng.standard_normal(n)
    x = (zt[:, None] + np.sqrt(ov) * rng.standard_normal((n, J))).astype(np.float32)
    rm, rv = np.float32(root[0]), np.float32(root[1])
    mu = (rm + np.sqrt(rv) * rng.standard_normal(K)).astype(np.float32)
    # a proposal near the conditional posterior z_i | mu, x_i = N((mu/gv + S_i/ov) / prec, 1/prec), jittered
    prec = 1.0 / gv + J / ov
    q = np.stack([x.sum(axis=1) / ov / prec + 0.1 * rng.standard_normal(n),
                  np.full(n, beta / gv / prec if beta else 0.0) * (1 + 0.2 * rng.standard_normal(n)),
                  (1.0 / prec) * np.exp(0.3 * rng.standard_normal(n))], axis=1)
    copy = oq.draw_copies(rng, n, K, scheme)
    eps = rng.standard_normal((n, K)).astype(np.float32)
    return dict(mu=mu, rm=rm, rv=rv, q=q, copy=copy, eps=eps, x=x, gv=gv, ov=ov)


# ------------------------------------------------------------------ oracle pins (CPU)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_beta_zero_is_the_factorised_q_of_the_c_oracle(scheme):
    """With beta_i = 0 the child ignores its parent copy, Q_MP is the factorised Q of the hot path
    and both schemes' densities are N(z; alpha_i, s_i): log Pe, weights and messages equal
    qem_oracle.c's nested sums (independent C code) on the same samples."""
    m = synth.config(1)  # n = 4, J = 5, K = 8, unit variances
    data = synth.make_data(m)
    c = _case(m.n, m.K, m.J, 11, scheme, beta=0.0)
    c["x"] = data.xg
    z = oq.sample_children(c["mu"], c["q"], c["copy"], c["eps"])
    out = oq.estep(c["mu"], c["rm"], c["rv"], c["q"], c["copy"], c["eps"], c["x"], scheme)
    ref = orc.estep(m, [c["mu"][None, :].astype(np.float64), z],
                    [(np.array([c["rm"]], np.float64), np.array([c["rv"]], np.float64)), (c["q"][:, 0], c["q"][:, 2])],
                    data)
    assert abs(out["log_pe"] - ref["log_pe"]) < 1e-10 * abs(ref["log_pe"])
    np.testing.assert_allclose(out["w_root"], ref["w"][0][0], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(out["w"], ref["w"][1], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(out["gm"][:, 0], ref["m1"][1], rtol=1e-9)
    np.testing.assert_allclose(out["gm"][:, 1], ref["m2"][1], rtol=1e-9)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_evidence_estimate_is_unbiased_under_both_schemes(scheme):
    """E_{Q_MP}[Pe(z)] = p(x) (the estimator's defining property; PAPER.md:139-150 with the Q_MP of
    App. A) against the closed-form evidence of the conjugate model, with a strongly parent-dependent
    proposal (beta = 0.8 of the conditional posterior's slope, broad root): a density that ignored the
    copy indices, used the wrong copy, or mixed the two schemes is biased here."""
    n, K, J, R = 2, 3, 2, 6000
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n, J)) + 0.5
    lpx = closed_form.log_evidence(x)
    prec = 1.0 + J
    q = np.stack([x.sum(axis=1) / prec, np.full(n, 0.8 / prec), np.full(n, 1.0 / prec)], axis=1)
    rm, rv = 0.2, 0.9
    ratios = np.empty(R)
    for r in range(R):
        mu = rm + np.sqrt(rv) * rng.standard_normal(K)
        copy = oq.draw_copies(rng, n, K, scheme)
        eps = rng.standard_normal((n, K))
        ratios[r] = np.exp(oq.estep(mu, rm, rv, q, copy, eps, x, scheme)["log_pe"] - lpx)
    se = ratios.std() / np.sqrt(R)
    assert abs(ratios.mean() - 1.0) < 4 * se + 1e-3, (ratios.mean(), se)
    # the same draws scored with the OTHER scheme's density are not an unbiased estimator in general;
    # here only check that the two densities really differ for K > 1
    mu = rm + np.sqrt(rv) * rng.standard_normal(K)
    copy = oq.draw_copies(rng, n, K, oq.PERMUTATION)
    z = oq.sample_children(mu, q, copy, rng.standard_normal((n, K)))
    assert np.abs(oq.log_qmp(z, mu, q, copy, oq.PERMUTATION) - oq.log_qmp(z, mu, q, copy, oq.MIXTURE)).max() > 1e-3


def test_wrong_copy_density_is_biased():
    """The pin above has teeth: scoring permutation draws at the identity copy (k' -> k') instead of
    the copy that was used is biased by many standard errors on the same model."""
    n, K, J, R = 2, 3, 2, 6000
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n, J)) + 0.5
    lpx = closed_form.log_evidence(x)
    prec = 1.0 + J
    q = np.stack([x.sum(axis=1) / prec, np.full(n, 0.8 / prec), np.full(n, 1.0 / prec)], axis=1)
    ident = np.tile(np.arange(K, dtype=np.int32), (n, 1))
    ratios = np.empty(R)
    for r in range(R):
        mu = 0.2 + np.sqrt(0.9) * rng.standard_normal(K)
        copy = oq.draw_copies(rng, n, K, oq.PERMUTATION)
        z = oq.sample_children(mu, q, copy, rng.standard_normal((n, K)))
        f_root, f = oq.make_tables(mu, 0.2, 0.9, q, ident, z, x, oq.PERMUTATION)
        from oracle import tables
        ratios[r] = np.exp(tables.estep_tables(f_root, f)["log_pe"] - lpx)
    se = ratios.std() / np.sqrt(R)
    assert abs(ratios.mean() - 1.0) > 6 * se


def test_single_copy_makes_the_schemes_equal_and_mixture_density_is_normalised():
    c = _case(3, 1, 2, 2, oq.PERMUTATION)
    z = oq.sample_children(c["mu"], c["q"], c["copy"], c["eps"])
    np.testing.assert_allclose(oq.log_qmp(z, c["mu"], c["q"], c["copy"], oq.PERMUTATION),
                               oq.log_qmp(z, c["mu"], c["q"], c["copy"], oq.MIXTURE), rtol=0, atol=1e-12)
    # int q_MP,i(z) dz = 1 for the mixture over K = 7 parent copies (trapezoid on a wide grid)
    c = _case(2, 7, 2, 3, oq.MIXTURE)
    grid = np.linspace(-12, 12, 24001)
    dens = np.exp(oq.log_qmp(np.tile(grid, (2, 1)), c["mu"], c["q"], c["copy"], oq.MIXTURE))
    np.testing.assert_allclose(np.trapezoid(dens, grid, axis=1), 1.0, rtol=1e-9)
    # and each permutation-scheme draw is the conditional at its own copy: residual / sd = eps
    c = _case(2, 7, 2, 4, oq.PERMUTATION)
    z = oq.sample_children(c["mu"], c["q"], c["copy"], c["eps"])
    lq = oq.log_qmp(z, c["mu"], c["q"], c["copy"], oq.PERMUTATION)
    np.testing.assert_allclose(lq, norm.logpdf(c["eps"].astype(np.float64)) - 0.5 * np.log(c["q"][:, 2:3]), atol=1e-9)


# ------------------------------------------------------------------ device parity (GPU)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("n,K,J", [(1, 1, 1), (4, 8, 5), (37, 96, 5), (300, 256, 7), (5, 1000, 3), (0, 16, 2)])
def test_device_qmp_estep_matches_oracle(n, K, J, scheme):
    import torch
    from paper_2503_08264_b200 import qem
    c = _case(n, K, J, 100 + n + K, scheme, gv=0.7, ov=1.3)
    ref = oq.estep(c["mu"], c["rm"], c["rv"], c["q"], c["copy"], c["eps"], c["x"], scheme,
                   prior_var=1.0, group_var=0.7, obs_var=1.3)
    dev = "cuda"
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(dev)  # noqa: E731
    out = qem.estep_qmp_gaussian(t(c["mu"], np.float32), t([c["rm"]], np.float32), t([c["rv"]], np.float32),
                                 t(c["q"].reshape(n, 3), np.float64), t(c["copy"].reshape(n, K), np.int32),
                                 t(c["eps"], np.float32), t(c["x"].reshape(n, J), np.float32), scheme,
                                 prior_var=1.0, group_var=0.7, obs_var=1.3)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    # fp64 on both sides; the device evaluates f = a_k + b_k z + psi (the square expanded), hence 1e-9
    assert abs(g["log_pe"][0] - ref["log_pe"]) <= 1e-9 * max(1.0, abs(ref["log_pe"]))
    np.testing.assert_allclose(g["w_root"], ref["w_root"], rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(g["root_m"], ref["root_m"], rtol=1e-9, atol=1e-12)
    if n:
        np.testing.assert_allclose(g["z"], ref["z"], rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(g["w"], ref["w"], rtol=1e-7, atol=1e-12)
        np.testing.assert_allclose(g["w"].sum(axis=1), 1.0, rtol=1e-12)
        np.testing.assert_allclose(g["g"], ref["g"], rtol=1e-10, atol=1e-9)
        np.testing.assert_allclose(g["gm"], ref["gm"], rtol=1e-8, atol=1e-12)


@pytest.mark.gpu
def test_device_qmp_rejects_bad_arguments():
    import torch
    from paper_2503_08264_b200 import _lib, qem
    c = _case(3, 8, 2, 1, oq.PERMUTATION)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to("cuda")  # noqa: E731
    args = [t(c["mu"], np.float32), t([c["rm"]], np.float32), t([c["rv"]], np.float32), t(c["q"], np.float64),
            t(c["copy"], np.int32), t(c["eps"], np.float32), t(c["x"], np.float32)]
    with pytest.raises(_lib.QemError, match="QEM_INVALID_ARGUMENT"):
        qem.estep_qmp_gaussian(*args, 2)
    with pytest.raises(_lib.QemError, match="QEM_INVALID_ARGUMENT"):
        qem.estep_qmp_gaussian(*args, oq.MIXTURE, group_var=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", SCHEMES)
def test_device_qmp_evidence_is_unbiased_with_device_drawn_normals(scheme):
    """End to end on the device, no host eps: root copies and child normals from qem_sample_normal
    (Philox), copy indices drawn with torch, qem_cols_qmp_gaussian -> qem_estep_separable; the mean of
    Pe / p(x) over 4000 independent draws is 1 within 4 standard errors (the property that holds at
    any size; closed-form evidence from oracle/closed_form.py)."""
    import ctypes
    import torch
    from paper_2503_08264_b200 import _lib, qem
    n, K, J, R = 2, 3, 2, 4000
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((n, J)) + 0.5).astype(np.float32)
    lpx = closed_form.log_evidence(x.astype(np.float64))
    prec = 1.0 + J
    q = np.stack([x.sum(axis=1) / prec, np.full(n, 0.8 / prec), np.full(n, 1.0 / prec)], axis=1)
    dev = "cuda"
    f32 = dict(dtype=torch.float32, device=dev)
    xq, qq = torch.from_numpy(x).to(dev), torch.from_numpy(q).to(dev)
    rm, rv = torch.full((1,), 0.2, **f32), torch.full((1,), 0.9, **f32)
    zero, one = torch.zeros(n, **f32), torch.ones(n, **f32)
    mu, eps = torch.empty(1, K, **f32), torch.empty(n, K, **f32)
    gen = torch.Generator(device=dev).manual_seed(9)
    L, s = _lib.lib(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    lpe = torch.empty(R, dtype=torch.float64, device=dev)
    for r in range(R):
        _lib.check(L.qem_sample_normal(1, K, 0, 77, r + 1, p(rm), p(rv), None, p(mu), s), "qem_sample_normal")
        _lib.check(L.qem_sample_normal(n, K, 1, 77, r + 1, p(zero), p(one), None, p(eps), s), "qem_sample_normal")
        if scheme == oq.PERMUTATION:
            copy = torch.argsort(torch.rand(n, K, generator=gen, device=dev), dim=1).to(torch.int32)
        else:
            copy = torch.randint(0, K, (n, K), generator=gen, device=dev, dtype=torch.int32)
        lpe[r] = qem.estep_qmp_gaussian(mu[0], rm, rv, qq, copy, eps, xq, scheme)["log_pe"][0]
    ratios = torch.exp(lpe - lpx).cpu().numpy()
    assert np.all(np.isfinite(ratios))
    se = ratios.std() / np.sqrt(R)
    assert abs(ratios.mean() - 1.0) < 4 * se + 1e-3, (ratios.mean(), se)
