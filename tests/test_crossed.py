"""Crossed effects (NEXT row f4; R33): the oracle pinned on CPU by
evidence unbiasedness against 4-D Gauss-Hermite quadrature, then the device calls against it."""
import itertools

import numpy as np
import pytest
from numpy.polynomial.hermite_e import hermegauss
from scipy.special import log_expit

from oracle import crossed as oc
from oracle import tables
from paper_2503_08264_b200 import synth


def _exact_evidence(cm, nodes=24):
    """One company, one journey type, one group: p(y) = int N(mu) N(cw) N(jw) N(w; mu, 1)
    prod_j Bern(y_j; sigmoid(w + cw + jw)) over (mu, cw, jw, w) by Gauss-Hermite (w = mu + e)."""
    t, wt = hermegauss(nodes)
    wt = wt / np.sqrt(2 * np.pi)
    y = cm.y[0].astype(np.float64)
    tot = 0.0
    for (a, wa), (b, wb), (c, wc) in itertools.product(zip(t, wt), repeat=3):
        w = a + t                                   # w = mu + e, e ~ N(0, 1)
        eta = w[:, None] + b + c
        lik = np.exp((y * log_expit(eta) + (1 - y) * log_expit(-eta)).sum(axis=1))
        tot += wa * wb * wc * (wt * lik).sum()
    return tot


def test_evidence_estimate_is_unbiased():
    cm = synth.bus_crossed(n=1, J=6, C=1, T=1, K=4, seed=3)
    exact = _exact_evidence(cm)
    rng = np.random.default_rng(8)
    rm = np.array([0.1, -0.2, 0.3], np.float32)
    rv = np.array([0.8, 1.3, 0.9], np.float32)
    qm, qv = np.array([0.2], np.float32), np.array([1.5], np.float32)
    vals = []
    for s in range(3000):
        rz = oc.oracle.sample(rm, rv, rng.normal(size=(cm.R, cm.K)).astype(np.float32))
        z = oc.oracle.sample(qm, qv, rng.normal(size=(cm.n, cm.K)).astype(np.float32))
        fr, f = oc.make_tables(cm, rz, rm, rv, z, qm, qv)
        vals.append(np.exp(tables.estep_tables(fr, f)["log_pe"]))
    vals = np.array(vals)
    se = vals.std() / np.sqrt(len(vals))
    assert abs(vals.mean() - exact) <= 4.5 * se, (vals.mean(), exact, se)


@pytest.mark.gpu
@pytest.mark.parametrize("use_tables", [False, True], ids=["on_chip", "tables"])
@pytest.mark.parametrize("n,J,C,T,K,steps", [(40, 12, 7, 3, 32, 3), (120, 40, 57, 6, 64, 2), (3, 1, 1, 1, 5, 2)])
def test_device_crossed_qem_teacher_forced(n, J, C, T, K, steps, use_tables):
    import torch
    from paper_2503_08264_b200.qem import CrossedQEM
    cm = synth.bus_crossed(n=n, J=J, C=C, T=T, K=K, seed=4)
    g = CrossedQEM(cm, tables=use_tables)
    state = oc.initial_state(cm)
    for t in range(1, steps + 1):
        g.set_state(state)
        rng = np.random.default_rng(100 + t)
        er = rng.normal(size=(cm.R, K)).astype(np.float32)
        eg = rng.normal(size=(n, K)).astype(np.float32)
        ref = oc.qem_step(cm, state, t, er, eg)
        g.step(t, 1, root_eps=torch.from_numpy(er).cuda(), eps=torch.from_numpy(eg).cuda())
        torch.cuda.synchronize()
        tag = f"crossed n{n} K{K} t={t}"
        np.testing.assert_array_equal(g.rz.cpu().numpy(), ref["rz"], err_msg=tag)
        np.testing.assert_array_equal(g.z.cpu().numpy(), ref["z"], err_msg=tag)
        if use_tables:
            np.testing.assert_allclose(g.f.cpu().numpy(), ref["f"], rtol=1e-11, atol=1e-10, err_msg=tag)
        else:  # no table: the plate messages g_i(k) = lse_k' f_i(k, k') - ln K of the oracle's tables
            np.testing.assert_allclose(g.g.cpu().numpy(), ref["est"]["g"], rtol=1e-11, atol=1e-10, err_msg=tag)
        assert abs(float(g.log_pe.item()) - ref["est"]["log_pe"]) <= 1e-10 * abs(ref["est"]["log_pe"]), tag
        np.testing.assert_allclose(g.w_root.cpu().numpy(), ref["est"]["w_root"], rtol=1e-9, atol=1e-13, err_msg=tag)
        np.testing.assert_allclose(g.w.cpu().numpy(), ref["est"]["w"], rtol=1e-9, atol=1e-13, err_msg=tag)
        np.testing.assert_allclose(g.root_m.cpu().numpy(), ref["root_m"], rtol=1e-9, atol=1e-12, err_msg=tag)
        nxt = ref["next"]
        np.testing.assert_allclose(g.root_mean.cpu().numpy(), nxt["root_mean"], rtol=1e-6, atol=1e-7, err_msg=tag)
        np.testing.assert_allclose(g.q_var.cpu().numpy(), nxt["q_var"], rtol=1e-6, err_msg=tag)
        state = nxt
