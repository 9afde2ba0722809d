"""E-step on explicit log-factor tables (qem_estep_tables; SURVEY.md §8(b) "from factors"):
the oracle's elimination pinned against literal enumeration and closed-form special cases (CPU),
then the device path against the oracle (GPU)."""
import numpy as np
import pytest
from scipy.special import logsumexp

from oracle import tables


def _rand(n, K, seed, scale=3.0):
    rng = np.random.default_rng(seed)
    return rng.normal(0, scale, K), rng.normal(0, scale, (n, K, K))


# ------------------------------------------------------------------ oracle pins (CPU)


@pytest.mark.parametrize("n,K", [(0, 3), (1, 5), (3, 4), (4, 3)])
def test_elimination_equals_enumeration(n, K):
    fr, f = _rand(n, K, 10 * n + K)
    a, b = tables.estep_tables(fr, f), tables.estep_tables_brute(fr, f)
    assert abs(a["log_pe"] - b["log_pe"]) < 1e-12
    np.testing.assert_allclose(a["w_root"], b["w_root"], atol=1e-13)
    np.testing.assert_allclose(a["w"], b["w"], atol=1e-13)


def test_zero_coupling_factorises():
    """f_i(k, k') = h_i(k') (the child ignores the root sample): the evidence estimate is the product
    of independent single-latent importance-sampling estimates."""
    rng = np.random.default_rng(1)
    K, n = 7, 5
    fr, h = rng.normal(0, 2, K), rng.normal(0, 2, (n, K))
    f = np.broadcast_to(h[:, None, :], (n, K, K))
    r = tables.estep_tables(fr, f)
    want = logsumexp(fr) - np.log(K) + sum(logsumexp(h[i]) - np.log(K) for i in range(n))
    assert abs(r["log_pe"] - want) < 1e-12
    np.testing.assert_allclose(r["w"], np.exp(h - logsumexp(h, axis=1, keepdims=True)), atol=1e-14)
    np.testing.assert_allclose(r["w_root"], np.exp(fr - logsumexp(fr)), atol=1e-14)


def test_single_sample():
    """K = 1: log Pe = log p(x, z) - log q(z) of the one tuple, every weight 1."""
    fr, f = _rand(6, 1, 2)
    r = tables.estep_tables(fr, f)
    assert abs(r["log_pe"] - (fr[0] + f[:, 0, 0].sum())) < 1e-12
    assert np.all(r["w"] == 1.0) and r["w_root"][0] == 1.0


def test_dead_root_sample_carries_no_weight():
    fr, f = _rand(3, 4, 3)
    fr[2] = -np.inf
    f[1, 1, :] = -np.inf  # root sample 1 kills instance 1's row
    a, b = tables.estep_tables(fr, f), tables.estep_tables_brute(fr, f)
    assert a["w_root"][1] == 0 and a["w_root"][2] == 0
    assert abs(a["log_pe"] - b["log_pe"]) < 1e-12
    np.testing.assert_allclose(a["w"], b["w"], atol=1e-13)
    np.testing.assert_allclose(a["w"].sum(axis=1), 1.0, atol=1e-14)


# ------------------------------------------------------------------ device path (GPU)


def _gpu(fr, f):
    import torch
    from paper_2503_08264_b200.qem import estep_tables
    dev = torch.device("cuda")
    out = estep_tables(torch.from_numpy(np.asarray(fr, np.float64)).to(dev),
                       torch.from_numpy(np.asarray(f, np.float64)).to(dev))
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("n,K,scale", [(37, 300, 3.0), (5, 1, 1.0), (0, 17, 2.0), (200, 33, 30.0), (3, 1024, 5.0),
                                       (1, 8192, 2.0)])
def test_device_tables_match_oracle(n, K, scale):
    fr, f = _rand(n, K, n + K, scale)
    ref = tables.estep_tables(fr, f)
    out = _gpu(fr, f)
    assert abs(out["log_pe"][0] - ref["log_pe"]) <= 1e-12 * max(1.0, abs(ref["log_pe"]))
    np.testing.assert_allclose(out["w_root"], ref["w_root"], rtol=1e-11, atol=1e-15)
    if n:
        np.testing.assert_allclose(out["g"], ref["g"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(out["w"], ref["w"], rtol=1e-11, atol=1e-15)
        np.testing.assert_allclose(out["w"].sum(axis=1), 1.0, atol=1e-12)


@pytest.mark.gpu
def test_device_tables_degenerate_and_dead_rows():
    fr, f = _rand(4, 64, 9)
    fr[5] = -np.inf
    f[2, 7, :] = -np.inf
    ref, out = tables.estep_tables(fr, f), _gpu(fr, f)
    assert out["w_root"][5] == 0 and out["w_root"][7] == 0
    np.testing.assert_allclose(out["w"], ref["w"], rtol=1e-11, atol=1e-15)
    # every root sample at -inf: degenerate evidence, reported as data
    out = _gpu(np.full(64, -np.inf), f)
    assert out["log_pe"][0] == -np.inf and np.all(np.isnan(out["w_root"]))


@pytest.mark.gpu
def test_device_tables_reject_bad_arguments():
    import torch
    from paper_2503_08264_b200 import _lib
    from paper_2503_08264_b200.qem import estep_tables
    dev = torch.device("cuda")
    with pytest.raises(_lib.QemError):
        estep_tables(torch.zeros(8193, dtype=torch.float64, device=dev), torch.zeros(0, dtype=torch.float64, device=dev))
