"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Tolerances (BASELINE.json north_star): log-marginal 1e-5 relative; per-sample
weights 1e-5 absolute; moments and M-step parameters 1e-4 relative (scale
max(|ref|, sd_ref) for means, R19).  Sample indexing and plate
bookkeeping are bit-exact (samples from host eps are compared with ==).
"""
import numpy as np
import pytest

from helpers import make_case, posterior_like_q
from oracle import oracle as orc
from paper_2503_08264_b200 import synth

pytestmark = pytest.mark.gpu

LOGPE_RTOL = 1e-5
W_ATOL = 1e-5
MOM_RTOL = 1e-4


def _qem(m, **kw):
    import torch
    from paper_2503_08264_b200.qem import QEM
    assert torch.cuda.is_available()
    return QEM(m, **kw)


def check_estep(m, gpu, ref, note=""):
    """Compare one E-step result dict (gpu.result()) with the oracle's."""
    lp, lr = gpu["log_pe"], ref["log_pe"]
    assert abs(lp - lr) <= LOGPE_RTOL * abs(lr), f"{note} log_pe {lp} vs {lr}"
    nlev = len(ref["w"])
    for l in range(nlev):
        wg = gpu["w"][l].reshape(ref["w"][l].shape)
        err = np.abs(wg - ref["w"][l]).max()
        assert err <= W_ATOL, f"{note} level {l} weights max err {err:.3g}"
        m1r, m2r = ref["m1"][l], ref["m2"][l]
        vr = m2r - m1r ** 2
        sd = np.sqrt(np.maximum(vr, 0))
        m1g, vg = gpu["m1"][l], gpu["v"][l]
        e1 = np.abs(m1g - m1r) / np.maximum(np.abs(m1r), sd)
        assert e1.max() <= MOM_RTOL, f"{note} level {l} m1 rel err {e1.max():.3g}"
        # second mean parameter E z^2 (R19: moments are the mean parameters (E z, E z^2))
        m2g = vg + m1g ** 2
        e2 = np.abs(m2g - m2r) / np.maximum(np.abs(m2r), 1e-300)
        assert e2.max() <= MOM_RTOL, f"{note} level {l} E z^2 rel err {e2.max():.3g}"


def run_case(m, data, q, eps, z, use_sampler=True):
    g = _qem(m)
    g.set_data(data)
    g.set_q(q)
    if use_sampler:
        g.sample_q(eps=eps)
    else:
        g.set_z(z)
    g.estep()
    out = g.result()
    flags, _ = g.read_flags()
    g.close()
    return out, flags


CASES = {
    "c1": dict(cid=1),
    "c2": dict(cid=2),
    "c3": dict(cid=3),
    "c4_n2000": dict(cid=4, n=2000),
    "c5_n24": dict(cid=5, n=24),
    "ragged_d3_K200": dict(cid=5, n=37, K=200, d=3, J=7),
    "ragged_d1_K77": dict(cid=4, n=53, K=77),
    "K1": dict(cid=4, n=9, K=1),
    "n1_K33": dict(cid=2, n=1, K=33, d=4),
    "d8_K512": dict(cid=5, n=11, K=512, d=8),
    # maximum K (QEM_MAX_K) on the FFMA tiles: d = 18 (config 2's dimension) and d = 3, ragged n
    "maxK_d18": dict(cid=2, n=29, K=1024),
    "maxK_d3_ragged": dict(cid=5, n=151, K=1024, d=3, J=9),
    # the rest of the compiled d menu (QEM_D_MENU): FFMA tiles at d = 5, 20, 32, tensor cores at d = 12
    "d5_K96": dict(cid=5, n=13, K=96, d=5, J=6),
    "d12_tc_K256": dict(cid=5, n=17, K=256, d=12, J=9),
    "d20_K64": dict(cid=2, n=7, K=64, d=20),
    "d32_K40": dict(cid=5, n=5, K=40, d=32, J=4),
}


def _model(spec):
    spec = dict(spec)
    return synth.config(spec.pop("cid"), **spec)


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("regime", ["prior_q", "posterior_q"])
def test_estep_parity(case, regime):
    m = _model(CASES[case])
    data = synth.make_data(m)
    if regime == "prior_q":
        q = synth.random_q(m, 11)
    else:
        q = posterior_like_q(m, data, seed=5)
    _, _, eps, _ = make_case(m, q=q)
    z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
    ref = orc.estep(m, z, q, data)
    gpu, flags = run_case(m, data, q, eps, z)
    # samples: bit-exact (same fp32 fmaf definition on both sides)
    for l, zz in enumerate(z):
        np.testing.assert_array_equal(gpu["z"][l].reshape(zz.shape), zz)
    check_estep(m, gpu, ref, note=f"{case}/{regime}")
    assert flags & 2 == 0


def test_weights_normalised_and_deterministic():
    m = synth.config(4, n=300, K=256)
    data = synth.make_data(m)
    q = posterior_like_q(m, data)
    _, _, eps, z = make_case(m, q=q)
    a, _ = run_case(m, data, q, eps, z)
    b, _ = run_case(m, data, q, eps, z)
    for l in range(2):
        np.testing.assert_allclose(a["w"][l].sum(axis=-1), 1.0, atol=2e-5)
        np.testing.assert_array_equal(a["w"][l], b["w"][l])
    assert a["log_pe"] == b["log_pe"]


def test_sampler_philox_matches_oracle_stream():
    """Philox mode: device eps (fp32 Box-Muller) vs the oracle's fp64 stream; integer part exact."""
    m = synth.config(5, n=6, K=64, d=3)
    g = _qem(m, group_begin=2, group_end=5)
    data = synth.make_data(m)
    g.set_data(data)
    q = synth.random_q(m, 3)
    g.set_q(q)
    g.sample_q(seed=0x1234567890ABCDEF, iter=7)
    out = g.result()
    qr, qg = q[0], q[1]
    # root
    eps = orc.normal_eps(0x1234567890ABCDEF, 7, 0, 0, m.R, m.K)
    zr = qr[0][:, None].astype(np.float64) + np.sqrt(qr[1].astype(np.float64))[:, None] * eps
    np.testing.assert_allclose(out["z"][0].reshape(m.R, m.K), zr, rtol=2e-6, atol=2e-6)
    for li, gi in enumerate(range(2, 5)):
        eps = orc.normal_eps(0x1234567890ABCDEF, 7, 1, gi, m.d, m.K)
        sl = slice(gi * m.d, (gi + 1) * m.d)
        zg = qg[0][sl, None].astype(np.float64) + np.sqrt(qg[1][sl].astype(np.float64))[:, None] * eps
        np.testing.assert_allclose(out["z"][1][li], zg, rtol=2e-6, atol=2e-6)
    g.close()


def test_mstep_parity():
    """EMA over mean parameters + Gaussian M-step vs the oracle (which EMAs (E z, E z^2))."""
    m = synth.config(2, n=50, K=8, d=4)
    g = _qem(m, new_weight=0.3)
    data = synth.make_data(m)
    g.set_data(data)
    rng = np.random.default_rng(0)
    shapes = synth.latent_shapes(m)
    m1 = [rng.standard_normal(n * d) for n, d in shapes]
    v = [np.exp(rng.standard_normal(n * d)) for n, d in shapes]
    m1n = [rng.standard_normal(n * d) for n, d in shapes]
    vn = [np.exp(rng.standard_normal(n * d)) * 1e-3 for n, d in shapes]
    vn[0][0] = 0.0
    v[0][0] = 0.0   # with equal means this forces a floor clamp
    m1n[0][0] = m1[0][0]
    g.set_state(list(zip(m1, v)))
    import torch
    for l, lv in enumerate(g.levels):
        lv["m1"].copy_(torch.as_tensor(m1n[l]))
        lv["v"].copy_(torch.as_tensor(vn[l]))
    g.mstep(3)
    out = g.result()
    flags, clamps = g.read_flags()
    lam = orc.lam(3, 0.3)
    for l in range(2):
        a, b = orc.ema(lam, m1[l], v[l] + m1[l] ** 2, m1n[l], vn[l] + m1n[l] ** 2)
        qm, qv, c = orc.mstep(a, b)
        np.testing.assert_allclose(out["ema_m1"][l], a, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(out["ema_v"][l], b - a ** 2, rtol=1e-9, atol=1e-12)
        np.testing.assert_array_equal(out["q_mean"][l], qm)
        np.testing.assert_allclose(out["q_var"][l], qv, rtol=2e-7)
    assert clamps >= 1 and (flags & 4)
    g.close()


def test_d_menu_validation():
    """d outside the compiled menu (QEM_D_MENU) is a model error, with the menu in the message; a
    K / d combination whose shared memory exceeds the device limit is rejected at creation."""
    from paper_2503_08264_b200 import _lib
    from paper_2503_08264_b200.qem import QEM, model_validate
    assert model_validate(synth.config(5, n=4, K=64, d=11)) and "QEM_D_MENU" in model_validate(synth.config(5, n=4, K=64, d=11))
    for d in (1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 18, 20, 24, 32):
        assert model_validate(synth.config(5 if d > 1 else 4, n=4, K=64, d=d)) is None, d
    with pytest.raises(_lib.QemError, match="shared memory"):
        QEM(synth.config(5, n=4, K=1024, d=32, J=5))
