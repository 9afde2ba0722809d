"""Numerical conditions reach the device flags, never a crash or a host exception (SURVEY.md
§8(b): degenerate evidence SPEC.md:317, NaN, variance clamps SPEC.md:436; include/qem.h
QEM_FLAG_*), on both pair paths (FFMA: config 4 shape; tensor cores: config 5 shape)."""
import numpy as np
import pytest

from helpers import make_case
from paper_2503_08264_b200 import synth

pytestmark = pytest.mark.gpu

DEGENERATE, NAN, CLAMP = 1, 2, 4


def _run(m, data, q, eps, **kw):
    from paper_2503_08264_b200.qem import QEM
    g = QEM(m, **kw)
    g.set_data(data)
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    g.mstep(1)
    out = g.result()
    flags, clamps = g.read_flags()
    g.close()
    return out, flags, clamps


@pytest.mark.parametrize("spec", [dict(cid=4, n=50, K=64), dict(cid=5, n=20, K=256)])
def test_clean_run_raises_no_flag(spec):
    m = synth.config(**spec)
    data, q, eps, z = make_case(m)
    out, flags, clamps = _run(m, data, q, eps)
    assert flags == 0 and clamps == 0 and np.isfinite(out["log_pe"])


def test_nan_observation_sets_the_nan_flag():
    m = synth.config(4, n=50, K=64)
    data, q, eps, z = make_case(m)
    data.xg = data.xg.copy()
    data.xg[7, 3] = np.nan
    out, flags, _ = _run(m, data, q, eps)
    assert flags & NAN, flags


@pytest.mark.parametrize("spec", [dict(cid=4, n=50, K=64), dict(cid=5, n=20, K=256)])
def test_nan_in_q_sets_the_nan_flag(spec):
    m = synth.config(**spec)
    data, q, eps, z = make_case(m)
    qm = q[1][0].copy()
    qm[3] = np.nan
    q = [q[0], (qm, q[1][1])]
    out, flags, _ = _run(m, data, q, eps)
    assert flags & NAN, flags


def test_impossible_observation_is_degenerate_evidence():
    """x = +inf: every sample's likelihood is 0, log Pe = -inf -> QEM_FLAG_DEGENERATE (as data)."""
    m = synth.config(4, n=50, K=64)
    data, q, eps, z = make_case(m)
    data.xg = data.xg.copy()
    data.xg[11, 0] = np.inf
    out, flags, _ = _run(m, data, q, eps)
    assert flags & DEGENERATE, flags
    assert not (out["log_pe"] > -np.inf)


@pytest.mark.parametrize("spec", [dict(cid=4, n=50, K=64), dict(cid=5, n=20, K=256)])
def test_variance_floor_clamps_are_counted(spec):
    m = synth.config(**spec)
    data, q, eps, z = make_case(m)
    out, flags, clamps = _run(m, data, q, eps, var_floor=100.0)
    n_latent = m.R + m.n * m.d
    assert flags & CLAMP and clamps == n_latent, (flags, clamps, n_latent)
    assert all(np.all(v == np.float32(100.0)) for v in out["q_var"])
