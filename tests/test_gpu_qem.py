"""Teacher-forced QEM trajectories on the GPU vs the oracle (R21).

For every iteration t of Algorithm 1 the GPU runs one
step -- sample (host eps) -> E-step -> EMA + M-step -- starting from the
ORACLE's state m_{t-1} and Q_t, and its outputs must meet the north-star
tolerances: log Pe 1e-5 relative, weights 1e-5 absolute, moments / EMA state /
M-step parameters 1e-4 relative.  This walks every regime of the run (one-hot
root weights early, spread weights at convergence), i.e. every forward tile
mode.  Free-running drift (GPU state fed back) is reported, not gated.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2503_08264_b200 import synth
from test_gpu_parity import check_estep

pytestmark = pytest.mark.gpu

CASES = {
    "c1_T20": (dict(cid=1), 20),
    "c2_T100": (dict(cid=2), 100),
    "c3_T30": (dict(cid=3), 30),
    "c4_n1000_T50": (dict(cid=4, n=1000), 50),
    "c5_n12_T10": (dict(cid=5, n=12), 10),
}


def _model(spec):
    spec = dict(spec)
    return synth.config(spec.pop("cid"), **spec)


def _rel(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / scale)) if np.size(a) else 0.0


@pytest.mark.parametrize("case", sorted(CASES))
def test_teacher_forced_trajectory(case):
    from paper_2503_08264_b200.qem import QEM
    spec, T = CASES[case]
    m = _model(spec)
    data = synth.make_data(m)
    seed = 100 + m.config_id
    ref_run = orc.run_qem(m, data, T, seed)
    g = QEM(m)
    g.set_data(data)
    state = orc.initial_state(m)
    q = [orc.mstep(a, b)[:2] for a, b in state]
    worst = dict(log_pe=0.0, w=0.0, m=0.0, q=0.0)
    for t in range(1, T + 1):
        ref = ref_run[t - 1]
        eps = orc.eps_for_iteration(m, t, seed)
        g.set_state([(a, b - a * a) for a, b in state])
        g.set_q(q)
        g.sample_q(eps=eps)
        g.estep()
        g.mstep(t)
        out = g.result()
        check_estep(m, out, ref["est"], note=f"{case} t={t}")
        est = ref["est"]
        worst["log_pe"] = max(worst["log_pe"], abs(out["log_pe"] - est["log_pe"]) / abs(est["log_pe"]))
        for lvl, ((m1r, m2r), (qm, qv)) in enumerate(zip(ref["state"], ref["q_next"])):
            vr = m2r - m1r * m1r
            sd = np.sqrt(np.maximum(vr, 0))
            e1 = _rel(out["ema_m1"][lvl], m1r, np.maximum(np.abs(m1r), sd))
            e2 = _rel(out["ema_v"][lvl] + out["ema_m1"][lvl] ** 2, m2r, np.abs(m2r))
            eq1 = _rel(out["q_mean"][lvl], qm, np.maximum(np.abs(qm), np.sqrt(qv)))
            eq2 = _rel(out["q_var"][lvl], qv, np.abs(qv))
            assert max(e1, e2) <= 1e-4, f"{case} t={t} level {lvl} EMA state rel err {max(e1, e2):.3g}"
            assert max(eq1, eq2) <= 1e-4, f"{case} t={t} level {lvl} M-step params rel err {max(eq1, eq2):.3g}"
            worst["m"] = max(worst["m"], e1, e2)
            worst["q"] = max(worst["q"], eq1, eq2)
        state, q = ref["state"], ref["q_next"]
    flags, _ = g.read_flags()
    assert flags & 2 == 0
    g.close()
    print(f"\n{case}: worst one-step errors {worst}")


@pytest.mark.parametrize("case", ["c1_T20", "c4_n1000_T50"])
def test_free_running_drift_reported(case):
    """GPU state fed back for T iterations with the same eps; drift vs the oracle's free run is
    reported (fp32 rounding is amplified ~10-50x per iteration), loosely bounded."""
    from paper_2503_08264_b200.qem import QEM
    spec, T = CASES[case]
    m = _model(spec)
    data = synth.make_data(m)
    seed = 100 + m.config_id
    ref_run = orc.run_qem(m, data, T, seed)
    g = QEM(m)
    g.set_data(data)
    state = orc.initial_state(m)
    g.set_state([(a, b - a * a) for a, b in state])
    g.set_q([orc.mstep(a, b)[:2] for a, b in state])
    drift = []
    for t in range(1, T + 1):
        g.sample_q(eps=orc.eps_for_iteration(m, t, seed))
        g.estep()
        g.mstep(t)
        out = g.result()
        m1r, m2r = ref_run[t - 1]["state"][0]
        sd = np.sqrt(np.maximum(m2r - m1r * m1r, 0))
        drift.append(_rel(out["ema_m1"][0], m1r, np.maximum(np.abs(m1r), sd)))
    g.close()
    print(f"\n{case}: free-running root-mean drift by iteration: " + " ".join(f"{d:.1e}" for d in drift))
    assert max(drift) < 0.05
