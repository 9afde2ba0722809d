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
    "c3_T100": (dict(cid=3), 100),
    "c4_n1000_T50": (dict(cid=4, n=1000), 50),
    "c5_n12_T10": (dict(cid=5, n=12), 10),
}


def _model(spec):
    spec = dict(spec)
    return synth.config(spec.pop("cid"), **spec)


def _rel(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / scale)) if np.size(a) else 0.0


def check_step(m, out, ref, note=""):
    """One teacher-forced iteration (gpu result() vs orc.qem_step): the E-step at the contract
    tolerances, then the EMA state m_t and the next Q (1e-4 relative).  Returns the worst errors."""
    check_estep(m, out, ref["est"], note=note)
    est = ref["est"]
    worst = dict(log_pe=abs(out["log_pe"] - est["log_pe"]) / abs(est["log_pe"]), w=0.0, m=0.0, q=0.0)
    for lvl, ((m1r, m2r), (qm, qv)) in enumerate(zip(ref["state"], ref["q_next"])):
        vr = m2r - m1r * m1r
        sd = np.sqrt(np.maximum(vr, 0))
        e1 = _rel(out["ema_m1"][lvl], m1r, np.maximum(np.abs(m1r), sd))
        e2 = _rel(out["ema_v"][lvl] + out["ema_m1"][lvl] ** 2, m2r, np.abs(m2r))
        eq1 = _rel(out["q_mean"][lvl], qm, np.maximum(np.abs(qm), np.sqrt(qv)))
        eq2 = _rel(out["q_var"][lvl], qv, np.abs(qv))
        assert max(e1, e2) <= 1e-4, f"{note} level {lvl} EMA state rel err {max(e1, e2):.3g}"
        assert max(eq1, eq2) <= 1e-4, f"{note} level {lvl} M-step params rel err {max(eq1, eq2):.3g}"
        worst["m"] = max(worst["m"], e1, e2)
        worst["q"] = max(worst["q"], eq1, eq2)
    return worst


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
        errs = check_step(m, out, ref, note=f"{case} t={t}")
        for k in worst:
            worst[k] = max(worst[k], errs[k])
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


def philox_eps(m, seed, t):
    """The oracle's own draw of the device sampler's Philox stream for iteration t (fp64 Box-Muller
    of the same counters, SURVEY.md §8(b) Determinism), rounded to fp32: one array per level."""
    out = []
    for lvl, (n, dd) in enumerate(synth.latent_shapes(m)):
        e = np.concatenate([orc.normal_eps(seed, t, lvl, i, dd, m.K) for i in range(n)], axis=0)
        out.append(e.astype(np.float32))
    return out


ITER_CASES = {
    "c1_T20": (dict(cid=1), 20),
    "c2_T20": (dict(cid=2), 20),
    "c3_T20": (dict(cid=3), 20),
    "c4_n500_T5": (dict(cid=4, n=500), 5),
    "c5_n8_T5": (dict(cid=5, n=8), 5),
}


@pytest.mark.parametrize("use_graph", [True, False], ids=["graph", "eager"])
@pytest.mark.parametrize("case", sorted(ITER_CASES))
def test_qem_iterate_teacher_forced(case, use_graph):
    """qem_iterate -- the library's own loop (sampler -> E-step -> EMA + M-step, captured in a CUDA
    graph or issued eagerly; Alg. 1) -- one iteration at a time from the oracle's
    state m_{t-1} and Q_t, on the SAME host eps as the oracle (the eps bank of qem_buffers): samples
    bit-exact, trace log Pe, weights, moments, EMA state and next Q at the contract tolerances."""
    from paper_2503_08264_b200.qem import QEM
    spec, T = ITER_CASES[case]
    m = _model(spec)
    data = synth.make_data(m)
    seed = 100 + m.config_id
    g = QEM(m, trace_len=1)
    g.set_data(data)
    state = orc.initial_state(m)
    q = [orc.mstep(a, b)[:2] for a, b in state]
    for t in range(1, T + 1):
        eps = orc.eps_for_iteration(m, t, seed)
        g.set_state([(a, b - a * a) for a, b in state])
        g.set_q(q)
        g.iterate(t, 1, seed=seed, use_graph=use_graph, eps_bank=[e[None] for e in eps])
        out = g.result()
        trace = float(g.trace[0].item())
        ref = orc.qem_step(m, state, q, eps, t, data=data)
        for lvl, zr in enumerate(ref["z"]):
            np.testing.assert_array_equal(out["z"][lvl].reshape(zr.shape), zr)
        assert trace == out["log_pe"]
        check_step(m, out, ref, note=f"{case} t={t} {'graph' if use_graph else 'eager'}")
        state, q = ref["state"], ref["q_next"]
    assert g.read_flags()[0] & 2 == 0
    g.close()


def test_qem_iterate_eps_bank_multi_iteration():
    """One qem_iterate call over T iterations with a T-slice eps bank == T single-iteration calls
    (the device iteration counter selects the slice), graph and eager bit-identical."""
    from paper_2503_08264_b200.qem import QEM
    m = synth.config(2, n=40)
    data = synth.make_data(m)
    T, seed = 6, 102
    eps = [orc.eps_for_iteration(m, t, seed) for t in range(1, T + 1)]
    bank = [np.stack([e[l] for e in eps]) for l in range(2)]
    outs = []
    for mode in ("graph_T", "eager_T", "graph_1"):
        g = QEM(m, trace_len=T)
        g.set_data(data)
        g.set_q(synth.initial_q(m))
        if mode == "graph_1":
            for t in range(1, T + 1):
                g.iterate(t, 1, seed=seed, use_graph=True, eps_bank=[b[t - 1:t] for b in bank])
        else:
            g.iterate(1, T, seed=seed, use_graph=mode == "graph_T", eps_bank=bank)
        outs.append(g.result())
        g.close()
    for o in outs[1:]:
        for l in range(2):
            np.testing.assert_array_equal(o["q_mean"][l], outs[0]["q_mean"][l])
            np.testing.assert_array_equal(o["w"][l], outs[0]["w"][l])


PHILOX_CASES = {"c1_T20": (dict(cid=1), 20), "c4_n500_T5": (dict(cid=4, n=500), 5), "c5_n8_T5": (dict(cid=5, n=8), 5)}


@pytest.mark.parametrize("case", sorted(PHILOX_CASES))
def test_qem_iterate_philox_stream(case):
    """qem_iterate with its device Philox sampler (the bench's mode): the oracle draws the same Philox
    counters itself (fp64 Box-Muller), the device's fp32 transform is within 2e-6 of it (DESIGN.md
    R27) plus fp32 rounding of z, and on these shapes the step still meets the contract tolerances
    (the samples differ by that rounding, so the comparison is not on identical samples)."""
    from paper_2503_08264_b200.qem import QEM
    spec, T = PHILOX_CASES[case]
    m = _model(spec)
    data = synth.make_data(m)
    seed = 0x5EED0000 + m.config_id
    g = QEM(m, trace_len=1)
    g.set_data(data)
    state = orc.initial_state(m)
    q = [orc.mstep(a, b)[:2] for a, b in state]
    for t in range(1, T + 1):
        g.set_state([(a, b - a * a) for a, b in state])
        g.set_q(q)
        g.iterate(t, 1, seed=seed, use_graph=True)
        out = g.result()
        eps = philox_eps(m, seed, t)
        ref = orc.qem_step(m, state, q, eps, t, data=data)
        for lvl, zr in enumerate(ref["z"]):
            zg = out["z"][lvl].reshape(zr.shape).astype(np.float64)
            sd = np.sqrt(np.asarray(q[lvl][1], np.float64))[:, None]
            tol = 2e-6 * sd + 2.0 * np.spacing(np.abs(zr).astype(np.float32)).astype(np.float64)  # + fp32 rounding of z
            assert np.all(np.abs(zg - zr) <= tol), f"{case} t={t} level {lvl} samples"
        assert float(g.trace[0].item()) == out["log_pe"]
        check_step(m, out, ref, note=f"{case} t={t} philox")
        state, q = ref["state"], ref["q_next"]
    g.close()
