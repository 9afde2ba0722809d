"""GPU parity of the tcgen05 tensor-core pair kernels (K % 256 == 0) vs the oracle: the split layout
(d = 16, Bernoulli observations, config 5's shape) and the compact layout (d = 1, Gaussian
observations, config 4's shape).

The tensor-core path has its own operand layouts,
warp-specialised pipeline and per-group tile modes, so it gets its own sweep:
every forward tile mode (expm1 polynomial degrees 3..9 and the online
log-sum-exp), K = 256 / 512 / 1024 (one to four column blocks), and more
groups than SMs (several groups per persistent CTA, ragged last wave), with
the north-star tolerances of tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

from helpers import make_case, posterior_like_q
from oracle import oracle as orc
from paper_2503_08264_b200 import synth
from test_gpu_parity import check_estep

pytestmark = pytest.mark.gpu

# (groups, K, Q regime): shrink = multiple of the posterior width of posterior_like_q;
# "prior" = random Q (one-hot root weights, online mode)
CASES = {
    "n40_K256_post1": (40, 256, 1.0),
    "n300_K512_post3": (300, 512, 3.0),
    "n161_K256_post10": (161, 256, 10.0),
    "n150_K1024_post1": (150, 1024, 1.0),
    "n301_K256_prior": (301, 256, None),
    "n23_K768_post0.3": (23, 768, 0.3),
    # very narrow Q: |D'| small enough for the expm1-polynomial tile modes
    "n60_K256_post0.2": (60, 256, 0.2),
    "n60_K256_post0.12": (60, 256, 0.12),
    "n60_K256_post0.08": (60, 256, 0.08),
    "n60_K256_post0.05": (60, 256, 0.05),
    "n60_K512_post0.01": (60, 512, 0.01),
    "n60_K256_post0.002": (60, 256, 0.002),
    "n60_K256_post0.0004": (60, 256, 0.0004),
}

_seen_modes = {4: np.zeros(8, np.int64), 5: np.zeros(8, np.int64)}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("cid", [5], ids=["split_d16"])
def test_tc_estep_parity(cid, case):
    from paper_2503_08264_b200.qem import QEM
    n, K, shrink = CASES[case]
    m = synth.config(cid, n=n, K=K)
    data = synth.make_data(m)
    q = synth.random_q(m, 11) if shrink is None else posterior_like_q(m, data, seed=7, shrink=shrink)
    _, _, eps, _ = make_case(m, q=q)
    z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
    ref = orc.estep(m, z, q, data)
    g = QEM(m)
    assert g.pair_path() == 1, "d=16 with K%256==0 must run the tensor-core kernels"
    g.set_data(data)
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    out = g.result()
    hist = np.asarray(g.mode_hist(), np.int64)
    dg, c = g.messages()
    flags, _ = g.read_flags()
    g.close()
    _seen_modes[cid][:] += hist
    assert hist[:6].sum() == n, hist  # one mode per group
    check_estep(m, out, ref, note=f"tc/{case}")
    assert flags & 2 == 0
    if shrink is None or shrink > 3:
        # one-hot regime with the reference row far from the weight mass: |lnP|, |D'|, |h| reach
        # O(500) on the dominant row, resolved to fp32; only the contract quantities are gated
        return
    # plate messages g_i(k) = c_i + dg_i(k) against the oracle's, on the rows the root
    # softmax can see (w_root > 1e-6; far rows carry O(1000) log-factors resolved to fp32)
    rows = ref["w"][0].reshape(-1) > 1e-6
    g_ref = ref["g"][:, rows]
    full = (c.cpu().numpy()[:, None] + dg.cpu().numpy().astype(np.float64))[:, rows]
    err = np.abs(full - g_ref) / (5e-6 + 1e-6 * np.abs(g_ref))
    assert err.max() <= 1.0, (case, float(err.max()))


@pytest.mark.parametrize("cid", [5])
def test_tc_modes_covered(cid):
    """The sweep above must have exercised the online mode and the polynomial modes."""
    seen = _seen_modes[cid]
    if seen[:6].sum() == 0:
        pytest.skip("run with the parity sweep")
    assert seen[5] > 0, seen
    assert (seen[:5] > 0).sum() >= 1, seen


COMPACT_CASES = ["n40_K256_post1", "n301_K256_prior", "n161_K256_post10", "n60_K256_post0.05", "n150_K1024_post1"]


def test_compact_tc_path_d1_opt_in():
    """The compact tensor-core layout for d = 1 (config 4's shape; opt-in with QEM_TC1=1, read once per
    process, so in a fresh process): E-step parity with the oracle on one-hot, spread, converged and
    polynomial-mode cases, and both polynomial and online tile modes exercised."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    cases = {c: CASES[c] for c in COMPACT_CASES}
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from helpers import make_case, posterior_like_q\n"
        "from oracle import oracle as orc\n"
        "from paper_2503_08264_b200 import synth\n"
        "from paper_2503_08264_b200.qem import QEM\n"
        "from test_gpu_parity import check_estep\n"
        "seen = np.zeros(8, np.int64)\n"
        "for name, (n, K, shrink) in %r.items():\n"
        "    m = synth.config(4, n=n, K=K); data = synth.make_data(m)\n"
        "    q = synth.random_q(m, 11) if shrink is None else posterior_like_q(m, data, seed=7, shrink=shrink)\n"
        "    _, _, eps, z = make_case(m, q=q)\n"
        "    g = QEM(m); assert g.pair_path() == 1\n"
        "    g.set_data(data); g.set_q(q); g.sample_q(eps=eps); g.estep(); out = g.result()\n"
        "    seen += np.asarray(g.mode_hist()); g.close()\n"
        "    check_estep(m, out, orc.estep(m, z, q, data), note='compact ' + name)\n"
        "assert seen[5:7].sum() > 0 and seen[:5].sum() > 0, seen\n"
        "print('COMPACT_OK', seen)\n" % (os.path.dirname(here), here, cases))
    env = dict(os.environ, QEM_TC1="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=900)
    assert "COMPACT_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("n,K", [(37, 256), (9, 1024)])
def test_fused_sampler_is_bit_identical(n, K):
    """qem_sample_estep_forward draws the level-1 samples inside the column prep: the bound z, the
    messages, log Pe, weights and moments equal qem_sample_q + qem_estep_forward's bit for bit
    (same Philox counters, same transform), on a sharded block too (global counters)."""
    from paper_2503_08264_b200.qem import QEM, shard_range
    m = synth.config(5, n=n, K=K)
    data = synth.make_data(m)
    q = synth.random_q(m, 5)
    for b, e in ((0, n), shard_range(n, 1, 2)):
        outs = []
        for fused in (False, True):
            g = QEM(m, group_begin=b, group_end=e)
            g.set_data(data)
            g.set_q(q)
            if fused:
                g.sample_estep_forward(91, 4)
            else:
                g.sample_q(seed=91, iter=4)
                g.estep_forward()
            dg, c = [x.cpu().numpy() for x in g.messages()]
            ps = g.plate_sum.cpu().numpy()
            if (b, e) == (0, n):
                g.estep_backward()
            r = g.result()
            r["dg"], r["c"], r["ps"] = dg, c, ps
            outs.append(r)
            g.close()
        a, f = outs
        for l in range(2):
            np.testing.assert_array_equal(a["z"][l], f["z"][l])
        np.testing.assert_array_equal(a["dg"], f["dg"])
        np.testing.assert_array_equal(a["c"], f["c"])
        np.testing.assert_array_equal(a["ps"], f["ps"])
        if (b, e) == (0, n):
            assert a["log_pe"] == f["log_pe"]
            for l in range(2):
                np.testing.assert_array_equal(a["w"][l], f["w"][l])
                np.testing.assert_array_equal(a["m1"][l], f["m1"][l])


def _lazy_cases(m):
    return (("initial", synth.initial_q(m)), ("random11", synth.random_q(m, 11)), ("random3", synth.random_q(m, 3)))


@pytest.mark.parametrize("forced", [False, True], ids=["default", "all_redone"])
def test_tc_lazy_max_redo_parity(forced):
    """The forward's max-free pass past a row's first column block (R41)
    redoes a 64-column chunk with the exact row max when its running sum passes 1e30.  In the one-hot
    regime (Q = N(0,1) and random Q, K = 1024: four column blocks) both the max-free chunks and
    (QEM_FWD_REDO_THR=0, read once per process: every max-free chunk redone) the redo path must meet
    the north-star tolerances.  (How often the default threshold redoes: tools/lazy_count.py with a
    QEM_FWD_REDO_COUNT=1 build -- 0.6 % of chunks at t = 1 of config 5, none from t = 3.)"""
    import os
    import subprocess
    import sys
    if not forced:
        from paper_2503_08264_b200.qem import QEM
        m = synth.config(5, n=200, K=1024)
        data = synth.make_data(m)
        for name, q in _lazy_cases(m):
            _, _, eps, _ = make_case(m, q=q)
            z = [orc.sample(qm, qv, e) for (qm, qv), e in zip(q, eps)]
            g = QEM(m)
            g.set_data(data)
            g.set_q(q)
            g.sample_q(eps=eps)
            g.estep()
            out = g.result()
            g.close()
            check_estep(m, out, orc.estep(m, z, q, data), note=f"lazy/{name}")
        return
    here = os.path.dirname(os.path.abspath(__file__))
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import test_gpu_tc as T\n"
        "T.test_tc_lazy_max_redo_parity(False)\n"
        "print('REDO_OK')\n" % (os.path.dirname(here), here))
    env = dict(os.environ, QEM_FWD_REDO_THR="0")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=900)
    assert "REDO_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
