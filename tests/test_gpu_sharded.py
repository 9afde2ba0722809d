"""The library's group-sharded path on one GPU.

Rank r of R owns groups qem_shard_range(n, r, R).  On one GPU the ranks are
*virtual*: R contexts over the shard blocks, their local plate sums
[G_r(0..K-1), sum_i c_i] added on the device in rank order (what the SUM
all-reduce computes), then every context runs the root + backward phase.  No
kernel waits on another rank's kernel, so this is the sharded data path without
standing in for an interconnect.  Checked:

* the Philox sampler keys every group's samples by its GLOBAL index: each shard's
  samples equal the single context's slice bit for bit;
* every group's forward message (Delta g_i, c_i) is bit-identical to the single
  context's (a group's message depends on its own data and the replicated root only);
* weights, moments and log Pe equal the single context's up to the fp64 order of the
  plate sum, and meet the oracle (Eq. 7a-c) at the contract tolerances;
* the in-library NCCL path: a 1-rank communicator (the only one one GPU admits) leaves the
  E-step and the captured qem_iterate loop bit-identical; the argument checks of the
  communicator / sharded entry points.
The multi-process variant (2 processes on the one GPU, plate sums over gloo) runs the
same phase API across real process boundaries.
"""
import os
import socket

import numpy as np
import pytest

from helpers import make_case, posterior_like_q
from oracle import oracle as orc
from paper_2503_08264_b200 import synth
from test_gpu_parity import check_estep

pytestmark = pytest.mark.gpu

SHAPES = {
    "tc_d16_K256": dict(cid=5, n=37, K=256),          # tcgen05 pair tiles
    "ffma_d1_K256": dict(cid=4, n=301, K=256),        # FFMA tiles, scalar latents (config 4's shape)
    "ffma_d18_K30": dict(cid=2, n=50),                # FFMA tiles, config 2's shape
}


def _model(spec):
    spec = dict(spec)
    return synth.config(spec.pop("cid"), **spec)


def _single(m, data, q, eps):
    from paper_2503_08264_b200.qem import QEM
    g = QEM(m)
    g.set_data(data)
    g.set_q(q)
    g.sample_q(eps=eps)
    g.estep()
    out = g.result()
    out["dg"], out["c"] = [t.cpu().numpy() for t in g.messages()]
    out["plate_sum"] = g.plate_sum.cpu().numpy()
    g.close()
    return out


def _virtual_ranks(m, data, q, eps, R):
    """R contexts over the shard blocks; device-side SUM of their plate sums between the phases."""
    import torch
    from paper_2503_08264_b200.qem import QEM, shard_range
    ctxs = []
    for r in range(R):
        b, e = shard_range(m.n, r, R)
        g = QEM(m, group_begin=b, group_end=e)
        g.set_data(data)
        g.set_q(q)
        g.sample_q(eps=eps)
        ctxs.append(g)
    for g in ctxs:
        g.estep_forward()
    total = torch.zeros_like(ctxs[0].plate_sum)
    for g in ctxs:  # rank order, like a deterministic all-reduce
        total += g.plate_sum
    outs = []
    for g in ctxs:
        g.plate_sum.copy_(total)
        g.estep_backward()
        o = g.result()
        o["dg"], o["c"] = [t.cpu().numpy() for t in g.messages()]
        outs.append(o)
        g.close()
    return outs, total.cpu().numpy()


def _concat(m, outs):
    """Stitch the shards' level-1 outputs back into global order."""
    res = dict(log_pe=outs[0]["log_pe"])
    for key in ("w", "m1", "v"):
        res[key] = [outs[0][key][0], np.concatenate([o[key][1] for o in outs], axis=0)]
    res["dg"] = np.concatenate([o["dg"] for o in outs], axis=0)
    res["c"] = np.concatenate([o["c"] for o in outs])
    return res


@pytest.mark.parametrize("R", [2, 3])
@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_virtual_ranks_match_single_context_and_oracle(shape, R):
    m = _model(SHAPES[shape])
    data = synth.make_data(m)
    # the converged regime (posterior-width Q): at 3x the width the d = 16 case sits at the edge of the
    # moment tolerance in the single context too (fp32 plate messages), which is not what this tests
    q = posterior_like_q(m, data, seed=4, shrink=1.0)
    _, _, eps, z = make_case(m, q=q)
    one = _single(m, data, q, eps)
    outs, total = _virtual_ranks(m, data, q, eps, R)
    sh = _concat(m, outs)
    # every rank holds the same root weights and log Pe (redundant root pass on identical bytes)
    for o in outs[1:]:
        np.testing.assert_array_equal(o["w"][0], outs[0]["w"][0])
        assert o["log_pe"] == outs[0]["log_pe"]
    # per-group forward messages: bit-identical to the single context
    np.testing.assert_array_equal(sh["dg"], one["dg"])
    np.testing.assert_array_equal(sh["c"], one["c"])
    # the reduced plate sum = the single context's up to the fp64 summation order
    np.testing.assert_allclose(total, one["plate_sum"], rtol=1e-12, atol=1e-9)
    # outputs: the single context's up to that order ...
    assert abs(sh["log_pe"] - one["log_pe"]) <= 1e-12 * abs(one["log_pe"])
    for l in range(2):
        np.testing.assert_allclose(sh["w"][l].reshape(one["w"][l].shape), one["w"][l], rtol=0, atol=1e-7)
        np.testing.assert_allclose(sh["m1"][l], one["m1"][l], rtol=1e-6, atol=1e-9)
        np.testing.assert_allclose(sh["v"][l], one["v"][l], rtol=1e-5, atol=1e-12)
    # ... and the oracle's at the contract tolerances
    check_estep(m, sh, orc.estep(m, z, q, data), note=f"{shape} R={R}")


@pytest.mark.parametrize("shape", ["tc_d16_K256", "ffma_d1_K256"])
def test_sharded_philox_samples_use_global_indices(shape):
    """Philox mode: a shard's samples are the single context's slice, bit for bit (counter keyed by
    the GLOBAL group index, SURVEY.md §8(b) Determinism)."""
    from paper_2503_08264_b200.qem import QEM, shard_range
    m = _model(SHAPES[shape])
    data = synth.make_data(m)
    q = synth.random_q(m, 5)
    full = QEM(m)
    full.set_data(data)
    full.set_q(q)
    full.sample_q(seed=77, iter=3)
    zf = full.result()["z"]
    full.close()
    for R in (2, 3):
        for r in range(R):
            b, e = shard_range(m.n, r, R)
            g = QEM(m, group_begin=b, group_end=e)
            g.set_data(data)
            g.set_q(q)
            g.sample_q(seed=77, iter=3)
            z = g.result()["z"]
            np.testing.assert_array_equal(z[0], zf[0])
            np.testing.assert_array_equal(z[1], zf[1][b:e])
            g.close()


def test_sharded_entry_points_need_a_communicator():
    from paper_2503_08264_b200 import _lib
    from paper_2503_08264_b200.qem import QEM, shard_range
    m = _model(SHAPES["ffma_d1_K256"])
    data = synth.make_data(m)
    b, e = shard_range(m.n, 1, 2)
    g = QEM(m, group_begin=b, group_end=e)
    g.set_data(data)
    g.set_q(synth.initial_q(m))
    g.sample_q(seed=1, iter=1)
    for call in (g.estep, g.estep_reduce, lambda: g.iterate(1, 1, seed=1)):
        with pytest.raises(_lib.QemError, match="QEM_UNSUPPORTED"):
            call()
    # a 1-rank communicator owns all groups, not this block
    with pytest.raises(_lib.QemError, match="QEM_INVALID_ARGUMENT"):
        g.nccl_init()
    g.close()


def test_nccl_single_rank_is_identity():
    """The in-library all-reduce on a 1-rank communicator: qem_estep and the CUDA-graph loop (which
    captures ncclAllReduce) give bit-identical results to the context without one."""
    from paper_2503_08264_b200.qem import QEM
    m = synth.config(5, n=40, K=256)
    data = synth.make_data(m)
    res = []
    for comm in (False, True):
        g = QEM(m)
        g.set_data(data)
        g.set_q(synth.initial_q(m))
        if comm:
            g.nccl_init()
            rank, world, ver = g.nccl_info()
            assert (rank, world) == (0, 1) and ver >= 22000
        g.sample_q(seed=9, iter=1)
        g.estep()
        a = g.result()
        g.iterate(2, 3, seed=9, use_graph=True)
        b = g.result()
        g.iterate(5, 2, seed=9, use_graph=False)
        c = g.result()
        res.append((a, b, c))
        g.close()
    for x, y in zip(res[0], res[1]):
        assert x["log_pe"] == y["log_pe"]
        for l in range(2):
            for key in ("w", "m1", "v", "q_mean", "q_var"):
                np.testing.assert_array_equal(x[key][l], y[key][l])


# ------------------------------------------------- two processes, one GPU, gloo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, spec, T, out_q):
    import sys
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_08264_b200 import dist as qdist
        from paper_2503_08264_b200.qem import QEM, shard_range
        m = _model(spec)
        data = synth.make_data(m)
        b, e = shard_range(m.n, rank, world)
        g = QEM(m, group_begin=b, group_end=e, device="cuda:0")
        g.set_data(data)
        g.set_q(synth.initial_q(m))
        runner = qdist.ShardedQEM(g)
        for t in range(1, T + 1):
            runner.step(t, seed=21)
        out = g.result()
        same = qdist.check_root_replicated(g.levels[0]["w"])
        out_q.put((rank, b, e, out["log_pe"], out["q_mean"], out["q_var"], out["w"][0], same))
        g.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_gloo_match_single_context():
    """2 processes on the one GPU, each a libqem context over its shard, the plate sums all-reduced
    over gloo between the library's phases (dist.ShardedQEM): T = 3 QEM iterations with device
    Philox samples equal the single-process run up to fp64 summation order."""
    import torch.multiprocessing as mp
    from paper_2503_08264_b200.qem import QEM
    spec, T, world = SHAPES["tc_d16_K256"], 3, 2
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, spec, T, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q_out.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = _model(spec)
    g = QEM(m)
    g.set_data(synth.make_data(m))
    g.set_q(synth.initial_q(m))
    for t in range(1, T + 1):
        g.sample_q(seed=21, iter=t)
        g.estep()
        g.mstep(t)
    one = g.result()
    g.close()
    assert all(r[7] for r in res)  # bit-identical root weights on both ranks
    for rank, b, e, lp, qm, qv, w_root, _ in res:
        assert abs(lp - one["log_pe"]) <= 1e-9 * abs(one["log_pe"])
        np.testing.assert_allclose(w_root, one["w"][0], atol=1e-6)
        np.testing.assert_allclose(qm[0], one["q_mean"][0], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(qm[1], one["q_mean"][1][b * m.d:e * m.d], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(qv[1], one["q_var"][1][b * m.d:e * m.d], rtol=1e-4, atol=1e-9)
