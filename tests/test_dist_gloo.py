"""Multi-rank (world_size 2, gloo, CPU) test of the group-sharded orchestration.

paper_2503_08264_b200.dist.ShardedQEM drives one QEM E-step across ranks:
local forward -> SUM all-reduce of the (K+1) fp64 plate sums -> redundant root
softmax on every rank -> local backward.  Here the per-rank compute backend is
the CPU oracle restricted to the rank's shard (no GPU on this box); the test
checks that the sharded result equals the single-process oracle E-step, that
the shards tile the groups exactly, and that every rank ends with bit-identical
root weights.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from scipy.special import logsumexp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShardBackend:
    """The QEM phase API on one shard, computed by the oracle (test stand-in for libqem)."""

    def __init__(self, m, data, q, z, begin, end):
        from paper_2503_08264_b200 import synth
        self.m_full = m
        self.m = synth.config(m.config_id, n=end - begin, K=m.K, J=m.J, d=m.d)
        d = m.d
        self.z = [z[0], z[1][begin * d:end * d]]
        self.q = [q[0], (q[1][0][begin * d:end * d], q[1][1][begin * d:end * d])]
        if data.xg is not None:
            self.data = synth.Data(xg=data.xg[begin:end])
        else:
            self.data = synth.Data(xb=data.xb[begin:end], yb=data.yb[begin:end])
        self.plate_sum = torch.zeros(m.K + 1, dtype=torch.float64)
        self.begin, self.end = begin, end

    def sample_q(self, seed=0, iter=1, eps=None):
        pass  # samples are given (host eps path)

    def estep_forward(self):
        from oracle import oracle as orc
        self.f_root, self.g = orc.forward2(self.m, self.z, self.q, self.data)
        self.plate_sum[: self.m.K] = torch.from_numpy(self.g.sum(axis=0))
        self.plate_sum[self.m.K] = 0.0

    def estep_backward(self):
        from oracle import oracle as orc
        a = self.f_root + self.plate_sum[: self.m.K].numpy()
        L = logsumexp(a)
        self.log_pe = L - np.log(self.m.K)
        self.w_root = torch.from_numpy(np.exp(a - L))
        self.w, self.m1, self.m2 = orc.backward2(self.m, self.z, self.q, self.data, self.w_root.numpy(), self.g)

    def evidence_root(self):
        a = self.f_root + self.plate_sum[: self.m.K].numpy()
        self.log_pe_fresh = logsumexp(a) - np.log(self.m.K)

    def mstep(self, t):
        pass

    def backward_resample(self, S, seed):
        from oracle import predict as op
        est = dict(w=[self.w_root.numpy()[None, :]], g=self.g)
        r = op.resample(self.m, self.z, self.q, self.data, est, S, seed, g_begin=self.begin)
        return torch.from_numpy(r["idx_root"]), torch.from_numpy(r["idx"])

    def predictive_loglik(self, idx, test):
        from oracle import predict as op
        part = op.test_loglik(self.m, self.z, self._test_shard(test), idx.numpy())
        return None, torch.from_numpy(part.sum(axis=1)), torch.from_numpy(part)

    def _test_shard(self, test):
        from paper_2503_08264_b200 import synth
        b, e = self.begin, self.end
        if test.xg is not None:
            return synth.Data(xg=test.xg[b:e])
        return synth.Data(xb=test.xb[b:e], yb=test.yb[b:e])

    def logmeanexp(self, ll_s):
        return float(logsumexp(ll_s.numpy()) - np.log(ll_s.numel()))


def _worker(rank, world, port, cid, n, K, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from helpers import make_case
        from paper_2503_08264_b200 import dist as qdist, synth
        m = synth.config(cid, n=n, K=K)
        data, q, eps, z = make_case(m)
        b, e = qdist.shard_range(m.n, rank, world)
        be = OracleShardBackend(m, data, q, z, b, e)
        runner = qdist.ShardedQEM(be)
        runner.estep()
        same = qdist.check_root_replicated(be.w_root)
        out_q.put((rank, b, e, be.log_pe, be.w_root.numpy(), be.w, be.m1, be.m2, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cid,n,K", [(4, 37, 16), (2, 9, 8)])
def test_two_rank_sharded_estep_matches_single_process(cid, n, K):
    from helpers import make_case
    from oracle import oracle as orc
    from paper_2503_08264_b200 import synth
    world = 2
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cid, n, K, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_out.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    m = synth.config(cid, n=n, K=K)
    data, q, eps, z = make_case(m)
    ref = orc.estep(m, z, q, data)
    covered = []
    for rank, b, e, log_pe, w_root, w, m1, m2, same in res:
        assert same, "root weights differ across ranks"
        covered.append((b, e))
        assert abs(log_pe - ref["log_pe"]) <= 1e-12 * abs(ref["log_pe"])
        np.testing.assert_allclose(w_root, ref["w"][0][0], atol=1e-13)
        np.testing.assert_allclose(w, ref["w"][1][b:e], atol=1e-13)
        np.testing.assert_allclose(m1, ref["m1"][1][b * m.d:e * m.d], rtol=1e-11, atol=1e-14)
        np.testing.assert_allclose(m2, ref["m2"][1][b * m.d:e * m.d], rtol=1e-11, atol=1e-14)
    assert covered[0][0] == 0 and covered[-1][1] == n and covered[0][1] == covered[1][0]


def _worker_evidence(rank, world, port, n, K, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from helpers import make_case
        from paper_2503_08264_b200 import dist as qdist, synth
        m = synth.config(4, n=n, K=K)
        data, q, eps, z_new = make_case(m, eps_seed=99)
        b, e = qdist.shard_range(m.n, rank, world)
        be = OracleShardBackend(m, data, q, z_new, b, e)
        qdist.ShardedQEM(be).evidence()
        out_q.put((rank, be.log_pe_fresh))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_evidence_pass():
    """Fresh-denominator evidence pass across 2 ranks: local forward, the same
    all-reduce, log Pe(z_new) on every rank equal to the single-process oracle's."""
    from helpers import make_case
    from oracle import oracle as orc
    from paper_2503_08264_b200 import synth
    world, n, K = 2, 23, 16
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_evidence, args=(r, world, port, n, K, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_out.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = synth.config(4, n=n, K=K)
    data, q, eps, z_new = make_case(m, eps_seed=99)
    ref = orc.estep(m, z_new, q, data)["log_pe"]
    for rank, lp in res:
        assert abs(lp - ref) <= 1e-12 * abs(ref), (rank, lp, ref)


def test_python_and_c_shard_ranges_agree():
    from paper_2503_08264_b200 import build, dist as qdist, qem
    build.build()
    for n in (1, 5, 100_000, 10_000, 12_345):
        for world in (1, 2, 3, 4, 8):
            for r in range(world):
                assert qdist.shard_range(n, r, world) == qem.shard_range(n, r, world)


def _worker_predict(rank, world, port, n, K, S, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from helpers import make_case
        from paper_2503_08264_b200 import dist as qdist, synth
        m = synth.config(4, n=n, K=K)
        data, q, eps, z = make_case(m)
        test = synth.make_test_data(m, data)
        b, e = qdist.shard_range(m.n, rank, world)
        be = OracleShardBackend(m, data, q, z, b, e)
        runner = qdist.ShardedQEM(be)
        runner.estep()
        pll, ll_s = runner.predictive_loglik(S, 13, test)
        out_q.put((rank, pll, ll_s.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_predictive_loglik():
    """Row f3 across 2 ranks: per-rank resampling of the local groups + the [S] all-reduce gives
    the single-process predictive log-likelihood (same draws: global instance keys)."""
    from helpers import make_case
    from oracle import oracle as orc
    from oracle import predict as op
    from paper_2503_08264_b200 import synth
    world, n, K, S = 2, 19, 16, 40
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_predict, args=(r, world, port, n, K, S, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_out.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = synth.config(4, n=n, K=K)
    data, q, eps, z = make_case(m)
    test = synth.make_test_data(m, data)
    est = orc.estep(m, z, q, data)
    r = op.resample(m, z, q, data, est, S, 13)
    pll_ref, ll_ref = op.predictive_loglik(op.test_loglik(m, z, test, r["idx"]))
    for rank, pll, ll_s in res:
        np.testing.assert_allclose(ll_s, ll_ref, rtol=1e-12)
        assert abs(pll - pll_ref) <= 1e-12 * abs(pll_ref), (rank, pll, pll_ref)
