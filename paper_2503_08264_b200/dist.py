"""Group-sharded QEM over torch.distributed (one process per GPU; NCCL over NVLink/NVSwitch).

The plate dimension partitions naturally: rank r owns the
contiguous block of level-1 groups ``qem_shard_range(n, r, world)``.  Per QEM
iteration the only exchange is one SUM all-reduce of the (K+1) fp64 plate sums
[G(0..K-1), sum_i c_i] that the local forward leaves in ``plate_sum``; it is
log-sum-exp-safe because the plate product is a plain sum of centred
log-messages (nothing is exponentiated before the reduction).  Every rank then
computes the root softmax, log Pe and the root M-step redundantly from the
identical reduced vector -- the "broadcast of the parent weights" of the
north star is therefore implicit (asserted by ``root_digest``).  Root samples
are regenerated identically on every rank from Philox keyed by global
indices, so no sample broadcast is needed either.

The compute backend is any object with the ``QEM`` phase API
(``sample_q / estep_forward / estep_backward / mstep`` and a ``plate_sum``
tensor); the product uses ``paper_2503_08264_b200.qem.QEM``.  A backend with
``estep_reduce`` and a library-owned communicator (``QEM.nccl_init``) runs the
all-reduce inside libqem (``ncclAllReduce`` on the compute stream, capturable
by ``qem_iterate``'s CUDA graph); otherwise the plate sums go through
``torch.distributed.all_reduce`` (e.g. gloo on CPU).
"""
from __future__ import annotations

import hashlib
from typing import Optional

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Contiguous block of groups owned by ``rank`` (same arithmetic as qem_shard_range)."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError(f"bad shard request n={n} rank={rank} world={world}")
    return n * rank // world, n * (rank + 1) // world


class ShardedQEM:
    """Drives one QEM iteration across ranks: local forward -> all-reduce -> local backward -> M-step."""

    def __init__(self, backend, group: Optional[dist.ProcessGroup] = None, in_library: bool = False):
        """in_library: attach a libqem-owned NCCL communicator to the backend (QEM.nccl_init) and
        let the library run the all-reduce (qem_estep_reduce); else torch.distributed does."""
        self.b = backend
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.in_library = bool(in_library)
        if self.in_library:
            backend.nccl_init(group)

    def allreduce_plate_sum(self) -> None:
        if self.in_library:
            self.b.estep_reduce()
        elif self.world > 1:
            t = self.b.plate_sum
            if t.is_cuda and dist.get_backend(self.group) == "gloo":  # gloo reduces host tensors
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def estep(self) -> None:
        self.b.estep_forward()
        self.allreduce_plate_sum()
        self.b.estep_backward()

    def evidence(self) -> None:
        """Fresh-denominator evidence pass on the bound samples: local forward,
        the same all-reduce, then log Pe(z_new) on every rank (no backward)."""
        self.b.estep_forward()
        self.allreduce_plate_sum()
        self.b.evidence_root()

    def step(self, t: int, seed: int, eps=None, eps_new=None, fresh: bool = False) -> None:
        """Iteration t of Algorithm 1 with Q_t already set: z ~ Q_t, E-step, EMA/M-step.
        fresh: first draw z_new (Philox stream bit 23, or eps_new) and run its evidence pass (R28)."""
        if fresh:
            if eps_new is None:
                self.b.sample_q(seed=seed, iter=t | (1 << 23))
            else:
                self.b.sample_q(eps=eps_new)
            self.evidence()
        if eps is None:
            self.b.sample_q(seed=seed, iter=t)
        else:
            self.b.sample_q(eps=eps)
        self.estep()
        self.b.mstep(t)


    def predictive_loglik(self, S: int, seed: int, test):
        """Row f3 across ranks: every rank draws S index tuples for its local
        groups (the root draws coincide: replicated root weights, the same Philox counters), sums
        its groups' held-out log-likelihood per draw, SUM-all-reduces the [S] partials and takes
        log mean exp.  Returns (pll, ll_s) on every rank."""
        idx_root, idx = self.b.backward_resample(S, seed)
        _, ll_s, _ = self.b.predictive_loglik(idx, test)
        if self.world > 1:
            dist.all_reduce(ll_s, op=dist.ReduceOp.SUM, group=self.group)
        return self.b.logmeanexp(ll_s), ll_s


def root_digest(root_weights: torch.Tensor) -> str:
    """Digest of this rank's root weights (must be identical on all ranks)."""
    return hashlib.sha256(root_weights.detach().cpu().numpy().tobytes()).hexdigest()


def check_root_replicated(root_weights: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> bool:
    """True iff every rank holds bit-identical root weights."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return True
    mine = root_digest(root_weights)
    allv = [None] * dist.get_world_size(group)
    dist.all_gather_object(allv, mine, group=group)
    return all(v == mine for v in allv)
