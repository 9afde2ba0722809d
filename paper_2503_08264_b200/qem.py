"""Python binding of the QEM C-ABI: same names as include/qem.h, argument marshalling only.

Torch supplies device memory and streams; every step of the hot path runs in
libqem.so kernels.  A ``QEM`` object owns one ``qem_ctx`` and the torch
buffers bound to it (Q parameters, EMA state, samples, weights, moments,
observations).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from . import synth


def _desc(m) -> _lib.ModelDesc:
    return _lib.ModelDesc(m.family, m.d if m.family == 2 else 1, m.scale_kind, m.obs_kind, m.n,
                          m.B, m.J, m.P, m.K, m.fixed_var, m.obs_var, m.top_var, m.sub_var,
                          m.prior_mean, m.prior_var)


def model_validate(m) -> Optional[str]:
    """None if the model is valid, else the library's one-line reason."""
    buf = ctypes.create_string_buffer(256)
    d = _desc(m)
    st = lib().qem_model_validate(ctypes.byref(d), buf, 256)
    return None if st == _lib.OK else buf.value.decode()


GAMMA, BETA, BERNOULLI, CATEGORICAL, DIRICHLET, BINOMIAL, MULTINOMIAL = 1, 2, 3, 4, 5, 6, 7


def mstep_family(family: int, lam: float, m_new: torch.Tensor, m_ema: torch.Tensor, C: int = 1, stream=None):
    """EMA over mean parameters + M-step of a non-Gaussian Q family (qem_mstep_family) on device
    tensors: m_new, m_ema float64 [n][S] (m_ema updated in place).  Returns (params [n][S], status [n])."""
    assert m_new.dtype == torch.float64 and m_ema.dtype == torch.float64 and m_new.is_cuda
    n = m_new.shape[0]
    params = torch.empty_like(m_ema)
    status = torch.empty(n, dtype=torch.int32, device=m_new.device)
    check(lib().qem_mstep_family(int(family), n, int(C), float(lam), ctypes.c_void_p(m_new.data_ptr()),
                                 ctypes.c_void_p(m_ema.data_ptr()), ctypes.c_void_p(params.data_ptr()),
                                 ctypes.c_void_p(status.data_ptr()), _stream(stream)), "qem_mstep_family")
    return params, status


def estep_tables(f_root: torch.Tensor, f: torch.Tensor, stream=None):
    """MPIW E-step on explicit log-factor tables (qem_estep_tables): f_root float64 [K], f float64
    [n][K][K] (device).  Returns dict(log_pe [1], w_root [K], w [n][K], g [n][K])."""
    assert f_root.dtype == torch.float64 and f.dtype == torch.float64 and f_root.is_cuda
    K = f_root.shape[0]
    n = f.shape[0] if f.numel() else 0
    assert f.numel() == 0 or tuple(f.shape) == (n, K, K)
    f_root, f = f_root.contiguous(), f.contiguous()
    dev = f_root.device
    out = dict(log_pe=torch.empty(1, dtype=torch.float64, device=dev),
               w_root=torch.empty(K, dtype=torch.float64, device=dev),
               w=torch.empty(n, K, dtype=torch.float64, device=dev),
               g=torch.empty(n, K, dtype=torch.float64, device=dev))
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t.numel() else None)  # noqa: E731
    check(lib().qem_estep_tables(n, K, ptr(f_root), ptr(f), ptr(out["g"]), ptr(out["log_pe"]), ptr(out["w_root"]),
                                 ptr(out["w"]), _stream(stream)), "qem_estep_tables")
    return out


def estep_separable(f_root: torch.Tensor, rows: torch.Tensor, cols: torch.Tensor, stream=None):
    """MPIW E-step on separable log-factors (qem_estep_separable): f_root [K], rows [K][1+R], cols
    [n][K][R+1] (float64 device).  Returns dict(log_pe [1], w_root [K], w [n][K], g [n][K])."""
    assert f_root.dtype == rows.dtype == cols.dtype == torch.float64 and f_root.is_cuda
    K, R = f_root.shape[0], rows.shape[1] - 1
    n = cols.shape[0] if cols.numel() else 0
    assert tuple(rows.shape) == (K, R + 1) and (n == 0 or tuple(cols.shape) == (n, K, R + 1))
    f_root, rows, cols = f_root.contiguous(), rows.contiguous(), cols.contiguous()
    dev = f_root.device
    out = dict(log_pe=torch.empty(1, dtype=torch.float64, device=dev),
               w_root=torch.empty(K, dtype=torch.float64, device=dev),
               w=torch.empty(n, K, dtype=torch.float64, device=dev),
               g=torch.empty(n, K, dtype=torch.float64, device=dev))
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t.numel() else None)  # noqa: E731
    check(lib().qem_estep_separable(n, K, R, ptr(f_root), ptr(rows), ptr(cols), ptr(out["g"]), ptr(out["log_pe"]),
                                    ptr(out["w_root"]), ptr(out["w"]), _stream(stream)), "qem_estep_separable")
    return out


QMP_PERMUTATION, QMP_MIXTURE = 0, 1


def estep_qmp_gaussian(mu: torch.Tensor, root_mean: torch.Tensor, root_var: torch.Tensor, q: torch.Tensor,
                       copy: torch.Tensor, eps: torch.Tensor, x: torch.Tensor, scheme: int, *, prior_var=1.0,
                       group_var=1.0, obs_var=1.0, stream=None):
    """MPIW E-step under the non-factorised Q_MP with a parent-copy scheme (App. A):
    qem_cols_qmp_gaussian (child draws + separable factors) -> qem_estep_separable -> qem_moments_qmp.
    mu [K] f32 root samples, root_mean / root_var [1] f32, q [n][3] f64 (alpha, beta, s), copy [n][K]
    int32, eps [n][K] f32, x [n][J] f32, all on the device.  Returns the E-step dict plus z [n][K],
    root_m [2], gm [n][2] (argument marshalling only: every step runs in libqem)."""
    K, n = mu.shape[0], q.shape[0]
    J = x.shape[1] if x.numel() else 0
    assert mu.dtype == eps.dtype == x.dtype == root_mean.dtype == root_var.dtype == torch.float32 and mu.is_cuda
    assert q.dtype == torch.float64 and copy.dtype == torch.int32
    assert tuple(q.shape) == (n, 3) and tuple(copy.shape) == (n, K) and tuple(eps.shape) == (n, K)
    mu, q, copy, eps, x = mu.contiguous(), q.contiguous(), copy.contiguous(), eps.contiguous(), x.contiguous()
    f64 = dict(dtype=torch.float64, device=mu.device)
    z, f_root = torch.empty(n, K, **f64), torch.empty(K, **f64)
    rows, cols = torch.empty(K, 2, **f64), torch.empty(n, K, 2, **f64)
    check(lib().qem_cols_qmp_gaussian(n, K, J, int(scheme), float(prior_var), float(group_var), float(obs_var),
                                      _ptr(mu), _ptr(root_mean), _ptr(root_var), _ptr(q), _ptr(copy), _ptr(eps),
                                      _ptr(x), _ptr(z), _ptr(f_root), _ptr(rows), _ptr(cols), _stream(stream)),
          "qem_cols_qmp_gaussian")
    out = estep_separable(f_root, rows, cols, stream=stream)
    out["z"], out["f_root"] = z, f_root
    out["root_m"], out["gm"] = torch.empty(2, **f64), torch.empty(n, 2, **f64)
    check(lib().qem_moments_qmp(n, K, _ptr(out["w_root"]), _ptr(mu), _ptr(out["w"]), _ptr(z), _ptr(out["root_m"]),
                                _ptr(out["gm"]), _stream(stream)), "qem_moments_qmp")
    return out


def logmeanexp(x: torch.Tensor, stream=None) -> torch.Tensor:
    """log (1/n) sum exp(x) of a float64 device vector (qem_logmeanexp); returns a [1] tensor."""
    assert x.dtype == torch.float64 and x.is_cuda
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    check(lib().qem_logmeanexp(x.numel(), _ptr(x.contiguous()), _ptr(out), _stream(stream)), "qem_logmeanexp")
    return out


def workspace_bytes(m, group_begin=0, group_end=None, *, new_weight=0.3, schedule_p=0.0, var_floor=1e-8,
                    fresh_denominator=False) -> int:
    """Device workspace a context over [group_begin, group_end) needs (qem_workspace_bytes)."""
    d = _desc(m)
    o = _lib.Opts(new_weight, schedule_p, var_floor, int(bool(fresh_denominator)), 0)
    nb = ctypes.c_size_t()
    check(lib().qem_workspace_bytes(ctypes.byref(d), ctypes.byref(o), int(group_begin),
                                    int(m.n if group_end is None else group_end), ctypes.byref(nb)),
          "qem_workspace_bytes")
    return nb.value


def shard_range(n: int, rank: int, world: int):
    b, e = ctypes.c_int64(), ctypes.c_int64()
    check(lib().qem_shard_range(n, rank, world, ctypes.byref(b), ctypes.byref(e)), "qem_shard_range")
    return b.value, e.value


def _ptr(t: Optional[torch.Tensor]) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() else None)


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class QEM:
    """One context over LOCAL level-1 instances [group_begin, group_end)."""

    def __init__(self, m, *, new_weight=0.3, schedule_p=0.0, var_floor=1e-8, group_begin=0, group_end=None,
                 device="cuda", trace_len=0, fresh_denominator=False, caller_workspace=False):
        if not torch.cuda.is_available():
            raise _lib.QemError("QEM needs a CUDA device (there is no CPU fallback)")
        self.m = m
        self.device = torch.device(device)
        if group_end is None:
            group_end = m.n
        self.g_begin, self.g_end = int(group_begin), int(group_end)
        self.n_local = self.g_end - self.g_begin
        d = _desc(m)
        o = _lib.Opts(new_weight, schedule_p, var_floor, int(bool(fresh_denominator)), 0)
        self.fresh = bool(fresh_denominator)
        ctx = ctypes.c_void_p()
        self._ws = None
        with torch.cuda.device(self.device):
            if caller_workspace:  # the context's buffers carved from a torch allocation (qem_create_in)
                nb = ctypes.c_size_t()
                check(lib().qem_workspace_bytes(ctypes.byref(d), ctypes.byref(o), self.g_begin, self.g_end,
                                                ctypes.byref(nb)), "qem_workspace_bytes")
                self._ws = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
                check(lib().qem_create_in(ctypes.byref(d), ctypes.byref(o), self.g_begin, self.g_end,
                                          ctypes.c_void_p(self._ws.data_ptr()), nb.value, ctypes.byref(ctx)),
                      "qem_create_in")
            else:
                check(lib().qem_create(ctypes.byref(d), ctypes.byref(o), self.g_begin, self.g_end,
                                       ctypes.byref(ctx)), "qem_create")
        self.ctx = ctx
        K = m.K
        f32 = dict(dtype=torch.float32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        shapes = synth.latent_shapes(m)
        if m.family == synth.FAMILY_TWO_LEVEL:
            shapes = [shapes[0], (self.n_local, m.d)]
        self.shapes = shapes
        self.levels = []
        for inst, dims in shapes:
            nl = inst * dims
            lv = dict(q_mean=torch.zeros(nl, **f32), q_var=torch.ones(nl, **f32),
                      ema_m1=torch.zeros(nl, **f64), ema_v=torch.ones(nl, **f64),
                      z=torch.zeros(inst, dims, K, **f32), w=torch.zeros(inst, K, **f32),
                      m1=torch.zeros(nl, **f64), v=torch.zeros(nl, **f64))
            self.levels.append(lv)
        self.log_pe = torch.zeros(1, **f64)
        self.log_pe_fresh = torch.zeros(1, **f64)
        self.plate_sum = torch.zeros(K + 1, **f64)
        self.trace = torch.zeros(max(trace_len, 1), **f64)
        self.x = self.y = None
        self._bound = False

    # ------------------------------------------------------------ buffers
    def set_data(self, data: synth.Data) -> None:
        """Upload the LOCAL shard of the observations (host numpy -> device)."""
        m, b, e = self.m, self.g_begin, self.g_end
        dev = self.device
        if m.obs_kind == synth.OBS_GAUSS:
            self.x = torch.from_numpy(np.ascontiguousarray(data.xg[b:e], np.float32)).to(dev)
            self.y = None
        elif m.obs_kind == synth.OBS_BERNOULLI_LOGIT:
            self.x = torch.from_numpy(np.ascontiguousarray(data.xb[b:e], np.uint8)).to(dev)
            self.y = torch.from_numpy(np.ascontiguousarray(data.yb[b:e], np.uint8)).to(dev)
        else:
            self.x = torch.from_numpy(np.ascontiguousarray(data.xp, np.float32)).to(dev)
            self.y = torch.from_numpy(np.ascontiguousarray(data.yp, np.int32)).to(dev)
        self.bind()

    def bind(self) -> None:
        b = _lib.Buffers()
        for l, lv in enumerate(self.levels):
            b.level[l] = _lib.Level(*[lv[k].data_ptr() for k in ("q_mean", "q_var", "ema_m1", "ema_v", "z", "w",
                                                                  "m1", "v")])
        b.x = self.x.data_ptr() if self.x is not None else None
        b.y = self.y.data_ptr() if self.y is not None else None
        b.log_pe = self.log_pe.data_ptr()
        b.trace = self.trace.data_ptr()
        b.trace_len = self.trace.numel()
        b.plate_sum = self.plate_sum.data_ptr()
        b.log_pe_fresh = self.log_pe_fresh.data_ptr()
        bank = getattr(self, "_eps_bank", None)
        if bank is not None:
            for l, t in enumerate(bank):
                b.eps_bank[l] = t.data_ptr()
            b.eps_bank_len = bank[0].shape[0]
        check(lib().qem_bind(self.ctx, ctypes.byref(b)), "qem_bind")
        self._bound = True

    def set_q(self, q: Sequence) -> None:
        """Q_t per level: (mean [inst*dims], var [inst*dims]) host arrays (local shard for level 1)."""
        for lv, (qm, qv) in zip(self.levels, self._local(q)):
            lv["q_mean"].copy_(torch.as_tensor(np.asarray(qm, np.float32)))
            lv["q_var"].copy_(torch.as_tensor(np.asarray(qv, np.float32)))

    def set_state(self, state: Sequence) -> None:
        """EMA state per level: (m1, v) fp64 host arrays."""
        for lv, (a, b) in zip(self.levels, self._local(state)):
            lv["ema_m1"].copy_(torch.as_tensor(np.asarray(a, np.float64)))
            lv["ema_v"].copy_(torch.as_tensor(np.asarray(b, np.float64)))

    def set_z(self, z: Sequence) -> None:
        """Samples per level [inst*dims][K] fp32 host arrays (bypasses the sampler)."""
        for lv, zz in zip(self.levels, self._local(z)):
            lv["z"].copy_(torch.as_tensor(np.asarray(zz, np.float32)).reshape(lv["z"].shape))

    def _bank_slices(self, nlev):
        """Row slices of each level's eps arrays that belong to this context's shard."""
        out = [slice(None)] * nlev
        if self.m.family == synth.FAMILY_TWO_LEVEL and nlev > 1:
            out[1] = slice(self.g_begin * self.m.d, self.g_end * self.m.d)
        return out

    def _local(self, per_level):
        out = list(per_level)
        if self.m.family == synth.FAMILY_TWO_LEVEL and len(out) > 1:
            d = self.m.d
            sl = slice(self.g_begin * d, self.g_end * d)

            def cut(a):
                if isinstance(a, tuple):
                    return tuple(np.asarray(x)[sl] for x in a)
                return np.asarray(a)[sl]
            out[1] = cut(out[1])
        return out

    # ---------------------------------------------------------- the C-ABI
    def sample_q(self, seed: int = 0, iter: int = 1, eps: Optional[Sequence] = None, stream=None) -> None:
        """K1: z = fmaf(sqrtf(v), eps, m); eps per level (host arrays) or Philox(seed, iter)."""
        keep = None
        arr = None
        if eps is not None:
            keep = [torch.as_tensor(np.asarray(e, np.float32)).to(self.device).contiguous()
                    for e in self._local(eps)]
            arr = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in keep] + [None] * (3 - len(keep)))
        check(lib().qem_sample_q(self.ctx, seed, iter, arr, _stream(stream)), "qem_sample_q")
        if keep is not None:
            torch.cuda.current_stream().synchronize()  # keep eps alive until consumed

    def estep(self, stream=None) -> None:
        check(lib().qem_estep(self.ctx, _stream(stream)), "qem_estep")

    def sample_estep_forward(self, seed: int, iter: int, stream=None) -> None:
        """qem_sample_estep_forward: Philox samples + forward phase (fused on the tensor-core path)."""
        check(lib().qem_sample_estep_forward(self.ctx, seed, iter, _stream(stream)), "qem_sample_estep_forward")

    def estep_forward(self, stream=None) -> None:
        check(lib().qem_estep_forward(self.ctx, _stream(stream)), "qem_estep_forward")

    def estep_reduce(self, stream=None) -> None:
        """The SUM all-reduce of the (K+1) plate sums over the attached communicator (qem_estep_reduce)."""
        check(lib().qem_estep_reduce(self.ctx, _stream(stream)), "qem_estep_reduce")

    # ------------------------------------------------------- communicator
    def nccl_init(self, group=None) -> None:
        """Attach a library-owned NCCL communicator over the ranks of `group` (torch.distributed,
        any backend; None = the default group, or a 1-rank communicator when torch.distributed is
        not initialised).  Collective: rank 0 draws the ncclUniqueId (qem_nccl_unique_id), the
        bytes travel over torch.distributed, every rank calls qem_nccl_init."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
        uid = (ctypes.c_char * _lib.NCCL_ID_BYTES)()
        if rank == 0:
            check(lib().qem_nccl_unique_id(uid), "qem_nccl_unique_id")
        if world > 1:
            box = [bytes(uid)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(box, src=src, group=group)
            ctypes.memmove(uid, box[0], _lib.NCCL_ID_BYTES)
        with torch.cuda.device(self.device):
            check(lib().qem_nccl_init(self.ctx, uid, int(rank), int(world)), "qem_nccl_init")

    def set_nccl_comm(self, comm_ptr) -> None:
        """Attach a caller-owned ncclComm_t (an integer handle; None detaches)."""
        check(lib().qem_set_nccl_comm(self.ctx, ctypes.c_void_p(comm_ptr)), "qem_set_nccl_comm")

    def nccl_info(self):
        """(rank, world, NCCL version code) of the attached communicator ((0, 1, 0) without one)."""
        r, w, v = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(lib().qem_nccl_info(self.ctx, ctypes.byref(r), ctypes.byref(w), ctypes.byref(v)), "qem_nccl_info")
        return r.value, w.value, v.value

    def estep_backward(self, stream=None) -> None:
        check(lib().qem_estep_backward(self.ctx, _stream(stream)), "qem_estep_backward")

    def estep_evidence(self, stream=None) -> None:
        """Fresh-denominator pass: log Pe of the bound samples -> log_pe_fresh."""
        check(lib().qem_estep_evidence(self.ctx, _stream(stream)), "qem_estep_evidence")

    def evidence_root(self, stream=None) -> None:
        """Phase 2 of the sharded evidence pass (after estep_forward + the all-reduce)."""
        check(lib().qem_evidence_root(self.ctx, _stream(stream)), "qem_evidence_root")

    def mstep(self, t: int, stream=None) -> None:
        check(lib().qem_mstep(self.ctx, t, _stream(stream)), "qem_mstep")

    def iterate(self, t0: int, T: int, seed: int, use_graph: bool = True, stream=None, eps_bank=None) -> None:
        """qem_iterate: T QEM iterations from t0.  eps_bank (parity mode): per level a host array
        [T][instances*dims][K] of N(0,1) draws (this context's shard for level 1) used instead of
        Philox; None restores Philox sampling."""
        rebind = False
        if T > self.trace.numel():
            self.trace = torch.zeros(T, dtype=torch.float64, device=self.device)
            rebind = True
        if eps_bank is not None:
            self._eps_bank = [torch.as_tensor(np.ascontiguousarray(np.asarray(e, np.float32)[:, sl])).to(self.device)
                              for e, sl in zip(eps_bank, self._bank_slices(len(eps_bank)))]
            rebind = True
        elif getattr(self, "_eps_bank", None) is not None:
            self._eps_bank = None
            rebind = True
        if rebind:
            self.bind()
        check(lib().qem_iterate(self.ctx, t0, T, seed, int(use_graph), _stream(stream)), "qem_iterate")

    def read_flags(self, stream=None):
        f, c = ctypes.c_uint32(), ctypes.c_int64()
        check(lib().qem_read_flags(self.ctx, _stream(stream), ctypes.byref(f), ctypes.byref(c)), "qem_read_flags")
        return f.value, c.value

    def mode_hist(self, stream=None):
        """Forward tile-mode histogram since the last call (diagnostics)."""
        h = (ctypes.c_uint64 * 8)()
        check(lib().qem_read_mode_hist(self.ctx, _stream(stream), h), "qem_read_mode_hist")
        return [int(v) for v in h]

    def set_kernel_events(self, events=None) -> None:
        """Record 4 torch.cuda.Event (fwd start/end, bwd start/end) around the pair-tile kernels."""
        if events is None:
            handles = [None] * 4
        else:
            events = list(events) + [None] * (4 - len(events))
            for e in events:  # torch creates the CUDA event lazily
                if e is not None:
                    e.record()
            handles = [ctypes.c_void_p(e.cuda_event) if e is not None else None for e in events]
        self._events = events
        check(lib().qem_set_kernel_events(self.ctx, *handles), "qem_set_kernel_events")

    def kernel_launches(self) -> int:
        return int(lib().qem_kernel_launches(self.ctx))

    def pair_path(self) -> int:
        """0 = FP32/SFU pair tiles, 1 = tcgen05 tensor-core pair tiles (d = 16)."""
        return int(lib().qem_pair_path(self.ctx))

    def messages(self):
        """(Delta g [n_local][K] f32, c [n_local] f64) of the last forward (device tensors)."""
        dg = torch.empty(self.n_local, self.m.K, dtype=torch.float32, device=self.device)
        c = torch.empty(self.n_local, dtype=torch.float64, device=self.device)
        check(lib().qem_copy_messages(self.ctx, dg.data_ptr(), c.data_ptr(), _stream()), "qem_copy_messages")
        return dg, c

    # ---------------------------------------------------------- readback
    def global_iw(self, stream=None):
        """Global importance weighting (App. A) on the bound samples after estep_forward / estep:
        returns dict(log_pe [1], w [K], m1 [n][d], diag [n][K])."""
        K, n, d = self.m.K, self.n_local, self.m.d
        f64 = dict(dtype=torch.float64, device=self.device)
        out = dict(log_pe=torch.empty(1, **f64), w=torch.empty(K, **f64), m1=torch.empty(n, d, **f64),
                   diag=torch.empty(n, K, **f64))
        scratch = torch.empty(n, K, **f64)
        check(lib().qem_global_iw(self.ctx, _ptr(out["diag"]), _ptr(scratch), _ptr(out["log_pe"]), _ptr(out["w"]),
                                  _ptr(out["m1"]), _stream(stream)), "qem_global_iw")
        self._gscratch = scratch
        return out

    def logmeanexp(self, x: torch.Tensor) -> torch.Tensor:
        return logmeanexp(x)

    def backward_resample(self, S: int, seed: int, stream=None):
        """S index tuples from the MPIW posterior after an E-step (qem_backward_resample):
        (idx_root [S], idx [S][n_local]) int32 device tensors."""
        idx_root = torch.empty(S, dtype=torch.int32, device=self.device)
        idx = torch.empty(S, self.n_local, dtype=torch.int32, device=self.device)
        check(lib().qem_backward_resample(self.ctx, int(S), int(seed), _ptr(idx_root), _ptr(idx), _stream(stream)),
              "qem_backward_resample")
        return idx_root, idx

    def set_test_data(self, test: "synth.Data") -> None:
        """Upload the LOCAL shard of held-out observations once (row f3)."""
        m, b, e = self.m, self.g_begin, self.g_end
        if m.obs_kind == synth.OBS_GAUSS:
            x = torch.from_numpy(np.ascontiguousarray(test.xg[b:e], np.float32)).to(self.device)
            y = None
        else:
            x = torch.from_numpy(np.ascontiguousarray(test.xb[b:e], np.uint8)).to(self.device)
            y = torch.from_numpy(np.ascontiguousarray(test.yb[b:e], np.uint8)).to(self.device)
        self._test = (x, y)

    def predictive_loglik(self, idx: torch.Tensor, test: Optional["synth.Data"] = None, stream=None):
        """Predictive log-likelihood of held-out observations of the local groups at the resampled
        latents (qem_predictive_loglik): returns (pll [1], ll_s [S], ll_part [S][n_local]).
        `test` uploads (and keeps) a held-out set; else the one from set_test_data is used."""
        if test is not None:
            self.set_test_data(test)
        x, y = self._test
        S = idx.shape[0]
        J = x.shape[1]
        f64 = dict(dtype=torch.float64, device=self.device)
        ll_part, ll_s, pll = torch.empty(S, self.n_local, **f64), torch.empty(S, **f64), torch.empty(1, **f64)
        check(lib().qem_predictive_loglik(self.ctx, int(S), _ptr(idx), int(J), _ptr(x), _ptr(y), _ptr(ll_part),
                                          _ptr(ll_s), _ptr(pll), _stream(stream)), "qem_predictive_loglik")
        return pll, ll_s, ll_part

    def result(self):
        """Host copies of the last E-step: log_pe, w / m1 / v per level, plus Q and EMA state."""
        torch.cuda.current_stream().synchronize()
        out = dict(log_pe=float(self.log_pe.item()))
        for key in ("w", "m1", "v", "q_mean", "q_var", "ema_m1", "ema_v", "z"):
            out[key] = [lv[key].cpu().numpy() for lv in self.levels]
        return out

    def close(self) -> None:
        if getattr(self, "ctx", None):
            lib().qem_destroy(self.ctx)
            self.ctx = None
            self._ws = None  # a caller workspace outlives the context

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CategoricalQEM:
    """QEM for discrete (categorical) latents under a Gaussian root (NEXT row f1, R30):
    one iteration = qem_sample_normal + qem_sample_categorical + qem_estep_categorical (or
    qem_tables_categorical + qem_estep_tables) + qem_moments_categorical + qem_mstep_categorical,
    all on device; this class only owns the buffers and sequences the calls (argument marshalling)."""

    def __init__(self, om, *, new_weight=0.3, schedule_p=0.0, var_floor=1e-8, device="cuda", tables=False):
        """tables=False: the factorised E-step (qem_estep_categorical, O(n K C)); True: the
        materialised log-factor tables + qem_estep_tables (O(n K^2), the generic engine)."""
        if not torch.cuda.is_available():
            raise _lib.QemError("CategoricalQEM needs a CUDA device (there is no CPU fallback)")
        self.om, self.device, self.tables = om, torch.device(device), bool(tables)
        self.new_weight, self.schedule_p, self.var_floor = new_weight, schedule_p, var_floor
        n, C, R, d, K = om.n, om.C, om.R, om.d, om.K
        f32 = dict(dtype=torch.float32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(self.device)  # noqa: E731
        self.x, self.logit, self.y = up(om.x, np.float64), up(om.logit, np.float64), up(om.y, np.uint8)
        self.L = torch.empty(n, C, **f64)
        check(lib().qem_loglik_bernoulli_states(n, C, R, _ptr(self.y), _ptr(self.logit), _ptr(self.L), _stream()),
              "qem_loglik_bernoulli_states")
        self.root_mean, self.root_var = torch.zeros(d, **f32), torch.ones(d, **f32)
        self.root_ema = torch.tensor([[0.0, 1.0]] * d, **f64)
        self.p = torch.full((n, C), 1.0 / C, **f64)
        self.p_ema = self.p.clone()
        self.root_z, self.z = torch.empty(d, K, **f32), torch.empty(n, K, dtype=torch.int32, device=self.device)
        self.f_root = torch.empty(K, **f64)
        self.f = torch.empty(n, K, K, **f64) if self.tables else None
        self.g, self.w = torch.empty(n, K, **f64), torch.empty(n, K, **f64)
        self.w_root, self.log_pe = torch.empty(K, **f64), torch.empty(1, **f64)
        self.root_m, self.pm = torch.empty(d, 2, **f64), torch.empty(n, C, **f64)
        self.clamps = torch.zeros(1, dtype=torch.int64, device=self.device)

    def lam(self, t: int) -> float:
        """History weight (R5; qem_history_weight): 1 - new_weight, or 1 - t^-p with a schedule."""
        return float(lib().qem_history_weight(int(t), float(self.new_weight), float(self.schedule_p)))

    def estep(self, t: int, seed: int, root_eps: Optional[torch.Tensor] = None, stream=None) -> None:
        om, L, s = self.om, lib(), _stream(stream)
        n, C, d, K = om.n, om.C, om.d, om.K
        eps = _ptr(root_eps) if root_eps is not None else None
        check(L.qem_sample_normal(d, K, 0, seed, t, _ptr(self.root_mean), _ptr(self.root_var), eps, _ptr(self.root_z),
                                  s), "qem_sample_normal")
        check(L.qem_sample_categorical(n, C, K, seed, t, _ptr(self.p), _ptr(self.z), s), "qem_sample_categorical")
        if self.tables:
            check(L.qem_tables_categorical(n, C, K, d, _ptr(self.root_z), _ptr(self.root_mean), _ptr(self.root_var),
                                           _ptr(self.x), _ptr(self.L), _ptr(self.p), _ptr(self.z), _ptr(self.f_root),
                                           _ptr(self.f), s), "qem_tables_categorical")
            check(L.qem_estep_tables(n, K, _ptr(self.f_root), _ptr(self.f), _ptr(self.g), _ptr(self.log_pe),
                                     _ptr(self.w_root), _ptr(self.w), s), "qem_estep_tables")
        else:
            check(L.qem_estep_categorical(n, C, K, d, _ptr(self.root_z), _ptr(self.root_mean), _ptr(self.root_var),
                                          _ptr(self.x), _ptr(self.L), _ptr(self.p), _ptr(self.z), _ptr(self.f_root),
                                          _ptr(self.g), _ptr(self.log_pe), _ptr(self.w_root), _ptr(self.w), s),
                  "qem_estep_categorical")
        check(L.qem_moments_categorical(n, C, K, d, _ptr(self.w_root), _ptr(self.root_z), _ptr(self.w), _ptr(self.z),
                                        _ptr(self.root_m), _ptr(self.pm), s), "qem_moments_categorical")

    def mstep(self, t: int, stream=None) -> None:
        om = self.om
        check(lib().qem_mstep_categorical(om.n, om.C, om.d, self.lam(t), self.var_floor, _ptr(self.root_m),
                                          _ptr(self.root_ema), _ptr(self.root_mean), _ptr(self.root_var),
                                          _ptr(self.pm), _ptr(self.p_ema), _ptr(self.p), _ptr(self.clamps),
                                          _stream(stream)), "qem_mstep_categorical")

    def step(self, t: int, seed: int, root_eps=None, stream=None) -> None:
        self.estep(t, seed, root_eps, stream)
        self.mstep(t, stream)

    def set_state(self, st: dict) -> None:
        """Teacher forcing (parity tests): Q and EMA state from host arrays."""
        for k in ("root_mean", "root_var", "root_ema", "p", "p_ema"):
            getattr(self, k).copy_(torch.from_numpy(np.asarray(st[k])).to(getattr(self, k).dtype))


class GammaPoissonQEM:
    """QEM with Gamma approximate posteriors (NEXT row f1, R32) on the Gamma-Poisson
    hierarchy of synth.gamma_poisson: one iteration = qem_sample_normal (root) + qem_sample_gamma
    + qem_tables_gamma_poisson + qem_estep_tables + qem_moments_gamma + qem_mstep_family (GAMMA)
    + qem_mstep_categorical (root only, n = 0), all on device (argument marshalling only)."""

    def __init__(self, gp, *, new_weight=0.3, var_floor=1e-8, device="cuda", tables=False):
        """tables=False (default): separable factors evaluated on chip (qem_cols_gamma_poisson +
        qem_estep_separable, no n x K x K array); True: the materialised fp64 tables
        (qem_tables_gamma_poisson + qem_estep_tables), kept for comparison."""
        if not torch.cuda.is_available():
            raise _lib.QemError("GammaPoissonQEM needs a CUDA device (there is no CPU fallback)")
        self.gp, self.device, self.tables = gp, torch.device(device), bool(tables)
        self.new_weight, self.var_floor = new_weight, var_floor
        n, K = gp.n, gp.K
        f32 = dict(dtype=torch.float32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        self.y = torch.from_numpy(np.ascontiguousarray(gp.y, np.int32)).to(self.device)
        self.root_mean, self.root_var = torch.zeros(1, **f32), torch.ones(1, **f32)
        self.root_ema = torch.tensor([[0.0, 1.0]], **f64)
        self.q = torch.ones(n, 2, **f64)                                   # Gamma(1, 1)
        self.g_ema = torch.tensor([[1.0, -0.5772156649015329]] * n, **f64)  # its (E l, E ln l)
        self.mu, self.z = torch.empty(1, K, **f32), torch.empty(n, K, **f64)
        self.f_root = torch.empty(K, **f64)
        if self.tables:
            self.f = torch.empty(n, K, K, **f64)
        else:
            self.rows, self.cols = torch.empty(K, 2, **f64), torch.empty(n, K, 2, **f64)
        self.g, self.w = torch.empty(n, K, **f64), torch.empty(n, K, **f64)
        self.w_root, self.log_pe = torch.empty(K, **f64), torch.empty(1, **f64)
        self.root_m, self.gm = torch.empty(1, 2, **f64), torch.empty(n, 2, **f64)
        self.status = torch.zeros(n, dtype=torch.int32, device=self.device)
        self.clamps = torch.zeros(1, dtype=torch.int64, device=self.device)

    def step(self, t: int, seed: int, root_eps: Optional[torch.Tensor] = None, stream=None) -> None:
        gp, L, s = self.gp, lib(), _stream(stream)
        n, K = gp.n, gp.K
        check(L.qem_sample_normal(1, K, 0, seed, t, _ptr(self.root_mean), _ptr(self.root_var),
                                  _ptr(root_eps) if root_eps is not None else None, _ptr(self.mu), s),
              "qem_sample_normal")
        check(L.qem_sample_gamma(n, K, seed, t, _ptr(self.q), _ptr(self.z), s), "qem_sample_gamma")
        if self.tables:
            check(L.qem_tables_gamma_poisson(n, K, gp.J, float(gp.alpha), _ptr(self.mu), _ptr(self.root_mean),
                                             _ptr(self.root_var), _ptr(self.y), _ptr(self.q), _ptr(self.z),
                                             _ptr(self.f_root), _ptr(self.f), s), "qem_tables_gamma_poisson")
            check(L.qem_estep_tables(n, K, _ptr(self.f_root), _ptr(self.f), _ptr(self.g), _ptr(self.log_pe),
                                     _ptr(self.w_root), _ptr(self.w), s), "qem_estep_tables")
        else:
            check(L.qem_cols_gamma_poisson(n, K, gp.J, float(gp.alpha), _ptr(self.mu), _ptr(self.root_mean),
                                           _ptr(self.root_var), _ptr(self.y), _ptr(self.q), _ptr(self.z),
                                           _ptr(self.f_root), _ptr(self.rows), _ptr(self.cols), s),
                  "qem_cols_gamma_poisson")
            check(L.qem_estep_separable(n, K, 1, _ptr(self.f_root), _ptr(self.rows), _ptr(self.cols), _ptr(self.g),
                                        _ptr(self.log_pe), _ptr(self.w_root), _ptr(self.w), s), "qem_estep_separable")
        check(L.qem_moments_gamma(n, K, _ptr(self.w_root), _ptr(self.mu), _ptr(self.w), _ptr(self.z),
                                  _ptr(self.root_m), _ptr(self.gm), s), "qem_moments_gamma")
        lam = L.qem_history_weight(int(t), float(self.new_weight), 0.0)
        check(L.qem_mstep_family(GAMMA, n, 1, lam, _ptr(self.gm), _ptr(self.g_ema), _ptr(self.q), _ptr(self.status),
                                 s), "qem_mstep_family")
        check(L.qem_mstep_gaussian(1, lam, self.var_floor, _ptr(self.root_m), _ptr(self.root_ema),
                                   _ptr(self.root_mean), _ptr(self.root_var), _ptr(self.clamps), s),
              "qem_mstep_gaussian")

    def set_state(self, st: dict) -> None:
        """Teacher forcing (parity tests): Q and EMA state from host arrays."""
        self.root_mean.fill_(float(st["root_mean"]))
        self.root_var.fill_(float(st["root_var"]))
        self.root_ema.copy_(torch.from_numpy(np.asarray(st["root_ema"], np.float64).reshape(1, 2)))
        self.q.copy_(torch.from_numpy(np.asarray(st["q"], np.float64)))
        self.g_ema.copy_(torch.from_numpy(np.asarray(st["g_ema"], np.float64)))


class BetaBinomialQEM:
    """QEM with Beta approximate posteriors (NEXT row f1, R32) on the Beta-Binomial
    hierarchy of synth.beta_binomial: qem_sample_normal (root) + qem_sample_beta +
    qem_tables_beta_binomial + qem_estep_tables + qem_moments_beta + qem_mstep_family (BETA) +
    qem_mstep_categorical (root only), all on device (argument marshalling only)."""

    def __init__(self, bb, *, new_weight=0.3, var_floor=1e-8, device="cuda", tables=False):
        """tables: as GammaPoissonQEM (False: qem_cols_beta_binomial + qem_estep_separable)."""
        if not torch.cuda.is_available():
            raise _lib.QemError("BetaBinomialQEM needs a CUDA device (there is no CPU fallback)")
        self.bb, self.device, self.tables = bb, torch.device(device), bool(tables)
        self.new_weight, self.var_floor = new_weight, var_floor
        n, K = bb.n, bb.K
        f32 = dict(dtype=torch.float32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        self.y = torch.from_numpy(np.ascontiguousarray(bb.y, np.int32)).to(self.device)
        self.N = torch.from_numpy(np.ascontiguousarray(bb.N, np.int32)).to(self.device)
        self.root_mean, self.root_var = torch.zeros(1, **f32), torch.ones(1, **f32)
        self.root_ema = torch.tensor([[0.0, 1.0]], **f64)
        self.q = torch.ones(n, 2, **f64)                                   # Beta(1, 1)
        self.g_ema = torch.tensor([[-1.0, -1.0]] * n, **f64)               # its (E ln p, E ln(1-p))
        self.mu, self.z = torch.empty(1, K, **f32), torch.empty(n, K, **f64)
        self.f_root = torch.empty(K, **f64)
        if self.tables:
            self.f = torch.empty(n, K, K, **f64)
        else:
            self.rows, self.cols = torch.empty(K, 3, **f64), torch.empty(n, K, 3, **f64)
        self.g, self.w = torch.empty(n, K, **f64), torch.empty(n, K, **f64)
        self.w_root, self.log_pe = torch.empty(K, **f64), torch.empty(1, **f64)
        self.root_m, self.gm = torch.empty(1, 2, **f64), torch.empty(n, 2, **f64)
        self.status = torch.zeros(n, dtype=torch.int32, device=self.device)
        self.clamps = torch.zeros(1, dtype=torch.int64, device=self.device)

    def step(self, t: int, seed: int, root_eps: Optional[torch.Tensor] = None, stream=None) -> None:
        bb, L, s = self.bb, lib(), _stream(stream)
        n, K = bb.n, bb.K
        check(L.qem_sample_normal(1, K, 0, seed, t, _ptr(self.root_mean), _ptr(self.root_var),
                                  _ptr(root_eps) if root_eps is not None else None, _ptr(self.mu), s),
              "qem_sample_normal")
        check(L.qem_sample_beta(n, K, seed, t, _ptr(self.q), _ptr(self.z), s), "qem_sample_beta")
        if self.tables:
            check(L.qem_tables_beta_binomial(n, K, float(bb.kappa), _ptr(self.mu), _ptr(self.root_mean),
                                             _ptr(self.root_var), _ptr(self.y), _ptr(self.N), _ptr(self.q),
                                             _ptr(self.z), _ptr(self.f_root), _ptr(self.f), s),
                  "qem_tables_beta_binomial")
            check(L.qem_estep_tables(n, K, _ptr(self.f_root), _ptr(self.f), _ptr(self.g), _ptr(self.log_pe),
                                     _ptr(self.w_root), _ptr(self.w), s), "qem_estep_tables")
        else:
            check(L.qem_cols_beta_binomial(n, K, float(bb.kappa), _ptr(self.mu), _ptr(self.root_mean),
                                           _ptr(self.root_var), _ptr(self.y), _ptr(self.N), _ptr(self.q), _ptr(self.z),
                                           _ptr(self.f_root), _ptr(self.rows), _ptr(self.cols), s),
                  "qem_cols_beta_binomial")
            check(L.qem_estep_separable(n, K, 2, _ptr(self.f_root), _ptr(self.rows), _ptr(self.cols), _ptr(self.g),
                                        _ptr(self.log_pe), _ptr(self.w_root), _ptr(self.w), s), "qem_estep_separable")
        check(L.qem_moments_beta(n, K, _ptr(self.w_root), _ptr(self.mu), _ptr(self.w), _ptr(self.z),
                                 _ptr(self.root_m), _ptr(self.gm), s), "qem_moments_beta")
        lam = L.qem_history_weight(int(t), float(self.new_weight), 0.0)
        check(L.qem_mstep_family(BETA, n, 1, lam, _ptr(self.gm), _ptr(self.g_ema), _ptr(self.q), _ptr(self.status),
                                 s), "qem_mstep_family")
        check(L.qem_mstep_gaussian(1, lam, self.var_floor, _ptr(self.root_m), _ptr(self.root_ema),
                                   _ptr(self.root_mean), _ptr(self.root_var), _ptr(self.clamps), s),
              "qem_mstep_gaussian")

    set_state = GammaPoissonQEM.set_state


class CrossedQEM:
    """QEM with crossed effects (NEXT row f4, R33) on synth.bus_crossed: one iteration =
    qem_sample_normal (root rows, level 0; group rows, level 1) + qem_tables_crossed +
    qem_estep_tables + qem_moments_gaussian + qem_mstep_categorical (n = 0: the Gaussian EMA +
    M-step of the root dims, then of the group latents), all on device."""

    def __init__(self, cm, *, new_weight=0.3, var_floor=1e-8, device="cuda", tables=True):
        """tables=True (default): the materialised fp64 tables (qem_tables_crossed + qem_estep_tables;
        n K^2 = 4 MB on the Bus shape, each pair's J-term sum evaluated once); False: qem_estep_crossed
        evaluates the K x K x J factor on chip, twice per pair (forward, backward) -- 3x the time here
        (R37)."""
        if not torch.cuda.is_available():
            raise _lib.QemError("CrossedQEM needs a CUDA device (there is no CPU fallback)")
        self.cm, self.device, self.tables = cm, torch.device(device), bool(tables)
        self.new_weight, self.var_floor = new_weight, var_floor
        n, K, R = cm.n, cm.K, cm.R
        f32 = dict(dtype=torch.float32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(self.device)  # noqa: E731
        self.comp, self.jtype, self.y = up(cm.comp, np.int32), up(cm.jtype, np.int32), up(cm.y, np.uint8)
        self.root_mean, self.root_var = torch.zeros(R, **f32), torch.ones(R, **f32)
        self.root_ema = torch.tensor([[0.0, 1.0]] * R, **f64)
        self.q_mean, self.q_var = torch.zeros(n, **f32), torch.ones(n, **f32)
        self.g_ema = torch.tensor([[0.0, 1.0]] * n, **f64)
        self.rz, self.z = torch.empty(R, K, **f32), torch.empty(n, K, **f32)
        self.f_root = torch.empty(K, **f64)
        self.f = torch.empty(n, K, K, **f64) if self.tables else None
        self.g, self.w = torch.empty(n, K, **f64), torch.empty(n, K, **f64)
        self.w_root, self.log_pe = torch.empty(K, **f64), torch.empty(1, **f64)
        self.root_m, self.gm = torch.empty(R, 2, **f64), torch.empty(n, 2, **f64)
        self.clamps = torch.zeros(1, dtype=torch.int64, device=self.device)

    def step(self, t: int, seed: int, root_eps: Optional[torch.Tensor] = None, eps: Optional[torch.Tensor] = None,
             stream=None) -> None:
        cm, L, s = self.cm, lib(), _stream(stream)
        n, K, R = cm.n, cm.K, cm.R
        check(L.qem_sample_normal(R, K, 0, seed, t, _ptr(self.root_mean), _ptr(self.root_var),
                                  _ptr(root_eps) if root_eps is not None else None, _ptr(self.rz), s),
              "qem_sample_normal")
        check(L.qem_sample_normal(n, K, 1, seed, t, _ptr(self.q_mean), _ptr(self.q_var),
                                  _ptr(eps) if eps is not None else None, _ptr(self.z), s), "qem_sample_normal")
        if self.tables:
            check(L.qem_tables_crossed(n, K, cm.J, cm.C, cm.T, _ptr(self.rz), _ptr(self.root_mean),
                                       _ptr(self.root_var), _ptr(self.z), _ptr(self.q_mean), _ptr(self.q_var),
                                       _ptr(self.comp), _ptr(self.jtype), _ptr(self.y), _ptr(self.f_root),
                                       _ptr(self.f), s), "qem_tables_crossed")
            check(L.qem_estep_tables(n, K, _ptr(self.f_root), _ptr(self.f), _ptr(self.g), _ptr(self.log_pe),
                                     _ptr(self.w_root), _ptr(self.w), s), "qem_estep_tables")
        else:
            check(L.qem_estep_crossed(n, K, cm.J, cm.C, cm.T, _ptr(self.rz), _ptr(self.root_mean), _ptr(self.root_var),
                                      _ptr(self.z), _ptr(self.q_mean), _ptr(self.q_var), _ptr(self.comp),
                                      _ptr(self.jtype), _ptr(self.y), _ptr(self.f_root), _ptr(self.g),
                                      _ptr(self.log_pe), _ptr(self.w_root), _ptr(self.w), s), "qem_estep_crossed")
        check(L.qem_moments_gaussian(n, K, R, _ptr(self.w_root), _ptr(self.rz), _ptr(self.w), _ptr(self.z),
                                     _ptr(self.root_m), _ptr(self.gm), s), "qem_moments_gaussian")
        lam = L.qem_history_weight(int(t), float(self.new_weight), 0.0)
        for m_new, ema, mean, var, d in ((self.root_m, self.root_ema, self.root_mean, self.root_var, R),
                                         (self.gm, self.g_ema, self.q_mean, self.q_var, n)):
            check(L.qem_mstep_gaussian(d, lam, self.var_floor, _ptr(m_new), _ptr(ema), _ptr(mean), _ptr(var),
                                       _ptr(self.clamps), s), "qem_mstep_gaussian")

    def set_state(self, st: dict) -> None:
        for k in ("root_mean", "root_var", "root_ema", "q_mean", "q_var", "g_ema"):
            getattr(self, k).copy_(torch.from_numpy(np.asarray(st[k])).to(getattr(self, k).dtype))
