"""ctypes binding of libqem.so (include/qem.h).  Argument marshalling only.

Loading fails loudly if the in-tree CUDA library is missing: there is no CPU
fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QEM_LIB_OVERRIDE") or os.path.join(HERE, "libqem.so")  # override: tuning experiments

FAMILY_TWO_LEVEL, FAMILY_THREE_LEVEL = 2, 3
OK, INVALID_ARGUMENT, INVALID_MODEL, UNSUPPORTED, CUDA_ERROR, NCCL_ERROR = 0, 1, 2, 3, 4, 5
NCCL_ID_BYTES = 128
FLAG_DEGENERATE, FLAG_NAN, FLAG_CLAMP = 1, 2, 4

# Every symbol include/qem.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "qem_model_validate", "qem_shard_range", "qem_create", "qem_workspace_bytes", "qem_create_in", "qem_destroy", "qem_bind", "qem_sample_q",
    "qem_estep", "qem_estep_forward", "qem_reduce_buffer", "qem_estep_reduce", "qem_estep_backward", "qem_estep_evidence",
    "qem_nccl_unique_id", "qem_nccl_init", "qem_set_nccl_comm", "qem_nccl_info",
    "qem_estep_separable", "qem_cols_gamma_poisson", "qem_cols_beta_binomial", "qem_mstep_gaussian",
    "qem_cols_qmp_gaussian", "qem_moments_qmp",
    "qem_history_weight", "qem_estep_crossed", "qem_sample_estep_forward",
    "qem_evidence_root", "qem_mstep", "qem_mstep_family", "qem_estep_tables", "qem_sample_normal",
    "qem_sample_categorical", "qem_tables_categorical", "qem_estep_categorical", "qem_moments_categorical", "qem_mstep_categorical",
    "qem_loglik_bernoulli_states", "qem_backward_resample", "qem_predictive_loglik", "qem_logmeanexp", "qem_global_iw", "qem_sample_gamma",
    "qem_tables_gamma_poisson", "qem_moments_gamma", "qem_sample_beta", "qem_tables_beta_binomial",
    "qem_moments_beta", "qem_tables_crossed", "qem_moments_gaussian", "qem_iterate",
    "qem_read_flags", "qem_read_mode_hist", "qem_set_kernel_events", "qem_kernel_launches", "qem_pair_path", "qem_copy_messages", "qem_status_str", "qem_last_error",
    "qem_version",
]


class ModelDesc(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("d", ctypes.c_int32), ("scale_kind", ctypes.c_int32),
                ("obs_kind", ctypes.c_int32), ("n", ctypes.c_int64), ("n_sub", ctypes.c_int32),
                ("n_obs", ctypes.c_int32), ("n_cov", ctypes.c_int32), ("K", ctypes.c_int32),
                ("fixed_var", ctypes.c_double), ("obs_var", ctypes.c_double), ("top_var", ctypes.c_double),
                ("sub_var", ctypes.c_double), ("prior_mean", ctypes.c_double), ("prior_var", ctypes.c_double)]


class Opts(ctypes.Structure):
    _fields_ = [("new_weight", ctypes.c_double), ("schedule_p", ctypes.c_double), ("var_floor", ctypes.c_double),
                ("fresh_denominator", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Level(ctypes.Structure):
    _fields_ = [("q_mean", ctypes.c_void_p), ("q_var", ctypes.c_void_p), ("ema_m1", ctypes.c_void_p),
                ("ema_v", ctypes.c_void_p), ("z", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("m1", ctypes.c_void_p), ("v", ctypes.c_void_p)]


class Buffers(ctypes.Structure):
    _fields_ = [("level", Level * 3), ("x", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("log_pe", ctypes.c_void_p), ("trace", ctypes.c_void_p), ("trace_len", ctypes.c_int64),
                ("plate_sum", ctypes.c_void_p), ("log_pe_fresh", ctypes.c_void_p),
                ("eps_bank", ctypes.c_void_p * 3), ("eps_bank_len", ctypes.c_int64)]


class QemError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QemError(f"{LIB_PATH} is missing: build it with `python -m paper_2503_08264_b200.build` "
                           "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        L.qem_model_validate.argtypes = [ctypes.POINTER(ModelDesc), ctypes.c_char_p, ctypes.c_size_t]
        L.qem_shard_range.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.qem_create.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(Opts), i64, i64, ctypes.POINTER(vp)]
        L.qem_workspace_bytes.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(Opts), i64, i64,
                                          ctypes.POINTER(ctypes.c_size_t)]
        L.qem_create_in.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(Opts), i64, i64, vp, ctypes.c_size_t,
                                    ctypes.POINTER(vp)]
        L.qem_estep_tables.argtypes = [i64, i32, vp, vp, vp, vp, vp, vp, vp]
        L.qem_estep_separable.argtypes = [i64, i32, i32] + [vp] * 8
        L.qem_sample_estep_forward.argtypes = [vp, u64, i32, vp]
        L.qem_estep_crossed.argtypes = [i64, i32, i32, i32, i32] + [vp] * 15
        L.qem_mstep_gaussian.argtypes = [i64, ctypes.c_double, ctypes.c_double] + [vp] * 6
        L.qem_history_weight.argtypes = [i32, ctypes.c_double, ctypes.c_double]
        L.qem_history_weight.restype = ctypes.c_double
        L.qem_cols_gamma_poisson.argtypes = [i64, i32, i32, ctypes.c_double] + [vp] * 10
        L.qem_cols_beta_binomial.argtypes = [i64, i32, ctypes.c_double] + [vp] * 11
        L.qem_cols_qmp_gaussian.argtypes = [i64, i32, i32, i32] + [ctypes.c_double] * 3 + [vp] * 12
        L.qem_moments_qmp.argtypes = [i64, i32] + [vp] * 7
        L.qem_sample_normal.argtypes = [i64, i32, i32, u64, i32, vp, vp, vp, vp, vp]
        L.qem_sample_categorical.argtypes = [i64, i32, i32, u64, i32, vp, vp, vp]
        L.qem_tables_categorical.argtypes = [i64, i32, i32, i32] + [vp] * 10
        L.qem_moments_categorical.argtypes = [i64, i32, i32, i32] + [vp] * 7
        L.qem_estep_categorical.argtypes = [i64, i32, i32, i32] + [vp] * 13
        L.qem_mstep_categorical.argtypes = [i64, i32, i32, ctypes.c_double, ctypes.c_double] + [vp] * 9
        L.qem_loglik_bernoulli_states.argtypes = [i64, i32, i32, vp, vp, vp, vp]
        L.qem_backward_resample.argtypes = [vp, i32, u64, vp, vp, vp]
        L.qem_predictive_loglik.argtypes = [vp, i32, vp, i32, vp, vp, vp, vp, vp, vp]
        L.qem_logmeanexp.argtypes = [i64, vp, vp, vp]
        L.qem_global_iw.argtypes = [vp] + [vp] * 6
        L.qem_sample_gamma.argtypes = [i64, i32, u64, i32, vp, vp, vp]
        L.qem_tables_gamma_poisson.argtypes = [i64, i32, i32, ctypes.c_double] + [vp] * 9
        L.qem_moments_gamma.argtypes = [i64, i32] + [vp] * 7
        L.qem_sample_beta.argtypes = [i64, i32, u64, i32, vp, vp, vp]
        L.qem_tables_beta_binomial.argtypes = [i64, i32, ctypes.c_double] + [vp] * 10
        L.qem_moments_beta.argtypes = [i64, i32] + [vp] * 7
        L.qem_tables_crossed.argtypes = [i64, i32, i32, i32, i32] + [vp] * 12
        L.qem_moments_gaussian.argtypes = [i64, i32, i32] + [vp] * 7
        L.qem_destroy.argtypes = [vp]
        L.qem_destroy.restype = None
        L.qem_bind.argtypes = [vp, ctypes.POINTER(Buffers)]
        L.qem_sample_q.argtypes = [vp, u64, i32, ctypes.POINTER(vp), vp]
        L.qem_estep.argtypes = [vp, vp]
        L.qem_estep_forward.argtypes = [vp, vp]
        L.qem_estep_backward.argtypes = [vp, vp]
        L.qem_reduce_buffer.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(i64)]
        L.qem_estep_reduce.argtypes = [vp, vp]
        L.qem_nccl_unique_id.argtypes = [vp]
        L.qem_nccl_init.argtypes = [vp, vp, i32, i32]
        L.qem_set_nccl_comm.argtypes = [vp, vp]
        L.qem_nccl_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.qem_mstep.argtypes = [vp, i32, vp]
        L.qem_mstep_family.argtypes = [i32, i64, i32, ctypes.c_double, vp, vp, vp, vp, vp]
        L.qem_mstep_family.restype = i32
        L.qem_estep_evidence.argtypes = [vp, vp]
        L.qem_evidence_root.argtypes = [vp, vp]
        L.qem_iterate.argtypes = [vp, i32, i32, u64, i32, vp]
        L.qem_read_flags.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(i64)]
        L.qem_read_mode_hist.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.qem_set_kernel_events.argtypes = [vp, vp, vp, vp, vp]
        L.qem_set_kernel_events.restype = i32
        L.qem_kernel_launches.argtypes = [vp]
        L.qem_kernel_launches.restype = i64
        L.qem_pair_path.argtypes = [vp]
        L.qem_pair_path.restype = i32
        L.qem_copy_messages.argtypes = [vp, vp, vp, vp]
        L.qem_status_str.argtypes = [i32]
        L.qem_status_str.restype = ctypes.c_char_p
        L.qem_last_error.restype = ctypes.c_char_p
        L.qem_version.restype = ctypes.c_char_p
        for name in ["qem_model_validate", "qem_shard_range", "qem_create", "qem_bind", "qem_sample_q", "qem_estep",
                     "qem_estep_forward", "qem_estep_backward", "qem_reduce_buffer", "qem_mstep", "qem_iterate",
                     "qem_estep_reduce", "qem_nccl_unique_id", "qem_nccl_init", "qem_set_nccl_comm", "qem_nccl_info",
                     "qem_read_flags", "qem_read_mode_hist", "qem_copy_messages", "qem_estep_evidence",
                     "qem_evidence_root", "qem_workspace_bytes", "qem_create_in", "qem_estep_tables",
                     "qem_sample_normal", "qem_sample_categorical", "qem_tables_categorical", "qem_estep_categorical",
                     "qem_moments_categorical", "qem_mstep_categorical", "qem_loglik_bernoulli_states",
                     "qem_backward_resample", "qem_predictive_loglik", "qem_logmeanexp", "qem_global_iw",
                     "qem_sample_gamma",
                     "qem_tables_gamma_poisson", "qem_moments_gamma", "qem_sample_beta",
                     "qem_tables_beta_binomial", "qem_moments_beta", "qem_tables_crossed",
                     "qem_moments_gaussian", "qem_estep_separable", "qem_cols_gamma_poisson",
                     "qem_cols_beta_binomial", "qem_mstep_gaussian", "qem_estep_crossed",
                     "qem_sample_estep_forward", "qem_cols_qmp_gaussian", "qem_moments_qmp"]:
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status != OK:
        L = lib()
        raise QemError(f"{what}: {L.qem_status_str(status).decode()}: {L.qem_last_error().decode()}")
