"""ctypes binding of the C-ABI library ``libpier_b200.so`` (include/pier_b200.h).

The product has no CPU fallback: if the library is missing the import of the
package fails loudly, and every entry point refuses tensors that are not on a
CUDA device.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, ProtocolError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpier_b200.so")

PIER_OK = 0
PIER_EINVAL = -1
PIER_ECUDA = -2
PIER_ENCCL = -3
PIER_EPROTOCOL = -4
PIER_ENOMEM = -5
PIER_EABORTED = -6


class PierCudaError(RuntimeError):
    """A CUDA or NCCL call inside the extension failed."""


class GroupAborted(RuntimeError):
    """Another rank of a virtual group failed and aborted the group's
    collectives (the reference's BrokenBarrierError, driver.py:494-501)."""


class PierAdamW(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double), ("step", C.c_int64)]


class PierClip(C.Structure):
    _fields_ = [("sqnorm", C.c_double), ("norm", C.c_double), ("scale", C.c_double),
                ("clipped", C.c_int32), ("nonfinite", C.c_int32)]


class PierTensorDesc(C.Structure):
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("exp_avg", C.c_void_p),
                ("exp_avg_sq", C.c_void_p), ("numel", C.c_int64)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
SZ = C.c_size_t
INT = C.c_int

# name -> (restype, argtypes); the exact list include/pier_b200.h declares
SIGNATURES = {
    "pier_last_error": (C.c_char_p, []),
    "pier_version": (INT, []),
    "pier_device_sm_count": (INT, [INT]),
    "pier_launch_count": (C.c_ulonglong, []),
    "pier_device_sync": (INT, []),
    "pier_pseudograd_f32": (INT, [P, P, P, I64, P]),
    "pier_pseudograd_f64": (INT, [P, P, P, I64, P]),
    "pier_fold_momentum_f32": (INT, [P, P, P, I64, D, P]),
    "pier_fold_momentum_f64": (INT, [P, P, P, I64, D, P]),
    "pier_outer_step_f32": (INT, [P, P, P, P, P, P, I64, D, D, P]),
    "pier_outer_step_f64": (INT, [P, P, P, P, P, P, I64, D, D, P]),
    "pier_outer_update_f32": (INT, [P, P, P, P, I64, D, D, I32, P]),
    "pier_outer_update_f64": (INT, [P, P, P, P, I64, D, D, I32, P]),
    "pier_warmup_fold_f32": (INT, [P, P, P, I64, D, P]),
    "pier_warmup_fold_f64": (INT, [P, P, P, I64, D, P]),
    "pier_mean_left_fold_f32": (INT, [P, I32, P, I64, P]),
    "pier_mean_left_fold_f64": (INT, [P, I32, P, I64, P]),
    "pier_norm_ws_bytes": (SZ, []),
    "pier_grad_sqnorm_f32": (INT, [P, I64, D, P, P]),
    "pier_grad_sqnorm_f64": (INT, [P, I64, D, P, P]),
    "pier_clip_finalize": (INT, [P, D, I32, P]),
    "pier_apply_clip_f32": (INT, [P, P, I64, P, P]),
    "pier_apply_clip_f64": (INT, [P, P, I64, P, P]),
    "pier_adamw_f32": (INT, [P, P, P, P, I64, C.POINTER(PierAdamW), P, P]),
    "pier_adamw_f64": (INT, [P, P, P, P, I64, C.POINTER(PierAdamW), P, P]),
    "pier_adamw_outer_f32": (INT, [P, P, P, P, P, P, I64, C.POINTER(PierAdamW), P, D, D, P]),
    "pier_adamw_outer_f64": (INT, [P, P, P, P, P, P, I64, C.POINTER(PierAdamW), P, D, D, P]),
    "pier_adamw_bf16_f32": (INT, [P, P, P, P, P, I64, C.POINTER(PierAdamW), P, P]),
    "pier_grad_sqnorm_bf16": (INT, [P, I64, D, P, P]),
    "pier_cast_bf16": (INT, [P, P, I64, P]),
    "pier_kernel_tune": (INT, [INT, INT]),
    "pier_tensor_list_create": (INT, [C.POINTER(PierTensorDesc), I32, I32, C.POINTER(P)]),
    "pier_tensor_list_destroy": (INT, [P]),
    "pier_grad_sqnorm_mt": (INT, [P, D, P, P]),
    "pier_adamw_mt": (INT, [P, C.POINTER(PierAdamW), P, P]),
    "pier_momentum_mu": (D, [I64, I64]),
    "pier_outer_lr": (INT, [I64, I64, C.POINTER(D)]),
    "pier_nccl_unique_id_bytes": (INT, []),
    "pier_nccl_get_unique_id": (INT, [P]),
    "pier_comm_init": (INT, [P, I32, I32, C.POINTER(P)]),
    "pier_comm_destroy": (INT, [P]),
    "pier_vgroup_create": (INT, [I32, C.POINTER(P)]),
    "pier_vgroup_abort": (INT, [P]),
    "pier_comm_is_virtual": (INT, [P]),
    "pier_comm_set_timeout": (INT, [P, D]),
    "pier_comm_diag": (INT, [P, C.POINTER(C.c_uint32)]),
    "pier_outer_step_sharded_f32": (INT, [P, P, P, P, I64, I64, D, D, P]),
    "pier_warmup_fold_sharded_f32": (INT, [P, P, P, P, I64, I64, D, P]),
    "pier_allreduce_mean_f32": (INT, [P, P, I64, I64, P]),
    "pier_shard_allgather_f32": (INT, [P, P, P, I64, I64, P]),
    "pier_allreduce_mean_bf16": (INT, [P, P, I64, I64, P]),
    "pier_comm_alloc_shared": (INT, [P, SZ, C.POINTER(P), C.POINTER(I32)]),
    "pier_comm_free_shared": (INT, [P, I32]),
    "pier_outer_step_p2p_f32": (INT, [P, I32, P, P, I64, I64, D, D, P]),
    "pier_outer_step_p2p_region_f32": (INT, [P, I32, I64, I64, P, P, I64, D, D, P]),
    "pier_outer_step_p2p_reps_f32": (INT, [P, I32, P, I32, P, P, P, I64, I64, D, D, P]),
    "pier_allreduce_mean_p2p_f32": (INT, [P, I32, I64, P]),
    "pier_allreduce_mean_norm_p2p_f32": (INT, [P, I32, I64, D, P, P]),
    "pier_lazy_step_p2p_f32": (INT, [P, I32, I32, P, P, I64, I64, C.POINTER(PierAdamW), D, P, P]),
    "pier_gather_p2p_f32": (INT, [P, I32, I64, I64, P]),
    "pier_lazy_step_p2p_team_f32": (INT, [P, I32, I32, P, I32, P, I32, P, P, I64, I64, C.POINTER(PierAdamW), D, P,
                                          P]),
    "pier_gather_p2p_team_f32": (INT, [P, I32, P, I32, I64, I64, P]),
    "pier_lazy_step_p2p_bf16": (INT, [P, I32, I32, I32, P, P, I64, I64, C.POINTER(PierAdamW), D, P, P]),
    "pier_lazy_pull_span_p2p_f32": (INT, [P, I32, P, I32, P, I64, I64, I32, P]),
    "pier_lazy_finish_staged_p2p_f32": (INT, [P, I32, I32, P, I32, P, I32, P, P, P, I64, I64, C.POINTER(PierAdamW),
                                              D, P, I32, P]),
    "pier_allgather_span_p2p_f32": (INT, [P, I32, P, I32, I64, I64, I32, P]),
    "pier_lazy_pull_span_p2p_bf16": (INT, [P, I32, P, I64, I64, I32, P]),
    "pier_lazy_finish_staged_p2p_bf16": (INT, [P, I32, I32, I32, P, P, P, I64, I64, C.POINTER(PierAdamW), D, P, P]),
    "pier_p2p_tune": (INT, [INT, INT, INT]),
    "pier_round_tune": (INT, [INT, INT]),
    "pier_round_split": (INT, [INT, INT]),
    "pier_outer_step_p2p_team_f32": (INT, [P, I32, P, I32, P, P, I64, I64, D, D, P]),
    "pier_allreduce_mean_p2p_team_f32": (INT, [P, I32, P, I32, I64, P]),
    "pier_allreduce_mean_p2p_bf16": (INT, [P, I32, I64, P]),
    "pier_allreduce_mean_norm_p2p_bf16": (INT, [P, I32, I64, D, P, P]),
    "pier_norm_allreduce_team": (INT, [P, P, I32, P, D, P]),
    "pier_round_fused_team_f32": (INT, [P, I32, P, I32, P, P, P, P, P, I64, I64, C.POINTER(PierAdamW), P, D, D,
                                        P]),
    "pier_round_sig_bytes": (SZ, []),
    "pier_p2p_virtual_f32": (INT, [I32, I32, P, P, P, I64, I64, D, D, P]),
    "pier_round_virtual_f32": (INT, [I32, P, P, P, P, P, P, P, I64, I64, C.POINTER(PierAdamW), P, D, D, I32, I32,
                                     P]),
    "pier_round_fused_f32": (INT, [P, I32, P, P, P, P, P, I64, I64, C.POINTER(PierAdamW), P, D, D, P]),
    "pier_round_fused_bf16_f32": (INT, [P, I32, P, P, P, P, P, I64, I64, C.POINTER(PierAdamW), P, D, D, P]),
    "pier_comm_alloc_window": (INT, [P, SZ, C.POINTER(P), C.POINTER(I32)]),
    "pier_outer_step_nvls_f32": (INT, [P, I32, P, P, I64, I64, D, D, P]),
    "pier_round_nvls_f32": (INT, [P, I32, P, P, P, P, P, I64, I64, C.POINTER(PierAdamW), P, D, D, P]),
    "pier_allreduce_mean_nvls_f32": (INT, [P, I32, I64, P]),
    "pier_round_p2p_f32": (INT, [P, I32, P, P, P, P, P, I64, I64, C.POINTER(PierAdamW), P, D, D, P]),
    "pier_offload_create": (INT, [I32, SZ, C.POINTER(P)]),
    "pier_offload_destroy": (INT, [P]),
    "pier_offload_park": (INT, [P, I32, P, SZ, P]),
    "pier_offload_fetch": (INT, [P, I32, P, SZ, P]),
    "pier_offload_prefetch": (INT, [P, I32, P, SZ, P]),
    "pier_offload_wait": (INT, [P, I32, P]),
    "pier_offload_sync": (INT, [P]),
    "pier_offload_counters": (INT, [P, C.POINTER(D)]),
    "pier_offload_host_ptr": (P, [P, I32]),
    "pier_offload_stream": (P, [P]),
    "pier_offload_stream_h2d": (P, [P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.pier_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a C status code to the reference's exception types (errors.py:4-23)."""
    if rc == PIER_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == PIER_EINVAL:
        raise ConfigError(msg)
    if rc == PIER_EPROTOCOL:
        raise ProtocolError(msg)
    if rc == PIER_ENOMEM:
        raise MemoryError(msg)
    if rc == PIER_EABORTED:
        raise GroupAborted(msg)
    raise PierCudaError(msg)
