"""ctypes binding of the in-tree C ABI libraries.

``libmimose_cuda.so`` (include/mimose_cuda.h) is the device side: budget
arena, sm_100a kernels, layer executor, trainer. ``libmimose_host.so``
(include/mimose_planner.h) is the host planner over include/mimose/*.hpp.

There is no fallback: if a library is missing, loading raises. Run
``make`` (or ``__graft_entry__.build()``) first.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MIMOSE_CUDA_LIB: alternate in-tree build (A/B kernel timing in tools/ only)
CUDA_LIB_PATH = os.environ.get("MIMOSE_CUDA_LIB", os.path.join(_HERE, "libmimose_cuda.so"))
HOST_LIB_PATH = os.path.join(_HERE, "libmimose_host.so")

_cuda = None
_host = None


class MimoseError(RuntimeError):
    pass


NUM_TAGS = 8
TAGS = ["param", "grad", "optim", "act", "boundary", "transient", "input", "other"]


class MemStats(C.Structure):
    _fields_ = [
        ("budget", C.c_int64),
        ("reserved", C.c_int64),
        ("peak_reserved", C.c_int64),
        ("requested", C.c_int64),
        ("peak_requested", C.c_int64),
        ("largest_free", C.c_int64),
        ("n_live", C.c_int64),
        ("n_allocs", C.c_int64),
        ("n_failures", C.c_int64),
        ("tag_requested", C.c_int64 * NUM_TAGS),
        ("tag_peak", C.c_int64 * NUM_TAGS),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("tag_")}
        d["tag_requested"] = {TAGS[i]: self.tag_requested[i] for i in range(NUM_TAGS)}
        d["tag_peak"] = {TAGS[i]: self.tag_peak[i] for i in range(NUM_TAGS)}
        return d


class GemmArgs(C.Structure):
    _fields_ = [
        ("M", C.c_int), ("N", C.c_int), ("K", C.c_int), ("nb1", C.c_int), ("nb2", C.c_int),
        ("a", C.c_void_p), ("a_rows", C.c_int64), ("a_cols", C.c_int64), ("lda", C.c_int64),
        ("a_bs1", C.c_int64), ("a_bs2", C.c_int64), ("a_mn", C.c_int),
        ("b", C.c_void_p), ("b_rows", C.c_int64), ("b_cols", C.c_int64), ("ldb", C.c_int64),
        ("b_bs1", C.c_int64), ("b_bs2", C.c_int64), ("b_mn", C.c_int),
        ("epi", C.c_int),
        ("out", C.c_void_p), ("out2", C.c_void_p), ("aux", C.c_void_p), ("bias", C.c_void_p),
        ("ldo", C.c_int64), ("obs1", C.c_int64), ("obs2", C.c_int64),
        ("alpha", C.c_float), ("beta", C.c_float),
        ("force_bn", C.c_int), ("direct_store", C.c_int),
        ("split_k", C.c_int), ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64),
        ("force_ew", C.c_int), ("force_cg", C.c_int),
        ("rowsum", C.c_void_p),
    ]


class ModelCfg(C.Structure):
    _fields_ = [
        ("layers", C.c_int), ("hidden", C.c_int), ("heads", C.c_int), ("ffn", C.c_int),
        ("vocab", C.c_int), ("max_pos", C.c_int), ("type_vocab", C.c_int),
        ("num_choices", C.c_int),
        ("hidden_dropout", C.c_float), ("attn_dropout", C.c_float), ("ln_eps", C.c_float),
        ("init_std", C.c_float),
        ("seed", C.c_uint64),
        ("arch", C.c_int), ("head", C.c_int), ("causal", C.c_int), ("gelu_tanh", C.c_int),
        ("pad_token_id", C.c_int),
    ]


class TrainCfg(C.Structure):
    _fields_ = [
        ("planner", C.c_int), ("batch", C.c_int), ("seq_min", C.c_int), ("seq_max", C.c_int),
        ("reserve_bytes", C.c_int64),
        ("bucket_tolerance", C.c_double), ("cache_tolerance", C.c_double),
        ("max_sheltered_iters", C.c_int), ("collect_new_sizes_always", C.c_int),
        ("estimator_order", C.c_int),
        ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
        ("weight_decay", C.c_float), ("max_grad_norm", C.c_float),
        ("attn_fused", C.c_int), ("reserve_per_size", C.c_int), ("ckpt_unit", C.c_int),
        ("ffn_regen_g", C.c_int),
    ]


class StepReport(C.Structure):
    _fields_ = [
        ("iter", C.c_int64), ("x", C.c_int64), ("batch", C.c_int), ("seq", C.c_int),
        ("phase", C.c_int), ("cache_hit", C.c_int), ("plan_size", C.c_int),
        ("insufficient", C.c_int), ("fit_order", C.c_int), ("loss", C.c_float),
        ("peak_requested", C.c_int64), ("peak_reserved", C.c_int64),
        ("predicted_kept", C.c_int64), ("budget", C.c_int64),
        ("plan_us", C.c_double), ("fit_us", C.c_double),
        ("dropped_mask_lo", C.c_uint64),
        ("pred_err_mean", C.c_double), ("pred_err_max", C.c_double), ("pred_layers", C.c_int),
        ("host_ms", C.c_double), ("reserve_bytes", C.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


GRAD_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
DP_REDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p)

_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)

class LayerIO(C.Structure):
    _fields_ = [
        ("tokens", C.c_void_p), ("types", C.c_void_p), ("labels", C.c_void_p),
        ("perm", C.c_void_p), ("seg", C.c_void_p), ("uid", C.c_void_p), ("n_unique", C.c_int),
        ("batch", C.c_int), ("seq", C.c_int), ("step", C.c_int64),
    ]


class AttnArgs(C.Structure):
    _fields_ = [
        ("B", C.c_int), ("S", C.c_int), ("nh", C.c_int), ("causal", C.c_int),
        ("scale", C.c_float), ("dropout_p", C.c_float),
        ("seed", C.c_uint64), ("stream_id", C.c_uint64),
        ("qkv", C.c_void_p), ("ctx", C.c_void_p), ("lse", C.c_void_p), ("keep_mask", C.c_void_p),
        ("dctx", C.c_void_p), ("dqkv", C.c_void_p),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64),
    ]


# (name, restype, argtypes) for every symbol include/mimose_cuda.h declares.
CUDA_SYMBOLS = [
    ("mimose_abi_version", C.c_int, []),
    ("mimose_last_error", C.c_char_p, []),
    ("mimose_launch_count", C.c_uint64, []),
    ("mimose_ctx_create", C.c_int, [C.c_int, C.c_int64, C.POINTER(C.c_void_p)]),
    ("mimose_ctx_destroy", C.c_int, [C.c_void_p]),
    ("mimose_alloc", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]),
    ("mimose_free", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mimose_mem_stats_get", C.c_int, [C.c_void_p, C.POINTER(MemStats)]),
    ("mimose_mem_reset_peak", C.c_int, [C.c_void_p]),
    ("mimose_book_create", C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    ("mimose_book_destroy", C.c_int, [C.c_void_p]),
    ("mimose_book_alloc", C.c_int64, [C.c_void_p, C.c_int64, C.c_int]),
    ("mimose_book_free", C.c_int, [C.c_void_p, C.c_int64]),
    ("mimose_book_stats", C.c_int, [C.c_void_p, C.POINTER(MemStats)]),
    ("mimose_gemm", C.c_int, [C.POINTER(GemmArgs), C.c_void_p]),
    ("mimose_flash_attn_fwd", C.c_int, [C.POINTER(AttnArgs), C.c_void_p]),
    ("mimose_flash_attn_bwd", C.c_int, [C.POINTER(AttnArgs), C.c_void_p]),
    ("mimose_gemm_profile_enable", C.c_int, [C.c_int]),
    ("mimose_gemm_profile_csv", C.c_int, [C.POINTER(C.c_void_p)]),
    ("mimose_gemm_profile_read", C.c_int,
     [C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    ("mimose_profile_enable", C.c_int, [C.c_int]),
    ("mimose_profile_read", C.c_int,
     [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
      C.POINTER(C.c_int64)]),
    ("mimose_profile_csv", C.c_int, [C.POINTER(C.c_void_p)]),
    ("mimose_trainer_create", C.c_int,
     [_P, C.POINTER(ModelCfg), C.POINTER(TrainCfg), C.POINTER(C.c_void_p)]),
    ("mimose_trainer_destroy", C.c_int, [_P]),
    ("mimose_trainer_step", C.c_int,
     [_P, _P, _P, _P, C.c_int, C.c_int, _P, C.POINTER(StepReport)]),
    ("mimose_trainer_step_async", C.c_int,
     [_P, _P, _P, _P, C.c_int, C.c_int, _P, C.POINTER(StepReport)]),
    ("mimose_trainer_loss", C.c_int, [_P, C.c_int64, C.POINTER(C.c_float)]),
    ("mimose_trainer_forward_backward", C.c_int,
     [_P, _P, _P, _P, C.c_int, C.c_int, _P, C.POINTER(StepReport)]),
    ("mimose_trainer_step_device", C.c_int,
     [_P, _P, _P, _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P,
      C.POINTER(StepReport)]),
    ("mimose_trainer_optimizer_step", C.c_int, [_P, C.c_float, _P]),
    ("mimose_trainer_force_plan", C.c_int, [_P, C.POINTER(C.c_int), C.c_int, C.c_int]),
    ("mimose_trainer_set_grad_hook", C.c_int, [_P, GRAD_HOOK, _P]),
    ("mimose_trainer_buffers", C.c_int,
     [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(C.c_int64),
      C.POINTER(_P), C.POINTER(_P)]),
    ("mimose_trainer_param_count", C.c_int, [_P]),
    ("mimose_trainer_param_info", C.c_int,
     [_P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("mimose_trainer_sync_params", C.c_int, [_P, _P]),
    ("mimose_trainer_samples_csv", C.c_int, [_P, C.POINTER(_P)]),
    ("mimose_trainer_estimator_text", C.c_int, [_P, C.POINTER(_P)]),
    ("mimose_trainer_model_text", C.c_int, [_P, C.POINTER(_P)]),
    ("mimose_trainer_report", C.c_int, [_P, C.POINTER(_P), C.POINTER(_P)]),
    ("mimose_trainer_info", C.c_int,
     [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
      C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("mimose_free_string", None, [_P]),
    ("mimose_build_token_tables", C.c_int,
     [_P, C.c_int64, C.c_int, _P, _P, _P, C.POINTER(C.c_int)]),
    ("mimose_trainer_units", C.c_int, [_P, C.POINTER(C.c_int)]),
    ("mimose_embed_fwd", C.c_int, [_P, C.POINTER(LayerIO), C.POINTER(_P), C.POINTER(_P), _P]),
    ("mimose_layer_fwd", C.c_int, [_P, C.c_int, C.POINTER(LayerIO), _P, _P, C.POINTER(_P), _P]),
    ("mimose_layer_recompute", C.c_int,
     [_P, C.c_int, C.POINTER(LayerIO), _P, _P, C.POINTER(_P), _P]),
    ("mimose_layer_release", C.c_int, [_P, C.c_int]),
    ("mimose_layer_bwd", C.c_int,
     [_P, C.c_int, C.POINTER(LayerIO), _P, _P, _P, C.POINTER(_P), _P]),
    ("mimose_head_fwd_bwd", C.c_int, [_P, C.POINTER(LayerIO), _P, C.POINTER(_P), _P]),
    ("mimose_embed_bwd", C.c_int, [_P, C.POINTER(LayerIO), _P, _P, _P, _P]),
    ("mimose_saved_free", C.c_int, [_P, _P]),
    ("mimose_adamw_step", C.c_int, [_P, C.c_float, _P]),
    ("mimose_event_create", C.c_int, [C.POINTER(_P)]),
    ("mimose_event_record", C.c_int, [_P, _P]),
    ("mimose_event_elapsed", C.c_int, [_P, _P, C.POINTER(C.c_float)]),
    ("mimose_event_destroy", C.c_int, [_P]),
    ("mimose_dp_unique_id", C.c_int, [_P]),
    ("mimose_dp_create", C.c_int, [C.c_int, _P, C.c_int, C.c_int, C.POINTER(_P)]),
    ("mimose_dp_create_custom", C.c_int,
     [C.c_int, C.c_int, C.c_int, DP_REDUCE, _P, C.POINTER(_P)]),
    ("mimose_dp_device_bytes", C.c_int, [_P, C.POINTER(C.c_int64)]),
    ("mimose_dp_destroy", C.c_int, [_P]),
    ("mimose_dp_allreduce", C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_int, _P]),
    ("mimose_trainer_attach_dp", C.c_int, [_P, _P, C.c_int64]),
    ("mimose_trainer_dp_buckets", C.c_int,
     [_P, C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int)]),
    ("mimose_dp_plan_buckets", C.c_int,
     [C.POINTER(C.c_int64), C.c_int, C.c_int64, C.POINTER(C.c_int64), C.c_int,
      C.POINTER(C.c_int)]),
]

ABI_VERSION = 7


def _bind(lib, symbols):
    for name, res, args in symbols:
        fn = getattr(lib, name)  # AttributeError == missing export: fail loudly
        fn.restype = res
        fn.argtypes = args


def cuda_lib():
    """Load libmimose_cuda.so (raises if it was not built)."""
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB_PATH):
            raise MimoseError(f"{CUDA_LIB_PATH} missing: run `make` (no CPU fallback exists)")
        lib = C.CDLL(CUDA_LIB_PATH)
        _bind(lib, CUDA_SYMBOLS)
        if lib.mimose_abi_version() != ABI_VERSION:
            raise MimoseError(f"{CUDA_LIB_PATH}: ABI {lib.mimose_abi_version()} != {ABI_VERSION}"
                              " (stale build: run make)")
        _cuda = lib
    return _cuda


def check(rc, lib=None):
    if rc != 0:
        lib = lib or cuda_lib()
        raise MimoseError(lib.mimose_last_error().decode())
    return rc


def take_string(lib, ptr):
    """Copy a library-allocated C string and free it."""
    try:
        return C.cast(ptr, C.c_char_p).value.decode()
    finally:
        lib.mimose_free_string(ptr)
