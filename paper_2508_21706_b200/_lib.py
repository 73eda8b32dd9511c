"""ctypes binding of libspecmoe.so (include/specmoe/c_api.h).

The library is the product: there is no fallback. If the shared object is
missing or a CUDA device is absent, every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPECMOE_LIB", os.path.join(HERE, "libspecmoe.so"))

SMO_OK, SMO_INVALID_ARG, SMO_CAPACITY, SMO_CUDA, SMO_NCCL, SMO_UNSUPPORTED = range(6)
EPI_BF16, EPI_F32, EPI_F32_ADD, EPI_SWIGLU, EPI_ARGMAX = range(5)
INIT_UNIFORM, INIT_GAUSSIAN = 0, 1  # smo_model_config.expert_init
ENGINE_DEBUG = 1

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_f32 = C.c_float
_sz = C.c_size_t


class SmoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class CapacityError(SmoError):
    """moeplan::CapacityError (memory.hpp:15) surfaced through the C-ABI."""


class AttnArgs(C.Structure):
    _fields_ = [("q", _vp), ("k_cache", _vp), ("v_cache", _vp), ("mask", _vp), ("prefix_len", _vp),
                ("out", _vp), ("b", _i32), ("n", _i32), ("n_q", _i32), ("n_kv", _i32), ("d", _i32),
                ("s_max", _i32), ("max_prefix", _i32), ("workspace", _vp), ("workspace_bytes", _sz),
                ("block_table", _vp), ("max_pages", _i32), ("num_pages", _i32)]


class GemmArgs(C.Structure):
    _fields_ = [("x", _vp), ("rows", _i32), ("K", _i32), ("N", _i32), ("groups", _i32),
                ("row_offsets", _vp), ("max_rows_per_group", _i32), ("w", _vp), ("w_up", _vp),
                ("w_block_stride", _u64), ("w_pool_blocks", _i32), ("w_index", _vp), ("epilogue", _i32),
                ("out", _vp), ("ldo", _i64), ("argmax_val", _vp), ("argmax_idx", _vp), ("split_k", _i32),
                ("workspace", _vp), ("workspace_bytes", _sz)]


class ModelConfig(C.Structure):
    _fields_ = [("hidden", _i32), ("inter", _i32), ("n_expert", _i32), ("top_k", _i32), ("n_layers", _i32),
                ("n_q_heads", _i32), ("n_kv_heads", _i32), ("head_dim", _i32), ("vocab", _i32),
                ("rope_theta", _f32), ("rms_eps", _f32), ("seed", _u64), ("lm_scale", _f32),
                ("router_scale", _f32), ("shared_inter", _i32), ("draft_layers", _i32), ("draft_inter", _i32),
                ("expert_init", _i32)]


class EngineOptions(C.Structure):
    _fields_ = [("max_batch", _i32), ("max_verify", _i32), ("max_seq", _i32), ("hbm_slots", _i32),
                ("expert_cache_bytes", _i64), ("host_alias_layers", _i32), ("device", _i32), ("flags", _i32),
                ("ep_rank", _i32), ("ep_size", _i32), ("nccl_comm", _vp), ("kv_pages", _i32),
                ("attn_cpu", _i32), ("moe_batching", _i32),
                ("compress_experts", _i32), ("micro_batches", _i32), ("draft_cpu_kv", _i32)]


class StreamerArgs(C.Structure):
    _fields_ = [("n_layers", _i32), ("n_experts", _i32), ("block_bytes", _u64), ("host_blocks", _vp),
                ("host_bytes", _vp), ("host_codes", _vp), ("hbm_slots", _i32), ("cache_bytes", _i64),
                ("device", _i32)]


class VerifyBatch(C.Structure):
    _fields_ = [("b", _i32), ("n", _i32), ("tokens", _vp), ("parent", _vp), ("prefix_len", _vp),
                ("on_device", _i32)]


class VerifyOutput(C.Structure):
    _fields_ = [("acc_len", _vp), ("bonus", _vp), ("keep", _vp), ("target", _vp), ("on_device", _i32)]


class StageTimes(C.Structure):
    _fields_ = [("target_total", C.c_double), ("attention", C.c_double), ("gpu_moe", C.c_double),
                ("h2d_transfer", C.c_double), ("others", C.c_double), ("h2d_bytes", C.c_double),
                ("launches", C.c_double), ("draft", C.c_double), ("h2d_raw_bytes", C.c_double),
                ("codec", C.c_double), ("codec_bytes", C.c_double), ("link_code", C.c_double),
                ("host_numa", C.c_double), ("code_bits", C.c_double)]


_SIGS = {
    "smo_last_error": (C.c_char_p, []),
    "smo_version": (C.c_char_p, []),
    "smo_launch_count": (_u64, []),
    "smo_device_sm_count": (C.c_int, [C.c_int]),
    "smo_fill_uniform_bf16": (C.c_int, [_vp, _u64, _u64, _u64, _u64, _f32, _vp]),
    "smo_fill_normal_bf16": (C.c_int, [_vp, _u64, _u64, _u64, _u64, _f32, _vp]),
    "smo_verify_attention_workspace": (_sz, [C.POINTER(AttnArgs)]),
    "smo_verify_attention": (C.c_int, [C.POINTER(AttnArgs), _vp]),
    "smo_cpu_verify_attention": (C.c_int, [C.POINTER(AttnArgs), _i32]),
    "smo_expert_code_bytes": (_sz, [_u64, _i32]),
    "smo_expert_coded_size": (_u64, [_vp, _u64, _i32]),
    "smo_expert_encode": (C.c_int, [_vp, _u64, _i32, _vp, _vp, _vp]),
    "smo_expert_decode": (C.c_int, [_vp, _u64, _i32, _vp, _vp]),
    "smo_tcode_max_bytes": (_sz, [_i32, _i32]),
    "smo_engine_set_draft_split": (C.c_int, [_vp, _i32]),
    "smo_engine_draft_split_times": (C.c_int, [_vp, _vp, _sz, _vp]),
    "smo_tcode_encode": (C.c_int, [_vp, _i32, _i32, _vp, _vp, _vp]),
    "smo_tcode_decode": (C.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "smo_moe_experts_coded": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "smo_tcode3_encode": (C.c_int, [_vp, _i32, _i32, _vp, _vp, _vp]),
    "smo_tcode3_decode": (C.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "smo_moe_experts_coded3": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "smo_chunked_attention_f64": (C.c_int, [_sz, _sz, _sz, _vp, _vp, _vp, _sz, _vp, _vp]),
    "smo_router_topk": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "smo_permute": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    "smo_unpermute_combine": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "smo_unpermute_combine_split": (C.c_int, [_vp, _i32, _u64, _vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "smo_moe_experts": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _u64, _i32, _vp, _vp, _vp, _i32, _vp, _vp,
                                  _vp]),
    "smo_gemm_workspace": (_sz, [C.POINTER(GemmArgs)]),
    "smo_gemm": (C.c_int, [C.POINTER(GemmArgs), _vp]),
    "smo_rmsnorm": (C.c_int, [_vp, _vp, _i32, _i32, _f32, _vp, _vp]),
    "smo_embed": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "smo_rope_append": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp]),
    "smo_fill_kv_prefix": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _u64, _u64, _vp]),
    "smo_argmax_reduce": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "smo_argmax_rows": (C.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "smo_greedy_accept": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "smo_kv_rollback": (C.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "smo_nccl_unique_id": (C.c_int, [_vp]),
    "smo_ep_nccl_create": (C.c_int, [_vp, _i32, _i32, C.POINTER(_vp)]),
    "smo_ep_loopback_create": (C.c_int, [_i32, C.POINTER(_vp)]),
    "smo_ep_group_destroy": (C.c_int, [_vp]),
    "smo_ep_ipc_handle_bytes": (_sz, []),
    "smo_ep_ipc_create": (C.c_int, [_i32, _i32, _u64, C.POINTER(_vp), _vp]),
    "smo_ep_ipc_connect": (C.c_int, [_vp, _vp, _vp, _vp]),
    "smo_engine_create": (C.c_int, [C.POINTER(ModelConfig), C.POINTER(EngineOptions), C.POINTER(_vp)]),
    "smo_engine_destroy": (C.c_int, [_vp]),
    "smo_ep_workspace": (_sz, [_i32, _i32, _i32, _i32, _i32, _i32]),
    "smo_ep_dispatch": (C.c_int, [_vp, _i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "smo_ep_combine": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "smo_streamer_create": (C.c_int, [_vp, _vp]),
    "smo_streamer_destroy": (C.c_int, [_vp]),
    "smo_streamer_enqueue_layer": (C.c_int, [_vp, _i32, _vp]),
    "smo_streamer_expert_ready_event": (C.c_int, [_vp, _i32, _vp]),
    "smo_streamer_wait_layer": (C.c_int, [_vp, _i32, _vp]),
    "smo_streamer_expert_ptr": (C.c_int, [_vp, _i32, _i32, _vp]),
    "smo_streamer_release_layer": (C.c_int, [_vp, _i32, _vp]),
    "smo_engine_fill_prefix": (C.c_int, [_vp, _vp, _i32]),
    "smo_engine_verify": (C.c_int, [_vp, C.POINTER(VerifyBatch), C.POINTER(VerifyOutput), _vp]),
    "smo_engine_last_times": (C.c_int, [_vp, C.POINTER(StageTimes)]),
    "smo_engine_prefill": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "smo_engine_decode_begin": (C.c_int, [_vp, _vp, _vp, _i32]),
    "smo_engine_decode_step": (C.c_int, [_vp, _i32, _vp, _vp]),
    "smo_engine_decode_run": (C.c_int, [_vp, _i32, _i32, _i32, _vp]),
    "smo_engine_decode_step_tree": (C.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "smo_engine_decode_read": (C.c_int, [_vp, _vp, _i32, _vp, _vp, _vp]),
    "smo_engine_draft_times": (C.c_int, [_vp, _vp, _sz, _vp]),
    "smo_engine_layer_times": (C.c_int, [_vp, _vp, _sz]),
    "smo_engine_last_micro_batches": (C.c_int, [_vp, _vp]),
    "smo_engine_set_micro_batches": (C.c_int, [_vp, _i32]),
    "smo_engine_debug_tensor": (C.c_int, [_vp, C.c_char_p, _i32, _vp, _sz]),
    "smo_engine_tensor_ptr": (C.c_int, [_vp, C.c_char_p, _i32, _i32, C.POINTER(_vp), C.POINTER(_sz)]),
}

_lib = None


def load(build_if_missing: bool = True):
    """Load libspecmoe.so (building it in-tree if absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from . import build as _b
        _b.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2508_21706_b200.build`")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status != SMO_OK:
        msg = load().smo_last_error().decode()
        if status == SMO_CAPACITY:
            raise CapacityError(status, msg)
        if status == SMO_INVALID_ARG:
            raise ValueError(msg)
        raise SmoError(status, msg)


def launch_count() -> int:
    return int(load().smo_launch_count())
