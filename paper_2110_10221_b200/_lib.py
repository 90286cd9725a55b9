"""ctypes view of libcora_b200.so (include/cora.h).  Argument marshalling only.

There is no fallback: if the shared library is missing or fails to load, importing the
binding raises.  Build it with `python paper_2110_10221_b200/build.py` (or
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CORA_LIB_PATH") or os.path.join(HERE, "libcora_b200.so")  # override: experiments

CORA_OK, CORA_ERR_INVALID, CORA_ERR_DATA, CORA_ERR_CUDA, CORA_ERR_UNSUPPORTED, CORA_ERR_NCCL = range(6)
CORA_DT_BF16, CORA_DT_F32 = 0, 1
CORA_ACT_NONE, CORA_ACT_RELU, CORA_ACT_GELU_ERF = 0, 1, 2
CORA_STATUS_BAD_LENGTH, CORA_STATUS_SUM_MISMATCH = 1, 2
TILE_ROWS = 128
LAYER_EVENTS = 8

# Every symbol include/cora.h declares (checked by tests/test_boundary.py on CPU).
EXPORTS = (
    "cora_layout_workspace_bytes", "cora_layout_build", "cora_layout_status", "cora_encoder_workspace_bytes",
    "cora_encoder_layer_fwd", "cora_encoder_layer_fwd_ex", "cora_encoder_layer_launches", "cora_encoder_stack_workspace_bytes", "cora_encoder_stack_fwd", "cora_encoder_forward_workspace_bytes", "cora_encoder_forward", "cora_forward_host_workspace_bytes",
    "cora_encoder_forward_host", "cora_linear_fwd", "cora_linear_residual_layernorm_fwd", "cora_vgemm_plan_bytes", "cora_vgemm_workspace_bytes", "cora_vgemm_plan", "cora_vgemm_fwd", "cora_trmm_fwd", "cora_ragged_attention_fwd", "cora_ragged_masked_attention_fwd", "cora_ragged_softmax_fwd",
    "cora_layernorm_fwd", "cora_shard_plan", "cora_shard_groups", "cora_encoder_stack_sharded_workspace_bytes",
    "cora_encoder_stack_sharded_fwd", "cora_comm_unique_id_bytes", "cora_comm_get_unique_id", "cora_comm_init", "cora_comm_destroy", "cora_allgather_ragged", "cora_status_string", "cora_device_sm_count", "cora_build_info",
)


class Layout(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("max_len", ctypes.c_int32),
        ("total_tokens", ctypes.c_int32),
        ("n_tiles_max", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("total_attn", ctypes.c_int64),
        ("lengths", ctypes.c_void_p),
        ("row_off", ctypes.c_void_p),
        ("attn_off", ctypes.c_void_p),
        ("seq_of_tok", ctypes.c_void_p),
        ("pos_in_seq", ctypes.c_void_p),
        ("tiles", ctypes.c_void_p),
        ("tile_seq", ctypes.c_void_p),
        ("n_tiles", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("n_units_max", ctypes.c_int32),
        ("_pad2", ctypes.c_int32),
        ("units", ctypes.c_void_p),
        ("unit_seq", ctypes.c_void_p),
        ("n_units", ctypes.c_void_p),
    ]


class EncoderParams(ctypes.Structure):
    _fields_ = [
        ("d_model", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("d_ff", ctypes.c_int32),
        ("ln_eps", ctypes.c_float),
        ("act", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ] + [(n, ctypes.c_void_p) for n in ("w_qkv", "b_qkv", "w_o", "b_o", "ln1_g", "ln1_b", "w1", "b1", "w2", "b2",
                                          "ln2_g", "ln2_b")]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python paper_2110_10221_b200/build.py`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, sz, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t, ctypes.c_float
        sig = {
            "cora_layout_workspace_bytes": (sz, [i32, i32, i32, i32]),
            "cora_layout_build": (i32, [vp, i32, i32, i32, i32, vp, sz, ctypes.POINTER(Layout), vp]),
            "cora_layout_status": (i32, [ctypes.POINTER(Layout), vp]),
            "cora_encoder_workspace_bytes": (sz, [ctypes.POINTER(EncoderParams), i32]),
            "cora_encoder_layer_fwd": (i32, [ctypes.POINTER(EncoderParams), ctypes.POINTER(Layout), vp, vp, vp, sz, vp]),
            "cora_encoder_layer_fwd_ex": (i32, [ctypes.POINTER(EncoderParams), ctypes.POINTER(Layout), vp, vp, vp, sz, vp,
                                                ctypes.POINTER(ctypes.c_void_p)]),
            "cora_encoder_layer_launches": (i32, [ctypes.POINTER(EncoderParams), i32]),
            "cora_encoder_forward_workspace_bytes": (sz, [ctypes.POINTER(EncoderParams), i32, i32, i32]),
            "cora_encoder_forward": (i32, [ctypes.POINTER(EncoderParams), vp, i32, i32, i32, vp, vp, vp, sz,
                                           ctypes.POINTER(Layout), vp]),
            "cora_encoder_stack_workspace_bytes": (sz, [ctypes.POINTER(EncoderParams), i32, i32]),
            "cora_encoder_stack_fwd": (i32, [ctypes.POINTER(EncoderParams), i32, ctypes.POINTER(Layout), vp, vp, vp, sz,
                                             vp]),
            "cora_forward_host_workspace_bytes": (sz, [ctypes.POINTER(EncoderParams), i32, i32, i32]),
            "cora_encoder_forward_host": (i32, [ctypes.POINTER(EncoderParams), vp, i32, i32, i32, vp, vp, vp, sz,
                                                ctypes.POINTER(Layout), vp]),
            "cora_linear_fwd": (i32, [vp, vp, vp, vp, vp, i32, i32, i32, i32, vp]),
            "cora_linear_residual_layernorm_fwd": (i32, [vp, vp, vp, vp, vp, vp, f32, vp, i32, i32, i32, i32, vp]),
            "cora_vgemm_plan_bytes": (sz, [i32, vp]),
            "cora_vgemm_workspace_bytes": (sz, [i32, vp]),
            "cora_vgemm_plan": (i32, [i32, vp, i32, i32, i32, vp, sz]),
            "cora_vgemm_fwd": (i32, [vp, vp, vp, vp, i32, i32, i32, vp, sz, vp]),
            "cora_trmm_fwd": (i32, [vp, vp, vp, i32, i32, vp]),
            "cora_ragged_attention_fwd": (i32, [ctypes.POINTER(Layout), vp, vp, i32, f32, vp]),
            "cora_ragged_masked_attention_fwd": (i32, [ctypes.POINTER(Layout), vp, vp, i32, f32, vp]),
            "cora_ragged_softmax_fwd": (i32, [ctypes.POINTER(Layout), vp, vp, i32, vp]),
            "cora_layernorm_fwd": (i32, [vp, vp, vp, vp, vp, i32, i32, f32, i32, vp]),
            "cora_shard_plan": (i32, [ctypes.POINTER(ctypes.c_int32), i32, i32, i32, i32, ctypes.POINTER(ctypes.c_int32),
                                      ctypes.POINTER(ctypes.c_int32)]),
            "cora_shard_groups": (i32, [ctypes.POINTER(ctypes.c_int32), i32, ctypes.POINTER(ctypes.c_int32), i32, i32,
                                        ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
            "cora_encoder_stack_sharded_workspace_bytes": (sz, [ctypes.POINTER(EncoderParams), i32, i32, i32, i32]),
            "cora_encoder_stack_sharded_fwd": (i32, [ctypes.POINTER(EncoderParams), i32, vp, ctypes.POINTER(ctypes.c_int32),
                                                     i32, i32, i32, vp, i32, vp, vp, vp, sz, vp]),
            "cora_comm_unique_id_bytes": (i32, []),
            "cora_comm_get_unique_id": (i32, [vp]),
            "cora_comm_init": (i32, [ctypes.POINTER(ctypes.c_void_p), vp, i32, i32]),
            "cora_comm_destroy": (i32, [vp]),
            "cora_allgather_ragged": (i32, [vp, ctypes.POINTER(ctypes.c_int32), vp, i32, i32, vp]),
            "cora_status_string": (ctypes.c_char_p, [i32]),
            "cora_device_sm_count": (i32, []),
            "cora_build_info": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class CoraError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = lib().cora_status_string(status).decode()
        super().__init__(f"{what}: {msg} (status {status})")
        self.status = status


def check(status: int, what: str) -> None:
    if status != CORA_OK:
        raise CoraError(status, what)
