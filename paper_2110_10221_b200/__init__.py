"""B200-native ragged transformer-encoder layer after CoRa (arXiv 2110.10221).

The product path is libcora_b200.so (C ABI, include/cora.h: hand-written sm_100a kernels);
this package is its thin ctypes binding.  Importing it loads the library and fails loudly if
it is missing -- there is no CPU or eager fallback.
"""
from . import _lib
from .api import (  # noqa: F401
    EncoderLayer,
    EncoderForward,
    EncoderParams,
    EncoderStack,
    HostForward,
    RaggedLayout,
    VgemmPlan,
    build_info,
    encoder_layer,
    layernorm,
    layout_build,
    linear,
    linear_residual_layernorm,
    ragged_attention,
    ragged_softmax,
    shard_groups,
    shard_plan,
    trmm,
    vgemm,
)

_lib.lib()  # load now: no silent fallback
