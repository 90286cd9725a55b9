"""CPU checks of the C-ABI boundary: the library loads, exports every declared symbol, and its
host-side logic (argument validation, shard plan) behaves; no device compute is called."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_declares_exactly_the_exported_symbols():
    from paper_2110_10221_b200 import _lib as C
    hdr = open(os.path.join(ROOT, "include", "cora.h")).read()
    declared = set(re.findall(r"\b(cora_[a-z_0-9]+)\s*\(", hdr)) - {"cora_status_t"}
    assert declared == set(C.EXPORTS)
    lib = C.lib()
    for name in declared:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess
    from paper_2110_10221_b200 import _lib as C
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", C.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", C.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):  # tcgen05.mma, TMA load/store, tcgen05.ld
        assert mnemonic in sass, mnemonic


def test_argument_validation_without_device():
    from paper_2110_10221_b200 import _lib as C
    L = C.lib()
    assert L.cora_layout_workspace_bytes(-1, 0, 8, 512) == 0
    assert L.cora_layout_workspace_bytes(4, 16, 0, 512) == 0
    assert L.cora_layout_workspace_bytes(4, 16, 2, 20000) == 0
    assert L.cora_layout_workspace_bytes(4, 16, 2, 512) > 0
    lay = C.Layout()
    assert L.cora_layout_build(None, 4, 16, 2, 512, None, 0, ctypes.byref(lay), None) == C.CORA_ERR_INVALID
    assert L.cora_linear_fwd(None, None, None, None, None, 4, 12, 16, 0, None) == C.CORA_ERR_INVALID  # n % 8
    assert L.cora_linear_fwd(None, None, None, None, None, 4, 16, 16, 7, None) == C.CORA_ERR_INVALID  # act
    assert L.cora_linear_fwd(None, None, None, None, None, 0, 16, 16, 0, None) == C.CORA_OK          # empty
    assert L.cora_layernorm_fwd(None, None, None, None, None, 4, 12, 1e-5, 0, None) == C.CORA_ERR_INVALID
    assert L.cora_layernorm_fwd(None, None, None, None, None, 0, 16, 1e-5, 0, None) == C.CORA_OK
    p = C.EncoderParams()
    p.d_model, p.heads, p.d_ff = 512, 7, 2048
    lay.total_tokens, lay.heads, lay.batch = 10, 7, 1
    assert L.cora_encoder_layer_fwd(ctypes.byref(p), ctypes.byref(lay), None, None, None, 0, None) == C.CORA_ERR_INVALID
    assert L.cora_status_string(2) == b"data error (bad lengths or sum(L) != T)"


@pytest.mark.parametrize("seed", range(8))
def test_shard_plan_matches_oracle(seed):
    import paper_2110_10221_b200 as P
    rng = np.random.default_rng(seed)
    B = int(rng.integers(0, 40))
    R = int(rng.integers(1, 9))
    L = [int(x) for x in rng.integers(0, 513, size=B)]
    assert P.shard_plan(L, 512, 2048, R) == oracle.shard_plan(L, 512, 2048, R)


def test_shard_plan_c4():
    import paper_2110_10221_b200 as P
    import synth
    L = [int(x) for x in synth.config("C4-wiki512")[0]]
    for R in (1, 2, 4, 8):
        assert P.shard_plan(L, 512, 2048, R) == oracle.shard_plan(L, 512, 2048, R)
