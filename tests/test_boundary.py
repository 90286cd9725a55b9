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


@pytest.mark.parametrize("seed", range(12))
def test_shard_plan_matches_oracle(seed):
    import paper_2110_10221_b200 as P
    rng = np.random.default_rng(seed)
    B = int(rng.integers(0, 40))
    R = int(rng.integers(1, 9))
    # mixes of long sequences and short ones that form windows (reading s2)
    pool = [0, 1, 5, 30, 64, 100, 128, 129, 300, 512] if seed % 2 else list(range(0, 513))
    L = [int(x) for x in rng.choice(pool, size=B)]
    plan, rows = P.shard_plan(L, 512, 2048, R, rows=True)
    assert plan == oracle.shard_plan(L, 512, 2048, R)
    ro = oracle.row_offsets(L)
    assert rows == [ro[b] for b in plan]


@pytest.mark.parametrize("cfg", ["C4-wiki512", "C4-race", "mnli-128", "cola-32", "C5-skewed-128"])
def test_shard_plan_paper_configs(cfg):
    import paper_2110_10221_b200 as P
    import synth
    L = [int(x) for x in synth.config(cfg)[0]]
    for R in (1, 2, 4, 8):
        assert P.shard_plan(L, 512, 2048, R) == oracle.shard_plan(L, 512, 2048, R)


def test_shard_plan_unconstrained_above_pack_limit():
    import paper_2110_10221_b200 as P
    L = [5] * 1100  # > CORA_PACK_MAX_BATCH: no windows, any cut is allowed
    plan = P.shard_plan(L, 512, 2048, 4)
    assert plan == [0, 275, 550, 825, 1100] == oracle.shard_plan(L, 512, 2048, 4)


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_shard_groups_partition_window_aligned(G):
    import paper_2110_10221_b200 as P
    import synth
    L = [int(x) for x in synth.config("mnli-128")[0]] + [300, 2, 3, 200]
    ok = oracle.shard.allowed_cuts(L)
    ro = oracle.row_offsets(L)
    for R in (1, 2, 3):
        plan = P.shard_plan(L, 512, 2048, R)
        gseq, grow = P.shard_groups(L, plan, G)
        for r in range(R):
            assert gseq[r][0] == plan[r] and gseq[r][G] == plan[r + 1] and gseq[r] == sorted(gseq[r])
            assert all(ok[c] for c in gseq[r])
            assert grow[r] == [ro[b] for b in gseq[r]]


def test_shard_entry_points_validate():
    from paper_2110_10221_b200 import _lib as C
    L = C.lib()
    lens = (ctypes.c_int32 * 3)(3, -1, 4)
    out = (ctypes.c_int32 * 3)()
    assert L.cora_shard_plan(lens, 3, 512, 2048, 2, out, None) == C.CORA_ERR_INVALID  # negative length
    assert L.cora_shard_plan(lens, 3, 512, 2048, 0, out, None) == C.CORA_ERR_INVALID  # no rank
    sb = (ctypes.c_int32 * 3)(0, 2, 1)
    gs = (ctypes.c_int32 * 8)()
    good = (ctypes.c_int32 * 3)(3, 1, 4)
    assert L.cora_shard_groups(good, 3, sb, 2, 3, gs, None) == C.CORA_ERR_INVALID  # decreasing plan
    p = C.EncoderParams()
    p.d_model, p.heads, p.d_ff = 512, 8, 2048
    assert L.cora_encoder_stack_sharded_workspace_bytes(ctypes.byref(p), 0, 4, 16, 512) == 0
    assert L.cora_encoder_stack_sharded_workspace_bytes(ctypes.byref(p), 2, 4, 16, 512) > 0


def test_vgemm_plan_host_logic():
    """cora_vgemm_plan (host-only): sizes, validation, and the serialised work list (longest reduction first)."""
    from paper_2110_10221_b200 import _lib as C
    L = C.lib()
    dims = [(300, 200, 256), (128, 264, 64), (0, 8, 64), (64, 64, 0)]
    dh = (ctypes.c_int32 * 12)(*[v for r in dims for v in r])
    n = L.cora_vgemm_plan_bytes(4, dh)
    units = sum(-(-m // 128) * -(-nn // 256) for m, nn, _ in dims)
    assert n == 16 + 16 * units + 8 * 4
    assert L.cora_vgemm_workspace_bytes(4, dh) == n
    buf = (ctypes.c_uint8 * n)()
    assert L.cora_vgemm_plan(4, dh, 300, 264, 256, buf, n) == C.CORA_OK
    h = np.frombuffer(bytes(buf), dtype=np.int32)
    assert h[1] == 4 and h[2] == units
    u = h[4:4 + 4 * units].reshape(units, 4)  # (problem, m0, n0, k-blocks)
    assert list(u[:, 3]) == sorted(u[:, 3], reverse=True)  # longest reduction first
    assert sorted(map(tuple, u[:, :3])) == sorted((p, m0, n0) for p, (m, nn, _k) in enumerate(dims)
                                                  for m0 in range(0, m, 128) for n0 in range(0, nn, 256))
    assert L.cora_vgemm_plan(4, dh, 300, 264, 256, buf, n - 1) == C.CORA_ERR_INVALID      # small buffer
    assert L.cora_vgemm_plan(4, dh, 200, 264, 256, buf, n) == C.CORA_ERR_INVALID          # M_i > m_max
    bad = (ctypes.c_int32 * 3)(64, 64, 100)
    assert L.cora_vgemm_plan(1, bad, 64, 64, 128, buf, n) == C.CORA_ERR_UNSUPPORTED       # partial k-block
    assert L.cora_vgemm_plan_bytes(1, (ctypes.c_int32 * 3)(-1, 8, 8)) == 0
