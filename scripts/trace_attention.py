"""Phase trace of the fused attention kernel (profiling build with -DCORA_ATTN_TRACE).

    python paper_2110_10221_b200/build.py -DCORA_ATTN_TRACE --out=variants/atrace.so
    CORA_LIB_PATH=variants/atrace.so python scripts/trace_attention.py [config] [causal]

Softmax warp 0 (lane 0) events: 9 tile start, 1 before s_full wait, 2 S ready, 3 S in registers,
4 row max done, 5 exponentials done, 6 PV_{j-1} done, 7 P handed over, 8 last PV done (epilogue).
MMA thread: 20 issue_s start, 21 K ready, 22 S buffer free, 23 P_j ready, 24 V ready, 25 PV issued.
"""
import ctypes
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P
from paper_2110_10221_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
causal = len(sys.argv) > 2 and sys.argv[2] == "causal"
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from attn_probe import lengths_of
lengths, d, H = lengths_of(cfg), 512, 8
T = int(lengths.sum())
qkv = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
lay = P.layout_build(torch.tensor(lengths, dtype=torch.int32, device="cuda"), T, H, max(512, int(lengths.max())))
o = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
lib = ctypes.CDLL(_lib.LIB_PATH)
NC, NL = 296, 2048
buf = np.zeros((NC, 2, NL), dtype=np.uint64)
cnt = np.zeros((NC, 2), dtype=np.int32)
for _ in range(3):
    P.ragged_attention(lay, qkv, 64, out=o, causal=causal)
torch.cuda.synchronize()
lib.cora_debug_attn_trace(buf.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))
P.ragged_attention(lay, qkv, 64, out=o, causal=causal)
torch.cuda.synchronize()
lib.cora_debug_attn_trace(buf.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))

def phases(role, pairs):
    acc = defaultdict(list)
    spans = []
    for c in range(NC):
        n = int(cnt[c, role])
        ev = [(int(x) >> 8, int(x) & 0xFF) for x in buf[c, role, :n]]
        if not ev:
            continue
        spans.append(ev[-1][0] - ev[0][0])
        for (t0, e0), (t1, e1) in zip(ev, ev[1:]):
            acc[(e0, e1)].append(t1 - t0)
    return acc, spans

names = {36: "PV1 mma start", 37: "PV1 mma end", 3: "token", 31: "K1 ready", 33: "P1 ready", 35: "PV1 issued", 9: "tile", 1: "pre-wait", 2: "S ready", 3: "S in regs", 4: "max", 5: "exps", 6: "PV done", 7: "P handed",
         8: "last PV", 20: "issue_s", 21: "K ready", 22: "S free", 23: "P ready", 24: "V ready", 25: "PV issued", 10: "O stored", 11: "loop top", 12: "meta ready", 13: "O in regs", 14: "masked", 26: "PV mma start", 27: "PV mma end"}
for role, title in ((0, "softmax warp 0"), (1, "MMA thread")):
    acc, spans = phases(role, None)
    print(f"== {title}: {len(spans)} CTAs, mean span {np.mean(spans):.0f} clk")
    tot = sum(sum(v) for v in acc.values())
    for (a, b), v in sorted(acc.items(), key=lambda t: -sum(t[1]))[:22]:
        print(f"  {names.get(a, a):>10} -> {names.get(b, b):<10} n={len(v):6d} mean {np.mean(v):7.0f} clk  share {sum(v) / tot:6.1%}")

if os.environ.get("TIMELINE"):
    # merged timeline of both roles of CTA c (same SM clock), steps s0..s0+n
    c = int(os.environ.get("TL_CTA", "0"))
    ev = []
    for role in (0, 1):
        n = int(cnt[c, role])
        ev += [(int(x) >> 8, int(x) & 0xFF, role) for x in buf[c, role, :n]]
    ev.sort()
    t0 = ev[0][0]
    lo, hi = int(os.environ.get("TL_FROM", "200")), int(os.environ.get("TL_TO", "260"))
    for k, (t, e, role) in enumerate(ev[lo:hi]):
        print(f"{t - t0:9d} {'  ' * 0 if role == 0 else ' ' * 40}{names.get(e, e)}")
