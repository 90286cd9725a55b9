"""Phase timeline of the last GEMM launch of a layer step (profiling build with -DCORA_GEMM_TRACE):
    CORA_LIB_PATH=variants/trace.so python scripts/trace_gemm.py [N] [rank]
Stamps (globaltimer, ns, per CTA): 0 entry, 1 setup done, 2 after griddepcontrol.wait, 3/4/5 MMA issuer
saw k-block 0 / K/2 / last of its first unit, 6 epilogue got the accumulator, 7 LN statistics exchanged,
8 first unit stored, 9 before the exit cluster barrier, 10 after it; 11 / 12 the accumulator of the
second / third unit ready (LN kernels), 13 / 14 the MMA issuer saw k-block 0 / last of its second unit.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P
from paper_2110_10221_b200 import _lib
from paper_2110_10221_b200.dist import shard_rows

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lengths, d, H, dff = synth.config("C4-wiki512")
lengths = np.asarray(lengths, np.int64)
plan, _ = shard_rows(list(lengths), d, dff, n)
L = lengths[plan[rank]:plan[rank + 1]]
T = int(L.sum())
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
fwd = P.EncoderForward(params)
Lt = torch.tensor(L, dtype=torch.int32, device="cuda")
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
lib = _lib.lib()
buf = (ctypes.c_ulonglong * (2048 * 16))()
for it in range(4):
    ctypes.memset(buf, 0, ctypes.sizeof(buf))
    fwd(Lt, T, x, out=y)
    torch.cuda.synchronize()
lib.cora_debug_gemm_trace(buf, 2048 * 16)
a = np.frombuffer(buf, dtype=np.uint64).reshape(2048, 16).astype(np.int64)
ctas = np.nonzero(a[:, 0])[0]
a = a[ctas]
t0 = a[:, 0].min()
rel = lambda k: (a[:, k] - t0) / 1000.0
print(f"N={n} rank={rank} T={T}: {len(ctas)} CTAs traced; times in us from the first CTA entry")
names = ["entry", "setup", "pdl_wait", "kb0", "kbK/2", "kblast", "acc", "xch", "stored", "exit_bar", "exit",
         "acc_u1", "acc_u2", "u1_kb0", "u1_kblast", "-"]
for k, nm in enumerate(names):
    v = rel(k)
    v = v[a[:, k] > 0]
    if len(v) and nm != "-":
        print(f"  {nm:9s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}  (n={len(v)})")
