"""Where the MMA thread of a GEMM launch waits (profiling build with -DCORA_GEMM_TRACE=<mode>; mode 1 FF2 + LN2,
2 out-proj + LN1, 3 plain GEMMs -- the last one of the layer, FF1):
    CORA_LIB_PATH=variants/gt3.so python scripts/gemm_waits.py [config]
Per CTA (clock64 cycles): producer waiting for free stages, MMA waiting for loaded stages / for a free
accumulator, MMA total, epilogue warp 0 waiting for its accumulator / total, units; medians over CTAs.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P
from paper_2110_10221_b200 import _lib
from kspan import lengths_of

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
lengths, d, H, dff = lengths_of(cfg)
lengths = [int(v) for v in lengths]
T = sum(lengths)
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
fwd = P.EncoderForward(params)
Lt = torch.tensor(lengths, dtype=torch.int32, device="cuda")
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
lib = _lib.lib()
buf = (ctypes.c_longlong * (2048 * 8))()
for _ in range(4):
    fwd(Lt, T, x, out=y)
torch.cuda.synchronize()
lib.cora_debug_gemm_waits(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(2048, 8)
mma = a[a[:, 3] > 0]
epi = a[a[:, 5] > 0]
print(f"{cfg} T={T}: {len(mma)} MMA CTAs, {len(epi)} epilogue records")
for nm, arr, k in [("producer wait empty", a[a[:, 0] > 0], 0), ("MMA wait full", mma, 1), ("MMA wait tmem_empty", mma, 2),
                   ("MMA total", mma, 3), ("epi wait tmem_full", epi, 4), ("epi total", epi, 5), ("units", mma, 6)]:
    if len(arr):
        v = arr[:, k]
        print(f"  {nm:22s} med {np.median(v):10.0f}  min {v.min():10.0f}  max {v.max():10.0f}")
