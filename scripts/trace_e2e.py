"""Timeline of the pipelined host-buffer forward (profiling helper): per chunk, ms from the start to its
H2D, layer and D2H completion (the directly enqueued pipeline, not the cached graph).

    python paper_2110_10221_b200/build.py -DCORA_HOST_TRACE --out=$PWD/variants/htrace.so
    CORA_LIB_PATH=variants/htrace.so CORA_HOST_CHUNKS=k python scripts/trace_e2e.py [config]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CORA_HOST_NO_GRAPH"] = "1"

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P
from paper_2110_10221_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
lengths, d, H, dff = synth.config(cfg)
T = int(lengths.sum())
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
hf = P.HostForward(params, len(lengths), T, 512)
len_h = torch.tensor(lengths, dtype=torch.int32).pin_memory()
x_h = torch.randn(T, d).to(torch.bfloat16).pin_memory()
y_h = torch.empty(T, d, dtype=torch.bfloat16).pin_memory()
for _ in range(5):
    hf(len_h, x_h, y_h)
torch.cuda.synchronize()
out = np.zeros(48, np.float32)
K = ctypes.CDLL(_lib.LIB_PATH).cora_debug_host_trace(out.ctypes.data_as(ctypes.c_void_p), 16)
print(f"{cfg} K={K}")
for c in range(K):
    print(f"chunk {c:2d}: h2d {out[c]:.3f}  layer {out[K + c]:.3f}  d2h {out[2 * K + c]:.3f}")
