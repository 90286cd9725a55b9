"""Time the fused attention kernel alone on a BASELINE config (profiling helper).

    python scripts/time_attention.py [config] [reps]
Env CORA_ATTN_MODE selects the profiling variants of attention_fwd_kernel (see attention.cu).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lengths, d, H, dff = synth.config(cfg)
T = int(lengths.sum())
qkv = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
lay = P.layout_build(torch.tensor(lengths, dtype=torch.int32, device="cuda"), T, H, 512)
o = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    P.ragged_attention(lay, qkv, 64, out=o)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(reps):
    P.ragged_attention(lay, qkv, 64, out=o)
ev[1].record()
torch.cuda.synchronize()
us = ev[0].elapsed_time(ev[1]) / reps * 1e3
S2 = int((lengths.astype(np.int64) ** 2).sum())
print(f"{cfg} mode={os.environ.get('CORA_ATTN_MODE', '0')} attention {us:.1f} us  {4 * d * S2 / us / 1e6:.1f} TFLOP/s")
