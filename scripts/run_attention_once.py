"""Run the fused attention kernel a few times on one configuration (ncu target; no timing).

    python scripts/run_attention_once.py [config] [reps] [causal]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
import paper_2110_10221_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
causal = len(sys.argv) > 3 and sys.argv[3] == "causal"
lengths, d, H, _ = synth.config(cfg)
T = int(lengths.sum())
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(T, 3 * d, device="cuda", generator=g).to(torch.bfloat16)
lay = P.layout_build(torch.tensor(lengths, dtype=torch.int32, device="cuda"), T, H, 512)
o = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
for _ in range(reps):
    P.ragged_attention(lay, qkv, 64, out=o, causal=causal)
torch.cuda.synchronize()
print("ok", cfg, T)
