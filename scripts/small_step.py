"""A few layer steps (prelude + layer, cora_encoder_forward) on one named configuration: a target for the
ncu launch list of small batches.

    python scripts/small_step.py [config] [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
import paper_2110_10221_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "cola-32"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg.count("-") == 1 and cfg.split("-")[1].isdigit() and not cfg.startswith("C"):
    ds, bs = cfg.split("-")
    lengths, d, H, dff = synth.dataset_lengths(ds, int(bs)), 512, 8, 2048
else:
    lengths, d, H, dff = synth.config(cfg)
T = int(sum(lengths))
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
fwd = P.EncoderForward(params)
Lt = torch.tensor(list(lengths), dtype=torch.int32, device="cuda")
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
for _ in range(iters):
    fwd(Lt, T, x, out=y)
torch.cuda.synchronize()
print(f"{cfg}: {len(lengths)} sequences, T={T}")
