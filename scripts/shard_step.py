"""Run one rank's shard of the C4 batch (cora_shard_plan at N ranks) through cora_encoder_forward a few
times: the launch list / ncu target for small-T (per-rank) kernels.

    python scripts/shard_step.py [N] [rank] [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P
from paper_2110_10221_b200.dist import shard_rows

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
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
for _ in range(iters):
    fwd(Lt, T, x, out=y)
torch.cuda.synchronize()
print(f"N={n} rank={rank}: {len(L)} sequences, T={T}")
