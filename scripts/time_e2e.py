"""Time cora_encoder_forward_host (pinned host buffers) alone (profiling helper).

    CORA_HOST_CHUNKS=k python scripts/time_e2e.py [config] [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lengths, d, H, dff = synth.config(cfg)
T = int(lengths.sum())
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
hf = P.HostForward(params, len(lengths), T, 512)
len_h = torch.tensor(lengths, dtype=torch.int32).pin_memory()
x_h = torch.randn(T, d).to(torch.bfloat16).pin_memory()
y_h = torch.empty(T, d, dtype=torch.bfloat16).pin_memory()
for _ in range(3):
    hf(len_h, x_h, y_h)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for _ in range(reps):
    hf(len_h, x_h, y_h)
t1 = time.perf_counter()
b.record()
b.synchronize()
print(f"{cfg} chunks={os.environ.get('CORA_HOST_CHUNKS', 'auto')}: {a.elapsed_time(b) / reps:.3f} ms per call "
      f"(host enqueue {(t1 - t0) / reps * 1e3:.3f} ms)")
