"""Expected strong scaling of the C4 step on one GPU: time every rank's shard (cora_shard_plan) of the
bs128 batch alone (prelude + layer, one CUDA graph, L2 flushed) and report the makespan per N.

    python scripts/time_shards.py [config] [reps]
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

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lengths, d, H, dff = synth.config(cfg)
lengths = np.asarray(lengths, np.int64)
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
S2 = lambda L: int((L ** 2).sum())
flops = lambda L: 2 * int(L.sum()) * (4 * d * d + 2 * d * dff) + 4 * d * S2(L)


def time_step(L):
    T = int(L.sum())
    fwd = P.EncoderForward(params)
    Lt = torch.tensor(L, dtype=torch.int32, device="cuda")
    x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    fwd(Lt, T, x, out=y)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fwd(Lt, T, x, out=y)
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.mean(ts)) * 1e3


t1 = time_step(lengths)
print(f"{cfg} N=1: {t1:.1f} us", flush=True)
for n in (2, 4, 8):
    plan, tok = shard_rows(list(lengths), d, dff, n)
    ts = [time_step(lengths[plan[r]:plan[r + 1]]) for r in range(n)]
    worst = max(ts)
    print(f"{cfg} N={n}: makespan {worst:.1f} us (ranks {', '.join(f'{t:.0f}' for t in ts)}), "
          f"scaling {t1 / worst:.2f}x, {flops(lengths) / worst / 1e6:.0f} TFLOP/s aggregate", flush=True)
