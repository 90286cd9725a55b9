"""How much of the timed step is the CUDA-graph launch?  A: L2 flush on the stream, event, graph replay of
the step, event (bench.py).  B: one graph holding the flush, an event-record node, the step and a second
event-record node (the graph's launch latency then precedes the flush).  20-step runs, alternating.
    python scripts/graph_launch_cost.py [config] [rounds]
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
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lengths, d, H, dff = synth.config(cfg)
T = int(lengths.sum())
fwd = P.EncoderForward(P.EncoderParams.from_host(synth.encoder_weights(d, H, dff)))
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
L = torch.tensor(lengths, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
acc = torch.empty((), dtype=torch.int64, device="cuda")


def flush_l2():
    flush.zero_()
    torch.sum(flush_rd, dim=0, out=acc)


for _ in range(3):
    fwd(L, T, x, out=y)
    flush_l2()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    fwd(L, T, x, out=y)
n = 20
evb = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
       for _ in range(n)]
for a, b in evb:
    a.record()
    b.record()
torch.cuda.synchronize()
gb = []
for i in range(n):
    gi = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gi):
        flush_l2()
        evb[i][0].record()
        fwd(L, T, x, out=y)
        evb[i][1].record()
    gb.append(gi)
for _ in range(3):
    g.replay()
    gb[0].replay()
torch.cuda.synchronize()
for r in range(rounds):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        flush_l2()
        ev[i][0].record()
        g.replay()
        ev[i][1].record()
    torch.cuda.synchronize()
    ta = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    time.sleep(2)
    for i in range(n):
        gb[i].replay()
    torch.cuda.synchronize()
    tb = np.array([a.elapsed_time(b) * 1e3 for a, b in evb])
    print(f"A (flush, event, replay, event): mean {ta.mean():.1f} p50 {np.median(ta):.1f} | "
          f"B (flush + events inside the graph): mean {tb.mean():.1f} p50 {np.median(tb):.1f}", flush=True)
    time.sleep(2)
