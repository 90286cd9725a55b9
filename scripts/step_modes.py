"""Step-time distribution of the graph-replayed C4 step: the per-step sequence (does the slow mode come in
runs, alternate, or drift?), with and without the L2 flush, and the flush's own time.
    python scripts/step_modes.py [config] [steps]
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
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
lengths, d, H, dff = synth.config(cfg)
T = int(lengths.sum())
params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
fwd = P.EncoderForward(params)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
L = torch.tensor(lengths, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
acc = torch.empty((), dtype=torch.int64, device="cuda")


def step():  # the bench's step: cora_encoder_forward (prelude + layer, QKV under the prelude)
    fwd(L, T, x, out=y)


for _ in range(3):
    step()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(10):
    g.replay()
torch.cuda.synchronize()


def run(mode):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n)]
    for i in range(n):
        ev[i][0].record()
        if mode != "noflush":
            flush.zero_()
            torch.sum(flush_rd, dim=0, out=acc)
        ev[i][1].record()
        g.replay()
        ev[i][2].record()
        if mode == "sync":
            ev[i][2].synchronize()
    torch.cuda.synchronize()
    st = np.array([e[1].elapsed_time(e[2]) * 1e3 for e in ev])
    fl = np.array([e[0].elapsed_time(e[1]) * 1e3 for e in ev])
    return st, fl


for mode in ("flush", "noflush", "sync", "flush"):
    st, fl = run(mode)
    q = np.percentile(st, [10, 50, 90])
    slow = st > (q[0] + q[2]) / 2
    print(f"{mode}: step mean {st.mean():.1f} p10/50/90 {q[0]:.1f}/{q[1]:.1f}/{q[2]:.1f}  flush mean {fl.mean():.1f} "
          f"p10/90 {np.percentile(fl, 10):.1f}/{np.percentile(fl, 90):.1f}  slow share {slow.mean():.2f}")
    print("  seq:", "".join("S" if s else "." for s in slow))
    if mode == "flush":
        print("  corr(step, flush) = %.2f" % np.corrcoef(st, fl)[0, 1])
