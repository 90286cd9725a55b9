"""Time the graph-captured step (prelude + layer) with and without per-kernel events (profiling helper).

    python scripts/time_layer.py [config] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth


def _config(name):
    """synth.config names, ds:<dataset>:<batch> (Table 3 length generator, d 512 / 8 heads / 2048), or
    shard<N> (rank 0's shard of C4 at N ranks)."""
    if name.startswith("shard"):
        from paper_2110_10221_b200.dist import shard_rows
        lengths, d, H, dff = synth.config("C4-wiki512")
        lengths = np.asarray(lengths, np.int64)
        plan, _ = shard_rows(list(lengths), d, dff, int(name[5:]))
        return lengths[plan[0]:plan[1]], d, H, dff
    if name.startswith("ds:"):
        _, ds, bs = name.split(":")
        return synth.dataset_lengths(ds, int(bs)), 512, 8, 2048
    return synth.config(name)
import paper_2110_10221_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
lengths, d, H, dff = _config(cfg)
T = int(lengths.sum())
w = synth.encoder_weights(d, H, dff)
params = P.EncoderParams.from_host(w)
layer = P.EncoderLayer(params)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
L = torch.tensor(lengths, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
for e in kev:
    e.record()


def step(ev=None):
    lay = P.layout_build(L, T, H, 512)
    layer(x, lay, out=y, events=ev)


for _ in range(3):
    step()
torch.cuda.synchronize()
S2 = int((lengths.astype(np.int64) ** 2).sum())
flops = 2 * T * (4 * d * d + 2 * d * dff) + 4 * d * S2
for name, ev in (("no-events", None), ("events", kev)):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(ev)
    for _ in range(3):
        g.replay()
    times = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
    ms = float(np.mean(times))
    extra = ""
    if ev is not None:  # per-kernel means of the last replays (events recorded inside the graph)
        per = []
        for _ in range(20):
            g.replay()
            torch.cuda.synchronize()
            per.append([kev[j].elapsed_time(kev[j + 1]) * 1e3 for j in range(7)])
        m = np.mean(per, axis=0)
        extra = "  [qkv %.1f attn %.1f oproj+ln1 %.1f ff1 %.1f ff2+ln2 %.1f]" % (m[0], m[1], m[2] + m[3], m[4], m[5] + m[6])
    print(f"{cfg} {name}: {ms * 1e3:.1f} us/step  {flops / ms / 1e9:.1f} TFLOP/s{extra}", flush=True)
