"""Time the device prelude (a1, cora_layout_build) alone: a CUDA graph of 20 builds (profiling helper).

    python scripts/time_prelude.py [config[,config...]]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth


def _config(name):
    """synth.config names, or ds:<dataset>:<batch> (Table 3 length generator, d 512 / 8 heads / 2048)."""
    if name.startswith("ds:"):
        _, ds, bs = name.split(":")
        return synth.dataset_lengths(ds, int(bs)), 512, 8, 2048
    return synth.config(name)
import paper_2110_10221_b200 as P

for cfg in (sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512,C2-mnli").split(","):
    lengths = _config(cfg)[0]
    L = torch.tensor(lengths, dtype=torch.int32, device="cuda")
    T = int(lengths.sum())
    lay = P.layout_build(L, T, 8, 512)
    assert lay.status() == 0
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            P.layout_build(L, T, 8, 512)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    b.synchronize()
    print(f"{cfg}: prelude {a.elapsed_time(b) / 200 * 1e3:.2f} us per build (B={len(lengths)}, T={T})", flush=True)
