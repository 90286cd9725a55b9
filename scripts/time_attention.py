"""Time the fused attention kernel alone (bidirectional and causal) on BASELINE configs (profiling helper).

    python scripts/time_attention.py [config[,config...]] [reps]
Useful FLOPs: 4 d sum L^2 (bidirectional), 4 d sum L(L+1)/2 (causal).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth


def _config(name):
    """synth.config names, or ds:<dataset>:<batch> (Table 3 length generator, d 512 / 8 heads / 2048)."""
    if name.startswith("ds:"):
        _, ds, bs = name.split(":")
        return synth.dataset_lengths(ds, int(bs)), 512, 8, 2048
    return synth.config(name)
import paper_2110_10221_b200 as P

cfgs = (sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512").split(",")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50


def time_us(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps * 1e3


for cfg in cfgs:
    if cfg.startswith("L"):  # "L<len>x<batch>": equal lengths
        ln, bs = cfg[1:].split("x")
        lengths, d, H = np.full(int(bs), int(ln), dtype=np.int64), 512, 8
    else:
        lengths, d, H, _ = _config(cfg)
    T = int(lengths.sum())
    qkv = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
    lay = P.layout_build(torch.tensor(lengths, dtype=torch.int32, device="cuda"), T, H, 512)
    o = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    L = lengths.astype(np.int64)
    full = time_us(lambda: P.ragged_attention(lay, qkv, 64, out=o))
    causal = time_us(lambda: P.ragged_attention(lay, qkv, 64, out=o, causal=True))
    f_full = 4 * d * int((L * L).sum())
    f_causal = 4 * d * int((L * (L + 1) // 2).sum())
    print(f"{cfg}: attention {full:.1f} us {f_full / full / 1e6:.1f} TFLOP/s | causal {causal:.1f} us "
          f"{f_causal / causal / 1e6:.1f} TFLOP/s | ratio {full / causal:.2f}x", flush=True)
