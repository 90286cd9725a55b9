"""Time the standalone LayerNorm (cora_layernorm_fwd, bf16 [T, 512]) and the GEMM kernels of the layer
alone, L2 flushed or warm (profiling helper).

    python scripts/time_ln.py [T]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_2110_10221_b200 as P

T = int(sys.argv[1]) if len(sys.argv) > 1 else 47283
x = torch.randn(T, 512, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
g = torch.randn(512, device="cuda")
b = torch.randn(512, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=50, do_flush=False):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        if do_flush:
            flush.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        e.synchronize()
        tot += a.elapsed_time(e)
    return tot / reps * 1e3


for fl in (False, True):
    us = t(lambda: P.layernorm(x, g, b, out=y), do_flush=fl)
    print(f"layernorm T={T} {'flushed' if fl else 'warm'}: {us:.1f} us  {2 * T * 512 * 2 / us / 1e3:.0f} GB/s", flush=True)
