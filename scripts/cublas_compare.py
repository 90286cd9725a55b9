"""cuBLAS (torch.matmul, bf16) vs the library's GEMMs on the layer's packed shapes (context for the GEMM rows
of the roofline table; cuBLAS is not on the product path).

    python scripts/cublas_compare.py [config] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
import paper_2110_10221_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lengths, d, H, dff = synth.config(cfg)
T = int(lengths.sum())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t_us(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1e3


for name, k, n in (("qkv", d, 3 * d), ("out_proj", d, d), ("ff1", d, dff), ("ff2", dff, d)):
    a = torch.randn(T, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    bias = torch.randn(n, device="cuda").to(torch.bfloat16)
    c = torch.empty(T, n, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * T * k * n
    tc = t_us(lambda: torch.matmul(a, w.t(), out=c))
    tca = t_us(lambda: torch.addmm(bias, a, w.t(), out=c))
    tl = t_us(lambda: P.linear(a, w, bias=bias, out=c))
    print(f"{name:9s} T={T} K={k} N={n}: cuBLAS {tc:6.1f} us ({fl / tc / 1e6:6.1f} TF/s)  cuBLAS+bias {tca:6.1f} us"
          f"  | cora {tl:6.1f} us ({fl / tl / 1e6:6.1f} TF/s)", flush=True)
