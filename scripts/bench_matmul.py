"""vgemm / trmm measurement (SURVEY f-3) on B200, one JSON line per case.

    python scripts/bench_matmul.py [--reps 20] [--out profiles/r1_matmul.jsonl]

vgemm: the paper's workload (dims uniform multiples of 128 in [512, 1408]) at batch
16 / 64 / 256; useful TFLOP/s = 2 sum M_i N_i K_i / time.  Context on the same GPU: the fully padded
batched GEMM (torch.bmm = cuBLAS on the [batch, M_max, K_max] buffers), the paper's "fully padded gemm".
trmm: tril(L) B with L [N, N], B [N, N], N = 1024..8192; useful FLOPs N (N+1) / 2 * N * 2; context:
cuBLAS dense GEMM of the same shape (torch.matmul), the paper's "fully-padded gemm".
Times: CUDA events over `reps` back-to-back launches after warm-up; L2 (126 MB) is not flushed, the
operands of the largest cases exceed it.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import synth
import paper_2110_10221_b200 as P


def time_ms(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    peak = peaks["bf16_tflops"]
    lines = []
    for batch in (16, 64, 256):
        d = synth.vgemm_dims(batch, seed=batch)
        dims = [tuple(map(int, r)) for r in d]
        mm, nn, kk = (int(d[:, j].max()) for j in range(3))
        a = torch.randn(batch, mm, kk, device="cuda").to(torch.bfloat16)
        b = torch.randn(batch, kk, nn, device="cuda").to(torch.bfloat16)
        c = torch.zeros(batch, mm, nn, dtype=torch.bfloat16, device="cuda")
        plan = P.VgemmPlan(dims, mm, nn, kk)  # built once on the host (pinned), reused by every call
        t = time_ms(lambda: P.vgemm(a, b, dims, out=c, plan=plan), args.reps)
        t_pad = time_ms(lambda: torch.bmm(a, b), args.reps)
        f = oracle.vgemm_flops(dims)
        tf = f / t / 1e9
        lines.append({"op": "vgemm", "batch": batch, "dims": "128*U{4..11} (PAPER.md:753-755)", "ms": t,
                      "useful_tflops": tf, "frac_of_burst_peak": tf / peak,
                      "padded_over_useful_flops": oracle.vgemm_padded_flops(dims) / f,
                      "cublas_padded_bmm_ms": t_pad, "speedup_vs_padded_bmm": t_pad / t})
        print(json.dumps(lines[-1]), flush=True)
    for n in (1024, 2048, 4096, 8192):
        l = torch.randn(n, n, device="cuda").to(torch.bfloat16)
        b = torch.randn(n, n, device="cuda").to(torch.bfloat16)
        c = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
        t = time_ms(lambda: P.trmm(l, b, out=c), args.reps)
        t_dense = time_ms(lambda: torch.matmul(l, b), args.reps)
        f = oracle.trmm_flops(n, n)
        tf = f / t / 1e9
        lines.append({"op": "trmm", "n": n, "n_cols": n, "ms": t, "useful_tflops": tf, "frac_of_burst_peak": tf / peak,
                      "cublas_dense_gemm_ms": t_dense, "speedup_vs_dense_gemm": t_dense / t})
        print(json.dumps(lines[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as fo:
            for ln in lines:
                fo.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
