"""Op-level measurements of every C entry point of the path against its roofline (one JSON line each).

    python scripts/time_ops.py [--out profiles/r1_ops.jsonl]

Each op is timed alone with CUDA events (20 launches after warm-up, L2 flushed before each) on the
BASELINE configurations: the prelude (a1), the packed GEMMs (a2, a4, a6, a7), fused GEMM + LayerNorm
(a4+a5, a7+a8), the fused attention (a3, bidirectional and causal: MUFU roofline), the standalone ragged
softmax (a3', HBM roofline: read + write of H * sum L^2 elements) and the standalone LayerNorm (HBM).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
    tensor_peak, hbm_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), pk["hbm_gbs"]
    sms = P._lib.lib().cora_device_sm_count()
    mufu_peak = 16.0 * sms * 1965e6 / 1e9  # Gexp/s at the B200 max SM clock
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def t_us(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            tot += a.elapsed_time(b)
        return tot / args.reps * 1e3

    lines = []

    def emit(**kw):
        lines.append(kw)
        print(json.dumps(kw), flush=True)

    for cfg in ("C2-mnli", "C3", "C4-wiki512"):
        lengths, d, H, dff = synth.config(cfg)
        T = int(lengths.sum())
        S2 = int((np.asarray(lengths, np.int64) ** 2).sum())
        Lt = torch.tensor(lengths, dtype=torch.int32, device="cuda")
        lay = P.layout_build(Lt, T, H, 512)
        emit(op="prelude (a1)", config=cfg, us=t_us(lambda: P.layout_build(Lt, T, H, 512)), bound="launch/latency")
        qkv = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
        o = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
        for causal in (False, True):
            us = t_us(lambda: P.ragged_attention(lay, qkv, 64, out=o, causal=causal))
            n_exp = H * (S2 if not causal else int((np.asarray(lengths, np.int64) * (np.asarray(lengths, np.int64) + 1) // 2).sum()))
            emit(op="attention (a3)" + (" causal (f-2)" if causal else ""), config=cfg, us=us, bound="alu (MUFU exp2)",
                 achieved_gexp_s=n_exp / us / 1e3, peak_gexp_s=mufu_peak, frac=n_exp / us / 1e3 / mufu_peak)
        # standalone ragged softmax over the materialised X[b, i, h, j] (bf16): read + write
        n = H * S2
        if n * 2 * 2 < (3 << 30):
            X = torch.randn(n, device="cuda").to(torch.bfloat16)
            Y = torch.empty_like(X)
            us = t_us(lambda: P.ragged_softmax(lay, X, out=Y))
            emit(op="ragged softmax (a3')", config=cfg, us=us, bound="hbm", achieved_gb_s=4 * n / us / 1e3,
                 peak_gb_s=hbm_peak, frac=4 * n / us / 1e3 / hbm_peak)
            del X, Y
        w = synth.encoder_weights(d, H, dff)
        prm = P.EncoderParams.from_host(w)
        x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        f = torch.randn(T, dff, device="cuda").to(torch.bfloat16)
        for name, a, wt, b, res, act, k, n_out in (
                ("QKV GEMM (a2)", x, prm.w_qkv, prm.b_qkv, None, "none", d, 3 * d),
                ("FF1 GEMM + ReLU (a6)", x, prm.w1, prm.b1, None, "relu", d, dff),
                ("out-proj GEMM + residual (a4)", x, prm.w_o, prm.b_o, x, "none", d, d),
                ("FF2 GEMM + residual (a7)", f, prm.w2, prm.b2, x, "none", dff, d)):
            c = torch.empty(T, n_out, dtype=torch.bfloat16, device="cuda")
            us = t_us(lambda: P.linear(a, wt, bias=b, residual=res, act=act, out=c))
            fl = 2.0 * T * k * n_out
            emit(op=name, config=cfg, us=us, bound="tensor", achieved_tflops=fl / us / 1e6, peak_tflops=tensor_peak,
                 frac=fl / us / 1e6 / tensor_peak)
        if T > 128:
            for name, a, wt, b, k in (("out-proj + residual + LayerNorm (a4+a5, f-1)", x, prm.w_o, prm.b_o, d),
                                      ("FF2 + residual + LayerNorm (a7+a8, f-1)", f, prm.w2, prm.b2, dff)):
                c = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
                us = t_us(lambda: P.linear_residual_layernorm(a, wt, x, prm.ln1_g, prm.ln1_b, bias=b, out=c))
                fl = 2.0 * T * k * d
                emit(op=name, config=cfg, us=us, bound="tensor", achieved_tflops=fl / us / 1e6,
                     peak_tflops=tensor_peak, frac=fl / us / 1e6 / tensor_peak)
        y = torch.empty_like(x)
        us = t_us(lambda: P.layernorm(x, prm.ln1_g, prm.ln1_b, out=y))
        emit(op="LayerNorm standalone (a5)", config=cfg, us=us, bound="hbm", achieved_gb_s=4 * T * d / us / 1e3,
             peak_gb_s=hbm_peak, frac=4 * T * d / us / 1e3 / hbm_peak)
    if args.out:
        with open(args.out, "w") as fo:
            for ln in lines:
                fo.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
