#!/usr/bin/env python
"""Config sweep: step time, useful TFLOP/s, padded/useful FLOP ratio and attention tile
waste for every BASELINE.json configuration, one GPU.  Writes JSON lines to stdout.

    python scripts/sweep.py [--steps K] [configs...]
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
from bench import tile_waste


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("configs", nargs="*")
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    configs = args.configs or (synth.SWEEP_CONFIGS + synth.TABLE4_CONFIGS)
    for cfg in configs:
        lengths, d, H, dff = synth.config(cfg)
        lengths = np.asarray(lengths, np.int64)
        T = int(lengths.sum())
        S2 = int((lengths ** 2).sum())
        w = synth.encoder_weights(d, H, dff)
        layer = P.EncoderLayer(P.EncoderParams.from_host(w))
        x = torch.tensor(synth.activations(T, d), dtype=torch.float32).to(torch.bfloat16).cuda()
        y = torch.empty_like(x)
        Lt = torch.tensor(lengths, dtype=torch.int32, device="cuda")

        def step():
            layer(x, P.layout_build(Lt, T, H, 512), out=y)

        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(3):
            g.replay()
        times = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b))
        ms = float(np.median(times))
        useful = 2 * T * (4 * d * d + 2 * d * dff) + 4 * d * S2
        Lp = int(lengths.max())
        padded = 2 * len(lengths) * Lp * (4 * d * d + 2 * d * dff) + 4 * d * len(lengths) * Lp * Lp
        # masked share of the attention work actually run, from the device work list (packed windows included)
        waste = tile_waste(P.layout_build(Lt, T, H, 512), H)
        print(json.dumps({
            "config": cfg, "batch": int(len(lengths)), "total_tokens": T, "sum_L2": S2, "max_len": Lp,
            "ms_per_step_p50": ms, "ms_p10": float(np.percentile(times, 10)), "ms_p90": float(np.percentile(times, 90)),
            "useful_tflops": useful / (ms * 1e-3) / 1e12,
            "frac_of_burst_peak": useful / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
            "padded_over_useful_flops": padded / useful,
            "attention_tile_waste": waste["waste"], "attention_work_items": waste["work_items"],
        }), flush=True)


if __name__ == "__main__":
    main()
