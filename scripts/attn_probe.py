"""Attention kernel alone, timed as a CUDA graph of back-to-back calls (profiling helper).

    python scripts/attn_probe.py [config[,config...]] [reps]
Configs: synth names (C4-wiki512, C3, ...), ds:<dataset>:<batch>, or L<len>x<batch> (equal lengths).
Prints per call: us, q-tiles, KV steps (128 x 128 score tiles), clk per score tile per SM at the
measured SM clock, useful exponentials / s.  Library variant: CORA_LIB_PATH=variants/<name>.so.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P


def lengths_of(name):
    if name.startswith("L"):
        ln, bs = name[1:].split("x")
        return np.full(int(bs), int(ln), dtype=np.int64)
    if name.startswith("ds:"):
        _, ds, bs = name.split(":")
        return synth.dataset_lengths(ds, int(bs))
    return synth.config(name)[0]


def main():
    cfgs = (sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512").split(",")
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    causal_too = os.environ.get("CAUSAL", "1") == "1"
    H, d = 8, 512
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk_ghz = float(os.environ.get("SM_GHZ", "1.965"))
    for cfg in cfgs:
        L = lengths_of(cfg).astype(np.int64)
        T = int(L.sum())
        maxlen = max(512, int(-(-int(L.max()) // 128) * 128))
        qkv = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
        lay = P.layout_build(torch.tensor(L, dtype=torch.int32, device="cuda"), T, H, maxlen)
        o = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
        nq = -(-L // 128)
        qtiles = int(nq.sum()) * H
        steps = int((nq * nq).sum()) * H
        steps_c = int((nq * (nq + 1) // 2).sum()) * H
        res = {}
        for causal in ((False, True) if causal_too else (False,)):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    P.ragged_attention(lay, qkv, 64, out=o, causal=causal, stream=s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    P.ragged_attention(lay, qkv, 64, out=o, causal=causal, stream=s)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e30
            for _ in range(3):
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
            st = steps_c if causal else steps
            clk = best * 1e-6 * clk_ghz * 1e9 * sms / st
            res["causal" if causal else "bidir"] = (best, st, clk)
        b = res["bidir"]
        line = (f"{cfg}: T {T} q-tiles {qtiles} steps {b[1]} | bidir {b[0]:.1f} us, {b[2]:.0f} clk/step/SM, "
                f"{H * int((L * L).sum()) / b[0] / 1e3:.0f} Gexp/s")
        if "causal" in res:
            c = res["causal"]
            line += f" | causal {c[0]:.1f} us, {c[1]} steps, {c[2]:.0f} clk/step/SM, ratio {c[0] / b[0]:.2f}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
