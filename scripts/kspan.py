"""Kernel spans of one layer step inside its CUDA graph (profiling build with -DCORA_KSPAN):
    CORA_LIB_PATH=variants/kspan.so python scripts/kspan.py [config[,config...]] [reps]
Configs: synth names (C4-wiki512, C2-mnli, ...), <dataset>-<batch> (mnli-32), or shard<N> (rank 0's shard
of C4 at N ranks).  Per kernel (slot order = launch order): first CTA entry, first / last return from
griddepcontrol.wait, last CTA exit, tail = last minus mean CTA exit, in us from the step's first entry; medians over reps, L2 flushed
(256 MB write + read) before each replay as in bench.py.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P
from paper_2110_10221_b200 import _lib
from paper_2110_10221_b200.dist import shard_rows

NAMES = ["prelude", "attention", "qkv", "outproj+ln1", "ff1", "ff2+ln2"]
ORDER = [0, 2, 1, 3, 4, 5]


def lengths_of(cfg):
    if cfg.startswith("shard"):
        n = int(cfg[5:])
        lengths, d, H, dff = synth.config("C4-wiki512")
        lengths = np.asarray(lengths, np.int64)
        plan, _ = shard_rows(list(lengths), d, dff, n)
        return lengths[plan[0]:plan[1]], d, H, dff
    if cfg.count("-") == 1 and cfg.split("-")[1].isdigit() and not cfg.startswith("C"):
        ds, bs = cfg.split("-")
        return synth.dataset_lengths(ds, int(bs)), 512, 8, 2048
    return synth.config(cfg)


def main():
    cfgs = (sys.argv[1] if len(sys.argv) > 1 else "C4-wiki512").split(",")
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
    lib = _lib.lib()
    tus = [getattr(lib, f"cora_debug_kspan_{t}") for t in ("prelude", "attn", "gemm")]
    buf = (ctypes.c_ulonglong * 48)()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg in cfgs:
        lengths, d, H, dff = lengths_of(cfg)
        lengths = [int(v) for v in lengths]
        T = sum(lengths)
        params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
        if os.environ.get("KSPAN_SPLIT"):  # prelude, then the layer (the QKV GEMM waits for the prelude)
            layer = P.EncoderLayer(params)

            def fwd(Lt, T, x, out):
                layer(x, P.layout_build(Lt, T, H, 512), out=out)
        else:
            fwd = P.EncoderForward(params)
        Lt = torch.tensor(lengths, dtype=torch.int32, device="cuda")
        x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        for _ in range(3):
            fwd(Lt, T, x, out=y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fwd(Lt, T, x, out=y)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        rows, steps = [], []
        for _ in range(reps):
            flush.fill_(1)
            flush.sum(dtype=torch.int32)
            for f in tus:
                f(buf, 1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            steps.append(e0.elapsed_time(e1) * 1e3)
            span = np.zeros((8, 6), dtype=np.int64)
            for si, f in enumerate(tus):
                f(buf, 0)
                a = np.frombuffer(buf, dtype=np.uint64).reshape(8, 6).astype(np.int64)
                # mean exit from the low 40 bits of the exits (the device sums those): max exit - its tail
                low = a[:, 1] & ((1 << 40) - 1)
                a[:, 4] = np.where(a[:, 5] > 0, a[:, 1] - (low - a[:, 4] // np.maximum(a[:, 5], 1)), 0)
                slots = [0] if si == 0 else ([1] if si == 1 else [2, 3, 4, 5])
                for s in slots:
                    span[s] = a[s]
            t0 = min(span[s][0] for s in range(6) if span[s][5] > 0)  # kernels that ran (the prelude may not)
            r = (span[:6, :5] - t0).astype(np.float64) / 1e3
            rows.append(r)
            ran = [span[s][5] > 0 for s in range(6)]
        med = np.median(np.stack(rows), axis=0)
        print(f"== {cfg}: B={len(lengths)} T={T}  step (events) median {np.median(steps):.1f} us")
        print(f"  {'kernel':<12} {'entry':>7} {'wait0':>7} {'wait1':>7} {'exit':>7} | {'wait1->exit':>11} {'tail':>6}")
        prev_exit = 0.0
        for s in ORDER:
            if not ran[s]:
                print(f"  {NAMES[s]:<12} (not launched: inside the QKV GEMM)")
                continue
            e, w1, w0, x_, xm = med[s][0], med[s][2], med[s][3], med[s][1], med[s][4]
            print(f"  {NAMES[s]:<12} {e:7.1f} {w0:7.1f} {w1:7.1f} {x_:7.1f} | {x_ - w1:11.1f} {x_ - xm:6.1f}")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
