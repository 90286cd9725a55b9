"""Small invocations of every entry point, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|initcheck|synccheck python scripts/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_2110_10221_b200 as P

# the third batch (T ~ 12k) gives the fused GEMM + LN kernels several 256-row units per cluster
for lengths, d, H, dff in ((list(synth.C1_LENGTHS), 16, 2, 32), ([3, 130, 1, 64, 0, 7], 512, 8, 2048),
                           (list(synth.uniform_lengths(40, 100, 512, seed=5)), 512, 8, 2048)):
    T = int(np.sum(lengths))
    w = synth.encoder_weights(d, H, dff)
    params = P.EncoderParams.from_host(w)
    L = torch.tensor(lengths, dtype=torch.int32, device="cuda")
    x = torch.tensor(synth.activations(T, d), dtype=torch.float32).to(torch.bfloat16).cuda()
    lay = P.layout_build(L, T, H, 512)
    y = P.encoder_layer(x, lay, params)
    y2 = P.EncoderForward(params)(L, T, x)
    y3 = P.EncoderStack([params, params])(x, lay)
    qkv = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
    o = P.ragged_attention(lay, qkv, d // H, causal=True)
    S2 = int(np.sum(np.asarray(lengths) ** 2))
    xs = torch.randn(H * S2, device="cuda").to(torch.bfloat16)
    ys = P.ragged_softmax(lay, xs)
    ln = P.layernorm(x, params.ln1_g, params.ln1_b)
    torch.cuda.synchronize()
    print("layer", lengths, float(y.float().abs().mean()), float(y2.float().abs().mean()), float(y3.float().abs().mean()),
          float(o.float().abs().mean()), float(ys.float().sum()), float(ln.float().abs().mean()), flush=True)
    # round 2: the sharded stack (gather groups, one rank), the causal kernel's chunk liveness
    from paper_2110_10221_b200.dist import ShardedStack
    y4 = ShardedStack([params, params], n_groups=3)(L, torch.tensor(lengths, dtype=torch.int32), x)
    o2 = P.ragged_attention(lay, qkv, d // H)
    torch.cuda.synchronize()
    print("round2", float(y4.float().abs().mean()), float(o2.float().abs().mean()), flush=True)
dims = [(130, 264, 128), (64, 8, 64), (64, 64, 0)]
a = torch.randn(3, 130, 128, device="cuda").to(torch.bfloat16)
b = torch.randn(3, 128, 264, device="cuda").to(torch.bfloat16)
c = P.vgemm(a, b, dims)
l = torch.randn(384, 384, device="cuda").to(torch.bfloat16)
bb = torch.randn(384, 64, device="cuda").to(torch.bfloat16)
t = P.trmm(l, bb)
torch.cuda.synchronize()
print("matmul", float(c.float().abs().mean()), float(t.float().abs().mean()))
