"""Layer outputs of a few configurations saved to a file (bitwise A/B of library variants):
    python scripts/dump_layer.py out.pt [config,...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
import paper_2110_10221_b200 as P
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from kspan import lengths_of

out = {}
for cfg in (sys.argv[2] if len(sys.argv) > 2 else "C4-wiki512,C2-mnli,shard8").split(","):
    lengths, d, H, dff = lengths_of(cfg)
    lengths = [int(v) for v in lengths]
    T = sum(lengths)
    torch.manual_seed(0)
    params = P.EncoderParams.from_host(synth.encoder_weights(d, H, dff))
    fwd = P.EncoderForward(params)
    Lt = torch.tensor(lengths, dtype=torch.int32, device="cuda")
    x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    out[cfg] = fwd(Lt, T, x).cpu()
torch.save(out, sys.argv[1])
