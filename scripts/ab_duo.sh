#!/bin/bash
# DUO LN GEMMs (CORA_LN_DUO=1) against the 4-CTA clusters: bitwise layer outputs, parity tests, kernel spans,
# bench steps.  Output under gpurun_out/duo/
mkdir -p gpurun_out/duo
timeout 120 python scripts/dump_layer.py gpurun_out/duo/base.pt
CORA_LN_DUO=1 timeout 120 python scripts/dump_layer.py gpurun_out/duo/duo.pt
python - <<'PY'
import torch
a, b = torch.load("gpurun_out/duo/base.pt"), torch.load("gpurun_out/duo/duo.pt")
for k in a:
    d = (a[k].float() - b[k].float()).abs()
    print(f"{k}: bitwise {torch.equal(a[k], b[k])}, differing {int((a[k] != b[k]).sum())} of {a[k].numel()}, max |d| {d.max().item():.3g}")
PY
CORA_LN_DUO=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "ln or layer or stack or host" -p no:cacheprovider 2>&1 | tail -3
for v in 0 1; do
  CORA_LN_DUO=$v CORA_LIB_PATH=variants/kspan.so timeout 200 python scripts/kspan.py C4-wiki512,shard8,C2-mnli 9 2>&1 | sed "s/^/duo=$v /"
done
for rep in 1 2; do for v in 0 1; do
  CORA_LN_DUO=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu --no-stack --no-ex2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('duo=$v', d['ms_per_step'], {k: round(v['ms']*1e3,1) for k, v in d.get('kernels', {}).items() if 'ms' in v} if isinstance(d.get('kernels'), dict) else '')"
done; done
