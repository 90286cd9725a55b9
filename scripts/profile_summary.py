#!/usr/bin/env python
"""Summarise a gpurun ncu capture into profiles/ (committed evidence).

    python scripts/profile_summary.py gpurun_out/<tag> profiles/<name>

Reads <tag>/launches.csv (ncu --metrics gpu__time_duration.sum launch list of one bench step)
and, if present, <tag>/prof.ncu-rep (ncu --set full capture), and writes
  profiles/<name>_launches.md   per-kernel launch times of one step and their shares
  profiles/<name>_ncu.md        per-kernel DRAM bytes, throughput, tensor/XU pipe use, stalls
  profiles/ncu_traffic.json     dram read+write bytes per launch for bench.py's roofline.traffic
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

# launch order of one layer step (prelude kernels first), see bench.py KERNELS
STEP_ORDER = ["prelude", "qkv_gemm", "attention", "out_proj_gemm", "layernorm1", "ff1_gemm", "ff2_gemm",
              "layernorm2"]

STEP_ORDER_FUSED = ["prelude", "qkv_gemm", "attention", "out_proj_gemm+ln1", "ff1_gemm", "ff2_gemm+ln2"]


def short(name: str) -> str:
    for key in ("layout_merged", "layout_scan", "fusion_maps", "gemm", "attention_fwd", "attention_simt", "layernorm",
                "ragged_softmax", "FillFunctor", "vectorized_elementwise", "reduce_kernel", "reduce"):
        if key in name:
            return key
    return name[:40]


def read_csv_after_header(path, first_col):
    lines = open(path).read().splitlines()
    for i, line in enumerate(lines):
        if line.startswith(f'"{first_col}"'):
            return list(csv.reader(io.StringIO("\n".join(lines[i:]))))
    return []


def launches(tag_dir):
    path = os.path.join(tag_dir, "launches.csv")
    if not os.path.exists(path):
        return None
    rows = read_csv_after_header(path, "ID")
    if not rows:
        return None
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    seq = [(short(r[ik]), float(r[iv]) / 1000.0) for r in rows[1:] if len(r) > iv]
    # keep our kernels of the LAST complete step (layout_scan starts a step)
    ours = [(k, t) for k, t in seq if k not in ("FillFunctor", "vectorized_elementwise", "reduce_kernel", "reduce")]
    starts = [i for i, (k, _) in enumerate(ours) if k in ("layout_merged", "layout_scan")]
    if not starts:
        # the prelude inside the QKV GEMM (cora_encoder_forward, <= 256 sequences): a step is the 5 kernels from
        # the GEMM launched right before an attention kernel
        att = [i for i, (k, _) in enumerate(ours) if k == "attention_fwd" and i >= 1]
        order = ["qkv_gemm+prelude", "attention", "out_proj_gemm+ln1", "ff1_gemm", "ff2_gemm+ln2"]
        for i in reversed(att):
            last = ours[i - 1:i - 1 + len(order)]
            if len(last) == len(order):
                return [(want, k, t) for (k, t), want in zip(last, order)]
        return None
    # the last step that has all its kernels (the launch list may end with an incomplete one)
    last = ours[starts[-1]:]
    if len(last) < len(STEP_ORDER_FUSED) and len(starts) > 1:
        last = ours[starts[-2]:starts[-1]]
    # 5 layer kernels: LayerNorm fused into the out-proj / FF2 GEMM epilogues (d_model 512)
    order = STEP_ORDER_FUSED if len(last) == len(STEP_ORDER_FUSED) else STEP_ORDER
    last = last[:len(order)]
    named = []
    for (k, t), want in zip(last, order):
        named.append((want, k, t))
    return named


def ncu_full(tag_dir):
    rep = os.path.join(tag_dir, "prof.ncu-rep")
    if not os.path.exists(rep):
        return None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = {
        "time_us": "gpu__time_duration.sum",
        "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "tensor_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "grid": "launch__grid_size",
        "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
    }
    stall_cols = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), j) for j, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    res = []
    for r in data:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, m in want.items():
            if m in hdr:
                j = hdr.index(m)
                v = r[j].replace(",", "")
                try:
                    val = float(v)
                except ValueError:
                    val = None
                u = units[j]
                if val is not None and k in ("dram_read", "dram_write"):
                    val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if val is not None and k == "time_us":
                    val *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
                d[k] = val
        stalls = sorted(((n, float(r[j] or 0)) for n, j in stall_cols), key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        d["top_stalls"] = [(n, round(100 * v / tot, 1)) for n, v in stalls[:5]]
        res.append(d)
    return res


def main():
    tag_dir, out_prefix = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.dirname(out_prefix) or ".", exist_ok=True)
    L = launches(tag_dir)
    if L:
        tot = sum(t for _, _, t in L)
        with open(out_prefix + "_launches.md", "w") as f:
            f.write(f"# Launch list of one bench step ({tag_dir}; ncu gpu__time_duration.sum, --clock-control none)\n\n")
            f.write("Cold-cache, serialised per-launch times under ncu: compare SHARES with bench.py's live numbers, "
                    "not absolutes.\n\n| step kernel | ncu kernel | us | share |\n|---|---|---:|---:|\n")
            for want, k, t in L:
                f.write(f"| {want} | {k} | {t:.1f} | {100 * t / tot:.1f}% |\n")
            f.write(f"| **sum** | | **{tot:.1f}** | 100% |\n")
    N = ncu_full(tag_dir)
    if N:
        with open(out_prefix + "_ncu.md", "w") as f:
            f.write(f"# ncu --set full summary ({tag_dir})\n\n| kernel | us | DRAM read MB | DRAM write MB | DRAM % | "
                    "tensor (UTCHMMA bf16) % | XU % | regs | warps active % | top stalls (% of samples) |\n"
                    "|---|---:|---:|---:|---:|---:|---:|---:|---:|---|\n")
            for d in N:
                f.write(f"| {d['kernel']} | {d.get('time_us') or 0:.1f} | {(d.get('dram_read') or 0) / 1e6:.1f} | "
                        f"{(d.get('dram_write') or 0) / 1e6:.1f} | {d.get('dram_pct') or 0:.1f} | "
                        f"{d.get('tensor_pct') or 0:.1f} | {d.get('xu_pct') or 0:.1f} | {int(d.get('regs') or 0)} | "
                        f"{d.get('warps_active_pct') or 0:.1f} | "
                        + ", ".join(f"{n} {v}" for n, v in d["top_stalls"]) + " |\n")
        # traffic per bench kernel key (ordered as captured: gemm x4 in step order, attention, layernorm x2)
        tp = os.path.join(os.path.dirname(out_prefix), "ncu_traffic.json")
        traffic = json.load(open(tp)) if os.path.exists(tp) else {}
        gemm_keys = iter(["qkv_gemm", "out_proj_gemm", "ff1_gemm", "ff2_gemm"])
        ln_keys = iter(["layernorm1", "layernorm2"])
        order = [d["kernel"] for d in N]
        for d in N:
            key = None
            if d["kernel"] == "gemm" and order.count("gemm") == 4:
                key = next(gemm_keys)
            elif d["kernel"] == "attention_fwd":
                key = "attention"
            elif d["kernel"] == "layernorm" and order.count("layernorm") == 2:
                key = next(ln_keys)
            if key and d.get("dram_read") is not None:
                traffic[key] = d["dram_read"] + (d.get("dram_write") or 0)
        if "layernorm" not in order and order.count("gemm") == 4:
            for k in ("layernorm1", "layernorm2"):  # fused into the GEMM epilogues: no kernel of their own
                traffic.pop(k, None)
        traffic["_source"] = f"ncu --set full capture {tag_dir} (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        json.dump(traffic, open(tp, "w"), indent=1)
    print("wrote", out_prefix, "launches" if L else "", "ncu" if N else "")


if __name__ == "__main__":
    main()
