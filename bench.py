#!/usr/bin/env python
"""Benchmark of the ragged encoder layer (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4-wiki512] [--impl cora|reference]

A "step" is one pass of the whole hot path over one synthetic ragged batch: the device prelude
(a1: offset tables + tile list) followed by the seven layer kernels (a2..a8), and for N > 1 the
final NCCL all-gather of the ragged outputs.  The batch is the configuration BASELINE.json's
metric is quoted on: bs 128, Wiki512-like lengths (configs[3], "C4").  Metric: useful (unpadded)
TFLOP/s = (2 T (4 d^2 + 2 d d_ff) + 4 d sum L^2) / step time; ms/step is reported beside it.

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on the launching
stream, with an L2 flush between steps (outside the events: 256 MB written, then 256 MB read so the flush's
dirty lines are written back before the step starts); barrier + synchronize on both
sides; the max over ranks.  `--impl reference` times the fp64 CPU oracle instead (the reference
arm of this tier: a deliberately slow program).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "ragged encoder layer useful TFLOP/s (bf16, unpadded FLOPs)"
KERNELS = ["qkv_gemm", "attention", "out_proj_gemm", "layernorm1", "ff1_gemm", "ff2_gemm", "layernorm2"]


def useful_flops(lengths, d, dff) -> int:
    T = int(np.sum(lengths))
    S2 = int(np.sum(np.asarray(lengths, np.int64) ** 2))
    return 2 * T * (4 * d * d + 2 * d * dff) + 4 * d * S2


def padded_flops(lengths, d, dff) -> int:
    Lp = int(np.max(lengths))
    return useful_flops([Lp] * len(lengths), d, dff)


def kernel_work(name, T, S2, d, dff, heads=8):
    """(bound, algorithmic amount per launch, unit) for each layer kernel."""
    if name == "qkv_gemm":
        return "tensor", 2.0 * T * d * 3 * d, "flop"
    if name == "attention":
        # MUFU-bound: one exp2 per useful score, H * sum L^2
        return "alu", float(heads) * S2, "exp"
    if name == "out_proj_gemm":
        # HBM-bound (AI 170 < ridge 249): reads O and the residual x, writes H1 (LayerNorm 1
        # fused into its epilogue), reads W_o once -- 3 T d + d^2 bf16 values
        return "hbm", 2.0 * (3.0 * T * d + d * d), "byte"
    if name == "ff1_gemm":
        return "tensor", 2.0 * T * d * dff, "flop"
    if name == "ff2_gemm":
        return "tensor", 2.0 * T * dff * d, "flop"
    # LayerNorm: read + write one bf16 row each, gamma/beta once
    return "hbm", 2.0 * T * d * 2 + 2 * d * 4, "byte"


def measured_ex2_peak():
    """Measured MUFU.EX2 rate of this GPU (scripts/micro/ex2_bench.cu, built by __graft_entry__.build()):
    the best Gex2/s over its configurations, or None when the binary is missing."""
    exe = os.path.join(ROOT, "scripts", "micro", "ex2_bench")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
    except Exception:
        return None
    best = None
    for line in out.splitlines():
        try:
            j = json.loads(line)
        except ValueError:
            continue
        if j.get("bench") == "ex2" and j.get("gex2_per_s", 0) < 1e5:
            if best is None or j["gex2_per_s"] > best["gex2_per_s"]:
                best = j
    return best


def tile_waste(lay, heads):
    """Masked-lane share of the attention work actually run (the analogue of the paper's partial-padding
    overhead), from the DEVICE work list the prelude built: every item covers
    32 * ceil(rows / 32) query rows (its live warps) times 128 keys per KV tile; the useful part is
    sum over sequences of L^2 per head."""
    tb = {k: v.cpu().numpy() for k, v in lay.tables().items()}
    n = int(tb["n_tiles"][0])
    words = tb["tiles"][:n].astype(np.int64)
    seq = tb["tile_seq"][:2 * n].reshape(-1, 2)
    computed = 0
    for wd, (_ro, L) in zip(words, seq):
        packed = wd < 0
        qt = (wd >> 24) & 0x7F
        rows = int(L) if packed else min(128, int(L) - 128 * int(qt))
        nkv = 1 if packed else -(-int(L) // 128)
        computed += 32 * (-(-rows // 32)) * 128 * nkv
    L = tb["row_off"][1:].astype(np.int64) - tb["row_off"][:-1].astype(np.int64)
    useful = heads * int((L * L).sum())
    return {"useful_scores": useful, "computed_lanes": computed, "waste": 1.0 - useful / computed if computed else 0.0,
            "work_items": n}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"bf16_tflops": j["bf16_tflops"], "bf16_tflops_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                "hbm_gbs": j["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    # B200_PROFILING.md fallback
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"], "samples": 0}
        time.sleep(0.05)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8 and f[0].replace(".", "").isdigit():
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows]
        reasons = set()
        for r in rows:
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": sorted(reasons),
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
                if any(r[2].replace(".", "").isdigit() for r in rows) else None}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count()


def oracle_sample(lengths, w, x, budget_s: float):
    """Time the fp64 oracle on a bounded sample of the workload's sequences (seeded order)."""
    import oracle

    ro = oracle.row_offsets(lengths)
    order = np.random.default_rng(0).permutation(len(lengths))
    done, flops, t_total, n = [], 0, 0.0, 0
    for b in order:
        L = int(lengths[b])
        if L == 0:
            continue
        t0 = time.perf_counter()
        oracle.encoder_layer(x[ro[b]:ro[b] + L], [L], w)
        t_total += time.perf_counter() - t0
        flops += useful_flops([L], w.d_model, w.d_ff)
        n += 1
        done.append(L)
        if t_total >= budget_s:
            break
    return flops, t_total, n, done


def run_reference(args, lengths, d, H, dff, world, rank):
    """The reference arm of this tier: the fp64 CPU oracle on the host cores, rank 0 only."""
    if rank != 0:
        return
    w = synth.encoder_weights(d, H, dff)
    x = synth.activations(int(lengths.sum()), d)
    per_step_budget = max(0.5, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(lengths, w, x, per_step_budget / 4)
    times, flops_all, nseq = [], [], 0
    for _ in range(args.steps):
        f, t, n, _ = oracle_sample(lengths, w, x, per_step_budget)
        times.append(t)
        flops_all.append(f)
        nseq = n
    value = sum(flops_all) / sum(times) / 1e12
    ms = 1e3 * sum(times) / len(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "batch": int(len(lengths)), "total_tokens": int(lengths.sum()),
                   "d_model": d, "heads": H, "d_ff": dff, "parallelism": "host"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": f"{nseq} of {len(lengths)} sequences per step (seeded permutation), fp64 NumPy"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C4-wiki512")
    ap.add_argument("--impl", default="cora", choices=["cora", "reference"])
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-stack", action="store_true", help="skip the 6-layer stack measurement")
    ap.add_argument("--groups", type=int, default=4,
                    help="N > 1 6-layer stack: groups per rank whose gather overlaps the next group's compute")
    ap.add_argument("--no-clocks", action="store_true", help="do not run the nvidia-smi sampler (use under ncu)")
    ap.add_argument("--prewarm", type=int, default=3,
                    help="untimed graph replays (each after an L2 flush) enqueued just before the timed steps")
    ap.add_argument("--no-ex2", action="store_true", help="skip the EX2 peak microbenchmark (use under ncu)")
    ap.add_argument("--debug-gloo", action="store_true",
                    help="N > 1 control-flow check on ONE GPU: ranks share the device, gloo process group, the "
                         "gather through torch.distributed (the library's NCCL path needs one GPU per rank); "
                         "not a measurement")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "cora" and os.environ.get("CORA_ALLOW_FEW_WARMUP") is None:
        args.warmup = 3

    world, rank, local = dist_setup()
    lengths, d, H, dff = synth.config(args.config)
    lengths = np.asarray(lengths, np.int64)

    if args.impl == "reference":
        run_reference(args, lengths, d, H, dff, world, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2110_10221_b200 as P
    from paper_2110_10221_b200.dist import NcclComm, ShardedStack, shard_rows

    if args.debug_gloo:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.debug_gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    # ---------------------------------------------------------------- workload (synthetic, seeded)
    w = synth.encoder_weights(d, H, dff)
    x_all = synth.activations(int(lengths.sum()), d)
    T_all = int(lengths.sum())
    # the library's plan: contiguous, FLOP-balanced, window-aligned sequence ranges and their packed rows
    plan, row_begin = shard_rows(list(lengths), d, dff, world)
    b0, b1 = plan[rank], plan[rank + 1]
    loc_len = lengths[b0:b1]
    T_loc = int(loc_len.sum())
    r0, r1 = row_begin[rank], row_begin[rank + 1]
    x_loc = x_all[r0:r1]
    params = P.EncoderParams.from_host(w, device=dev)
    layer = P.EncoderLayer(params)
    layer_launches = layer.launches(T_loc) if T_loc else layer.launches(T_all)  # 5: GEMM + LN fused, else 7
    fused_ln = layer_launches == 5
    # cora_encoder_forward: batches of <= 256 sequences build the layout in the QKV GEMM's epilogue warps (no
    # prelude kernel, csrc/api.cu forward_impl); larger batches launch the prelude kernel beside the QKV GEMM
    prelude_in_gemm = 1 <= len(loc_len) <= 256 and T_loc > 0 and os.environ.get("CORA_QKV_PRELUDE", "1") != "0"
    prelude_launches = 0 if prelude_in_gemm else 1
    len_dev = torch.tensor(loc_len, dtype=torch.int32, device=dev)
    # every rank holds the whole [T, d] input and output; its own rows are contiguous views of them, so the
    # gather lands in place (no copy)
    x_full = torch.tensor(x_all, dtype=torch.float32).to(torch.bfloat16).to(dev)
    y_full = torch.empty(T_all, d, dtype=torch.bfloat16, device=dev)
    x_dev, y_dev = x_full[r0:r1], y_full[r0:r1]
    # L2 flush between timed steps: write a 256 MB buffer (> the 126 MB L2), then read a second one, so the
    # flush's own dirty lines are written back to HBM before the step's events -- the step starts with a
    # cold L2 holding no line of its inputs and no dirty data of the flush
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(32 << 20, dtype=torch.int64, device=dev)
    flush_acc = torch.empty((), dtype=torch.int64, device=dev)

    def flush_l2():
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=flush_acc)
    stream = torch.cuda.current_stream()

    lay_holder = {}

    fwd = P.EncoderForward(params)

    def step(events=None, pre_event=None):
        if pre_event is not None:
            pre_event.record()
        if events is None and T_loc:
            # the timed step: prelude + layer in one call (cora_encoder_forward: QKV runs under the prelude)
            fwd(len_dev, T_loc, x_dev, out=y_dev)
            return fwd
        # the instrumented step: separate calls, events between the kernels
        lay = P.layout_build(len_dev, T_loc, H, 512) if T_loc else None
        lay_holder["lay"] = lay
        if lay is not None:
            layer(x_dev, lay, out=y_dev, events=events)
        elif events is not None:
            for e in events:
                e.record()
        return lay

    # N > 1: the library's own NCCL communicator and in-place ragged all-gather (cora_allgather_ragged)
    lib_comm = NcclComm(rank, world) if world > 1 and not args.debug_gloo else None

    def gather():
        if lib_comm is not None:
            lib_comm.allgather_ragged(y_full, row_begin)
        else:  # --debug-gloo: the same in-place schedule through torch.distributed
            for r in range(world):
                if row_begin[r + 1] > row_begin[r]:
                    dist.broadcast(y_full[row_begin[r]:row_begin[r + 1]], src=r)

    # correctness gate on the benchmarked configuration (status word)
    lay = step()
    if lay is not None:
        assert lay.status() == 0, "layout status != 0"
    if world > 1:
        gather()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    n_ev = P._lib.LAYER_EVENTS
    pre_ev = torch.cuda.Event(enable_timing=True, external=True)  # external: a graph node when captured
    kev = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    for e in [pre_ev] + kev:  # torch creates events lazily: materialise them before capture
        e.record()
    torch.cuda.synchronize()
    graph = graph_ev = None
    if not args.no_graph and T_loc:
        # the step as ONE CUDA graph: prelude (a1) + the layer kernels, chained with programmatic
        # dependent launch.  graph_ev is the same step with event-record nodes between the kernels (for
        # the per-kernel breakdown; those nodes break the PDL overlap, so it is timed separately).
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph_ev = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_ev):
            step(kev, pre_ev)
        for _ in range(args.warmup):
            graph.replay()
            graph_ev.replay()
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()

    def timed(run, n, per_step=None):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i in range(n):
            if not args.no_flush:
                flush_l2()
            evs[i][0].record(stream)
            run()
            evs[i][1].record(stream)
            if per_step is not None:
                evs[i][1].synchronize()
                per_step()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    kern_rec, pre_rec = [], []

    def read_kernel_events():
        kern_rec.append([kev[j].elapsed_time(kev[j + 1]) for j in range(n_ev - 1)])
        pre_rec.append(pre_ev.elapsed_time(kev[0]))

    sampler = ClockSampler(local)
    if not args.no_clocks:
        sampler.start()
        time.sleep(0.1)
    try:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # warm-up replays enqueued right before the timed steps (outside the events), so the timed region
        # does not start on a GPU that idled while the clock sampler started
        if graph is not None:
            for _ in range(args.prewarm):
                if not args.no_flush:
                    flush_l2()
                graph.replay()
        # ---- the timed region: exactly K steps
        if graph is not None:
            step_ms = timed(graph.replay, args.steps)
        elif T_loc:
            step_ms = timed(lambda: step(kev, pre_ev), args.steps, read_kernel_events)
        else:  # a rank with no sequences: nothing to launch, it only joins the barriers and the gather
            step_ms = timed(lambda: None, args.steps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    finally:
        clocks = sampler.stop()
    # ---- per-kernel breakdown (instrumented replays of the same step)
    if graph_ev is not None:
        kern_step_ms = timed(graph_ev.replay, args.steps, read_kernel_events)
    else:
        kern_step_ms = step_ms

    ms_local = float(np.mean(step_ms))
    kern_ms = {k: float(np.mean([rec[j] for rec in kern_rec])) if kern_rec else 0.0 for j, k in enumerate(KERNELS)}
    prelude_ms = float(np.mean(pre_rec)) if pre_rec else 0.0
    pct_local = [float(np.percentile(step_ms, q)) for q in (10, 50, 90)]
    if world > 1:
        t = torch.tensor([ms_local] + pct_local, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, *pct = (float(v) for v in t.tolist())
    else:
        ms, pct = ms_local, pct_local

    # ---------------------------------------------------------------- N > 1: the all-gather
    # `value` is the compute makespan (max over ranks from a common barrier, the scaling
    # target); the NCCL all-gather of the ragged outputs is timed alone (ii) and with the step (iii)
    gather_info = None
    if world > 1:
        run_step = graph.replay if graph is not None else ((lambda: step()) if T_loc else (lambda: None))
        for _ in range(args.warmup):
            gather()
        torch.cuda.synchronize()
        dist.barrier()
        g_ms = float(np.mean(timed(gather, args.steps)))
        dist.barrier()

        def step_and_gather():
            run_step()
            gather()

        sg_ms = float(np.mean(timed(step_and_gather, args.steps)))
        t = torch.tensor([g_ms, sg_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        g_ms, sg_ms = (float(v) for v in t.tolist())
        gather_info = {"allgather_ms": g_ms, "bytes_received_per_rank": int((T_all - T_loc) * d * 2),
                       "path": ("torch.distributed gloo broadcasts (--debug-gloo control-flow check, ranks share one GPU)"
                                if args.debug_gloo else
                                "cora_allgather_ragged (the library's NCCL communicator, grouped in-place broadcasts)"),
                       "with_gather": {"ms_per_step": sg_ms,
                                       "value": useful_flops(lengths, d, dff) / (sg_ms * 1e-3) / 1e12,
                                       "unit": "TFLOP/s"},
                       "note": "value / ms_per_step: (i) compute makespan (prelude + layer per rank, max over "
                               "ranks); (ii) allgather_ms: the gather alone; (iii) with_gather: the step then the "
                               "gather, end to end; stack6: the 6-layer model with the gather overlapped"}

    # ---------------------------------------------------------------- the paper's 6-layer model (SURVEY f-4)
    # one layout (prelude) per batch shared by 6 layers, one CUDA graph per
    # step, L2 flushed between steps like the headline number; reported beside it, not instead of it
    stack = None
    if not args.no_stack and not (world > 1 and args.debug_gloo):
        stack_params = [P.EncoderParams.from_host(synth.encoder_weights(d, H, dff, seed=200 + i), device=dev)
                        for i in range(6)]
        n_stack = max(3, min(args.steps, 50))
        if world == 1:
            enc_stack = P.EncoderStack(stack_params)
            y_stack = torch.empty_like(y_dev)

            def stack_step():
                enc_stack(x_dev, P.layout_build(len_dev, T_loc, H, 512), out=y_stack)

            stack_step()
            torch.cuda.synchronize()
            g_stack = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_stack):
                stack_step()
            for _ in range(args.warmup):
                g_stack.replay()
            torch.cuda.synchronize()
            st_ms = float(np.mean(timed(g_stack.replay, n_stack)))
            what = "prelude(a1) once + 6 encoder layers, one CUDA graph"
            # the same 6 layers cut into the gather groups the sharded stack uses at N > 1 (no communicator):
            # the price of the group split that lets the gather overlap the compute
            sh1 = ShardedStack(stack_params, n_groups=args.groups)
            len_h1 = torch.tensor(loc_len, dtype=torch.int32)
            y_sh1 = torch.empty_like(y_dev)
            sh1(len_dev, len_h1, x_dev, out=y_sh1)
            torch.cuda.synchronize()
            g_sh1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_sh1):
                sh1(len_dev, len_h1, x_dev, out=y_sh1)
            for _ in range(args.warmup):
                g_sh1.replay()
            torch.cuda.synchronize()
            grouped_ms = float(np.mean(timed(g_sh1.replay, n_stack)))
        else:
            # every rank: its sequences in `groups` window-aligned groups, each one layout through the 6
            # layers; group g's rows are gathered (NCCL, side stream) while group g + 1 computes
            sh = ShardedStack(stack_params, n_groups=args.groups)
            len_all_dev = torch.tensor(lengths, dtype=torch.int32, device=dev)
            len_all_host = torch.tensor(lengths, dtype=torch.int32)
            y_sh = torch.empty_like(y_full)

            def stack_step():
                sh(len_all_dev, len_all_host, x_full, comm=lib_comm, out=y_sh)

            for _ in range(args.warmup):
                stack_step()
            torch.cuda.synchronize()
            dist.barrier()
            st_ms = float(np.mean(timed(stack_step, n_stack)))
            t = torch.tensor([st_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            st_ms = float(t.item())
            what = (f"cora_encoder_stack_sharded_fwd: per rank {args.groups} groups x (prelude + 6 layers), each "
                    "group's outputs all-gathered while the next computes; every rank ends with all T rows")
        stack = {"layers": 6, "ms_per_step": st_ms, "steps": n_stack,
                 "value": 6 * useful_flops(lengths, d, dff) / (st_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                 "step": what}
        if world == 1:
            stack["grouped"] = {"groups": args.groups, "ms_per_step": grouped_ms,
                                "note": "cora_encoder_stack_sharded_fwd with one rank: the batch in window-aligned "
                                        "groups, each one layout through the 6 layers (the N > 1 overlap schedule "
                                        "without the gather)"}

    # ---------------------------------------------------------------- e2e: host buffers through the C ABI
    e2e = None
    if not args.no_e2e:
        e2e_ms, h2d, d2h = 0.0, 0, 0
        if T_loc:
            hf = P.HostForward(params, len(loc_len), T_loc, 512, device=dev)
            len_h = torch.tensor(loc_len, dtype=torch.int32).pin_memory()
            x_h = torch.tensor(x_loc, dtype=torch.float32).to(torch.bfloat16).pin_memory()
            y_h = torch.empty(T_loc, d, dtype=torch.bfloat16).pin_memory()
            for _ in range(args.warmup):
                hf(len_h, x_h, y_h)
            torch.cuda.synchronize()
            assert hf.status() == 0
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            for i in range(args.steps):
                if not args.no_flush:
                    flush_l2()
                ev[i][0].record(stream)
                hf(len_h, x_h, y_h)
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            e2e_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
            h2d, d2h = int(x_h.numel() * 2 + len_h.numel() * 4), int(y_h.numel() * 2)
        if world > 1:  # every rank joins (an empty rank contributes 0), so none waits forever
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": useful_flops(lengths, d, dff) / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "cora_encoder_forward_host (pinned host buffers)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    ex2 = None if args.no_ex2 else measured_ex2_peak()
    total_flops = useful_flops(lengths, d, dff)
    value = total_flops / (ms * 1e-3) / 1e12
    T, S2 = int(loc_len.sum()), int((loc_len ** 2).sum())
    sm_count = int(P._lib.lib().cora_device_sm_count())
    kernels = {}
    for k in KERNELS:
        bound, work, unit = kernel_work(k, T, S2, d, dff, H)
        dur = kern_ms[k] * 1e-3
        if k.startswith("layernorm") and fused_ln:
            # LayerNorm runs in the preceding GEMM's epilogue (cora_linear_residual_layernorm_fwd): no
            # kernel of its own; its time is inside that GEMM's interval (the events around it coincide)
            kernels[k] = {"fused_into": "out_proj_gemm" if k == "layernorm1" else "ff2_gemm"}
            continue
        if bound == "tensor":
            ach = work / dur / 1e12
            peak = peaks["bf16_tflops_sustained"]
            kernels[k] = {"ms": kern_ms[k], "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                          "frac": ach / peak}
        elif bound == "alu":
            # exponentials vs the MUFU.EX2 rate measured on this GPU (scripts/micro/ex2_bench.cu), else the
            # nominal 16 / clk / SM x SMs x max SM clock (2x on B300 only)
            ach = work / dur / 1e9
            if ex2 is not None:
                peak = ex2["gex2_per_s"]
                src = (f"measured: scripts/micro/ex2_bench.cu ({ex2['ex2_per_clk_per_sm_at_max_clock']:.2f} "
                       "EX2/clk/SM at the max clock)")
            else:
                peak = 16.0 * sm_count * (clocks.get("sm_max_mhz") or 1965.0) * 1e6 / 1e9
                src = "nominal: 16 MUFU.EX2/clk/SM x SMs x max SM clock (ex2 microbenchmark missing)"
            tf = 4.0 * d * S2 / dur / 1e12
            kernels[k] = {"ms": kern_ms[k], "bound": "alu", "achieved": ach, "peak": peak, "unit": "Gexp/s",
                          "frac": ach / peak, "peak_source": src,
                          "tensor_view": {"achieved": tf, "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                                          "frac": tf / peaks["bf16_tflops_sustained"]}}
        else:
            ach = work / dur / 1e9
            peak = peaks["hbm_gbs"]
            kernels[k] = {"ms": kern_ms[k], "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                          "frac": ach / peak}
            if k == "out_proj_gemm":
                tf = 2.0 * T * d * d / dur / 1e12
                kernels[k]["tensor_view"] = {"achieved": tf, "peak": peaks["bf16_tflops_sustained"],
                                             "unit": "TFLOP/s", "frac": tf / peaks["bf16_tflops_sustained"]}
    for k in ("out_proj_gemm", "ff2_gemm"):
        if fused_ln:
            kernels[k]["epilogue"] = "bias + residual + LayerNorm (fused)"
    dom = max((k for k in KERNELS if "achieved" in kernels[k]), key=lambda k: kern_ms[k])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)
    roofline = {"kernel": dom, "bound": kernels[dom]["bound"], "achieved": kernels[dom]["achieved"],
                "peak": kernels[dom]["peak"], "unit": kernels[dom]["unit"], "frac": kernels[dom]["frac"],
                "traffic": traffic,
                "peak_source": kernels[dom].get("peak_source") or (
                    peaks["source"] + (" sustained" if kernels[dom]["bound"] == "tensor" else ""))}

    waste = tile_waste(P.layout_build(len_dev, T_loc, H, 512), H) if T_loc else None

    cpu = None
    if world == 1 and not args.no_cpu:
        lengths_c, _, _, _ = synth.config(args.config)
        f, t, n, _ = oracle_sample(np.asarray(lengths_c), w, x_all, args.cpu_budget)
        cpu = {"value": f / t / 1e12, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"{n} of {len(lengths)} sequences of {args.config} (seeded permutation), fp64 NumPy, "
                         f"{t:.1f} s"}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": args.config, "batch": int(len(lengths)), "total_tokens": int(lengths.sum()),
                   "sum_L2": int((lengths ** 2).sum()), "max_len": int(lengths.max()), "d_model": d, "heads": H,
                   "d_ff": dff, "parallelism": f"seq-shard{world}" if world > 1 else "single",
                   "l2": "no flush" if args.no_flush else ("flushed between steps: 256 MB written, then 256 MB read "
                                                            "(the flush's dirty lines leave L2 before the step)"),
                   "step": ("prelude(a1) in the QKV GEMM's epilogue warps + " if prelude_in_gemm else "prelude(a1) + ")
                   + f"{layer_launches} layer kernels (a2..a8"
                   + (", LayerNorm fused into the out-proj / FF2 GEMM epilogues)" if fused_ln else ")") + (" per rank; NCCL all-gather timed separately (multi_gpu)" if world > 1 else ""),
                   "launch": "eager" if args.no_graph else "CUDA graph replay per step, programmatic dependent launch"},
        "frac_of_peak": {"burst": value / peaks["bf16_tflops"], "sustained": value / peaks["bf16_tflops_sustained"],
                         "source": peaks["source"]},
        "ms_percentiles": {"p10": pct[0], "p50": pct[1], "p90": pct[2]},
        "padded_over_useful_flops": padded_flops(lengths, d, dff) / total_flops,
        "attention_tile_waste": waste,
        "roofline": roofline,
        "kernels": kernels,
        "prelude_ms": prelude_ms,
        "stack6": stack,
        "multi_gpu": gather_info,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": (prelude_launches + layer_launches) * args.steps,
        "kernel_timing": ("CUDA events between the kernels in an instrumented replay of the same graph, "
                          f"{args.steps} steps after the timed region; those event nodes disable the PDL overlap, so "
                          "per-kernel times are upper bounds (instrumented step "
                          f"{float(np.mean(kern_step_ms)):.4f} ms vs timed {ms:.4f} ms)"),
        "clocks": clocks,
        "paper_context": {"cora_v100_fp32_ms_wiki512_bs128": 32.17, "ft_eff_v100_fp32_ms": 33.66,
                          "source": "PAPER.md:870-872 (Table 4), other hardware and precision"},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
