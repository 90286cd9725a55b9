"""Multi-process (gloo, CPU) tests of the sharded path's host logic and its gather schedule.

Every rank derives the plan (cora_shard_plan) and the groups (cora_shard_groups) from the library itself --
host-only C entry points, no GPU -- computes its own groups (the fp64 oracle stands in for the device
layers), and after each group issues the same set of in-place broadcasts (one per root rank, that root's
rows of the group) that cora_encoder_stack_sharded_fwd issues over NCCL.  Every rank must end with the
whole batch's output, equal to the single-process result; a rank that owns no sequence must not stall the
others.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stack(x, lengths, ws):
    for w in ws:
        x = oracle.encoder_layer(x, lengths, w)
    return x


def _worker(rank, world, port, lengths, n_groups, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_10221_b200.api import shard_groups
        from paper_2110_10221_b200.dist import shard_rows

        lengths = np.asarray(lengths)
        d, H, dff = 16, 2, 32
        ws = [synth.encoder_weights(d, H, dff, seed=s) for s in (1, 2)]
        T = int(lengths.sum())
        x = synth.activations(T, d)
        plan, rows = shard_rows(list(lengths), d, dff, world)
        gseq, grow = shard_groups(list(lengths), plan, n_groups)
        y_full = torch.zeros(T, d, dtype=torch.float64)
        for g in range(n_groups):
            b0, b1 = gseq[rank][g], gseq[rank][g + 1]
            r0, r1 = grow[rank][g], grow[rank][g + 1]
            if r1 > r0:  # this rank's group g: one ragged batch through every layer
                y_full[r0:r1] = torch.from_numpy(_stack(x[r0:r1], lengths[b0:b1], ws))
            for r in range(world):  # the group's gather: every root's rows of group g, same order on every rank
                if grow[r][g + 1] > grow[r][g]:
                    dist.broadcast(y_full[grow[r][g]:grow[r][g + 1]], src=r)
        ref = _stack(x, lengths, ws)
        q.put((rank, plan, rows, gseq, bool(np.array_equal(y_full.numpy(), ref))))
    finally:
        dist.destroy_process_group()


def _run(world, lengths, n_groups):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lengths, n_groups, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,n_groups", [(2, 1), (2, 3)])
def test_sharded_stack_gather_cpu(world, n_groups):
    lengths = [5, 0, 140, 3, 12, 1, 200, 7, 40, 130, 9, 60]
    res = _run(world, lengths, n_groups)
    assert len({tuple(pl) for _, pl, _, _, _ in res}) == 1  # every rank derives the same plan
    plan = res[0][1]
    assert plan == oracle.shard_plan(lengths, 16, 32, world)
    assert res[0][2] == [oracle.row_offsets(lengths)[b] for b in plan]
    for _, _, _, gseq, _ in res:  # groups partition every rank's range, window-aligned
        ok = oracle.shard.allowed_cuts(lengths)
        for r in range(world):
            assert gseq[r][0] == plan[r] and gseq[r][-1] == plan[r + 1] and gseq[r] == sorted(gseq[r])
            assert all(ok[c] for c in gseq[r])
    assert all(good for *_, good in res)


def test_sharded_gather_with_an_empty_rank_cpu():
    # 3 ranks, 2 indivisible units (a long sequence and one window of short ones): rank 2 owns nothing and
    # must still take part in every group's broadcasts without stalling the others
    lengths = [300, 2, 3]
    res = _run(3, lengths, 2)
    plan = res[0][1]
    assert plan[-2] == plan[-1] == 3  # the last rank is empty
    assert all(good for *_, good in res)
