"""World-size-2 gloo test of the multi-GPU host path on CPU: FLOP-balanced contiguous shard plan,
per-rank work on its own sequence range, in-place ragged all-gather -> the full batch in order."""
import os
import socket

import numpy as np
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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_10221_b200.dist import allgather_ragged, shard_rows

        lengths = np.array([5, 0, 9, 3, 12, 1, 7])
        d, H, dff = 16, 2, 32
        w = synth.encoder_weights(d, H, dff)
        x = synth.activations(int(lengths.sum()), d)
        plan, tok = shard_rows(list(lengths), d, dff, world)
        b0, b1 = plan[rank], plan[rank + 1]
        # each rank computes only its own sequences (the oracle stands in for the device layer here)
        y_loc = torch.from_numpy(oracle.encoder_layer(x[tok[rank]:tok[rank + 1]], lengths[b0:b1], w))
        y_full = torch.zeros(int(lengths.sum()), d, dtype=torch.float64)
        allgather_ragged(y_full, y_loc, tok, rank, world)
        ref = oracle.encoder_layer(x, lengths, w)
        q.put((rank, plan, bool(np.array_equal(y_full.numpy(), ref))))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_cpu():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plans = {tuple(pl) for _, pl, _ in res}
    assert len(plans) == 1  # every rank derives the same plan
    assert plans.pop() == tuple(oracle.shard_plan([5, 0, 9, 3, 12, 1, 7], 16, 32, 2))
    assert all(ok for _, _, ok in res)
