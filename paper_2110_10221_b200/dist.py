"""Sequence-sharded multi-GPU plumbing.

Sequences are independent, so each rank runs the one-GPU layer on a contiguous sequence range
chosen by `cora_shard_plan` (FLOP-balanced); the only exchange is the final all-gather of the
ragged outputs, done in place as one broadcast per rank (NCCL over NVLink on GPUs; gloo in the CPU
tests).  This module holds host bookkeeping and the collective call only -- no layer arithmetic.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from .api import shard_plan


def shard_rows(lengths: Sequence[int], d_model: int, d_ff: int, world: int) -> Tuple[List[int], List[int]]:
    """(seq_begin[world+1], tok_begin[world+1]): rank r owns sequences [seq_begin[r], seq_begin[r+1])
    = packed rows [tok_begin[r], tok_begin[r+1])."""
    plan = shard_plan(list(lengths), d_model, d_ff, world)
    ro = [0]
    for L in lengths:
        ro.append(ro[-1] + int(L))
    return plan, [ro[b] for b in plan]


def allgather_ragged(y_full, y_local, tok_begin: Sequence[int], rank: int, world: int, group=None) -> None:
    """Gather every rank's packed rows into y_full[T, d] in original order (in place)."""
    import torch.distributed as dist

    if tok_begin[rank + 1] > tok_begin[rank]:
        y_full[tok_begin[rank]:tok_begin[rank + 1]].copy_(y_local)
    for r in range(world):
        if tok_begin[r + 1] > tok_begin[r]:
            dist.broadcast(y_full[tok_begin[r]:tok_begin[r + 1]], src=r, group=group)


class NcclComm:
    """The library's own NCCL communicator (cora_comm_init): rank 0 draws the unique id, torch.distributed
    (already initialised: the process group is only used to ship the id) broadcasts it, every rank joins."""

    def __init__(self, rank: int, world: int, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib as C

        n = C.lib().cora_comm_unique_id_bytes()
        buf = (ctypes.c_uint8 * n)()
        if rank == 0:
            C.check(C.lib().cora_comm_get_unique_id(buf), "cora_comm_get_unique_id")
        if world > 1:
            t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            buf = (ctypes.c_uint8 * n)(*t.cpu().tolist())
        self.comm = ctypes.c_void_p()
        C.check(C.lib().cora_comm_init(ctypes.byref(self.comm), buf, world, rank), "cora_comm_init")
        self.world = world

    def allgather_ragged(self, out, row_off: Sequence[int], seq_begin: Sequence[int], stream=None) -> None:
        """In place: rows of rank r's sequences broadcast from r (cora_allgather_ragged)."""
        import ctypes

        import torch

        from . import _lib as C

        ro = (ctypes.c_int32 * len(row_off))(*[int(v) for v in row_off])
        sb = (ctypes.c_int32 * len(seq_begin))(*[int(v) for v in seq_begin])
        dt = C.CORA_DT_BF16 if out.dtype == torch.bfloat16 else C.CORA_DT_F32
        s = torch.cuda.current_stream() if stream is None else stream
        C.check(C.lib().cora_allgather_ragged(self.comm, ro, sb, ctypes.c_void_p(out.data_ptr()), out.shape[1], dt,
                                              ctypes.c_void_p(s.cuda_stream)), "cora_allgather_ragged")

    def close(self) -> None:
        from . import _lib as C

        if self.comm:
            C.lib().cora_comm_destroy(self.comm)
            self.comm = None
