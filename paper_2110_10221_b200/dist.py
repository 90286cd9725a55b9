"""Sequence-sharded multi-GPU plumbing over the library's C entry points.

Sequences are independent, so each rank runs the one-GPU layers on a contiguous, window-aligned sequence
range chosen by `cora_shard_plan` (FLOP-balanced, row offsets included); the only exchange is the all-gather
of the ragged outputs, done in place as one broadcast per rank by the library's own NCCL communicator
(`cora_allgather_ragged`), or overlapped with the compute group by group inside
`cora_encoder_stack_sharded_fwd`.  torch.distributed only ships the NCCL unique id.  This module holds
argument marshalling only -- the plan, the groups and the collectives are in libcora_b200.so.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

from .api import _expect, _ptr, _stream, shard_plan


def shard_rows(lengths: Sequence[int], d_model: int, d_ff: int, world: int) -> Tuple[List[int], List[int]]:
    """(seq_begin[world+1], row_begin[world+1]) of cora_shard_plan: rank r owns sequences
    [seq_begin[r], seq_begin[r+1]) = packed rows [row_begin[r], row_begin[r+1])."""
    return shard_plan(list(lengths), d_model, d_ff, world, rows=True)


class NcclComm:
    """The library's own NCCL communicator (cora_comm_init): rank 0 draws the unique id, torch.distributed
    (already initialised: the process group is only used to ship the id) broadcasts it, every rank joins."""

    def __init__(self, rank: int, world: int, group=None):
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
        self.world, self.rank = world, rank

    def allgather_ragged(self, out, row_begin: Sequence[int], stream=None) -> None:
        """In place: rank r's rows [row_begin[r], row_begin[r+1]) broadcast from r (cora_allgather_ragged)."""
        import torch

        from . import _lib as C

        if len(row_begin) != self.world + 1 or out.dim() != 2 or int(row_begin[-1]) > out.shape[0]:
            raise ValueError("row_begin: [world + 1] row offsets within out")
        _expect(out, tuple(out.shape), out.dtype, "out")
        rb = (ctypes.c_int32 * len(row_begin))(*[int(v) for v in row_begin])
        dt = C.CORA_DT_BF16 if out.dtype == torch.bfloat16 else C.CORA_DT_F32
        C.check(C.lib().cora_allgather_ragged(self.comm, rb, _ptr(out), out.shape[1], dt, _stream(stream)),
                "cora_allgather_ragged")

    def close(self) -> None:
        from . import _lib as C

        if self.comm:
            C.lib().cora_comm_destroy(self.comm)
            self.comm = None


class ShardedStack:
    """cora_encoder_stack_sharded_fwd: this rank's sequences through every layer, one layout per group, and the
    groups' outputs gathered to every rank while the next group computes.  comm=None: one rank."""

    def __init__(self, params, max_len: int = 512, n_groups: int = 4):
        from . import _lib as C

        self.params = list(params)
        self.cps = (C.EncoderParams * len(self.params))(*[p.cstruct() for p in self.params])
        self.max_len, self.n_groups = int(max_len), int(n_groups)
        self.ws = None

    def __call__(self, lengths, lengths_host, x, comm: Optional[NcclComm] = None, out=None, stream=None):
        import torch

        from . import _lib as C

        B = int(lengths.numel())
        T = int(lengths_host.sum())
        d = self.params[0].d_model
        _expect(lengths, (B,), torch.int32, "lengths")
        _expect(lengths_host, (B,), torch.int32, "lengths_host", host=True)
        _expect(x, (T, d), torch.bfloat16, "x", lengths.device)
        _expect(out, (T, d), torch.bfloat16, "out", lengths.device)
        n = len(self.params)
        nbytes = int(C.lib().cora_encoder_stack_sharded_workspace_bytes(self.cps, n, B, T, self.max_len))
        if nbytes == 0:
            raise C.CoraError(C.CORA_ERR_INVALID, "cora_encoder_stack_sharded_workspace_bytes")
        if self.ws is None or self.ws.numel() < nbytes or self.ws.device != x.device:
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        y = torch.empty_like(x) if out is None else out
        lh = (ctypes.c_int32 * max(B, 1))(*[int(v) for v in lengths_host.tolist()])
        C.check(C.lib().cora_encoder_stack_sharded_fwd(self.cps, n, _ptr(lengths), lh, B, T, self.max_len,
                                                       comm.comm if comm is not None else None, self.n_groups,
                                                       _ptr(x), _ptr(y), _ptr(self.ws), self.ws.numel(),
                                                       _stream(stream)), "cora_encoder_stack_sharded_fwd")
        return y
