"""Host-side collectives for rpc_create_hostcoll (include/rpchol_gpu.h) over
torch.distributed (any CPU backend, e.g. gloo).

The library's per-round exchange is two collectives: an allgather of
per-shard slots and an "owner" reduce in which at most one rank holds a non-zero
64-bit word per position.  The owner reduce is a bitwise OR here (exact for that
pattern: the owner's bit pattern comes back unchanged).  With the NCCL context the
same two steps run on the device; this adapter exists for CPU transports and for
running several ranks on one GPU in tests.
"""
from __future__ import annotations

import numpy as np


class TorchHostCollectives:
    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist = dist
        self._group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)

    def allgather(self, send: np.ndarray) -> np.ndarray:
        import torch
        t = torch.from_numpy(np.ascontiguousarray(send, dtype=np.uint8))
        out = torch.empty(t.numel() * self.nranks, dtype=torch.uint8)
        self._dist.all_gather_into_tensor(out, t, group=self._group)
        return out.numpy()

    def allreduce_or(self, buf: np.ndarray) -> None:
        import torch
        t = torch.from_numpy(buf.view(np.int64).copy())
        self._dist.all_reduce(t, op=self._dist.ReduceOp.BOR, group=self._group)
        buf[:] = t.numpy().view(np.uint64)
