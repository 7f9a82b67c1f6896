"""Host-side tensor-parallel plumbing: one process per GPU, torch.distributed for
bootstrap and timing only — every data-path collective (per-layer all-reduce of the O-proj and
down-proj partials, max-reduce of the packed argmax keys, all-gather of the head's softmax
statistics) runs inside libsirius on the NCCL communicator this module creates.

  nccl_bootstrap(lib, tp, rank)  rank 0 draws an ncclUniqueId through the library, the 128-byte id
                                 is broadcast over the default process group, every rank calls
                                 ncclCommInitRank (sirius_nccl_comm_init); returns the comm handle
  par_bootstrap(ctx)             fused peer all-reduce (SURVEY.md §8(e) phase 2): every rank exports
                                 its comm-buffer CUDA-IPC handle, the handles are all-gathered in rank
                                 order, every rank maps its peers' buffers (sirius_par_enable)
  max_over_ranks(x)              device timings are reported as the max over ranks
"""
from __future__ import annotations

import ctypes
from typing import Callable, Optional

NCCL_ID_BYTES = 128


def broadcast_id(rank: int, make_id: Callable[[], bytes]) -> bytes:
    """Rank 0's id (make_id() is called on rank 0 only) on every rank of the default group."""
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != NCCL_ID_BYTES:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def nccl_bootstrap(lib, tp: int, rank: int) -> int:
    def make_id() -> bytes:
        buf = (ctypes.c_char * NCCL_ID_BYTES)()
        if lib.sirius_nccl_unique_id(buf) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        return bytes(buf)

    uid = broadcast_id(rank, make_id)
    buf = (ctypes.c_char * NCCL_ID_BYTES)()
    ctypes.memmove(buf, uid, NCCL_ID_BYTES)
    h = ctypes.c_void_p()
    if lib.sirius_nccl_comm_init(tp, buf, rank, ctypes.byref(h)) != 0:
        raise RuntimeError("ncclCommInitRank failed")
    return h.value


def exchange_handles(handle: bytes, size: int) -> list:
    """Every rank's `size`-byte handle, in rank order, on every rank of the default group."""
    import torch.distributed as dist
    if not isinstance(handle, (bytes, bytearray)) or len(handle) != size:
        raise RuntimeError("bad handle")
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [bytes(handle)]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, bytes(handle))
    if any(not isinstance(h, bytes) or len(h) != size for h in out):
        raise RuntimeError("bad handle from a peer")
    return out


def par_bootstrap(ctx) -> None:
    """Collective: map every rank's comm buffer and switch the decode step to the fused all-reduce."""
    from . import sirius as S
    handles = exchange_handles(ctx.sirius_par_export(), S.PAR_HANDLE_BYTES)
    ctx.sirius_par_enable(handles)
    barrier()  # no rank decodes before every rank has mapped its peers


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
