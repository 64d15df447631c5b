"""Multi-GPU bootstrap: one process per GPU (torchrun), torch.distributed for
the control plane (rendezvous, NCCL unique-id broadcast, barriers, max-over-ranks
timing); the iteration's data exchange itself is NCCL inside the C++ solver
graph (csrc/comm.cpp)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _lib as L


@dataclass
class DistContext:
    rank: int
    world: int
    local_rank: int
    nccl_id: Optional[bytes]
    dist: object  # torch.distributed module or None


def env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str = "gloo", need_nccl_id: bool = True) -> DistContext:
    rank, world, local = env()
    if world <= 1:
        return DistContext(0, 1, local, None, None)
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if not dist.is_initialized():
        dist.init_process_group(backend)
    ctx = DistContext(rank, world, local, None, dist)
    if need_nccl_id:
        ctx.nccl_id = new_nccl_id(ctx)
    return ctx


def new_nccl_id(ctx: DistContext) -> Optional[bytes]:
    """A fresh NCCL unique id, drawn on rank 0 and broadcast (collective over
    the process group).  An id bootstraps ONE communicator: every solver after
    the first needs a new one (reusing an id leaves ncclCommInitRank waiting
    for a bootstrap root that has already exited)."""
    if ctx.world <= 1:
        return None
    buf = C.create_string_buffer(128)
    if ctx.rank == 0:
        L.check(L.lib().pdd_nccl_unique_id(buf))
    lst = [bytes(buf.raw) if ctx.rank == 0 else None]
    ctx.dist.broadcast_object_list(lst, src=0)
    return lst[0]


@dataclass
class RankLayout:
    local_subs: List[int]
    local_pairs: List[int]
    exchange: List[tuple]  # (local pair index, peer rank, my side)


def rank_layout(plan, rank: int, world: int) -> RankLayout:
    """The C++ layout layer's ownership and exchange schedule (host only)."""
    D, P = plan.D, len(plan.overlaps)
    ns, npairs, nex = C.c_int32(), C.c_int32(), C.c_int32()
    subs = np.zeros(max(D, 1), np.int32)
    pairs = np.zeros(max(P, 1), np.int32)
    ex = np.zeros((max(P, 1), 3), np.int32)
    L.check(L.lib().pdd_rank_layout(plan.handle, C.c_int32(rank), C.c_int32(world), C.byref(ns), L.ptr(subs),
                                    C.byref(npairs), L.ptr(pairs), C.byref(nex), L.ptr(ex)))
    return RankLayout([int(x) for x in subs[: ns.value]], [int(x) for x in pairs[: npairs.value]],
                      [tuple(int(v) for v in r) for r in ex[: nex.value]])
