"""Multi-GPU partitioned Newton steps: one process per GPU.

The scene's per-pair work (primitive pairs, pair blocks, CCD, contact and
friction energies) is split across ranks by overlap body pair
(`abd_scene_set_comm_*`, csrc/comm.cu); the assembled system, the energies and
the CCD bound are all-reduced, and the factorisation and the Newton update run
replicated, so every rank holds the same state after each step.

    import torch.distributed as dist
    dist.init_process_group("nccl")            # bootstrap only
    attach_nccl(model)                         # NCCL from the library itself
    state, stats = advance_step(model, state, params)

`attach_torch` routes the reductions through a torch.distributed group instead
(host round trip per reduction; used by the gloo tests with ranks sharing one GPU).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native

__all__ = ["attach_nccl", "attach_torch", "detach"]

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int)
_keep = {}  # scene ptr -> callback object (must outlive the scene's use of it)


class _DevArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    _types = {0: "<f8", 1: "<i4", 2: "<i8"}

    def __init__(self, ptr, count, dtype):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": self._types[dtype],
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def attach_nccl(model, group=None):
    """Partition `model`'s scene over the ranks of the default (or given) process group."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    sc = model.gpu_scene()
    L = _native.lib()
    uid = C.create_string_buffer(128)
    if rank == 0:
        _native.check(L.abd_nccl_unique_id(uid))
    obj = [bytes(uid.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    _native.check(L.abd_scene_set_comm_nccl(sc.ptr, obj[0], rank, world))
    return rank, world


def attach_torch(model, group=None):
    """Partition with reductions through torch.distributed (e.g. gloo, CPU staging)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    sc = model.gpu_scene()
    ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MIN, 2: dist.ReduceOp.MAX}

    def cb(user, ptr, count, dtype, op):
        try:
            dev = torch.as_tensor(_DevArray(ptr, count, dtype), device="cuda")
            host = dev.cpu()
            dist.all_reduce(host, op=ops[op], group=group)
            dev.copy_(host)
            torch.cuda.synchronize()
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed collective
            return 1

    fn = ALLREDUCE_FN(cb)
    _keep[sc.ptr] = fn
    _native.check(_native.lib().abd_scene_set_comm_callback(sc.ptr, rank, world, C.cast(fn, C.c_void_p), None))
    return rank, world


def detach(model):
    """Back to a single-rank scene."""
    sc = model.gpu_scene()
    _native.check(_native.lib().abd_scene_set_comm_callback(sc.ptr, 0, 1, None, None))
    _keep.pop(sc.ptr, None)


def owned_bodies(n_bodies, rank, world):
    """Bodies whose body terms a rank would own under body partitioning (reporting helper)."""
    return np.arange(rank, n_bodies, world)
