"""Multi-GPU plumbing.

Rendering shards at frame granularity with the scene replicated on every GPU
and no collective (`frame_shard`). Training is data parallel: every rank
steps on its batch shard; gradients (and, for parity with the single-process
reference, the batch-norm statistics = SyncBN) are all-reduced over NCCL on
NVLink/NVSwitch inside libdrcb (`attach_nccl`), or — without an in-library
communicator — over torch.distributed (`dp_step`'s external path).
"""

from __future__ import annotations

import ctypes as C

from . import _lib


def frame_shard(n_frames, rank, world):
    """Contiguous block of frame indices for `rank` (weak scaling: callers
    usually pass n_frames = frames_per_rank * world)."""
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def share_unique_id(provider, group=None):
    """Rank 0 creates the 128-byte NCCL unique id (provider()), every rank
    receives it through torch.distributed (works with gloo or nccl)."""
    import torch.distributed as dist

    obj = [provider() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _lib.call("drcb_nccl_unique_id", C.cast(buf, C.c_void_p))
    return bytes(buf)


class NcclComm:
    """An NCCL communicator owned by libdrcb (one per rank, device already
    selected)."""

    def __init__(self, uid, world, rank):
        h = C.c_void_p()
        idb = (C.c_uint8 * 128).from_buffer_copy(uid)
        _lib.call("drcb_nccl_comm_create", C.cast(idb, C.c_void_p), int(world), int(rank),
                  C.byref(h))
        self.handle, self.world, self.rank = h, int(world), int(rank)

    def close(self):
        if self.handle:
            _lib.call("drcb_nccl_comm_destroy", self.handle)
            self.handle = None


def attach_nccl(trainer, group=None, uid=None):
    """Create a libdrcb NCCL communicator over the torch.distributed group (or
    a single-rank one when torch.distributed is not initialised) and attach it
    to the trainer: SyncBN + gradient all-reduce inside the step."""
    try:
        import torch.distributed as dist

        initialised = dist.is_initialized()
    except Exception:  # pragma: no cover
        initialised = False
    if initialised:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = uid or share_unique_id(nccl_unique_id, group)
    else:
        world, rank = 1, 0
        uid = uid or nccl_unique_id()
    comm = NcclComm(uid, world, rank)
    _lib.call("drcb_trainer_set_comm", trainer.handle, comm.handle, world)
    trainer._comm = comm
    return comm


def dp_step(trainer, x, y, group=None):
    """One data-parallel optimisation step on this rank's shard.

    With a communicator attached (attach_nccl) the library does SyncBN and the
    gradient all-reduce itself. Otherwise the flat gradient buffer is summed
    with torch.distributed and Adam applies it scaled by 1/world (plain DDP:
    per-replica BN statistics)."""
    if getattr(trainer, "_comm", None) is not None:
        return trainer.step(x, y, apply=True)
    import torch.distributed as dist

    loss = trainer.step(x, y, apply=False)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world > 1:
        dist.all_reduce(trainer.grad_tensor(), op=dist.ReduceOp.SUM, group=group)
    trainer.apply(1.0 / world)
    return loss


# ---------------------------------------------------------------------------
# reduction hooks (drcb_trainer_set_reducer): the same SyncBN + gradient
# all-reduce points NCCL serves, through another transport

# int fn(void* user, void* buf, int64_t count, int32_t is_double, void* stream)
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)


def attach_reducer(trainer, fn, user, world):
    """Route the trainer's reductions through `fn` (a REDUCE_FN or the address
    of a C function) with context `user`."""
    _lib.call("drcb_trainer_set_reducer", trainer.handle,
              C.cast(fn, C.c_void_p) if not isinstance(fn, int) else C.c_void_p(fn),
              C.c_void_p(user) if not isinstance(user, C.c_void_p) else user, int(world))
    trainer._reducer = fn  # keep a Python callback alive


class LoopbackGroup:
    """`world` data-parallel ranks as host threads of one process (e.g. two
    half-batch trainers on one GPU): libdrcb's loopback all-reduce sums the
    ranks' buffers in rank order — SyncBN and the gradient all-reduce exactly
    where NCCL would run them."""

    def __init__(self, world):
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.drcb_loopback_create(int(world), C.byref(h)), "drcb_loopback_create")
        self.handle, self.world = h, int(world)
        self._ranks = []

    def attach(self, trainer, rank):
        lib = _lib.load()
        ctx = C.c_void_p()
        _lib.call("drcb_loopback_rank", self.handle, int(rank), C.byref(ctx))
        self._ranks.append(ctx)
        addr = C.cast(lib.drcb_loopback_reduce, C.c_void_p).value
        attach_reducer(trainer, addr, ctx, self.world)

    def close(self):
        if self.handle:
            arr = (C.c_void_p * len(self._ranks))(*[r.value for r in self._ranks])
            _lib.load().drcb_loopback_destroy(self.handle, arr, len(self._ranks))
            self.handle = None


def host_reducer(group=None, device=True):
    """A REDUCE_FN doing a host-staged torch.distributed all-reduce (sum):
    device buffer -> host -> all_reduce (gloo or any backend) -> device. With
    device=False the buffer is host memory (CPU tests call it directly)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    def reduce(user, buf, count, is_double, stream):
        try:
            dt = np.float64 if is_double else np.float32
            host = np.empty(int(count), dtype=dt)
            nbytes = host.nbytes
            if device:
                _lib.call("drcb_copy_sync", host.ctypes.data_as(C.c_void_p), C.c_void_p(buf), nbytes,
                          C.c_void_p(stream))
            else:
                C.memmove(host.ctypes.data, buf, nbytes)
            t = torch.from_numpy(host)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            if device:
                _lib.call("drcb_copy_sync", C.c_void_p(buf), host.ctypes.data_as(C.c_void_p), nbytes,
                          C.c_void_p(stream))
            else:
                C.memmove(buf, host.ctypes.data, nbytes)
            return 0
        except Exception:  # the library reports a failed hook as an error
            return 1

    return REDUCE_FN(reduce)
