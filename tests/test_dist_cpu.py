"""Multi-process host logic of the multi-GPU paths on CPU (gloo, world 2):
frame sharding, NCCL unique-id distribution, and the data-parallel step's
gradient all-reduce + 1/world scaling (checked against a full-batch step)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_02480_b200.dist import dp_step, frame_shard, share_unique_id


def test_frame_shards_partition():
    for n in (1, 7, 8, 32, 64):
        for world in (1, 2, 4, 8):
            shards = [frame_shard(n, r, world) for r in range(world)]
            flat = [f for s in shards for f in s]
            assert flat == list(range(n))
            assert max(map(len, shards)) - min(map(len, shards)) <= 1


class _CpuTrainer:
    """Stand-in exposing DeviceTrainer's step/grad_tensor/apply interface on a
    tiny CPU model (plain SGD so the update is linear in the gradient)."""

    def __init__(self, seed=0):
        g = torch.Generator().manual_seed(seed)
        self.w = torch.randn(5, 3, generator=g)
        self.g = torch.zeros(15)

    def step(self, x, y, apply=True):
        w = self.w.clone().requires_grad_(True)
        loss = torch.nn.functional.l1_loss(torch.as_tensor(x) @ w, torch.as_tensor(y))
        loss.backward()
        self.g.copy_(w.grad.reshape(-1))
        if apply:
            self.apply(1.0)
        return float(loss)

    def grad_tensor(self):
        return self.g

    def apply(self, scale):
        self.w -= 0.1 * scale * self.g.reshape(self.w.shape)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(0)
    return (rng.normal(size=(8, 5)).astype(np.float32), rng.normal(size=(8, 3)).astype(np.float32))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = share_unique_id(
            lambda: bytes(np.random.default_rng(1).integers(0, 256, 128, dtype=np.uint8)))
        x, y = _data()
        tr = _CpuTrainer()
        shard = frame_shard(8, rank, world)
        dp_step(tr, x[shard], y[shard])
        out[rank] = (uid, tr.w.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_dp_step_matches_full_batch_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] and len(res[0][0]) == 128
    x, y = _data()
    ref = _CpuTrainer()
    ref.step(x, y, apply=True)
    # equal shards of an L1 mean: full-batch gradient == mean of shard grads
    assert np.allclose(res[0][1], ref.w.numpy(), atol=1e-6)
    assert np.array_equal(res[0][1], res[1][1])


def _host_reducer_worker(rank, world, port, out):
    import ctypes as C

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1910_02480_b200.dist import host_reducer

        fn = host_reducer(device=False)  # the REDUCE_FN libdrcb calls (host buffers here)
        for dt, is_double in ((np.float32, 0), (np.float64, 1)):
            buf = (np.arange(10, dtype=dt) + 100 * rank).copy()
            rc = fn(None, buf.ctypes.data_as(C.c_void_p).value, len(buf), is_double, None)
            out.put((rank, str(dt), rc, buf.tolist()))
    finally:
        dist.destroy_process_group()


def test_host_staged_reduction_hook_world2_gloo():
    """The reduction hook the trainer calls at every SyncBN / gradient
    reduction point (drcb_trainer_set_reducer), backed by a gloo all-reduce:
    both ranks receive the sum, in both precisions."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_host_reducer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(4)]
    for p in ps:
        p.join(timeout=60)
    want = (2 * np.arange(10) + 100).tolist()
    for rank, dt, rc, buf in res:
        assert rc == 0 and buf == want, (rank, dt, rc, buf)
