"""The autoencoder's training step on the B200 — the drop-in for
drc_trainer.train's inner step (trainer/src/drc_trainer/train.py:97-103):

    optimizer.zero_grad(); loss = L1(model(x), y); loss.backward(); optimizer.step()

`DeviceTrainer` keeps fp32 master weights, gradients and Adam moments in HBM
(drcb_trainer_*); BN runs in train mode (batch statistics, momentum 0.1).
Parameters are laid out in torch's named_parameters() order of
MapAutoencoder (model.py:54-88) so gradients and updates compare 1:1.

Data parallelism: each rank steps on its shard with apply=False, the flat
gradient buffer is all-reduced (sum) over NCCL, then `apply(1/world)`.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cnn import architecture, load_weights, save_weights

_LAYERS = ["enc1.conv1", "enc1.conv2", "enc2.conv1", "enc2.conv2", "enc3.conv1", "enc3.conv2",
           "bott.conv1", "bott.conv2", "dec3.deconv1", "dec3.deconv2", "dec2.deconv1",
           "dec2.deconv2", "dec1.deconv1", "dec1.deconv2", "head.deconv1", "head.deconv2",
           "head.conv_out"]


def _bn_of(layer):
    if layer == "head.conv_out":
        return None
    mod, conv = layer.split(".")
    return f"{mod}.bn{conv[-1]}"


def param_layout(k):
    """[(torch name, drcw name, shape, offset)] in named_parameters() order."""
    arch = architecture(k)
    out, off = [], 0
    for layer in _LAYERS:
        for suffix in ("weight", "bias"):
            shape = arch[f"{layer}.{suffix}"]
            out.append((f"{layer}.{suffix}", f"{layer}.{suffix}", shape, off))
            off += int(np.prod(shape))
        bn = _bn_of(layer)
        if bn:
            for tsuf, dsuf in (("weight", "gamma"), ("bias", "beta")):
                shape = arch[f"{bn}.{dsuf}"]
                out.append((f"{bn}.{tsuf}", f"{bn}.{dsuf}", shape, off))
                off += int(np.prod(shape))
    return out


class DeviceTrainer:
    """mode "fp32": CUDA-core engine (the parity engine); "bf16": the NHWC
    tensor-core engine (drcb_train_tc.cu: forward, dgrad and wgrad of every
    3x3 layer on tcgen05, activations and gradients NHWC bf16, batch
    statistics / Adam / master weights fp32; BASELINE config 5: bf16 compute,
    fp32 master weights; k = 64)."""

    def __init__(self, net_or_drcw, lr=6e-5, betas=(0.9, 0.999), eps=1e-8, mode="fp32"):
        lib = _lib.load()
        raw = net_or_drcw if isinstance(net_or_drcw, (bytes, bytearray)) else save_weights(net_or_drcw)
        h = C.c_void_p()
        _lib.check(lib.drcb_trainer_create(bytes(raw), len(raw), float(lr), float(betas[0]),
                                           float(betas[1]), float(eps), C.byref(h)),
                   "drcb_trainer_create")
        self.handle = h
        info = (C.c_int64 * 4)()
        _lib.call("drcb_trainer_info", h, info)
        self.k, self.n_params, self.n_running = int(info[0]), int(info[1]), int(info[2])
        self.layout = param_layout(self.k)
        if mode not in ("fp32", "bf16"):
            raise ValueError("trainer mode must be 'fp32' or 'bf16'")
        self.mode = mode
        _lib.call("drcb_trainer_set_mode", h, 0 if mode == "fp32" else 2)

    # -- steps ---------------------------------------------------------------
    def step(self, x, y, apply=True, want_loss=True):
        """One step on x (n,7,32,32), y (n,3,32,32) (CUDA tensors or numpy).
        Returns the batch L1 loss (float) or None."""
        import torch

        xd = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, np.float32))
        yd = y if isinstance(y, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(y, np.float32))
        xd = xd.to(device="cuda", dtype=torch.float32).contiguous()
        yd = yd.to(device="cuda", dtype=torch.float32).contiguous()
        loss = C.c_double(0.0)
        key = getattr(self, "_graph_key", None)
        if key is not None and int(xd.shape[0]) > key[2]:
            # a larger batch can regrow the engine's buffers under the graph
            self._graph = self._graph_key = None
        self._last_n_pad = (int(xd.shape[0]) + 7) // 8 * 8
        _lib.call("drcb_trainer_step", self.handle, _lib.ptr(xd), _lib.ptr(yd), int(xd.shape[0]),
                  C.byref(loss) if want_loss else None, int(bool(apply)), _lib.stream_ptr())
        return float(loss.value) if want_loss else None

    def step_graph(self, x, y, want_loss=False):
        """One full step (apply=True) replayed from a captured CUDA graph —
        the bf16 engine's ~350 launches per step cost one graph launch, which
        is what small batches (BASELINE config 5's 64) are bound by. x, y are
        device fp32 contiguous tensors the caller refills in place; the first
        call with a new (x, y, n) runs the step eagerly (engine setup) and
        captures the next one. Bit-identical to step(x, y): same kernels, same
        order; the Adam step counter is on the device."""
        import torch

        if self.mode != "bf16":
            raise ValueError("step_graph needs the bf16 tensor-core engine")
        if not (x.is_cuda and y.is_cuda and x.dtype == torch.float32 and y.dtype == torch.float32
                and x.is_contiguous() and y.is_contiguous()):
            raise ValueError("step_graph takes contiguous float32 CUDA tensors")
        key = (x.data_ptr(), y.data_ptr(), int(x.shape[0]))
        if getattr(self, "_graph_key", None) != key:
            loss = self.step(x, y, apply=True, want_loss=want_loss)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                _lib.call("drcb_trainer_step", self.handle, _lib.ptr(x), _lib.ptr(y),
                          int(x.shape[0]), None, 1, _lib.stream_ptr())
            self._graph, self._graph_key = g, key
            return loss
        self._graph.replay()
        return self.last_loss() if want_loss else None

    def steps_taken(self):
        """Adam steps applied so far (the device counter; synchronises)."""
        info = (C.c_int64 * 4)()
        _lib.call("drcb_trainer_info", self.handle, info)
        return int(info[3])

    def last_loss(self):
        """The batch L1 loss of the last bf16 step (synchronises)."""
        loss = C.c_double(0.0)
        _lib.call("drcb_trainer_last_loss", self.handle, C.byref(loss), _lib.stream_ptr())
        return float(loss.value)

    def debug_z(self, layer):
        """(test hook, bf16 engine) the pre-BN conv output of 3x3 layer
        `layer` (0..15) from the last step, or (16) the head's input
        activation: float32 CUDA tensor (n_pad, hw, hw, c_pad)."""
        import torch

        cout = [self.k, self.k, 2 * self.k, 2 * self.k, 4 * self.k, 4 * self.k, 8 * self.k,
                8 * self.k, 4 * self.k, 4 * self.k, 2 * self.k, 2 * self.k, self.k, self.k,
                self.k // 2, self.k // 4, self.k // 4][layer]
        hw = [32, 32, 16, 16, 8, 8, 4, 4, 8, 8, 16, 16, 32, 32, 32, 32, 32][layer]
        cpad = (cout + 63) // 64 * 64
        n = self._last_n_pad
        out = torch.empty((n, hw, hw, cpad), dtype=torch.bfloat16, device="cuda")
        _lib.call("drcb_trainer_debug_z", self.handle, int(layer), _lib.ptr(out), _lib.stream_ptr())
        return out.float()

    def apply(self, grad_scale=1.0):
        _lib.call("drcb_trainer_apply", self.handle, float(grad_scale), _lib.stream_ptr())

    # -- buffers -------------------------------------------------------------
    def _buffers(self):
        p, g, r = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _lib.call("drcb_trainer_buffers", self.handle, C.byref(p), C.byref(g), C.byref(r))
        return p.value, g.value, r.value

    def grad_tensor(self):
        """The flat fp32 gradient buffer as a CUDA tensor view (for NCCL)."""
        return _device_view(self._buffers()[1], self.n_params)

    def _host(self, which):
        import torch

        ptr = self._buffers()[which]
        torch.cuda.current_stream().synchronize()
        return _device_view(ptr, self.n_params).cpu().numpy()

    def params(self):
        flat = self._host(0)
        return {n: flat[o:o + int(np.prod(s))].reshape(s).copy() for n, _, s, o in self.layout}

    def running(self):
        """Batch-norm running statistics, flat fp32 (DRCW order of the layers)."""
        import torch

        ptr = self._buffers()[2]
        torch.cuda.current_stream().synchronize()
        return _device_view(ptr, self.n_running).cpu().numpy()

    def grads(self):
        flat = self._host(1)
        return {n: flat[o:o + int(np.prod(s))].reshape(s).copy() for n, _, s, o in self.layout}

    def export(self):
        size = _lib.load().drcb_trainer_export(self.handle, None, 0)
        buf = (C.c_uint8 * size)()
        _lib.load().drcb_trainer_export(self.handle, buf, size)
        return bytes(buf)

    def network(self):
        return load_weights(self.export())

    def close(self):
        self._graph = self._graph_key = None
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.drcb_trainer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_view(ptr, n):
    """Zero-copy torch view of library-owned device memory."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_CAI(), device="cuda")


@dataclass
class TrainConfig:
    """TrainConfig (train.py:19-36)."""

    learning_rate: float = 6e-5
    batch_size: int = 32
    epochs: int = 3
    ablation: tuple = ()
    seed: int = 0
    val_fraction: float = 0.1
    k: int = 64
    slope: float = 0.01


def train_step(trainer, x, y):
    """train.py:97-103 on the device; returns the loss."""
    return trainer.step(x, y, apply=True)


def torch_default_network(k=64, slope=0.01):
    """The initial weights of a freshly constructed MapAutoencoder
    (model.py:20-88) under the current torch RNG state: the same torch modules
    (default Kaiming-uniform conv init, unit/zero batch norm) built in the same
    order, exported to a DRCW Network. Weight initialisation only; nothing here
    runs on the training path."""
    import torch
    from torch import nn

    from .cnn import Network

    tensors = {}

    def conv(name, cin, cout, transposed, ks=3):
        if transposed:
            m = nn.ConvTranspose2d(cin, cout, ks, stride=1, padding=1)
        else:
            m = nn.Conv2d(cin, cout, ks, padding=1 if ks == 3 else 0)
        tensors[f"{name}.weight"] = m.weight.detach().numpy().astype(np.float32)
        tensors[f"{name}.bias"] = m.bias.detach().numpy().astype(np.float32)

    def bn(name, c):
        m = nn.BatchNorm2d(c, eps=1e-5)
        tensors[f"{name}.gamma"] = m.weight.detach().numpy().astype(np.float32)
        tensors[f"{name}.beta"] = m.bias.detach().numpy().astype(np.float32)
        tensors[f"{name}.running_mean"] = m.running_mean.numpy().astype(np.float32)
        tensors[f"{name}.running_var"] = m.running_var.numpy().astype(np.float32)

    with torch.no_grad():
        for name, cin, cout, tr in (("enc1", 7, k, False), ("enc2", k, 2 * k, False),
                                    ("enc3", 2 * k, 4 * k, False), ("bott", 4 * k, 8 * k, False),
                                    ("dec3", 12 * k, 4 * k, True), ("dec2", 6 * k, 2 * k, True),
                                    ("dec1", 3 * k, k, True)):
            kind = "deconv" if tr else "conv"
            conv(f"{name}.{kind}1", cin, cout, tr)
            bn(f"{name}.bn1", cout)
            conv(f"{name}.{kind}2", cout, cout, tr)
            bn(f"{name}.bn2", cout)
        conv("head.deconv1", k, k // 2, True)
        bn("head.bn1", k // 2)
        conv("head.deconv2", k // 2, k // 4, True)
        bn("head.bn2", k // 4)
        conv("head.conv_out", k // 4, 3, False, ks=1)
    return Network(tensors=tensors, k=k, slope=float(np.float32(slope)))


def evaluate(trainer, dev_examples, batch_size, ablation=()):
    """_evaluate (train.py:56-64): eval-mode (running statistics) L1 over
    batches, weighted by batch length."""
    import torch

    from .cnn import DeviceNet

    net = DeviceNet(trainer.export())
    total, count = 0.0, 0
    for b0 in range(0, dev_examples.n, batch_size):
        idx = list(range(b0, min(b0 + batch_size, dev_examples.n)))
        x, y = dev_examples.gather(idx, None, ablation)
        pred = net.forward_device(x, mode="fp32")
        total += float(torch.nn.functional.l1_loss(pred, y)) * len(idx)
        count += len(idx)
    net.close()
    return total / max(count, 1)


def train(examples, config, weights_out=None, curves_out=None, log=print):
    """drc_trainer.train.train (train.py:65-116) on the device: by-scene
    split, 8 augmentation variants per training example gathered and
    transformed per batch by the device pipeline (data.DeviceExamples), the
    reference's shuffling (torch.randperm with the seeded loader generator),
    one DeviceTrainer step per batch, validation once per epoch. Returns
    (trainer, history) with history rows (step, split, loss)."""
    import csv
    import os

    import torch

    from . import data

    if config.learning_rate <= 0:
        raise ValueError("learning rate must be > 0")
    if config.batch_size < 1 or config.epochs < 1:
        raise ValueError("batch size and epochs must be >= 1")
    if set(config.ablation) - {"normals", "distance"}:
        raise ValueError("ablation mask must be within {normals, distance}")
    torch.manual_seed(config.seed)
    np.random.seed(config.seed)
    train_ex, val_ex = data.split_by_scene(examples, config.val_fraction, config.seed)
    if not val_ex:  # single-scene corpus: fall back to an example split
        cut = max(1, len(examples) // 10)
        train_ex, val_ex = examples[cut:], examples[:cut]
    trainer = DeviceTrainer(torch_default_network(config.k, config.slope), lr=config.learning_rate)
    dtrain, dval = data.DeviceExamples(train_ex), data.DeviceExamples(val_ex)
    n_items = 8 * len(train_ex)
    gen = torch.Generator().manual_seed(config.seed)
    history = []
    step = 0
    val0 = evaluate(trainer, dval, config.batch_size, config.ablation)
    history.append((step, "val", val0))
    log(f"initial val L1 {val0:.5f} ({n_items} augmented train, {len(val_ex)} val examples)")
    for epoch in range(config.epochs):
        # the DataLoader's draws per epoch: the iterator's base seed, the
        # RandomSampler permutation, and the sampler's trailing (empty-slice)
        # randperm when it is exhausted (torch/utils/data/sampler.py)
        torch.empty((), dtype=torch.int64).random_(generator=gen)
        perm = torch.randperm(n_items, generator=gen).tolist()
        torch.randperm(n_items, generator=gen)
        for b0 in range(0, n_items, config.batch_size):
            items = perm[b0:b0 + config.batch_size]
            x, y = dtrain.gather([i // 8 for i in items], [i % 8 for i in items], config.ablation)
            loss = trainer.step(x, y, apply=True)
            step += 1
            history.append((step, "train", loss))
        val = evaluate(trainer, dval, config.batch_size, config.ablation)
        history.append((step, "val", val))
        log(f"epoch {epoch + 1}/{config.epochs}: val L1 {val:.5f}")
    if curves_out:
        with open(curves_out, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["step", "split", "loss"])
            w.writerows(history)
    if weights_out:
        tmp = f"{weights_out}.tmp"
        with open(tmp, "wb") as f:
            f.write(trainer.export())
        os.replace(tmp, weights_out)
    return trainer, history
