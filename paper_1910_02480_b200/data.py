"""The trainer's input pipeline: the drop-in for
drc_trainer.data (trainer/src/drc_trainer/data.py).

DRCD containers are parsed on the host (the same byte format and error
messages as read_drcd, data.py:42-74); the examples are uploaded once as a
resident base set and every training batch is gathered, augmented (azimuthal
column shift by {0, 8, 16, 24} + optional flip with the frame-local normals
re-expressed, data.py:77-104) and ablated (data.py:106-117) on the device by
one libdrcb kernel (drcb_augment_gather), straight into the step's input
buffers.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import io
import struct
from dataclasses import replace

import numpy as np

from . import _lib
from .dataset import TrainingExample as Example
from .errors import DrcError

DRCD_MAGIC = b"DRCD"
DRCD_VERSION = 1
SHIFTS = (0, 8, 16, 24)
ABLATABLE = {"normals": slice(3, 6), "distance": slice(6, 7)}
_ABLATE_BITS = {"normals": 1, "distance": 2}


class DatasetError(DrcError):
    """data.py DatasetError: malformed DRCD or unknown ablation channel."""


def read_drcd(src):
    """Parse a DRCD file (path or bytes) into Examples (data.py:42-74)."""
    if isinstance(src, str):
        with open(src, "rb") as f:
            raw = f.read()
    else:
        raw = src
    buf = io.BytesIO(raw)

    def take(n, what):
        b = buf.read(n)
        if len(b) != n:
            raise DatasetError(f"truncated while reading {what} at byte {buf.tell()}")
        return b

    if take(4, "magic") != DRCD_MAGIC:
        raise DatasetError("bad magic, not a DRCD file")
    version, count, res = struct.unpack("<IIH", take(10, "header"))
    if version != DRCD_VERSION:
        raise DatasetError(f"unsupported DRCD version {version}")
    out = []
    for _ in range(count):
        (slen,) = struct.unpack("<I", take(4, "scene-id length"))
        sid = take(slen, "scene id").decode("utf-8")
        px, py = struct.unpack("<II", take(8, "pixel"))
        s_r, s_d = struct.unpack("<ff", take(8, "scales"))
        inp = np.frombuffer(take(7 * res * res * 4, "input"), dtype="<f4")
        tgt = np.frombuffer(take(3 * res * res * 4, "target"), dtype="<f4")
        out.append(Example(input=inp.reshape(7, res, res).copy(),
                           target=tgt.reshape(3, res, res).copy(),
                           s_r=s_r, s_d=s_d, scene_id=sid, pixel=(px, py)))
    if buf.read(1):
        raise DatasetError("trailing bytes after last example")
    return out


def write_drcd(examples, path=None):
    """DRCD writer (the renderer side's write_dataset, dataset.py:133-154)."""
    if not examples:
        raise DatasetError("refusing to write an empty dataset")
    res = examples[0].input.shape[1]
    buf = io.BytesIO()
    buf.write(DRCD_MAGIC)
    buf.write(struct.pack("<IIH", DRCD_VERSION, len(examples), res))
    for e in examples:
        sid = e.scene_id.encode("utf-8")
        buf.write(struct.pack("<I", len(sid)))
        buf.write(sid)
        buf.write(struct.pack("<II", int(e.pixel[0]), int(e.pixel[1])))
        buf.write(struct.pack("<ff", e.s_r, e.s_d))
        buf.write(np.ascontiguousarray(e.input, dtype="<f4").tobytes())
        buf.write(np.ascontiguousarray(e.target, dtype="<f4").tobytes())
    raw = buf.getvalue()
    if path is None:
        return raw
    with open(path, "wb") as f:
        f.write(raw)
    return None


def ablation_bits(mask):
    unknown = set(mask) - set(ABLATABLE)
    if unknown:
        raise DatasetError(f"unknown ablation channels {sorted(unknown)}")
    return sum(_ABLATE_BITS[m] for m in set(mask))


def split_by_scene(examples, val_fraction=0.1, seed=0):
    """Deterministic train/validation split on whole scenes (data.py:124-140)."""
    scenes = sorted({e.scene_id for e in examples})
    if len(scenes) < 2:
        return examples, []
    n_val = max(1, int(round(val_fraction * len(scenes))))
    ranked = sorted(scenes, key=lambda s: hashlib.sha256(f"{seed}:{s}".encode()).hexdigest())
    val_scenes = set(ranked[:n_val])
    train = [e for e in examples if e.scene_id not in val_scenes]
    val = [e for e in examples if e.scene_id in val_scenes]
    return train, val


def _trig():
    t = _lib.AugmentTrig()
    for i, s in enumerate(SHIFTS):
        alpha = 2.0 * np.pi * s / 32
        t.cos_a[i] = float(np.cos(alpha))
        t.sin_a[i] = float(np.sin(alpha))
    return t


class DeviceExamples:
    """Examples resident in HBM as x (N,7,32,32) and y (N,3,32,32) fp32."""

    def __init__(self, examples):
        import torch

        if not examples:
            raise DatasetError("no examples")
        res = examples[0].input.shape[-1]
        if res != 32:
            raise DatasetError(f"the device pipeline needs 32x32 maps, got {res}")
        self.n = len(examples)
        self.x = torch.from_numpy(np.stack([e.input for e in examples]).astype(np.float32)).cuda()
        self.y = torch.from_numpy(np.stack([e.target for e in examples]).astype(np.float32)).cuda()
        self._trig = _trig()

    def gather(self, base, variant=None, ablate=(), out=None):
        """Batch of base[i] under augmentation variant[i] (v = 2 * shift index
        + flip, augment()'s order) with the ablation mask -> (x, y) CUDA."""
        import torch

        base_t = torch.as_tensor(np.asarray(base, dtype=np.int64)).cuda()
        n = int(base_t.numel())
        var_t = None
        if variant is not None:
            var_t = torch.as_tensor(np.asarray(variant, dtype=np.int32)).cuda()
            if var_t.numel() != n:
                raise DatasetError("variant and base lengths differ")
        if out is None:
            out = (torch.empty((n, 7, 32, 32), dtype=torch.float32, device="cuda"),
                   torch.empty((n, 3, 32, 32), dtype=torch.float32, device="cuda"))
        _lib.call("drcb_augment_gather", _lib.ptr(self.x), _lib.ptr(self.y), _lib.ptr(base_t),
                  _lib.ptr(var_t) if var_t is not None else None, n, C.byref(self._trig),
                  ablation_bits(ablate), _lib.ptr(out[0]), _lib.ptr(out[1]), _lib.stream_ptr())
        return out


def transform_example(example, shift=0, flip=False):
    """One augmentation variant of one example (data.py:86-100), on the device."""
    if shift not in SHIFTS:
        raise DatasetError(f"shift must be one of {SHIFTS}")
    x, y = DeviceExamples([example]).gather([0], [2 * SHIFTS.index(shift) + int(bool(flip))])
    return replace(example, input=x[0].cpu().numpy(), target=y[0].cpu().numpy())


def augment(example):
    """All rotation/flip variants of one example, identity first (data.py:103-104)."""
    x, y = DeviceExamples([example]).gather([0] * 8, list(range(8)))
    xs, ys = x.cpu().numpy(), y.cpu().numpy()
    return [replace(example, input=xs[v], target=ys[v]) for v in range(8)]


def ablate(example, mask):
    """Zero the masked auxiliary input channels (data.py:106-117)."""
    bits = ablation_bits(mask)
    if not bits:
        return example
    inp = example.input.copy()
    for name in mask:
        inp[ABLATABLE[name]] = 0.0
    return replace(example, input=inp)
