"""Reference-mode training examples on the B200:
the drop-in for drc.dataset.generate_examples (dataset.py:53-104).

For every grid pixel whose camera chain finds a non-specular surface: the
1-spp 7-channel input stack and a ref_spp ground-truth radiance map in the
same hemisphere frame (_reference_map, dataset.py:107-127), both path traced
by libdrcb; the target is normalised by the input's s_r.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib, render
from .errors import ConfigError, FormatError
from .scene import device_scene

DATASET_KEY_BASE = 1 << 42
SAMPLER_KINDS = ("independent", "stratified")


@dataclass(frozen=True)
class TrainingExample:
    input: np.ndarray   # (7, res, res) float32
    target: np.ndarray  # (3, res, res) float32, normalised by s_r
    s_r: float
    s_d: float
    scene_id: str
    pixel: tuple

    def __post_init__(self):
        if self.input.ndim != 3 or self.input.shape[0] != 7:
            raise FormatError("input stack must be (7,res,res)")
        if self.target.shape != (3,) + self.input.shape[1:]:
            raise FormatError("target must be (3,res,res) matching the input")
        object.__setattr__(self, "s_r", float(np.float32(self.s_r)))
        object.__setattr__(self, "s_d", float(np.float32(self.s_d)))


def generate_examples(scene, grid, ref_spp, sampler_variants=None, seed=0, config=None,
                      progress=None, precision=64):
    cfg = config or render.RenderConfig()
    nx, ny = grid
    if nx < 1 or ny < 1:
        raise ConfigError("grid must be at least 1x1")
    if ref_spp < 256:
        raise ConfigError("ref_spp must be >= 256")
    kinds = list(sampler_variants or SAMPLER_KINDS)
    w, h = scene.camera.resolution
    xs = ((np.arange(nx) + 0.5) * w / nx).astype(np.int64)
    ys = ((np.arange(ny) + 0.5) * h / ny).astype(np.int64)
    gx, gy = np.meshgrid(xs, ys)
    gx, gy = gx.ravel(), gy.ravel()
    import math

    f, r, u = scene.camera.basis()
    th = math.tan(math.radians(scene.camera.fov) * 0.5)
    ndc_x = ((gx + 0.5) / w * 2.0 - 1.0) * th * (w / h)
    ndc_y = (1.0 - (gy + 0.5) / h * 2.0) * th
    d = f + ndc_x[:, None] * r + ndc_y[:, None] * u
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    geo = render.primary_chain_batch(scene, np.broadcast_to(scene.camera.position, d.shape), d,
                                     precision=precision)
    import torch

    ds = device_scene(scene)
    rd = torch.float64 if precision == 64 else torch.float32
    found = [i for i in range(len(gx)) if geo["found"][i]]
    n = len(found)
    examples = []
    if n == 0:
        return examples
    # every point's stacks and reference map are enqueued back to back and
    # read back once (no host round trip per example)
    P = torch.from_numpy(np.ascontiguousarray(geo["position"][found])).to("cuda", rd)
    N = torch.from_numpy(np.ascontiguousarray(geo["normal"][found])).to("cuda", rd)
    keys = torch.tensor([DATASET_KEY_BASE + i for i in found], dtype=torch.int64, device="cuda")
    stacks = torch.zeros((n, 7, 32, 32), dtype=torch.float32, device="cuda")
    s_r = torch.zeros(n, dtype=rd, device="cuda")
    s_d = torch.zeros(n, dtype=rd, device="cuda")
    frames = torch.zeros((n, 9), dtype=rd, device="cuda")
    ref = torch.zeros((n, 1024, 3), dtype=rd, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    fields = [k for k in render.RenderConfig.__dataclass_fields__ if hasattr(cfg, k)]
    for j, i in enumerate(found):
        kind = kinds[i % len(kinds)]
        c = render.RenderConfig(**{k: getattr(cfg, k) for k in fields})
        c.sampler_kind, c.seed, c.precision = kind, seed + i, precision
        st = render._cfg_struct(c, precision)
        st.map_spp = int(ref_spp)
        _lib.call("drcb_render_stacks", ds.handle, C.byref(st), _lib.ptr(P[j]), _lib.ptr(N[j]),
                  _lib.ptr(keys[j:j + 1]), 1, _lib.ptr(stacks[j]), _lib.ptr(s_r[j]),
                  _lib.ptr(s_d[j]), _lib.ptr(frames[j]), _lib.ptr(nf), _lib.stream_ptr())
        _lib.call("drcb_reference_map", ds.handle, C.byref(st), _lib.ptr(P[j]), _lib.ptr(N[j]),
                  C.c_uint64(DATASET_KEY_BASE + i), int(ref_spp), _lib.ptr(ref[j]), _lib.ptr(nf),
                  _lib.stream_ptr())
    stacks_h = stacks.cpu().numpy()
    s_r_h, s_d_h = s_r.double().cpu().numpy(), s_d.double().cpu().numpy()
    ref_h = ref.double().cpu().numpy()
    for j, i in enumerate(found):
        sr = float(s_r_h[j])
        target = ref_h[j].reshape(32, 32, 3) / sr
        examples.append(TrainingExample(
            input=stacks_h[j],
            target=np.moveaxis(target, -1, 0).astype(np.float32),
            s_r=sr, s_d=float(s_d_h[j]), scene_id=getattr(scene, "name", "scene"),
            pixel=(int(gx[i]), int(gy[i]))))
        if progress is not None:
            progress(len(examples), n)
    return examples
