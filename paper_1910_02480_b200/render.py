"""Frame driver and stage entry points — the drop-in surfaces of the
reference's rendering path, executed on the B200 through libdrcb.

  render_drc(scene, config, net)          drc/cache.py:377-470
  render(scene, config, mode, weights)    drc/integrators.py:662-722 (drc/direct)
  intersect_batch / primary_chain_batch / li_direct_batch /
  trace_radiance_batch / render_input_stacks / shade_indirect_batch
                                          stage-level parity surfaces

Host-side here is only integer control logic: the progressive pass plan
(cache.py:59-113), the task order and the per-point sample keys
(cache.py:42, 243, 279). Everything per ray, per texel, per map and per
pixel runs in CUDA; there is no CPU fallback.
"""

from __future__ import annotations

import dataclasses

import ctypes as C
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cnn import MODES, device_net
from .errors import ConfigError, ContractError, FormatError
from .scene import camera_struct, device_scene

T_EPS = 1e-4
ENTRY_KEY_BASE = 1 << 40
FALLBACK_KEY_BASE = 1 << 41
SAMPLER_KINDS = ("independent", "stratified")

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_SEED0 = np.uint64(0x853C49E6748FEA9B)


def hash_u64(*keys):
    """Keyed splitmix-style hash (sampler.py:25-37), host side, for the pass
    plan only (device kernels carry their own copy)."""
    h = _SEED0
    with np.errstate(over="ignore"):
        for k in keys:
            z = (h * _M2) ^ np.asarray(k, dtype=np.uint64)
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            h = z ^ (z >> np.uint64(31))
    return h


@dataclass
class RenderConfig:
    """RenderConfig (integrators.py:41-72) plus two B200 knobs:
    precision (64 = fp64 parity build, 32 = fp32 fast build) and net_mode
    ("fp32" exact SIMT, "tf32" / "bf16" tcgen05)."""

    spp: int = 16
    direct_spp: int = 8
    indirect_tasks: int = 5
    passes: int | None = None
    max_path_depth: int = 8
    map_resolution: int = 32
    mis_samples: int = 16
    rr_start: int = 5
    seed: int = 0
    threads: int = 0
    r0: int = 16
    tile: int = 64
    exposure: float = 1.0
    sampler_kind: str = "independent"
    precision: int = 64
    net_mode: str = "fp32"

    def __post_init__(self):
        for name in ("spp", "direct_spp", "indirect_tasks", "max_path_depth", "mis_samples",
                     "rr_start", "r0", "tile"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be >= 1")
        if self.mis_samples < 2:
            raise ConfigError("mis_samples must be >= 2")
        if self.r0 < 2 or (self.r0 & (self.r0 - 1)) != 0:
            raise ConfigError("r0 must be a power of two >= 2")
        if self.passes is not None and self.passes < 1:
            raise ConfigError("passes must be >= 1")
        if self.sampler_kind not in SAMPLER_KINDS:
            raise ConfigError(f"unknown sampler kind {self.sampler_kind!r}")
        if self.precision not in (32, 64):
            raise ConfigError("precision must be 32 or 64")
        if self.net_mode not in MODES:
            raise ConfigError(f"unknown net_mode {self.net_mode!r}")


def _cfg_struct(config, precision=None):
    if getattr(config, "map_resolution", 32) != 32:
        raise ConfigError("map_resolution must be 32 (the network's input size)")
    mis = int(config.mis_samples)
    if mis > 64:
        raise ConfigError("mis_samples above 64 is not supported on the device")
    c = _lib.RenderCfg()
    c.direct_spp = int(config.direct_spp)
    c.max_path_depth = int(config.max_path_depth)
    c.mis_samples = mis
    c.rr_start = int(config.rr_start)
    c.sampler_kind = SAMPLER_KINDS.index(config.sampler_kind)
    c.precision = int(precision or getattr(config, "precision", 64))
    c.tile = int(config.tile)
    c.seed = int(config.seed)
    return c


# ---------------------------------------------------------------------------
# progressive plan (cache.py:59-113, 371-374): integer host logic

@dataclass(frozen=True)
class PassPlan:
    pass_index: int
    r: int
    offset: tuple
    grid_x: np.ndarray
    grid_y: np.ndarray
    subgrids: tuple

    @property
    def task_count(self):
        return len(self.subgrids)

    def task_points(self, t):
        a, b = self.subgrids[t]
        step = len(self.subgrids) and int(round(np.sqrt(len(self.subgrids))))
        xs = self.grid_x[a::step] if step > 1 else self.grid_x
        ys = self.grid_y[b::step] if step > 1 else self.grid_y
        return xs, ys


def _ceil_div(a, b):
    return -(-a // b)


def plan_pass(image_size, pass_index, r0=16, jitter_seed=0):
    if r0 < 2 or (r0 & (r0 - 1)) != 0:
        raise ConfigError("r0 must be a power of two >= 2")
    w, h = image_size
    r = r0
    off = [int(hash_u64(jitter_seed, 0, 101) % np.uint64(r)),
           int(hash_u64(jitter_seed, 1, 101) % np.uint64(r))]
    for k in range(1, pass_index + 1):
        r = max(1, _ceil_div(r0, 1 << k))
        off = [(off[0] + (r + 1) // 2) % r, (off[1] + (r + 1) // 2) % r]
    r = max(1, _ceil_div(r0, 1 << pass_index))
    grid_x = np.arange(off[0], w, r, dtype=np.int64)
    grid_y = np.arange(off[1], h, r, dtype=np.int64)
    step = min(1 << pass_index, r0)
    cells = [(a, b) for a in range(step) for b in range(step)]
    order = np.argsort([int(hash_u64(jitter_seed, 7, a * step + b)) for a, b in cells],
                       kind="stable")
    return PassPlan(pass_index, r, (off[0], off[1]), grid_x, grid_y,
                    tuple(cells[i] for i in order))


def task_budget(config):
    if config.passes is not None:
        return sum(min(4 ** k, config.r0 ** 2) for k in range(config.passes))
    return config.indirect_tasks


def plan_points(size, config):
    """All cache points of a frame in the reference's evaluation order:
    pass by pass, task by task, meshgrid(xs, ys) y-major (cache.py:274-280,
    436-452). Returns px, py (int32), keys (uint64), r_final, pass records."""
    w, h = size
    budget = task_budget(config)
    pxs, pys, keys, passes = [], [], [], []
    done, k, r_final = 0, 0, None
    while done < budget:
        plan = plan_pass((w, h), k, config.r0, jitter_seed=config.seed)
        base = ENTRY_KEY_BASE + plan.pass_index * w * h * 4
        executed = 0
        for t in range(plan.task_count):
            if done >= budget:
                break
            xs, ys = plan.task_points(t)
            gx, gy = np.meshgrid(xs, ys)
            gx, gy = gx.ravel(), gy.ravel()
            pxs.append(gx)
            pys.append(gy)
            keys.append((base + gy * w + gx).astype(np.uint64))
            done += 1
            executed += 1
        passes.append({"index": k, "r": plan.r, "tasks": executed,
                       "points": int(sum(len(a) for a in pxs))})
        r_final = plan.r
        k += 1
    cat = (lambda a, dt: np.ascontiguousarray(np.concatenate(a).astype(dt)) if a
           else np.zeros(0, dt))
    return cat(pxs, np.int32), cat(pys, np.int32), cat(keys, np.uint64), r_final, passes


# ---------------------------------------------------------------------------
# frame driver

@dataclasses.dataclass(frozen=True)
class CacheEntry:
    """drc.cache.CacheEntry (cache.py:50-55)."""

    pixel: tuple
    position: np.ndarray
    normal: np.ndarray
    indirect_radiance: np.ndarray
    specular_throughput: np.ndarray


class FrameState:
    """Telemetry view of a finished frame (the reference returns its DrcState).
    The entry pool is copied out only when the frame was rendered with
    entries=True (render_drc does); otherwise only its size is known."""

    def __init__(self, entries, points, pool=None):
        self.entry_count = entries
        self.planned_points = points
        self._pool = pool

    def entries(self):
        """DrcState.entries (cache.py:196-201), in append (task) order."""
        if self._pool is None:
            raise ContractError("entry pool not collected (render with entries=True)")
        px, py, pos, nrm, rad, thr = self._pool
        return [CacheEntry(pixel=(int(px[i]), int(py[i])), position=pos[i], normal=nrm[i],
                           indirect_radiance=rad[i], specular_throughput=thr[i])
                for i in range(self.entry_count)]


DRCC_MAGIC = b"DRCC"
DRCC_VERSION = 1


def write_cache_dump(entries, path):
    """Little-endian entry records: pixel, position, normal, radiance
    (cache.py:476-485)."""
    import struct

    with open(path, "wb") as f:
        f.write(DRCC_MAGIC)
        f.write(struct.pack("<II", DRCC_VERSION, len(entries)))
        for e in entries:
            f.write(struct.pack("<II", int(e.pixel[0]), int(e.pixel[1])))
            f.write(np.asarray(e.position, dtype="<f4").tobytes())
            f.write(np.asarray(e.normal, dtype="<f4").tobytes())
            f.write(np.asarray(e.indirect_radiance, dtype="<f4").tobytes())


def read_cache_dump(path):
    """cache.py:488-507 (FormatError with byte offsets)."""
    import struct

    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != DRCC_MAGIC:
        raise FormatError("bad magic, not a DRCC dump", offset=0)
    version, count = struct.unpack("<II", raw[4:12])
    if version != DRCC_VERSION:
        raise FormatError(f"unsupported DRCC version {version}", offset=4)
    rec = 8 + 9 * 4
    if len(raw) != 12 + count * rec:
        raise FormatError("truncated cache dump", offset=len(raw))
    out = []
    for i in range(count):
        o = 12 + i * rec
        x, y = struct.unpack("<II", raw[o:o + 8])
        vals = np.frombuffer(raw[o + 8:o + rec], dtype="<f4").astype(np.float64)
        out.append(CacheEntry(pixel=(x, y), position=vals[0:3], normal=vals[3:6],
                              indirect_radiance=vals[6:9], specular_throughput=np.ones(3)))
    return out


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise ContractError("libdrcb needs a CUDA device (there is no CPU path)")
    return torch


def render_drc_device(scene, config, net, camera=None, out=None, precision=None, plan=None,
                      telemetry=True, entries=False):
    """One DRC frame, result left on the device: (image (H,W,3) CUDA tensor,
    telemetry dict). `camera` overrides scene.camera (multi-frame benches);
    `plan` reuses a plan_points() result; telemetry=False enqueues the frame
    without any host synchronisation."""
    torch = _torch()
    prec = int(precision or getattr(config, "precision", 64))
    dtype = torch.float64 if prec == 64 else torch.float32
    cam = camera or scene.camera
    w, h = cam.resolution
    ds = device_scene(scene)
    cfg = _cfg_struct(config, prec)
    px, py, keys, r_final, passes = plan or plan_points((w, h), config)
    net_mode = getattr(config, "net_mode", "fp32")
    dn = device_net(net) if len(px) else None
    if out is None:
        out = torch.empty((h, w, 3), dtype=dtype, device="cuda")
    tel = (C.c_int64 * 10)() if (telemetry or entries) else None
    t0 = time.time()
    args = (ds.handle, dn.handle if dn else None, C.byref(camera_struct(cam)), C.byref(cfg),
            px.ctypes.data_as(C.c_void_p), py.ctypes.data_as(C.c_void_p),
            keys.ctypes.data_as(C.c_void_p), len(px), int(r_final or 1), MODES[net_mode],
            _lib.ptr(out), tel)
    pool = None
    if entries:
        n = max(len(px), 1)
        bufs = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(2)] + \
               [torch.zeros((n, 3), dtype=dtype, device="cuda") for _ in range(4)]
        ent = _lib.Entries(*[C.c_void_p(b.data_ptr()) for b in bufs])
        _lib.call("drcb_render_drc_entries", *args, C.byref(ent), _lib.stream_ptr())
        m = int(tel[0])
        pool = [b[:m].cpu().numpy().astype(np.float64 if b.dim() == 2 else np.int64) for b in bufs]
    else:
        _lib.call("drcb_render_drc", *args, _lib.stream_ptr())
    if tel is None:
        return out, None
    telemetry = {
        "mode": "drc", "direct_spp": config.direct_spp,
        "geometry_seconds": 0.0, "direct_seconds": 0.0,
        "passes": [dict(p, entries=None, seconds=None) for p in passes],
        "nonfinite": int(tel[2]), "entries": int(tel[0]),
        "fallback_pixels": int(tel[1]), "tasks": sum(p["tasks"] for p in passes),
        "seconds": time.time() - t0,
        "stage_us": {"gbuffer_direct": int(tel[4]), "maps": int(tel[5]), "network": int(tel[6]),
                     "shade_interp": int(tel[7])},
        "substage_us": {"shade": int(tel[8]), "interp": int(tel[9])},
    }
    telemetry["state"] = FrameState(int(tel[0]), int(tel[3]), pool)
    return out, telemetry


class DeviceFrame:
    """A DRC frame in progress on the device (drcb_frame_*): G-buffer + direct
    at construction, then cache points in any number of submissions, then
    composites at a pass spacing r. The host pass loop of render_drc drives
    it (cache.py:426-469)."""

    def __init__(self, scene, config, net, camera=None, max_points=0):
        torch = _torch()
        self.prec = int(getattr(config, "precision", 64))
        self.dtype = torch.float64 if self.prec == 64 else torch.float32
        self.cam = camera or scene.camera
        self.w, self.h = self.cam.resolution
        self.net_mode = MODES[getattr(config, "net_mode", "fp32")]
        dn = device_net(net) if max_points else None
        self._keep = (dn,)
        h = C.c_void_p()
        _lib.call("drcb_frame_begin", device_scene(scene).handle, dn.handle if dn else None,
                  C.byref(camera_struct(self.cam)), C.byref(_cfg_struct(config, self.prec)),
                  self.net_mode, int(max_points), C.byref(h), _lib.stream_ptr())
        self.handle = h
        self.max_points = int(max_points)

    def add_points(self, px, py, keys):
        px = np.ascontiguousarray(px, dtype=np.int32)
        py = np.ascontiguousarray(py, dtype=np.int32)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        if len(px):
            _lib.call("drcb_frame_add_points", self.handle, px.ctypes.data_as(C.c_void_p),
                      py.ctypes.data_as(C.c_void_p), keys.ctypes.data_as(C.c_void_p), len(px),
                      _lib.stream_ptr())

    def composite(self, r, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty((self.h, self.w, 3), dtype=self.dtype, device="cuda")
        _lib.call("drcb_frame_composite", self.handle, int(r), _lib.ptr(out), _lib.stream_ptr())
        return out

    def info(self):
        o = (C.c_int64 * 4)()
        _lib.call("drcb_frame_info", self.handle, o, _lib.stream_ptr())
        return {"entries": int(o[0]), "nonfinite": int(o[1]), "points": int(o[2])}

    def entries(self):
        torch = _torch()
        n = max(self.max_points, 1)
        bufs = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(2)] + \
               [torch.zeros((n, 3), dtype=self.dtype, device="cuda") for _ in range(4)]
        ent = _lib.Entries(*[C.c_void_p(b.data_ptr()) for b in bufs])
        _lib.call("drcb_frame_entries", self.handle, C.byref(ent), _lib.stream_ptr())
        m = self.info()["entries"]
        return [b[:m].cpu().numpy().astype(np.float64 if b.dim() == 2 else np.int64) for b in bufs]

    def close(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.drcb_frame_end(self.handle, _lib.stream_ptr())
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def render_drc(scene, config, net, interrupt=None, snapshots=None):
    """Drop-in for drc.cache.render_drc (cache.py:377-470): (image (H,W,3)
    float64, telemetry).

    The reference's progressive control plane on the host: pass by pass and
    task by task (plan_pass, cache.py:96-113), each pass's cache points
    evaluated on the device in one submission (split at snapshot budgets);
    `snapshots` budgets are composited mid-run from the entries so far (the
    reference's append-only pool makes them equal to clean runs,
    cache.py:381-385, 450-452); `interrupt` is polled after every pass and
    finalises the frame at that pass (cache.py:460-461). Telemetry carries
    per-pass {index, r, tasks, entries, seconds}."""
    w, h = scene.camera.resolution
    t0 = time.time()
    budget = task_budget(config)
    px_all, _, _, _, _ = plan_points((w, h), config)
    frame = DeviceFrame(scene, config, net, max_points=len(px_all))
    try:
        _torch().cuda.current_stream().synchronize()
        geo_direct_s = time.time() - t0
        snaps = sorted(set(snapshots)) if snapshots else []
        snap_images = {}
        passes = []
        done, k, r = 0, 0, None
        while done < budget:
            plan = plan_pass((w, h), k, config.r0, jitter_seed=config.seed)
            tp = time.time()
            base = ENTRY_KEY_BASE + plan.pass_index * w * h * 4
            seg = ([], [], [])
            executed = 0
            for t in range(plan.task_count):
                if done >= budget:
                    break
                xs, ys = plan.task_points(t)
                gx, gy = np.meshgrid(xs, ys)
                gx, gy = gx.ravel(), gy.ravel()
                seg[0].append(gx)
                seg[1].append(gy)
                seg[2].append((base + gy * w + gx).astype(np.uint64))
                done += 1
                executed += 1
                if done in snaps:
                    frame.add_points(*(np.concatenate(a) for a in seg))
                    seg = ([], [], [])
                    snap_images[done] = frame.composite(plan.r).double().cpu().numpy()
            if seg[0]:
                frame.add_points(*(np.concatenate(a) for a in seg))
            r = plan.r
            info = frame.info()  # synchronises: the pass is finished
            passes.append({"index": k, "r": plan.r, "tasks": executed, "entries": info["entries"],
                           "seconds": time.time() - tp})
            k += 1
            if interrupt is not None and interrupt():
                break  # this pass is finalised: composite below
        image = frame.composite(r or 1).double().cpu().numpy()
        info = frame.info()
        pool = frame.entries() if frame.max_points else [np.zeros(0, np.int64)] * 2 + \
            [np.zeros((0, 3))] * 4
    finally:
        frame.close()
    tel = {"mode": "drc", "direct_spp": config.direct_spp,
           "geometry_seconds": geo_direct_s, "direct_seconds": 0.0,
           "passes": passes, "nonfinite": info["nonfinite"], "entries": info["entries"],
           "fallback_pixels": 0, "tasks": done, "seconds": time.time() - t0}
    if snap_images:
        tel["snapshots"] = snap_images
    tel["state"] = FrameState(info["entries"], info["points"], pool)
    return image, tel


def _replace(config, **kw):
    import dataclasses

    if dataclasses.is_dataclass(config):
        return dataclasses.replace(config, **kw)
    d = dict(config.__dict__)
    d.update(kw)
    return RenderConfig(**{k: v for k, v in d.items() if k in RenderConfig.__dataclass_fields__})


def render(scene, config, mode="pt", weights=None, interrupt=None):
    """Drop-in for drc.integrators.render for the modes on the hot path."""
    if mode not in ("pt", "direct", "drc"):
        raise ConfigError(f"unknown render mode {mode!r}")
    if mode == "drc":
        if weights is None:
            raise ConfigError("drc mode requires a weights network")
        return render_drc(scene, config, weights, interrupt=interrupt)
    if mode == "direct":
        t0 = time.time()
        torch = _torch()
        prec = int(getattr(config, "precision", 64))
        dtype = torch.float64 if prec == 64 else torch.float32
        w, h = scene.camera.resolution
        gb = GBufferTensors(w * h, dtype)
        direct = torch.empty((h, w, 3), dtype=dtype, device="cuda")
        nf = torch.zeros(1, dtype=torch.int64, device="cuda")
        cfg = _cfg_struct(config, prec)
        cfg.include_background = 1
        _lib.call("drcb_gbuffer_direct", device_scene(scene).handle,
                  C.byref(camera_struct(scene.camera)), C.byref(cfg), C.byref(gb.struct()),
                  _lib.ptr(direct), _lib.ptr(nf), _lib.stream_ptr())
        return direct.double().cpu().numpy(), {"mode": "direct", "spp": config.direct_spp,
                                               "seconds": time.time() - t0,
                                               "nonfinite": int(nf.item())}
    # mode == "pt": spp jittered paths per pixel (integrators.py:678-722)
    t0 = time.time()
    torch = _torch()
    prec = int(getattr(config, "precision", 64))
    dtype = torch.float64 if prec == 64 else torch.float32
    w, h = scene.camera.resolution
    image = torch.empty((h, w, 3), dtype=dtype, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cfg = _cfg_struct(config, prec)
    cfg.direct_spp = int(config.spp)
    _lib.call("drcb_render_pt", device_scene(scene).handle, C.byref(camera_struct(scene.camera)),
              C.byref(cfg), _lib.ptr(image), _lib.ptr(nf), _lib.stream_ptr())
    return image.double().cpu().numpy(), {"mode": "pt", "spp": config.spp,
                                          "seconds": time.time() - t0,
                                          "nonfinite": int(nf.item())}


# ---------------------------------------------------------------------------
# stage-level surfaces (numpy in / numpy out, for parity tests)

def gbuffer_direct(scene, config, camera=None, include_background=False):
    """The frame's first stage on its own: DrcState's G-buffer (the
    unjittered centre chains, cache.py:157-176) and the direct pass averaged
    per pixel (cache.py:393-423) -> (G-buffer dict of (W*H, ...) arrays,
    direct (H, W, 3) float64)."""
    torch = _torch()
    prec = int(getattr(config, "precision", 64))
    dtype = torch.float64 if prec == 64 else torch.float32
    cam = camera or scene.camera
    w, h = cam.resolution
    gb = GBufferTensors(w * h, dtype)
    direct = torch.empty((h, w, 3), dtype=dtype, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cfg = _cfg_struct(config, prec)
    cfg.include_background = int(bool(include_background))
    _lib.call("drcb_gbuffer_direct", device_scene(scene).handle, C.byref(camera_struct(cam)),
              C.byref(cfg), C.byref(gb.struct()), _lib.ptr(direct), _lib.ptr(nf), _lib.stream_ptr())
    return gb.numpy(), direct.double().cpu().numpy()


class GBufferTensors:
    def __init__(self, n, dtype):
        torch = _torch()
        dev = "cuda"
        self.found = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.escaped = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.position = torch.zeros((n, 3), dtype=dtype, device=dev)
        self.normal = torch.zeros((n, 3), dtype=dtype, device=dev)
        self.throughput = torch.zeros((n, 3), dtype=dtype, device=dev)
        self.direction = torch.zeros((n, 3), dtype=dtype, device=dev)
        self.t_total = torch.zeros(n, dtype=dtype, device=dev)
        self.mat = torch.zeros(n, dtype=torch.int32, device=dev)

    def struct(self):
        g = _lib.GBuffer()
        for f in ("found", "escaped", "position", "normal", "throughput", "direction",
                  "t_total", "mat"):
            setattr(g, f, getattr(self, f).data_ptr())
        return g

    def numpy(self):
        return {
            "found": self.found.cpu().numpy().astype(bool),
            "escaped": self.escaped.cpu().numpy().astype(bool),
            "position": self.position.double().cpu().numpy(),
            "normal": self.normal.double().cpu().numpy(),
            "mat": self.mat.cpu().numpy().astype(np.int64),
            "throughput": self.throughput.double().cpu().numpy(),
            "direction": self.direction.double().cpu().numpy(),
            "t_total": self.t_total.double().cpu().numpy(),
        }


class _Keep(list):
    """Holds device temporaries until the library call has been issued and
    the stream synchronised (a bare `ptr(_dev(...))` would let torch recycle
    the block before the kernel reads it)."""

    def dev(self, a, dtype):
        torch = _torch()
        t = torch.from_numpy(np.array(a, copy=True, order="C")).to(device="cuda", dtype=dtype)
        self.append(t)
        return _lib.ptr(t)


def _dev(a, dtype):
    torch = _torch()
    return torch.from_numpy(np.array(a, copy=True, order="C")).to(device="cuda", dtype=dtype)


# drcb_intersect's mixed mode: the fp32 build's traversal of fp64 rays, with
# undecided / near-tie candidates re-tested in fp64 (include/drcb.h)
PREC_MIXED = 3264


def _rdtype(precision):
    torch = _torch()
    return torch.float64 if precision in (64, PREC_MIXED) else torch.float32


def intersect_batch(scene, origins, directions, t_min=T_EPS, t_max=np.inf, record=True,
                    precision=64):
    """geometry.intersect_batch on the device: dict(hit, t, prim[, mat,
    position, normal]). precision: 64 (fp64 build), 32 (fp32 build on
    fp32-rounded rays) or PREC_MIXED (fp32 build on the fp64 rays, the
    G-buffer's primary-cast mode)."""
    torch = _torch()
    rd = _rdtype(precision)
    O = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    D = np.atleast_2d(np.asarray(directions, dtype=np.float64))
    n = len(O)
    Od, Dd = _dev(O, rd), _dev(D, rd)
    tmin = _dev(np.broadcast_to(np.asarray(t_min, dtype=np.float64), (n,)), rd)
    tmax = _dev(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,)), rd)
    hit = torch.zeros(n, dtype=torch.uint8, device="cuda")
    t = torch.zeros(n, dtype=rd, device="cuda")
    prim = torch.zeros(n, dtype=torch.int64, device="cuda")
    mat = torch.zeros(n, dtype=torch.int32, device="cuda") if record else None
    pos = torch.zeros((n, 3), dtype=rd, device="cuda") if record else None
    nrm = torch.zeros((n, 3), dtype=rd, device="cuda") if record else None
    _lib.call("drcb_intersect", device_scene(scene).handle, precision, _lib.ptr(Od), _lib.ptr(Dd),
              n, _lib.ptr(tmin), _lib.ptr(tmax), int(bool(record)), _lib.ptr(hit), _lib.ptr(t),
              _lib.ptr(prim), _lib.ptr(mat), _lib.ptr(pos), _lib.ptr(nrm), _lib.stream_ptr())
    out = {"hit": hit.cpu().numpy().astype(bool), "t": t.double().cpu().numpy(),
           "prim": prim.cpu().numpy()}
    if record:
        out["mat"] = mat.cpu().numpy().astype(np.int64)
        out["position"] = pos.double().cpu().numpy()
        out["normal"] = nrm.double().cpu().numpy()
    return out


def primary_chain_batch(scene, origins, directions, precision=64):
    K = _Keep()
    rd = _rdtype(precision)
    O = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    D = np.atleast_2d(np.asarray(directions, dtype=np.float64))
    gb = GBufferTensors(len(O), rd)
    _lib.call("drcb_primary_chain", device_scene(scene).handle, precision, K.dev(O, rd),
              K.dev(D, rd), len(O), C.byref(gb.struct()), _lib.stream_ptr())
    return gb.numpy()


def _sampler_cfg(sampler, precision, **kw):
    cfg = RenderConfig(direct_spp=max(int(getattr(sampler, "spp", 1)), 1),
                       sampler_kind=getattr(sampler, "kind", "independent"),
                       seed=int(getattr(sampler, "seed", 0)), precision=precision, **kw)
    return _cfg_struct(cfg, precision)


def li_direct_batch(scene, origins, directions, pixel_keys, sample_keys, sampler,
                    include_background=True, stats=None, precision=64):
    K = _Keep()
    torch = _torch()
    rd = _rdtype(precision)
    O = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    n = len(O)
    L = torch.zeros((n, 3), dtype=rd, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cfg = _sampler_cfg(sampler, precision)
    _lib.call("drcb_li_direct", device_scene(scene).handle, C.byref(cfg), K.dev(O, rd),
              K.dev(np.asarray(directions, dtype=np.float64), rd),
              K.dev(np.asarray(pixel_keys, dtype=np.uint64).view(np.int64), torch.int64),
              K.dev(np.asarray(sample_keys, dtype=np.uint64).view(np.int64), torch.int64),
              n, int(bool(include_background)), _lib.ptr(L), _lib.ptr(nf), _lib.stream_ptr())
    if stats is not None:
        stats["nonfinite"] = stats.get("nonfinite", 0) + int(nf.item())
    return L.double().cpu().numpy()


def trace_radiance_batch(scene, origins, directions, pixel_keys, sample_keys, sampler, max_depth,
                         skip_first_emission=False, rr_start=5, stats=None, precision=64):
    K = _Keep()
    torch = _torch()
    if max_depth < 1:
        raise ContractError("max_depth must be >= 1")
    rd = _rdtype(precision)
    O = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    n = len(O)
    L = torch.zeros((n, 3), dtype=rd, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cfg = _sampler_cfg(sampler, precision)
    _lib.call("drcb_trace_radiance", device_scene(scene).handle, C.byref(cfg),
              K.dev(O, rd), K.dev(np.asarray(directions, dtype=np.float64), rd),
              K.dev(np.asarray(pixel_keys, dtype=np.uint64).view(np.int64), torch.int64),
              K.dev(np.asarray(sample_keys, dtype=np.uint64).view(np.int64), torch.int64),
              n, int(max_depth), int(bool(skip_first_emission)), int(rr_start), _lib.ptr(L),
              _lib.ptr(nf), _lib.stream_ptr())
    if stats is not None:
        stats["nonfinite"] = stats.get("nonfinite", 0) + int(nf.item())
    return L.double().cpu().numpy()


def render_input_stacks(scene, positions, normals, keys, config, precision=64):
    """render_input_stacks_batch (hemimap.py:229-281) for n hits given as
    front-facing positions/normals. Returns stacks (n,7,32,32) float32,
    s_r (n,), s_d (n,), frames (n,3,3) rows t,b,n."""
    K = _Keep()
    torch = _torch()
    rd = _rdtype(precision)
    P = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    n = len(P)
    stacks = torch.zeros((n, 7, 32, 32), dtype=torch.float32, device="cuda")
    s_r = torch.zeros(n, dtype=rd, device="cuda")
    s_d = torch.zeros(n, dtype=rd, device="cuda")
    frames = torch.zeros((n, 9), dtype=rd, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cfg = _cfg_struct(config, precision)
    _lib.call("drcb_render_stacks", device_scene(scene).handle, C.byref(cfg),
              K.dev(P, rd), K.dev(np.asarray(normals, dtype=np.float64), rd),
              K.dev(np.asarray(keys, dtype=np.uint64).view(np.int64), torch.int64), n,
              _lib.ptr(stacks), _lib.ptr(s_r), _lib.ptr(s_d), _lib.ptr(frames), _lib.ptr(nf),
              _lib.stream_ptr())
    return (stacks.cpu().numpy(), s_r.double().cpu().numpy(), s_d.double().cpu().numpy(),
            frames.double().cpu().numpy().reshape(n, 3, 3))


def shade_indirect_batch(scene, pred, s_r, frames, wo, mats, keys, config, precision=64):
    """shade_indirect (integrators.py:564-614) for n cache points at once.
    pred (n,3,32,32) float32 normalised prediction; frames (n,3,3)."""
    K = _Keep()
    torch = _torch()
    rd = _rdtype(precision)
    pred = np.ascontiguousarray(pred, dtype=np.float32)
    n = len(pred)
    L = torch.zeros((n, 3), dtype=rd, device="cuda")
    cfg = _cfg_struct(config, precision)
    _lib.call("drcb_shade", device_scene(scene).handle, C.byref(cfg),
              K.dev(pred, torch.float32), K.dev(np.asarray(s_r, np.float64), rd),
              K.dev(np.asarray(frames, np.float64).reshape(n, 9), rd),
              K.dev(np.asarray(wo, np.float64).reshape(n, 3), rd),
              K.dev(np.asarray(mats, np.int32), torch.int32),
              K.dev(np.asarray(keys, dtype=np.uint64).view(np.int64), torch.int64), n,
              _lib.ptr(L), _lib.stream_ptr())
    return L.double().cpu().numpy()
