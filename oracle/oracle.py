"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_build/liboracle.so,
the scalar fp64 C restatement of the reference renderer (drc_oracle.c).

Functions mirror the reference's numpy signatures (numpy in, numpy out) so
tests read like the reference's own. Pinned against the reference's golden
vectors in tests/test_oracle.py.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
vp = C.c_void_p


class OrSceneDesc(C.Structure):
    _fields_ = [("n_spheres", C.c_int32), ("n_quads", C.c_int32), ("n_tris", C.c_int32),
                ("n_materials", C.c_int32), ("n_point_lights", C.c_int32)] + \
        [(n, vp) for n in ("sph_center", "sph_radius", "sph_mat", "quad_corner", "quad_eu",
                           "quad_ev", "quad_mat", "tri_v0", "tri_v1", "tri_v2", "tri_mat",
                           "mat_kind", "mat_albedo", "mat_exponent", "mat_ior", "mat_emission",
                           "point_pos", "point_intensity")] + \
        [("global_up", C.c_double * 3), ("rotated_up", C.c_double * 3),
         ("environment", C.c_double * 3)]


class OrCamera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("forward", C.c_double * 3),
                ("right", C.c_double * 3), ("up", C.c_double * 3), ("tan_half", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class OrCfg(C.Structure):
    _fields_ = [("direct_spp", C.c_int32), ("max_path_depth", C.c_int32),
                ("mis_samples", C.c_int32), ("rr_start", C.c_int32),
                ("sampler_kind", C.c_int32), ("tile", C.c_int32), ("seed", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            import subprocess

            subprocess.check_call(["make"], cwd=HERE)
        _lib = C.CDLL(LIB)
        _lib.or_scene_create.restype = vp
        _lib.or_scene_create.argtypes = [C.POINTER(OrSceneDesc)]
        _lib.or_net_create.restype = vp
        _lib.or_net_create.argtypes = [C.c_char_p, C.c_int64]
        _lib.or_li_direct.restype = C.c_int64
        _lib.or_trace_radiance.restype = C.c_int64
        _lib.or_gbuffer_direct.restype = C.c_int64
        _lib.or_render_stacks.restype = C.c_int64
        for f in ("or_scene_destroy", "or_net_destroy"):
            getattr(_lib, f).argtypes = [vp]
    return _lib


def set_threads(n):
    lib().or_set_threads(int(n))


def P(a):
    return a.ctypes.data_as(vp) if a is not None and a.size else None


class OracleScene:
    def __init__(self, scene):
        from paper_1910_02480_b200.scene import flatten

        self.scene = scene
        f = flatten(scene)
        d = OrSceneDesc()
        d.n_spheres, d.n_quads, d.n_tris = len(f["sph_radius"]), len(f["quad_mat"]), len(f["tri_mat"])
        d.n_materials, d.n_point_lights = len(f["mat_kind"]), len(f["point_pos"])
        self._keep = {}
        for k, _ in OrSceneDesc._fields_[5:-3]:
            a = np.ascontiguousarray(f[k])
            self._keep[k] = a
            setattr(d, k, P(a))
        for k in ("global_up", "rotated_up", "environment"):
            for i in range(3):
                getattr(d, k)[i] = float(f[k][i])
        self.env = np.asarray(f["environment"], dtype=np.float64)
        self.h = vp(lib().or_scene_create(C.byref(d)))

    def __del__(self):
        try:
            lib().or_scene_destroy(self.h)
        except Exception:
            pass


def camera(cam):
    fwd, right, up = cam.basis()
    c = OrCamera()
    for k in range(3):
        c.position[k], c.forward[k], c.right[k], c.up[k] = (float(cam.position[k]), float(fwd[k]),
                                                           float(right[k]), float(up[k]))
    c.tan_half = math.tan(math.radians(cam.fov) * 0.5)
    c.width, c.height = int(cam.resolution[0]), int(cam.resolution[1])
    return c


def cfg_of(config=None, sampler=None):
    c = OrCfg()
    if config is not None:
        c.direct_spp, c.max_path_depth = int(config.direct_spp), int(config.max_path_depth)
        c.mis_samples, c.rr_start = int(config.mis_samples), int(config.rr_start)
        c.sampler_kind = ("independent", "stratified").index(config.sampler_kind)
        c.tile, c.seed = int(config.tile), int(config.seed)
    if sampler is not None:
        c.direct_spp = max(int(sampler.spp), 1)
        c.sampler_kind = ("independent", "stratified").index(sampler.kind)
        c.seed = int(sampler.seed)
        c.tile = c.tile or 64
    return c


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape else a


def intersect_batch(osc, O, D, t_min=1e-4, t_max=np.inf, record=True):
    O, D = _f64(np.atleast_2d(O)), _f64(np.atleast_2d(D))
    n = len(O)
    tmin = _f64(np.broadcast_to(np.asarray(t_min, dtype=np.float64), (n,)))
    tmax = _f64(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,)))
    hit, t, prim = np.zeros(n, np.uint8), np.zeros(n), np.zeros(n, np.int64)
    mat, pos, nrm = np.zeros(n, np.int32), np.zeros((n, 3)), np.zeros((n, 3))
    lib().or_intersect(osc.h, P(O), P(D), C.c_int64(n), P(tmin), P(tmax), int(record), P(hit),
                       P(t), P(prim), P(mat), P(pos), P(nrm))
    out = {"hit": hit.astype(bool), "t": t, "prim": prim}
    if record:
        out.update(mat=mat.astype(np.int64), position=pos, normal=nrm)
    return out


def primary_chain_batch(osc, O, D):
    O, D = _f64(np.atleast_2d(O)), _f64(np.atleast_2d(D))
    n = len(O)
    g = _gbuf(n)
    lib().or_primary_chain(osc.h, P(O), P(D), C.c_int64(n), *[P(g[k]) for k in GB_KEYS])
    return _gfix(g)


GB_KEYS = ("found", "escaped", "position", "normal", "mat", "throughput", "direction", "t_total")


def _gbuf(n):
    return {"found": np.zeros(n, np.uint8), "escaped": np.zeros(n, np.uint8),
            "position": np.zeros((n, 3)), "normal": np.zeros((n, 3)), "mat": np.zeros(n, np.int32),
            "throughput": np.zeros((n, 3)), "direction": np.zeros((n, 3)), "t_total": np.zeros(n)}


def _gfix(g):
    g = dict(g)
    g["found"] = g["found"].astype(bool)
    g["escaped"] = g["escaped"].astype(bool)
    g["mat"] = g["mat"].astype(np.int64)
    return g


def li_direct_batch(osc, O, D, pix, smp, sampler, include_background=True):
    O, D = _f64(np.atleast_2d(O)), _f64(np.atleast_2d(D))
    n = len(O)
    L = np.zeros((n, 3))
    pix = np.ascontiguousarray(pix, dtype=np.uint64)
    smp = np.ascontiguousarray(smp, dtype=np.uint64)
    lib().or_li_direct(osc.h, C.byref(cfg_of(sampler=sampler)), P(O), P(D), P(pix), P(smp),
                       C.c_int64(n), int(include_background), P(L))
    return L


def trace_radiance_batch(osc, O, D, pix, smp, sampler, max_depth, skip_first_emission=False,
                         rr_start=5):
    O, D = _f64(np.atleast_2d(O)), _f64(np.atleast_2d(D))
    n = len(O)
    L = np.zeros((n, 3))
    pix = np.ascontiguousarray(pix, dtype=np.uint64)
    smp = np.ascontiguousarray(smp, dtype=np.uint64)
    lib().or_trace_radiance(osc.h, C.byref(cfg_of(sampler=sampler)), P(O), P(D), P(pix), P(smp),
                            C.c_int64(n), int(max_depth), int(skip_first_emission), int(rr_start),
                            P(L))
    return L


def gbuffer_direct(osc, cam, config, p0=0, p1=None):
    """DrcState geo + direct pass (cache.py:157-176, 393-423) for pixels
    [p0, p1) of the camera's image; other rows stay zero."""
    w, h = cam.resolution
    n = w * h
    p1 = n if p1 is None else p1
    g = _gbuf(n)
    direct = np.zeros((n, 3))
    lib().or_gbuffer_direct(osc.h, C.byref(camera(cam)), C.byref(cfg_of(config)), C.c_int64(p0),
                            C.c_int64(p1), *[P(g[k]) for k in GB_KEYS], P(direct))
    return _gfix(g), direct


def render_stacks(osc, pos, nrm, keys, config):
    pos, nrm = _f64(np.atleast_2d(pos)), _f64(np.atleast_2d(nrm))
    n = len(pos)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    stacks = np.zeros((n, 7, 32, 32), np.float32)
    s_r, s_d, frames = np.zeros(n), np.zeros(n), np.zeros((n, 9))
    lib().or_render_stacks(osc.h, C.byref(cfg_of(config)), P(pos), P(nrm), P(keys), C.c_int64(n),
                           P(stacks), P(s_r), P(s_d), P(frames))
    return stacks, s_r, s_d, frames.reshape(n, 3, 3)


def shade(osc, pred, s_r, frames, wo, mats, keys, config):
    pred = np.ascontiguousarray(pred, dtype=np.float32)
    n = len(pred)
    L = np.zeros((n, 3))
    lib().or_shade(osc.h, C.byref(cfg_of(config)), P(pred), P(_f64(s_r)), P(_f64(frames, (n, 9))),
                   P(_f64(wo, (n, 3))), P(np.ascontiguousarray(mats, dtype=np.int32)),
                   P(np.ascontiguousarray(keys, dtype=np.uint64)), C.c_int64(n), P(L))
    return L


class OracleNet:
    def __init__(self, drcw_bytes):
        self.h = vp(lib().or_net_create(bytes(drcw_bytes), len(drcw_bytes)))
        if not self.h:
            raise ValueError("oracle: bad DRCW bytes")

    def forward(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.zeros((len(x), 3, 32, 32), np.float32)
        lib().or_net_forward(self.h, P(x), P(y), C.c_int64(len(x)))
        return y

    def __del__(self):
        try:
            lib().or_net_destroy(self.h)
        except Exception:
            pass


def interp_composite(geo, size, env, epx, epy, en, erad, r, direct):
    w, h = size
    image = np.zeros((w * h, 3))
    m = len(epx)
    lib().or_interp_composite(
        int(w), int(h), P(np.ascontiguousarray(geo["found"], np.uint8)),
        P(np.ascontiguousarray(geo["escaped"], np.uint8)), P(_f64(geo["normal"])),
        P(_f64(geo["throughput"])), P(_f64(env)), P(np.ascontiguousarray(epx, np.int32)),
        P(np.ascontiguousarray(epy, np.int32)), P(_f64(en, (max(m, 0), 3))),
        P(_f64(erad, (max(m, 0), 3))), C.c_int64(m), int(r),
        P(_f64(direct, (w * h, 3))) if direct is not None else None, P(image))
    return image.reshape(h, w, 3)


def render_drc(osc, config, onet, cam=None):
    """Whole DRC frame (cache.py:377-470) on the CPU oracle; the pass plan
    comes from the host planner (integer logic shared with the product)."""
    from paper_1910_02480_b200.render import plan_points

    cam = cam or osc.scene.camera
    w, h = cam.resolution
    geo, direct = gbuffer_direct(osc, cam, config)
    px, py, keys, r_final, _ = plan_points((w, h), config)
    idx = py.astype(np.int64) * w + px
    live = geo["found"][idx]
    px, py, keys, idx = px[live], py[live], keys[live], idx[live]
    if len(px):
        stacks, s_r, _, frames = render_stacks(osc, geo["position"][idx], geo["normal"][idx], keys,
                                               config)
        pred = onet.forward(stacks)
        L = shade(osc, pred, s_r, frames, -geo["direction"][idx], geo["mat"][idx], keys, config)
        en = geo["normal"][idx]
    else:
        L = en = np.zeros((0, 3))
    img = interp_composite(geo, (w, h), osc.env, px, py, en, L, r_final or 1, direct)
    return img, {"entries": int(len(px))}
