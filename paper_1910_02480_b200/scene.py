"""Scene documents and their upload to the device.

`parse_scene` reads the reference's JSON scene format (drc/scene.py:286-331:
camera, materials, shapes, point_lights, global_up, optional environment) into
plain dataclasses whose attribute names match the reference's `Scene`, so a
reference `drc.scene.Scene` object can be passed anywhere a scene is expected
(duck typing). `DeviceScene` packs any such scene into the SoA description of
include/drcb.h and builds the device BVH once (drcb_scene_create).

Host-side constants that feed every ray (camera basis, the rotated reference
up of bsdf._rotated_up) are computed here with numpy using the same
expressions as the reference, so they are bit-identical to it.
"""

from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import SceneParseError, SceneValidationError

MATERIAL_KINDS = ("diffuse", "glossy", "mirror", "transmission")
KIND_CODE = {"diffuse": 0, "glossy": 1, "mirror": 2, "transmission": 3}


def _normalize(v):
    n = float(np.linalg.norm(v))
    if n < 1e-12:
        raise ValueError("cannot normalize a zero-length vector")
    return v / n


@dataclass(frozen=True)
class Material:
    name: str
    kind: str
    albedo: np.ndarray
    roughness: float | None = None
    ior: float | None = None
    emission: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def is_specular(self):
        return self.kind in ("mirror", "transmission")

    @property
    def is_emitter(self):
        return bool(np.any(self.emission > 0))


@dataclass(frozen=True)
class Camera:
    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    fov: float
    resolution: tuple

    def basis(self):
        """scene.py:70-74: forward, right, cam_up."""
        forward = _normalize(self.look_at - self.position)
        right = _normalize(np.cross(forward, self.up))
        return forward, right, np.cross(right, forward)


@dataclass(frozen=True)
class Sphere:
    center: np.ndarray
    radius: float
    material: str


@dataclass(frozen=True)
class Quad:
    corner: np.ndarray
    edge_u: np.ndarray
    edge_v: np.ndarray
    material: str


@dataclass(frozen=True)
class Mesh:
    vertices: np.ndarray
    triangles: np.ndarray
    material: str


@dataclass(frozen=True)
class PointLight:
    position: np.ndarray
    intensity: np.ndarray


@dataclass(frozen=True)
class Scene:
    camera: Camera
    materials: tuple
    shapes: tuple
    point_lights: tuple
    global_up: np.ndarray
    environment: np.ndarray
    name: str = "scene"

    def material_index(self, name):
        for i, m in enumerate(self.materials):
            if m.name == name:
                return i
        raise SceneValidationError(f"material {name!r} is not declared")


# ---------------------------------------------------------------------------
# parsing (the document format of drc/scene.py; validation rules restated)

def _keys(obj, required, optional, where):
    if not isinstance(obj, dict):
        raise SceneValidationError(f"{where}: expected an object")
    unknown = set(obj) - set(required) - set(optional)
    if unknown:
        raise SceneValidationError(f"{where}: unknown keys {sorted(unknown)}")
    missing = set(required) - set(obj)
    if missing:
        raise SceneValidationError(f"{where}: missing keys {sorted(missing)}")


def _vec(v, where):
    try:
        a = np.asarray(v, dtype=np.float64)
    except (TypeError, ValueError):
        raise SceneValidationError(f"{where}: expected a 3-array of reals")
    if a.shape != (3,):
        raise SceneValidationError(f"{where}: expected a 3-array of reals")
    return a


def _color(v, where, lo=0.0, hi=None):
    c = _vec(v, where)
    if not np.all(np.isfinite(c)):
        raise SceneValidationError(f"{where}: non-finite components")
    if np.any(c < lo) or (hi is not None and np.any(c > hi)):
        raise SceneValidationError(f"{where}: components out of range")
    return c


def _material(name, spec):
    where = f"materials[{name!r}]"
    _keys(spec, ["kind", "albedo"], ["roughness", "ior", "emission"], where)
    kind = spec["kind"]
    if kind not in MATERIAL_KINDS:
        raise SceneValidationError(f"{where}: unknown kind {kind!r}")
    albedo = _color(spec["albedo"], f"{where}.albedo", 0.0, 1.0)
    emission = _color(spec.get("emission", [0, 0, 0]), f"{where}.emission", 0.0)
    if not np.any(emission > 0) and np.any(albedo >= 1.0):
        raise SceneValidationError(f"{where}: non-emitter albedo must be < 1 componentwise")
    rough, ior = spec.get("roughness"), spec.get("ior")
    if kind == "glossy" and (rough is None or not (0.0 < rough <= 1.0)):
        raise SceneValidationError(f"{where}: glossy needs roughness in (0,1]")
    if kind != "glossy" and rough is not None:
        raise SceneValidationError(f"{where}: roughness is glossy-only")
    if kind == "transmission" and (ior is None or not ior > 0):
        raise SceneValidationError(f"{where}: transmission needs ior > 0")
    if kind != "transmission" and ior is not None:
        raise SceneValidationError(f"{where}: ior is transmission-only")
    return Material(name, kind, albedo, rough, ior, emission)


def _shape(i, spec, names):
    where = f"shapes[{i}]"
    if not isinstance(spec, dict) or "type" not in spec:
        raise SceneValidationError(f"{where}: expected an object with a 'type' key")
    t = spec["type"]
    if t == "sphere":
        _keys(spec, ["type", "center", "radius", "material"], [], where)
        r = float(spec["radius"])
        if r <= 0:
            raise SceneValidationError(f"{where}: radius must be > 0")
        s = Sphere(_vec(spec["center"], where), r, spec["material"])
    elif t == "quad":
        _keys(spec, ["type", "corner", "edge_u", "edge_v", "material"], [], where)
        eu, ev = _vec(spec["edge_u"], where), _vec(spec["edge_v"], where)
        if np.linalg.norm(np.cross(eu, ev)) < 1e-12:
            raise SceneValidationError(f"{where}: degenerate quad (parallel edges)")
        s = Quad(_vec(spec["corner"], where), eu, ev, spec["material"])
    elif t == "mesh":
        _keys(spec, ["type", "vertices", "triangles", "material"], [], where)
        v = np.asarray(spec["vertices"], dtype=np.float64)
        tr = np.asarray(spec["triangles"], dtype=np.int64)
        if v.ndim != 2 or v.shape[1] != 3 or tr.ndim != 2 or tr.shape[1] != 3:
            raise SceneValidationError(f"{where}: vertices must be Nx3, triangles Mx3")
        if tr.size and (tr.min() < 0 or tr.max() >= len(v)):
            raise SceneValidationError(f"{where}: triangle index out of range")
        s = Mesh(v, tr, spec["material"])
    else:
        raise SceneValidationError(f"{where}: unknown shape type {t!r}")
    if s.material not in names:
        raise SceneValidationError(f"{where}: material {s.material!r} is not declared")
    return s


def scene_from_doc(doc, name="scene"):
    _keys(doc, ["camera", "materials", "shapes", "point_lights", "global_up"],
          ["environment"], "document")
    cam = doc["camera"]
    _keys(cam, ["position", "look_at", "up", "fov", "resolution"], [], "camera")
    fov = float(cam["fov"])
    if not (0.0 < fov < 180.0):
        raise SceneValidationError(f"camera.fov must be in (0, 180), got {fov}")
    res = cam["resolution"]
    if (not isinstance(res, (list, tuple)) or len(res) != 2
            or any((not isinstance(v, int)) or v < 1 for v in res)):
        raise SceneValidationError("camera.resolution must be two positive integers")
    pos, look = _vec(cam["position"], "camera"), _vec(cam["look_at"], "camera")
    if np.linalg.norm(look - pos) < 1e-12:
        raise SceneValidationError("camera.look_at coincides with camera.position")
    camera = Camera(pos, look, _normalize(_vec(cam["up"], "camera")), fov,
                    (int(res[0]), int(res[1])))
    if not isinstance(doc["materials"], dict) or not doc["materials"]:
        raise SceneValidationError("materials must be a non-empty object")
    mats = tuple(_material(n, s) for n, s in doc["materials"].items())
    names = {m.name for m in mats}
    if not isinstance(doc["shapes"], list):
        raise SceneValidationError("shapes must be an array")
    shapes = tuple(_shape(i, s, names) for i, s in enumerate(doc["shapes"]))
    if not isinstance(doc["point_lights"], list):
        raise SceneValidationError("point_lights must be an array")
    lights = []
    for i, l in enumerate(doc["point_lights"]):
        _keys(l, ["position", "intensity"], [], f"point_lights[{i}]")
        lights.append(PointLight(_vec(l["position"], "light"),
                                 _color(l["intensity"], f"point_lights[{i}].intensity", 0.0)))
    env = _color(doc.get("environment", [0, 0, 0]), "environment", 0.0)
    return Scene(camera, mats, shapes, tuple(lights), _normalize(_vec(doc["global_up"], "up")),
                 env, name)


def parse_scene(text, name="scene"):
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneParseError(f"syntax error at line {e.lineno} column {e.colno}: {e.msg}")
    return scene_from_doc(doc, name)


def load_scene(path):
    with open(path, "r", encoding="utf-8") as f:
        return parse_scene(f.read(), os.path.splitext(os.path.basename(path))[0])


# ---------------------------------------------------------------------------
# device upload

def rotated_up(up):
    """bsdf._rotated_up (bsdf.py:45-53), numpy expressions kept identical."""
    up = np.asarray(up, dtype=np.float64)
    for axis in (np.array([0.0, 1.0, 0.0]), np.array([1.0, 0.0, 0.0])):
        w = axis - (axis @ up) * up
        norm = np.linalg.norm(w)
        if norm > 1e-6:
            return w / norm
    return np.array([0.0, 0.0, 1.0])


def _is_sphere(s):
    return hasattr(s, "radius")


def _is_quad(s):
    return hasattr(s, "edge_u")


def flatten(scene):
    """Scene -> dict of contiguous numpy arrays in global prim-id order
    [spheres | quads | triangles] (geometry.py:52-66)."""
    mat_index = {m.name: i for i, m in enumerate(scene.materials)}
    sc, sr, sm, qc, qu, qv, qm, t0, t1, t2, tm = ([] for _ in range(11))
    for s in scene.shapes:
        mi = mat_index[s.material]
        if _is_sphere(s):
            sc.append(np.asarray(s.center, dtype=np.float64))
            sr.append(float(s.radius))
            sm.append(mi)
        elif _is_quad(s):
            qc.append(np.asarray(s.corner, dtype=np.float64))
            qu.append(np.asarray(s.edge_u, dtype=np.float64))
            qv.append(np.asarray(s.edge_v, dtype=np.float64))
            qm.append(mi)
        else:
            v = np.asarray(s.vertices, dtype=np.float64)
            tr = np.asarray(s.triangles, dtype=np.int64).reshape(-1, 3)
            if len(tr):
                t0.append(v[tr[:, 0]])
                t1.append(v[tr[:, 1]])
                t2.append(v[tr[:, 2]])
                tm.append(np.full(len(tr), mi, dtype=np.int32))

    def a3(lst):
        return np.ascontiguousarray(np.array(lst, dtype=np.float64).reshape(-1, 3))

    def cat3(lst):
        return np.ascontiguousarray(np.concatenate(lst).reshape(-1, 3)) if lst else np.zeros((0, 3))

    mats = scene.materials
    out = {
        "sph_center": a3(sc), "sph_radius": np.array(sr, dtype=np.float64),
        "sph_mat": np.array(sm, dtype=np.int32),
        "quad_corner": a3(qc), "quad_eu": a3(qu), "quad_ev": a3(qv),
        "quad_mat": np.array(qm, dtype=np.int32),
        "tri_v0": cat3(t0), "tri_v1": cat3(t1), "tri_v2": cat3(t2),
        "tri_mat": np.concatenate(tm).astype(np.int32) if tm else np.zeros(0, np.int32),
        "mat_kind": np.array([KIND_CODE[m.kind] for m in mats], dtype=np.int32),
        "mat_albedo": a3([m.albedo for m in mats]),
        "mat_exponent": np.array([(2.0 / (m.roughness * m.roughness) - 2.0)
                                  if m.kind == "glossy" else 0.0 for m in mats]),
        "mat_ior": np.array([m.ior if m.ior else 1.0 for m in mats], dtype=np.float64),
        "mat_emission": a3([m.emission for m in mats]),
        "point_pos": a3([l.position for l in scene.point_lights]),
        "point_intensity": a3([l.intensity for l in scene.point_lights]),
        "global_up": np.asarray(scene.global_up, dtype=np.float64),
        "rotated_up": rotated_up(scene.global_up),
        "environment": np.asarray(scene.environment, dtype=np.float64),
    }
    return out


def camera_struct(camera):
    fwd, right, up = camera.basis()
    cam = _lib.Camera()
    for k in range(3):
        cam.position[k] = float(camera.position[k])
        cam.forward[k] = float(fwd[k])
        cam.right[k] = float(right[k])
        cam.up[k] = float(up[k])
    cam.tan_half = math.tan(math.radians(camera.fov) * 0.5)
    cam.width, cam.height = int(camera.resolution[0]), int(camera.resolution[1])
    return cam


def desc_from_flat(flat):
    d = _lib.SceneDesc()
    d.n_spheres = len(flat["sph_radius"])
    d.n_quads = len(flat["quad_mat"])
    d.n_tris = len(flat["tri_mat"])
    d.n_materials = len(flat["mat_kind"])
    d.n_point_lights = len(flat["point_pos"])
    keep = []
    for name in ("sph_center", "sph_radius", "sph_mat", "quad_corner", "quad_eu", "quad_ev",
                 "quad_mat", "tri_v0", "tri_v1", "tri_v2", "tri_mat", "mat_kind",
                 "mat_albedo", "mat_exponent", "mat_ior", "mat_emission", "point_pos",
                 "point_intensity"):
        arr = np.ascontiguousarray(flat[name])
        keep.append(arr)
        setattr(d, name, arr.ctypes.data_as(C.c_void_p) if arr.size else None)
    for name in ("global_up", "rotated_up", "environment"):
        for k in range(3):
            getattr(d, name)[k] = float(flat[name][k])
    return d, keep


class DeviceScene:
    """A scene resident in HBM: prim tables + BVH (drcb_scene_create).
    Immutable after construction; safe to share across streams."""

    def __init__(self, scene):
        lib = _lib.load()
        self.scene = scene
        self.flat = flatten(scene)
        desc, keep = desc_from_flat(self.flat)
        h = C.c_void_p()
        _lib.check(lib.drcb_scene_create(C.byref(desc), C.byref(h)), "drcb_scene_create")
        del keep
        self.handle = h

    def stats(self):
        out = (C.c_int64 * 8)()
        _lib.call("drcb_scene_stats", self.handle, out)
        keys = ("n_prims", "n_nodes", "n_leaves", "max_depth", "n_lights", "bytes", "n_refs")
        return {k: int(out[i]) for i, k in enumerate(keys)}

    def close(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.drcb_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_CACHE_ATTR = "_drcb_device_scene"


def device_scene(scene):
    """Cached DeviceScene for a scene object (built lazily once, like
    Scene.geometry in scene.py:140-149)."""
    ds = scene.__dict__.get(_CACHE_ATTR) if hasattr(scene, "__dict__") else None
    if ds is None:
        ds = DeviceScene(scene)
        try:
            object.__setattr__(scene, _CACHE_ATTR, ds)
        except Exception:
            pass
    return ds
