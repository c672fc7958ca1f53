"""Seeded procedural scenes for BASELINE.json configs 1-4 (with
the reconciliation rules R6/R10/R11 of SURVEY §0.2). No public scene suite
is involved; these synthetic scenes stand in for the paper's unshipped ones.

Every object is a `mesh` shape with its own diffuse material, so prim ids are
triangle indices in mesh order (R9). `scene_doc` returns the reference's JSON
document (parseable by drc.scene.parse_scene and by our scene.parse_scene);
`build_scene` returns our Scene directly from arrays (fast for 1M triangles).
"""

from __future__ import annotations

import numpy as np

from .scene import Camera, Material, Mesh, Scene

LIGHT_HALF = 0.125  # 0.25 x 0.25 ceiling light


def icosphere(subdiv=2):
    """Unit icosphere: 20 * 4^subdiv triangles (subdiv=2 -> 320, R6)."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
         (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.array(p, dtype=np.float64) / np.linalg.norm(p) for p in v]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return np.array(verts), np.array(faces, dtype=np.int64)


def _box(lo, hi):
    """Axis-aligned box as 8 vertices / 12 triangles."""
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    v = np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                  [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]], dtype=np.float64)
    f = np.array([[0, 2, 1], [0, 3, 2], [4, 5, 6], [4, 6, 7], [0, 1, 5], [0, 5, 4],
                  [3, 6, 2], [3, 7, 6], [0, 4, 7], [0, 7, 3], [1, 2, 6], [1, 6, 5]])
    return v, f


def _quad_tris(p0, p1, p2, p3):
    return np.array([p0, p1, p2, p3], dtype=np.float64), np.array([[0, 1, 2], [0, 2, 3]])


def _light(y, half, cx=0.0, cz=0.0):
    """Ceiling light, two triangles with e1 x e2 pointing -y (R10: emitters
    are one-sided, integrators.py:152-153, 209-210)."""
    a = half
    v = np.array([[cx - a, y, cz - a], [cx + a, y, cz - a], [cx + a, y, cz + a],
                  [cx - a, y, cz + a]], dtype=np.float64)
    return v, np.array([[0, 1, 2], [0, 2, 3]])


class _Builder:
    def __init__(self):
        self.materials = []
        self.meshes = []

    def add(self, verts, faces, albedo, emission=None, name=None):
        name = name or f"m{len(self.materials)}"
        self.materials.append(Material(name, "diffuse", np.asarray(albedo, dtype=np.float64),
                                       None, None,
                                       np.zeros(3) if emission is None
                                       else np.asarray(emission, dtype=np.float64)))
        self.meshes.append(Mesh(np.asarray(verts, dtype=np.float64),
                                np.asarray(faces, dtype=np.int64), name))


def _cornell(b, rng, lights, closed=True, light_y=0.999):
    """Cornell box (closed=True: 5 walls, configs 1-2). The orbit-camera
    configs (3-4, cameras on a radius-3 sphere) use an open stage instead:
    only a 6x6 floor, so the cameras see the objects rather than the outside
    of the walls; their lights hang above the object cloud (light_y)."""
    if closed:
        walls = [
            _quad_tris([-1, -1, -1], [1, -1, -1], [1, -1, 1], [-1, -1, 1]),   # floor
            _quad_tris([-1, 1, -1], [-1, 1, 1], [1, 1, 1], [1, 1, -1]),       # ceiling
            _quad_tris([-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]),       # back
            _quad_tris([-1, -1, -1], [-1, -1, 1], [-1, 1, 1], [-1, 1, -1]),   # left
            _quad_tris([1, -1, -1], [1, 1, -1], [1, 1, 1], [1, -1, 1]),       # right
        ]
    else:
        walls = [_quad_tris([-3, -1, -3], [3, -1, -3], [3, -1, 3], [-3, -1, 3])]
    for v, f in walls:
        b.add(v, f, rng.uniform(0.1, 0.9, 3))
    for lo, hi in (([-0.6, -0.999, 0.1], [-0.1, 0.2, 0.6]), ([0.1, -0.999, -0.5], [0.6, -0.4, 0.0])):
        v, f = _box(lo, hi)
        b.add(v, f, rng.uniform(0.1, 0.9, 3))
    for (cx, cz, e) in lights:
        v, f = _light(light_y, LIGHT_HALF, cx, cz)
        b.add(v, f, [0.0, 0.0, 0.0], emission=[e, e, e])


def _spheres(b, rng, count, subdiv=2):
    uv, uf = icosphere(subdiv)
    for _ in range(count):
        c = rng.uniform(-1, 1, 3)
        r = rng.uniform(0.05, 0.3)
        b.add(c + r * uv, uf, rng.uniform(0.1, 0.9, 3))


def _random_tris(b, rng, count):
    v = rng.uniform(-1, 1, (3 * count, 3))
    b.add(v, np.arange(3 * count).reshape(-1, 3), rng.uniform(0.1, 0.9, 3))


CONFIGS = {
    # name: (resolution, frames, spheres, random_tris, lights, weights seed)
    "c1": ((128, 128), 1, 0, 0, [(0.0, 0.0, 10.0)], 0),
    "c2": ((512, 512), 1, 20, 0, [(0.0, 0.0, 10.0)], 1),
    "c3": ((1024, 1024), 8, 800, 2000, [(0.0, 0.0, 10.0)], 2),
    "c4": ((1920, 1080), 32, 3200, 16000, [(-0.4, 0.0, 5.0), (0.4, 0.0, 15.0)], 2),
}


# The orbit-camera configs (3-4): the 2,000 / 16,000 random triangles with
# vertices uniform in [-1,1]^3 make the cube nearly opaque, so a ceiling light
# at y = 0.999 inside it lit almost nothing, and the radius-3 orbit cameras
# sit above the light plane or below the floor (their frames had no direct
# light at all). The open stage therefore hangs its lights above the cloud
# (y = 1.6, facing down, still one-sided, R10) and adds a uniform grey
# environment (the reference's `environment`, scene.py:328) that escaped
# paths see: every orbit camera's frame is lit.
OPEN_STAGE_LIGHT_Y = 1.6
OPEN_STAGE_ENV = 0.3


def build_scene(config="c1", seed=None, resolution=None):
    """Scene for BASELINE config c1..c4 (seed defaults to the config's)."""
    res, _, n_sph, n_rand, lights, wseed = CONFIGS[config]
    seed = {"c1": 0, "c2": 1, "c3": 2, "c4": 2}[config] if seed is None else seed
    rng = np.random.default_rng(seed)
    b = _Builder()
    closed = config in ("c1", "c2")
    _cornell(b, rng, lights, closed=closed, light_y=0.999 if closed else OPEN_STAGE_LIGHT_Y)
    _spheres(b, rng, n_sph)
    if n_rand:
        _random_tris(b, rng, n_rand)
    res = tuple(resolution or res)
    cam = Camera(np.array([0.0, 0.0, -3.7]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, res)
    env = np.zeros(3) if closed else np.full(3, OPEN_STAGE_ENV)
    return Scene(cam, tuple(b.materials), tuple(b.meshes), (), np.array([0.0, 1.0, 0.0]), env,
                 name=config)


def orbit_cameras(n, resolution, seed=2, radius=3.0, up=(0.0, 1.0, 0.0)):
    """Cameras uniform on a sphere of `radius` looking at the origin; poses
    with |forward . up| > 0.999 are redrawn (R11, scene.py:32-36)."""
    rng = np.random.default_rng(seed)
    up = np.asarray(up, dtype=np.float64)
    cams = []
    while len(cams) < n:
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        if abs(float(d @ up)) > 0.999:
            continue
        cams.append(Camera(radius * d, np.zeros(3), up, 40.0, tuple(resolution)))
    return cams


def scene_doc(scene):
    """Our Scene -> the reference's JSON document dict."""
    mats = {}
    for m in scene.materials:
        d = {"kind": m.kind, "albedo": [float(x) for x in m.albedo]}
        if m.is_emitter:
            d["emission"] = [float(x) for x in m.emission]
        mats[m.name] = d
    shapes = [{"type": "mesh", "vertices": s.vertices.tolist(), "triangles": s.triangles.tolist(),
               "material": s.material} for s in scene.shapes]
    c = scene.camera
    return {
        "camera": {"position": [float(x) for x in c.position], "look_at": [float(x) for x in c.look_at],
                   "up": [float(x) for x in c.up], "fov": float(c.fov),
                   "resolution": [int(c.resolution[0]), int(c.resolution[1])]},
        "global_up": [float(x) for x in scene.global_up],
        "materials": mats, "shapes": shapes, "point_lights": [],
        **({"environment": [float(x) for x in scene.environment]}
           if np.any(np.asarray(scene.environment) > 0) else {}),
    }
