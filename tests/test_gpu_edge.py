"""Edge cases the reference's own tests exercise (pkg/tests/test_cache.py
test_all_rays_escape_yields_background / test_drc_smoke_nonnegative_and_
tile_invariant, pkg/tests/test_geometry.py test_batch_respects_bounds), on the
device path: empty scenes (no cache points at all), the (t_min, t_max]
bound, the direct-pass tile only splitting work, a ragged frame size against
the oracle, zero-length batches; and the analytic cases of
pkg/tests/test_integrators.py / test_dataset.py (furnace, no light = exact
zero, point light under a Lambertian floor, unlit dataset = zero targets)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1910_02480_b200 import cnn, render  # noqa: E402
from paper_1910_02480_b200.scene import scene_from_doc  # noqa: E402

MATS = {"matte": {"kind": "diffuse", "albedo": [0.65, 0.6, 0.55]},
        "rust": {"kind": "diffuse", "albedo": [0.5, 0.2, 0.1]},
        "glow": {"kind": "diffuse", "albedo": [0.4, 0.4, 0.4], "emission": [8.0, 7.5, 7.0]}}


def _doc(shapes, res=(16, 16), env=(0.0, 0.0, 0.0), lights=()):
    return {"camera": {"position": [0.0, 1.2, -3.0], "look_at": [0.0, 0.8, 0.5], "up": [0, 1, 0],
                       "fov": 50.0, "resolution": list(res)},
            "materials": MATS, "shapes": list(shapes), "point_lights": list(lights),
            "global_up": [0, 1, 0], "environment": list(env)}


def _room(res):
    """An open box (floor, back and side walls), a ball and a ceiling panel."""
    return scene_from_doc(_doc([
        {"type": "quad", "corner": [-2.5, 0, -1], "edge_u": [5, 0, 0], "edge_v": [0, 0, 4],
         "material": "matte"},
        {"type": "quad", "corner": [-2.5, 0, 3], "edge_u": [5, 0, 0], "edge_v": [0, 2.5, 0],
         "material": "matte"},
        {"type": "quad", "corner": [-2.5, 0, -1], "edge_u": [0, 0, 4], "edge_v": [0, 2.5, 0],
         "material": "rust"},
        {"type": "sphere", "center": [0.5, 0.6, 1.2], "radius": 0.6, "material": "matte"},
        {"type": "mesh", "vertices": [[-1.2, 0, 0.5], [-0.2, 0, 0.9], [-0.8, 1.1, 0.8]],
         "triangles": [[0, 1, 2]], "material": "rust"},
        {"type": "quad", "corner": [-0.5, 2.4, 0.5], "edge_u": [1, 0, 0], "edge_v": [0, 0, 1],
         "material": "glow"},
    ], res=res, env=(0.05, 0.06, 0.08), lights=[{"position": [1.5, 2.0, 0.0],
                                                  "intensity": [2.0, 2.0, 2.0]}]), name="room")


@pytest.mark.parametrize("precision", [64, 32])
def test_all_rays_escape_yields_background(precision):
    """No geometry at all: no cache point survives the plan, the indirect
    layer is the environment times the (unit) throughput, and the direct
    pass adds nothing (background excluded in DRC)."""
    env = (0.3, 0.5, 0.7)
    sc = scene_from_doc(_doc([], env=env), name="empty")
    cfg = render.RenderConfig(indirect_tasks=1, direct_spp=2, precision=precision)
    img, tel = render.render_drc(sc, cfg, cnn.make_blur_network(k=16))
    assert tel["entries"] == 0
    assert np.allclose(img, np.broadcast_to(env, img.shape), rtol=1e-6, atol=0)


@pytest.mark.parametrize("precision", [64, 32])
def test_intersect_bound_is_half_open(precision):
    """t in (t_min, t_max]: a hit exactly at t_max counts, one beyond it does
    not (geometry.py's batch bound)."""
    sc = scene_from_doc(_doc([{"type": "sphere", "center": [0, 0, 0], "radius": 1.0,
                               "material": "matte"}]), name="ball")
    o = np.array([[0.0, 0.0, -5.0]])
    d = np.array([[0.0, 0.0, 1.0]])
    miss = render.intersect_batch(sc, o, d, t_max=3.0, precision=precision)
    hit = render.intersect_batch(sc, o, d, t_max=4.0, precision=precision)
    assert not miss["hit"][0]
    assert hit["hit"][0] and hit["t"][0] == 4.0
    assert np.allclose(hit["normal"][0], [0, 0, -1])


def test_zero_length_batches():
    sc = _room((16, 16))
    empty = np.zeros((0, 3))
    r = render.intersect_batch(sc, empty, empty)
    assert len(r["hit"]) == 0 and len(r["t"]) == 0


def test_direct_tile_only_splits_work():
    """RenderConfig.tile groups the direct pass's per-pixel sample sums; it
    must not change the frame beyond summation rounding."""
    sc = _room((48, 40))
    net = cnn.make_blur_network(k=16)
    base = dict(indirect_tasks=2, direct_spp=3, mis_samples=8, precision=64)
    a, ta = render.render_drc(sc, render.RenderConfig(tile=64, **base), net)
    b, tb = render.render_drc(sc, render.RenderConfig(tile=24, **base), net)
    assert ta["entries"] == tb["entries"] > 0
    assert np.all(np.isfinite(a)) and np.all(a >= 0)
    assert np.allclose(a, b, rtol=0, atol=1e-6 * max(1.0, float(np.abs(a).max())))


def test_ragged_frame_matches_oracle():
    """A frame size that is a multiple of nothing (37 x 23: partial pixel
    blocks, partial buckets, clamped plan grid) against the oracle."""
    sc = _room((37, 23))
    cfg = render.RenderConfig(direct_spp=2, indirect_tasks=3, mis_samples=8, precision=64,
                              net_mode="fp32")
    net = cnn.random_network(16, 3)
    img, tel = render.render_drc(sc, cfg, net)
    O.set_threads(0)
    ref, otel = O.render_drc(O.OracleScene(sc), cfg, O.OracleNet(cnn.save_weights(net)))
    assert img.shape == (23, 37, 3)
    assert tel["entries"] == otel["entries"] > 0
    err = np.abs(img - ref).max() / max(np.abs(ref).max(), 1e-30)
    assert err <= 1e-4, err


class _Sampler:
    def __init__(self, kind="independent", spp=1, seed=0):
        self.kind, self.spp, self.seed = kind, spp, seed


def _ball(env=(0.0, 0.0, 0.0), lights=()):
    doc = _doc([{"type": "sphere", "center": [0, 0, 0], "radius": 1.0, "material": "half"}],
               env=env, lights=lights)
    doc["materials"] = {"half": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5]}}
    return scene_from_doc(doc, name="ball")


def _centre_rays(n):
    o = np.tile([0.0, 0.0, -5.0], (n, 1))
    d = np.tile([0.0, 0.0, 1.0], (n, 1))
    return o, d, np.zeros(n, np.uint64), np.arange(n, dtype=np.uint64)


@pytest.mark.parametrize("precision,tol", [(64, 1e-12), (32, 1e-6)])
def test_furnace_every_path_reflects_the_albedo(precision, tol):
    """A convex Lambertian ball (albedo 0.5) in a unit environment: cosine
    sampling makes every path's throughput exactly the albedo and the bounce
    escapes, so every path (not just the mean) returns 0.5."""
    o, d, pix, smp = _centre_rays(4096)
    L = render.trace_radiance_batch(_ball(env=(1.0, 1.0, 1.0)), o, d, pix, smp, _Sampler(seed=1),
                                    max_depth=4, precision=precision)
    assert np.allclose(L, 0.5, rtol=tol, atol=0)


@pytest.mark.parametrize("precision", [64, 32])
def test_no_lights_no_environment_is_exactly_zero(precision):
    o, d, pix, smp = _centre_rays(1024)
    L = render.trace_radiance_batch(_ball(), o, d, pix, smp, _Sampler(), max_depth=6,
                                    precision=precision)
    assert np.all(L == 0.0)


@pytest.mark.parametrize("precision,tol", [(64, 1e-9), (32, 1e-5)])
def test_direct_point_light_analytic(precision, tol):
    """A Lambertian floor point straight below a point light: L = albedo/pi *
    I / d^2 (the NEE estimate of a delta light is exact)."""
    doc = _doc([{"type": "quad", "corner": [-40, 0, -40], "edge_u": [80, 0, 0],
                 "edge_v": [0, 0, 80], "material": "half"}],
               lights=[{"position": [0.0, 2.5, 0.0], "intensity": [6.0, 5.0, 4.0]}])
    doc["materials"] = {"half": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5]}}
    sc = scene_from_doc(doc, name="floor")
    o = np.array([[0.0, 2.0, -2.0]])
    d = np.array([[0.0, -2.0, 2.0]]) / np.sqrt(8.0)
    L = render.li_direct_batch(sc, o, d, np.zeros(1, np.uint64), np.zeros(1, np.uint64),
                               _Sampler(seed=3), precision=precision)
    want = 0.5 / np.pi * np.array([6.0, 5.0, 4.0]) / 2.5 ** 2
    assert np.allclose(L[0], want, rtol=tol, atol=0)


def test_dataset_of_an_unlit_scene_has_zero_targets():
    from paper_1910_02480_b200 import dataset

    ex = dataset.generate_examples(_room_unlit(), (2, 2), 256, seed=2,
                                   config=render.RenderConfig(max_path_depth=3, rr_start=3))
    assert len(ex) > 0
    for e in ex:
        assert e.target.shape == (3, 32, 32) and np.all(e.target == 0.0)
        assert np.all(e.input[:3] == 0.0)  # radiance channels


def _room_unlit():
    doc = _doc([
        {"type": "quad", "corner": [-2.5, 0, -1], "edge_u": [5, 0, 0], "edge_v": [0, 0, 4],
         "material": "matte"},
        {"type": "sphere", "center": [0.5, 0.6, 1.2], "radius": 0.6, "material": "rust"},
    ], res=(24, 24))
    return scene_from_doc(doc, name="unlit")
