"""Edge cases the reference's own tests exercise (pkg/tests/test_cache.py
test_all_rays_escape_yields_background / test_drc_smoke_nonnegative_and_
tile_invariant, pkg/tests/test_geometry.py test_batch_respects_bounds), on the
device path: empty scenes (no cache points at all), the (t_min, t_max]
bound, the direct-pass tile only splitting work, a ragged frame size against
the oracle, and zero-length batches."""

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
