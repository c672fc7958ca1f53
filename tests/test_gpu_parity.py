"""libdrcb (CUDA, sm_100a) against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py). fp64 build: the reference's own
arithmetic, compared at 1e-9 relative; fp32 build: prim ids exact except
documented near-ties, continuous outputs at 1e-4 relative."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1910_02480_b200 import cnn, render  # noqa: E402
from paper_1910_02480_b200.scene import scene_from_doc  # noqa: E402


def _scene(g):
    return scene_from_doc(g["doc"])


def rel_err(a, b, floor=1e-12):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), floor)


def test_intersect_fp64_matches_reference_exactly():
    g = load_golden("geometry_mixed.npz")
    sc = _scene(g)
    r = render.intersect_batch(sc, g["O"], g["D"], precision=64)
    assert np.array_equal(r["hit"], g["hit"])
    assert np.array_equal(r["prim"], g["prim"])
    h = g["hit"]
    assert np.array_equal(r["mat"][h], g["mat"][h])
    assert np.max(rel_err(r["t"][h], g["t"][h])) <= 1e-12
    assert np.allclose(r["position"], g["position"], rtol=1e-12, atol=1e-12)
    assert np.allclose(r["normal"], g["normal"], rtol=1e-12, atol=1e-12)
    s = render.intersect_batch(sc, g["O"], g["D"], t_max=g["tmax"], record=False, precision=64)
    assert np.array_equal(s["hit"], g["shadow_hit"])


def test_intersect_fp32_prims_match_except_near_ties():
    g = load_golden("geometry_mixed.npz")
    sc = _scene(g)
    r = render.intersect_batch(sc, g["O"], g["D"], precision=32)
    mism = np.count_nonzero(r["prim"] != g["prim"])
    assert mism <= max(1, int(1e-3 * len(g["prim"])))
    ok = (r["prim"] == g["prim"]) & g["hit"]
    assert np.max(rel_err(r["t"][ok], g["t"][ok])) < 1e-4


@pytest.mark.parametrize("name", ["frame_c1.npz", "frame_cornell.npz", "frame_glossybox.npz",
                                  "frame_room.npz", "frame_furnace.npz", "frame_glass.npz"])
def test_gbuffer_and_direct_fp64(name):
    g = load_golden(name)
    sc = _scene(g)
    cfg = render.RenderConfig(**g["cfg"], precision=64)
    img, _ = render.render(sc, cfg, "direct")
    assert np.allclose(img, g["direct"], rtol=1e-9, atol=1e-12)
    w, h = sc.camera.resolution
    xs, ys = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    f, r_, u = sc.camera.basis()
    import math
    th = math.tan(math.radians(sc.camera.fov) * 0.5)
    ndc_x = ((xs.ravel() + 0.5) / w * 2.0 - 1.0) * th * (w / h)
    ndc_y = (1.0 - (ys.ravel() + 0.5) / h * 2.0) * th
    d = f + ndc_x[:, None] * r_ + ndc_y[:, None] * u
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    o = np.broadcast_to(sc.camera.position, d.shape)
    geo = render.primary_chain_batch(sc, o, d, precision=64)
    for key in ("found", "escaped", "mat"):
        assert np.array_equal(geo[key], g[key]), key
    for key in ("position", "normal", "throughput", "direction", "t_total"):
        assert np.allclose(geo[key], g[key], rtol=1e-9, atol=1e-12), key


@pytest.mark.parametrize("name", ["frame_c1.npz", "frame_cornell.npz", "frame_glossybox.npz",
                                  "frame_room.npz", "frame_glass.npz"])
def test_stacks_cnn_shade_fp64(name):
    g = load_golden(name)
    sc = _scene(g)
    cfg = render.RenderConfig(**g["cfg"], precision=64)
    pts = g["pts"]
    w = sc.camera.resolution[0]
    idx = pts[:, 1] * w + pts[:, 0]
    stacks, s_r, s_d, frames = render.render_input_stacks(
        sc, g["position"][idx], g["normal"][idx], g["keys"], cfg, precision=64)
    assert np.allclose(s_r, g["s_r"], rtol=1e-9)
    assert np.allclose(s_d, g["s_d"], rtol=1e-9)
    assert np.allclose(frames, g["frames"], rtol=1e-12, atol=1e-12)
    assert np.allclose(stacks, g["stacks"], rtol=1e-6, atol=1e-7)
    net = cnn.random_network(int(g["k"]), int(g["seed_w"])) if name != "frame_room.npz" \
        else cnn.make_blur_network(16)
    pred = cnn.forward_batch(net, g["stacks"], mode="fp32")
    assert np.max(np.abs(pred - g["preds"])) <= 1e-4 * max(1.0, np.abs(g["preds"]).max())
    L = render.shade_indirect_batch(sc, g["preds"], g["s_r"], g["frames"], -g["direction"][idx],
                                    g["mat"][idx], g["keys"], cfg, precision=64)
    assert np.allclose(L, g["shade"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", ["frame_c1.npz", "frame_cornell.npz", "frame_glossybox.npz",
                                  "frame_room.npz", "frame_furnace.npz", "frame_glass.npz"])
def test_render_drc_fp64_image(name):
    g = load_golden(name)
    sc = _scene(g)
    cfg = render.RenderConfig(**g["cfg"], precision=64, net_mode="fp32")
    net = cnn.random_network(int(g["k"]), int(g["seed_w"])) if name != "frame_room.npz" \
        else cnn.make_blur_network(16)
    img, tel = render.render_drc(sc, cfg, net)
    assert tel["entries"] == int(g["entries"])
    assert tel["tasks"] == int(g["tasks"])
    err = np.abs(img - g["image"]).max() / max(1e-6, np.abs(g["image"]).max())
    assert err <= 1e-4, err


def test_trace_and_direct_paths_fp64():
    g = load_golden("trace_c1.npz")
    sc = _scene(g)

    class S:
        kind, seed, spp = "independent", 3, 1

    L0 = render.trace_radiance_batch(sc, g["O"], g["D"], g["pix"], g["smp"], S, 8, False, 5)
    L1 = render.trace_radiance_batch(sc, g["O"], g["D"], g["pix"], g["smp"], S, 8, True, 5)
    assert np.allclose(L0, g["L_full"], rtol=1e-9, atol=1e-12)
    assert np.allclose(L1, g["L_skip"], rtol=1e-9, atol=1e-12)

    class S4:
        kind, seed, spp = "stratified", 5, 4

    Ld = render.li_direct_batch(sc, g["O"], g["D"], g["pix"], g["smp"] % np.uint64(4), S4, True)
    assert np.allclose(Ld, g["L_direct_strat"], rtol=1e-9, atol=1e-12)


def test_cnn_fp32_matches_reference_k8_k64():
    g = load_golden("cnn.npz")
    for k, seed in ((8, 5), (64, 1)):
        net = cnn.random_network(k, seed)
        y = cnn.forward_batch(net, g[f"x_k{k}"], mode="fp32")
        ref = g[f"y_k{k}"]
        assert np.max(np.abs(y - ref)) <= 1e-4 * max(1.0, np.abs(ref).max())
    blur = cnn.make_blur_network(16)
    y = cnn.forward_batch(blur, g["blur_x"], mode="fp32")
    assert np.allclose(y, g["blur_y"], rtol=1e-5, atol=1e-6)


def test_glass_chains_paths_direct_fp64():
    """Transmission: chains, paths and direct estimates through the glass
    sphere of the reference's refraction test scene (plus a lamp) against the
    reference's own batch functions (golden glass_chain.npz)."""
    g = load_golden("glass_chain.npz")
    sc = _scene(g)
    ch = render.primary_chain_batch(sc, g["O"], g["D"], precision=64)
    for k in ("found", "escaped", "mat"):
        assert np.array_equal(ch[k], g[f"chain_{k}"]), k
    for k in ("position", "normal", "throughput", "direction", "t_total"):
        assert np.allclose(ch[k], g[f"chain_{k}"], rtol=1e-9, atol=1e-12), k

    class S:
        kind, seed, spp = "independent", 3, 1

    L = render.trace_radiance_batch(sc, g["O"], g["D"], g["pix"], g["smp"], S, 8, False, 5)
    assert np.allclose(L, g["L"], rtol=1e-9, atol=1e-12)
    Ld = render.li_direct_batch(sc, g["O"], g["D"], g["pix"], g["smp"], S, True)
    assert np.allclose(Ld, g["L_direct"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("precision", [64, 32])
def test_refraction_chain_matches_manual_snell_walk(precision):
    """pkg/tests/test_integrators.py:132-170: a ray entering the unit glass
    sphere above its centre is bent down and lands on the floor (y = -3)
    where an independent step-by-step Snell walk says (atol 1e-3)."""
    g = load_golden("glass_chain.npz")
    sc = _scene(g)
    origin = np.array([0.0, 0.3, -5.0])
    direction = np.array([0.0, 0.0, 1.0])
    res = render.primary_chain_batch(sc, origin[None], direction[None], precision=precision)
    assert res["found"][0]

    def refract(d, n, eta):
        ci = -d @ n
        s2 = eta * eta * (1 - ci * ci)
        if s2 >= 1:
            return d + 2 * ci * n
        return eta * d + (eta * ci - np.sqrt(1 - s2)) * n

    p1 = origin + direction * (5.0 - np.sqrt(1 - 0.09))
    n1 = p1 / np.linalg.norm(p1)
    d1 = refract(direction, n1, 1 / 1.5)
    d1 /= np.linalg.norm(d1)
    p2 = p1 + (-2.0 * (p1 @ d1)) * d1
    n2 = -(p2 / np.linalg.norm(p2))
    d2 = refract(d1, n2, 1.5)
    d2 /= np.linalg.norm(d2)
    target = p2 + ((-3.0 - p2[1]) / d2[1]) * d2
    assert np.allclose(res["position"][0], target, atol=1e-3)
    assert np.all(res["throughput"][0] < 0.95)  # two transmission links (1 - Fresnel) * albedo
