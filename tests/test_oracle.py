"""Pin the C oracle (oracle/drc_oracle.c) against golden vectors produced by
the unmodified reference (tests/golden/make_golden.py). CPU only."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from paper_1910_02480_b200 import cnn
from paper_1910_02480_b200.render import RenderConfig
from paper_1910_02480_b200.scene import scene_from_doc


def _osc(g):
    return O.OracleScene(scene_from_doc(g["doc"]))


def test_intersect_matches_reference_exactly():
    g = load_golden("geometry_mixed.npz")
    osc = _osc(g)
    r = O.intersect_batch(osc, g["O"], g["D"])
    assert np.array_equal(r["hit"], g["hit"])
    assert np.array_equal(r["prim"], g["prim"])
    h = g["hit"]
    assert np.array_equal(r["t"][h], g["t"][h])
    assert np.array_equal(r["mat"][h], g["mat"][h])
    assert np.allclose(r["normal"], g["normal"], rtol=0, atol=1e-15)
    s = O.intersect_batch(osc, g["O"], g["D"], t_max=g["tmax"], record=False)
    assert np.array_equal(s["hit"], g["shadow_hit"])


FRAMES = ["frame_c1.npz", "frame_cornell.npz", "frame_glossybox.npz", "frame_room.npz",
          "frame_furnace.npz", "frame_glass.npz"]


@pytest.mark.parametrize("name", FRAMES)
def test_gbuffer_direct(name):
    g = load_golden(name)
    osc = _osc(g)
    cfg = RenderConfig(**g["cfg"])
    geo, direct = O.gbuffer_direct(osc, osc.scene.camera, cfg)
    for k in ("found", "escaped", "mat"):
        assert np.array_equal(geo[k], g[k]), k
    for k in ("position", "normal", "throughput", "direction", "t_total"):
        assert np.allclose(geo[k], g[k], rtol=1e-9, atol=1e-12), k
    # render(mode="direct") in the golden includes the background; the
    # DRC direct pass does not — only compare where no env is visible
    env = np.any(osc.env > 0)
    if not env:
        w, h = osc.scene.camera.resolution
        assert np.allclose(direct.reshape(h, w, 3), g["direct"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", FRAMES[:4] + ["frame_glass.npz"])
def test_stacks_shade(name):
    g = load_golden(name)
    osc = _osc(g)
    cfg = RenderConfig(**g["cfg"])
    w = osc.scene.camera.resolution[0]
    idx = g["pts"][:, 1] * w + g["pts"][:, 0]
    stacks, s_r, s_d, frames = O.render_stacks(osc, g["position"][idx], g["normal"][idx], g["keys"], cfg)
    assert np.allclose(s_r, g["s_r"], rtol=1e-9)
    assert np.allclose(s_d, g["s_d"], rtol=1e-9)
    assert np.allclose(frames, g["frames"], rtol=1e-12, atol=1e-12)
    assert np.allclose(stacks, g["stacks"], rtol=1e-6, atol=1e-7)
    L = O.shade(osc, g["preds"], g["s_r"], g["frames"], -g["direction"][idx], g["mat"][idx],
                g["keys"], cfg)
    assert np.allclose(L, g["shade"], rtol=1e-9, atol=1e-12)


def test_paths():
    g = load_golden("trace_c1.npz")
    osc = _osc(g)

    class S:
        kind, seed, spp = "independent", 3, 1

    class S4:
        kind, seed, spp = "stratified", 5, 4

    assert np.allclose(O.trace_radiance_batch(osc, g["O"], g["D"], g["pix"], g["smp"], S, 8),
                       g["L_full"], rtol=1e-9, atol=1e-12)
    assert np.allclose(O.trace_radiance_batch(osc, g["O"], g["D"], g["pix"], g["smp"], S, 8, True),
                       g["L_skip"], rtol=1e-9, atol=1e-12)
    assert np.allclose(O.li_direct_batch(osc, g["O"], g["D"], g["pix"], g["smp"] % np.uint64(4), S4),
                       g["L_direct_strat"], rtol=1e-9, atol=1e-12)
    ch = O.primary_chain_batch(osc, g["O"], g["D"])
    assert np.array_equal(ch["found"], g["chain_found"])
    assert np.allclose(ch["position"], g["chain_position"], rtol=1e-12, atol=1e-12)


def test_cnn_k8_and_blur():
    g = load_golden("cnn.npz")
    net = cnn.random_network(8, 5)
    y = O.OracleNet(cnn.save_weights(net)).forward(g["x_k8"])
    assert np.max(np.abs(y - g["y_k8"])) <= 1e-4 * max(1.0, np.abs(g["y_k8"]).max())
    y = O.OracleNet(cnn.save_weights(cnn.make_blur_network(16))).forward(g["blur_x"])
    assert np.allclose(y, g["blur_y"], rtol=1e-5, atol=1e-6)


def test_glass_chains_paths_direct():
    """Transmission (dielectric) rays through the reference's refraction-test
    lens scene (pkg/tests/test_integrators.py:132-170, plus a lamp)."""
    g = load_golden("glass_chain.npz")
    osc = _osc(g)

    class S:
        kind, seed, spp = "independent", 3, 1

    ch = O.primary_chain_batch(osc, g["O"], g["D"])
    for k in ("found", "escaped", "mat"):
        assert np.array_equal(ch[k], g[f"chain_{k}"]), k
    for k in ("position", "normal", "throughput", "direction", "t_total"):
        assert np.allclose(ch[k], g[f"chain_{k}"], rtol=1e-9, atol=1e-12), k
    assert np.allclose(O.trace_radiance_batch(osc, g["O"], g["D"], g["pix"], g["smp"], S, 8),
                       g["L"], rtol=1e-9, atol=1e-12)
    assert np.allclose(O.li_direct_batch(osc, g["O"], g["D"], g["pix"], g["smp"], S),
                       g["L_direct"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", ["frame_c1.npz", "frame_cornell.npz", "frame_furnace.npz",
                                  "frame_glass.npz"])
def test_render_drc_frame(name):
    g = load_golden(name)
    osc = _osc(g)
    cfg = RenderConfig(**g["cfg"])
    net = cnn.random_network(int(g["k"]), int(g["seed_w"]))
    img, tel = O.render_drc(osc, cfg, O.OracleNet(cnn.save_weights(net)))
    assert tel["entries"] == int(g["entries"])
    err = np.abs(img - g["image"]).max() / max(1e-6, np.abs(g["image"]).max())
    assert err <= 1e-4, err
