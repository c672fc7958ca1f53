"""libdrcb against the C oracle at BASELINE configuration sizes, plus
size-independent properties (determinism, precision agreement, flip rates).

The oracle (oracle/drc_oracle.c) is itself pinned to the reference's golden
vectors in tests/test_oracle.py."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1910_02480_b200 import cnn, render, scenegen  # noqa: E402


def _rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def c1():
    return scenegen.build_scene("c1")


def test_config1_full_frame_fp64_matches_oracle(c1):
    """BASELINE config 1 (128^2, 36 triangles), 4 indirect tasks, fp32 U-Net
    (k=64, weights seed 0): GPU fp64 build vs the oracle frame."""
    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=4, precision=64, net_mode="fp32")
    net = cnn.random_network(64, 0)
    img, tel = render.render_drc(c1, cfg, net)
    O.set_threads(0)
    osc = O.OracleScene(c1)
    ref, otel = O.render_drc(osc, cfg, O.OracleNet(cnn.save_weights(net)))
    assert tel["entries"] == otel["entries"]
    err = np.abs(img - ref).max() / np.abs(ref).max()
    assert err <= 1e-4, err


def test_config1_gbuffer_direct_bit_level(c1):
    cfg = render.RenderConfig(direct_spp=2, precision=64)
    img, _ = render.render(c1, cfg, "direct")
    osc = O.OracleScene(c1)
    _, direct = O.gbuffer_direct(osc, c1.camera, cfg)
    w, h = c1.camera.resolution
    assert np.allclose(img, direct.reshape(h, w, 3), rtol=1e-9, atol=1e-12)


def _camera_rays_of(cam, px, py):
    from stacks_util import centre_rays

    return centre_rays(cam, px, py)


def _flip_stats(r64, r32):
    diff = r64["prim"] != r32["prim"]
    hit_flip = r64["hit"] != r32["hit"]          # silhouette grazes
    both = r64["hit"] & r32["hit"]
    rel_t = np.zeros(len(diff))
    rel_t[both] = np.abs(r32["t"][both] - r64["t"][both]) / r64["t"][both]
    same_surface = diff & both & (rel_t < 1e-5)  # shared-edge near-ties
    other = diff & ~hit_flip & ~same_surface     # a genuinely different surface
    return diff, both, rel_t, (diff.mean(), hit_flip.mean(), same_surface.mean(), other.mean())


@pytest.mark.parametrize("config", ["c2", "c3"])
def test_fp32_primary_prim_ids_match_fp64_except_near_ties(config):
    """Every primary ray of config 2 (512^2, 6,436 tris) / config 3's first
    camera above the floor (1024^2, 258,028 tris): the fp32 build's primary
    casts (fp32 traversal of the fp64 camera rays; candidates whose fp32
    decision lies within its rounding bound, and near-ties with the nearest
    hit, re-tested in fp64 — render.PREC_MIXED, what the G-buffer kernels do)
    vs the fp64 build. BASELINE bar: hit triangle ids bit-exact except
    near-ties <= 1e-4 of pixels."""
    from stacks_util import camera_for

    sc, cam = camera_for(config)
    w, h = cam.resolution
    px, py = np.meshgrid(np.arange(w), np.arange(h))
    o, d = _camera_rays_of(cam, px.ravel(), py.ravel())
    r64 = render.intersect_batch(sc, o, d, precision=64)
    rmx = render.intersect_batch(sc, o, d, precision=render.PREC_MIXED)
    diff, both, rel_t, stats = _flip_stats(r64, rmx)
    # the plain fp32 build on fp32-rounded rays (map / bounce casts), reported
    _, _, _, plain = _flip_stats(r64, render.intersect_batch(sc, o, d, precision=32))
    print(f"{config}: mixed flips {stats}; plain fp32 flips {plain}")
    assert diff.mean() <= 1e-4, stats
    assert rel_t[both & ~diff].max() < 1e-4, stats


def test_config2_fp32_gbuffer_and_direct_agree_with_fp64():
    sc = scenegen.build_scene("c2")
    cfg64 = render.RenderConfig(direct_spp=1, precision=64)
    cfg32 = render.RenderConfig(direct_spp=1, precision=32)
    d64, _ = render.render(sc, cfg64, "direct")
    d32, _ = render.render(sc, cfg32, "direct")
    # per-pixel 1e-4 relative except pixels whose discrete decisions flipped
    rel = np.abs(d32 - d64) / np.maximum(np.abs(d64), 1e-3)
    flips = (rel > 1e-4).any(axis=2).mean()
    assert flips <= 1e-3, flips
    assert _rel_l2(d32, d64) <= 1e-2


def test_frames_bit_identical_across_runs_and_streams(c1):
    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=2, precision=32, net_mode="bf16")
    net = cnn.random_network(64, 0)
    a, _ = render.render_drc(c1, cfg, net)
    b, _ = render.render_drc(c1, cfg, net)
    assert np.array_equal(a, b)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out, _ = render.render_drc_device(c1, cfg, net)
    s.synchronize()
    assert np.array_equal(out.double().cpu().numpy(), a)


@pytest.mark.parametrize("precision", [32, 64])
def test_fused_gbuffer_direct_bit_identical_to_split_passes(c1, precision, monkeypatch):
    # direct_spp = 1: centre chain + li_direct path in one kernel vs the
    # k_gbuffer / k_direct_samples / k_direct_reduce passes (direct_spp > 1
    # always takes the split passes)
    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=2, precision=precision, net_mode="fp32")
    net = cnn.random_network(64, 0)
    fused, tf = render.render_drc(c1, cfg, net)
    monkeypatch.setenv("DRCB_SPLIT_DIRECT", "1")
    split, ts = render.render_drc(c1, cfg, net)
    assert tf["entries"] == ts["entries"] and tf["nonfinite"] == ts["nonfinite"]
    if precision == 64:  # -fmad=false build: the same operations bit for bit
        assert np.array_equal(fused, split)
    else:  # the fp32 build contracts FMAs per kernel: last-ulp differences only
        rel = np.abs(fused - split) / np.maximum(np.abs(split), 1e-3)
        assert (rel > 1e-4).any(axis=2).mean() <= 1e-3
        assert np.linalg.norm(fused - split) <= 1e-5 * np.linalg.norm(split)


def test_bf16_and_tf32_frames_within_bar(c1):
    """Whole frame with the tensor-core U-Net vs the fp32 engine (config 3's
    bench weights, seed 2): relative L2 of the image."""
    net = cnn.random_network(64, 2)
    base = render.RenderConfig(direct_spp=1, indirect_tasks=4, precision=32)
    ref, _ = render.render_drc(c1, base, net)
    for mode, bar in (("bf16", 1e-2), ("tf32", 2e-3)):
        cfg = render.RenderConfig(direct_spp=1, indirect_tasks=4, precision=32, net_mode=mode)
        img, _ = render.render_drc(c1, cfg, net)
        assert _rel_l2(img, ref) <= bar, (mode, _rel_l2(img, ref))


def test_config3_frame_properties():
    """Config 3 (1024^2, 258k triangles) cannot run on the CPU oracle; check
    size-independent properties: fp32 vs fp64 image agreement, non-negative
    finite output, entry count == found cache points."""
    sc = scenegen.build_scene("c3")
    cam = scenegen.orbit_cameras(8, (1024, 1024), seed=2)[2]
    net = cnn.random_network(64, 2)
    out = {}
    for prec in (32, 64):
        cfg = render.RenderConfig(direct_spp=1, indirect_tasks=1, precision=prec, net_mode="bf16")
        img, tel = render.render_drc_device(sc, cfg, net, camera=cam)
        out[prec] = (img.double().cpu().numpy(), tel)
    a, b = out[32][0], out[64][0]
    assert np.all(np.isfinite(a)) and a.min() >= 0
    assert out[32][1]["entries"] == out[64][1]["entries"] > 0
    assert _rel_l2(a, b) <= 2e-2, _rel_l2(a, b)


def test_frames_from_concurrent_host_threads_bit_identical(c1):
    """Two host threads render on their own streams at once (the C-ABI's
    per-device launch state is shared): same bits as a
    sequential render."""
    import threading

    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=2, precision=32, net_mode="fp16")
    net = cnn.random_network(64, 0)
    ref, _ = render.render_drc(c1, cfg, net)
    out = [None, None]

    def work(i):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            img, _ = render.render_drc_device(c1, cfg, net)
            res = img.double().cpu().numpy()
        s.synchronize()
        out[i] = res

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert np.array_equal(out[0], ref) and np.array_equal(out[1], ref)
