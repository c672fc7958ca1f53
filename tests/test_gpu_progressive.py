"""The progressive control plane of render_drc (drc/cache.py:426-469) on the
device: the host pass loop over drcb_frame_* — per-pass telemetry, mid-run
snapshots and interrupts — against the reference's own run (golden
drc_progressive.npz, tests/golden/make_golden.py:progressive_fixture), and
the reference's invariants: snapshots equal clean runs
(pkg/tests/test_cache.py:246-255), an interrupt finalises the current pass and
equals a clean run of the passes done (pkg/tests/test_cli.py:154-168)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1910_02480_b200 import cnn, render, scenegen  # noqa: E402
from paper_1910_02480_b200.scene import scene_from_doc  # noqa: E402


@pytest.fixture(scope="module")
def prog():
    g = load_golden("drc_progressive.npz")
    return g, scene_from_doc(g["doc"]), cnn.random_network(int(g["k"]), int(g["seed_w"]))


def _cfg(g, **kw):
    c = dict(g["cfg"])
    c.update(kw)
    return render.RenderConfig(**c, precision=64, net_mode="fp32")


def _rel(a, b):
    return np.abs(a - b).max() / max(1e-6, np.abs(b).max())


def test_passes_and_snapshots_match_reference(prog):
    g, sc, net = prog
    img, tel = render.render_drc(sc, _cfg(g), net, snapshots=[int(b) for b in g["snap_budgets"]])
    got = np.array([[p["index"], p["r"], p["tasks"], p["entries"]] for p in tel["passes"]])
    assert np.array_equal(got, g["passes"])
    assert all(p["seconds"] >= 0 for p in tel["passes"])
    assert tel["tasks"] == int(g["tasks"]) and tel["entries"] == int(g["entries"])
    assert _rel(img, g["image"]) <= 1e-4
    assert sorted(tel["snapshots"]) == [int(b) for b in g["snap_budgets"]]
    for b, ref in zip(g["snap_budgets"], g["snaps"]):
        assert _rel(tel["snapshots"][int(b)], ref) <= 1e-4, int(b)


@pytest.mark.parametrize("net_mode,precision", [("fp32", 64), ("fp16", 32)])
def test_snapshots_equal_clean_runs(prog, net_mode, precision):
    g, sc, net = prog
    if net_mode != "fp32":  # the tensor-core engines are built for k = 64
        net = cnn.random_network(64, 2)
    cfg = render.RenderConfig(**g["cfg"], precision=precision, net_mode=net_mode)
    img, tel = render.render_drc(sc, cfg, net, snapshots=[2, 5, 21])
    for b in (2, 5):
        clean, _ = render.render_drc(sc, render.RenderConfig(
            **{**g["cfg"], "passes": None}, indirect_tasks=b, precision=precision,
            net_mode=net_mode), net)
        assert np.array_equal(tel["snapshots"][b], clean), b
    assert np.array_equal(tel["snapshots"][21], img)


def test_interrupt_finalises_the_current_pass(prog):
    g, sc, net = prog
    polls = []

    def interrupt():
        polls.append(1)
        return len(polls) >= 2

    img, tel = render.render_drc(sc, _cfg(g), net, interrupt=interrupt)
    got = np.array([[p["index"], p["r"], p["tasks"], p["entries"]] for p in tel["passes"]])
    assert np.array_equal(got, g["passes_interrupted"])
    assert tel["tasks"] == int(g["tasks_interrupted"])
    assert _rel(img, g["image_interrupted"]) <= 1e-4
    clean, _ = render.render_drc(sc, _cfg(g, passes=2), net)
    assert np.array_equal(img, clean)
    now, tel_now = render.render_drc(sc, _cfg(g), net, interrupt=lambda: True)
    one, _ = render.render_drc(sc, _cfg(g, passes=1), net)
    assert np.array_equal(now, one) and len(tel_now["passes"]) == 1


@pytest.mark.parametrize("net_mode,precision", [("fp32", 64), ("bf16", 32), ("fp16", 32)])
def test_pass_loop_equals_single_submission(prog, net_mode, precision):
    """The per-pass submissions (drcb_frame_*) and the one-call frame
    (drcb_render_drc, the bench path) are the same computation."""
    g, sc, net = prog
    if net_mode != "fp32":  # the tensor-core engines are built for k = 64
        net = cnn.random_network(64, 2)
    cfg = render.RenderConfig(**g["cfg"], precision=precision, net_mode=net_mode)
    a, ta = render.render_drc(sc, cfg, net)
    b, tb = render.render_drc_device(sc, cfg, net)
    assert np.array_equal(a, b.double().cpu().numpy())
    assert ta["entries"] == tb["entries"]


def test_config3_progressive_frame():
    """A bench-size frame (C3 scene, 1024^2) through the pass loop: two passes
    with a snapshot; finite, entries monotone, equal to the one-call frame."""
    sc = scenegen.build_scene("c3")
    cam = scenegen.orbit_cameras(8, (1024, 1024), seed=2)[1]
    import dataclasses

    sc = dataclasses.replace(sc, camera=cam)
    net = cnn.random_network(64, 2)
    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=5, precision=32, net_mode="fp16")
    img, tel = render.render_drc(sc, cfg, net, snapshots=[1])
    ents = [p["entries"] for p in tel["passes"]]
    assert ents == sorted(ents) and len(ents) == 2
    assert np.all(np.isfinite(img)) and img.min() >= 0
    one, _ = render.render_drc_device(sc, cfg, net)
    assert np.array_equal(img, one.double().cpu().numpy())
