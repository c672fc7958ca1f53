"""SURVEY §8f "next" rows on the B200: render(mode="pt") and reference-mode
dataset generation, against the unmodified reference (golden vectors)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1910_02480_b200 import dataset, render  # noqa: E402
from paper_1910_02480_b200.scene import scene_from_doc  # noqa: E402


@pytest.fixture(scope="module")
def g():
    return load_golden("pt_dataset.npz")


def test_pt_mode_fp64_matches_reference(g):
    sc = scene_from_doc(g["doc"])
    cfg = render.RenderConfig(spp=3, max_path_depth=5, rr_start=3, seed=4, precision=64)
    img, tel = render.render(sc, cfg, "pt")
    assert tel["mode"] == "pt"
    assert np.allclose(img, g["pt"], rtol=1e-9, atol=1e-12)


def test_reference_mode_examples_match_reference(g):
    sc = scene_from_doc(g["doc2"])
    cfg = render.RenderConfig(max_path_depth=4, rr_start=3)
    ex = dataset.generate_examples(sc, (2, 2), 256, seed=5, config=cfg)
    assert [e.pixel for e in ex] == [tuple(p) for p in g["ex_pixel"]]
    assert np.allclose([e.s_r for e in ex], g["ex_sr"], rtol=1e-6)
    assert np.allclose([e.s_d for e in ex], g["ex_sd"], rtol=1e-6)
    assert np.allclose(np.stack([e.input for e in ex]), g["ex_input"], rtol=1e-6, atol=1e-7)
    assert np.allclose(np.stack([e.target for e in ex]), g["ex_target"], rtol=1e-6, atol=1e-7)
