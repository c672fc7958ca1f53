"""Host-side logic and the C-ABI boundary, CPU only (no compute calls)."""

import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

from conftest import REPO, load_golden
from paper_1910_02480_b200 import cnn, render, scenegen
from paper_1910_02480_b200.errors import ConfigError, FormatError, SceneValidationError
from paper_1910_02480_b200.scene import flatten, parse_scene, scene_from_doc


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(REPO, "include", "drcb.h")).read()
    names = set(re.findall(r"\b(drcb_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 15
    lib = ctypes.CDLL(os.path.join(REPO, "paper_1910_02480_b200", "libdrcb.so"))
    for n in sorted(names):
        assert hasattr(lib, n), n
    from paper_1910_02480_b200 import _lib

    assert names == set(_lib.EXPORTED)


def test_random_network_is_bit_identical_to_reference():
    g = load_golden("cnn.npz")
    for k, seed in ((8, 5), (64, 1)):
        raw = cnn.save_weights(cnn.random_network(k, seed))
        assert hashlib.sha256(raw).digest() == bytes(g[f"sha_k{k}"])


def test_drcw_round_trip_and_errors():
    net = cnn.random_network(8, 2)
    raw = cnn.save_weights(net)
    assert cnn.save_weights(cnn.load_weights(raw)) == raw
    with pytest.raises(FormatError):
        cnn.load_weights(raw[:-3])
    with pytest.raises(FormatError):
        cnn.load_weights(b"XXXX" + raw[4:])
    with pytest.raises(FormatError):
        cnn.load_weights(raw + b"\x00")


def test_plan_matches_reference_entry_counts():
    for name in ("frame_c1.npz", "frame_cornell.npz", "frame_room.npz"):
        g = load_golden(name)
        sc = scene_from_doc(g["doc"])
        cfg = render.RenderConfig(**g["cfg"])
        px, py, keys, r, passes = render.plan_points(sc.camera.resolution, cfg)
        w = sc.camera.resolution[0]
        found = g["found"][py.astype(np.int64) * w + px]
        assert int(found.sum()) == int(g["entries"])
        assert sum(p["tasks"] for p in passes) == int(g["tasks"])
        assert np.all(keys >= np.uint64(1 << 40))


def test_flatten_prim_order_and_lights():
    sc = scenegen.build_scene("c1")
    f = flatten(sc)
    assert len(f["tri_mat"]) == 36
    em = f["mat_emission"][f["tri_mat"]].sum(axis=1) > 0
    assert em.sum() == 2 and np.all(np.nonzero(em)[0] == [34, 35])
    # emitters face down (R10)
    n = np.cross(f["tri_v1"] - f["tri_v0"], f["tri_v2"] - f["tri_v0"])
    assert np.all(n[em][:, 1] < 0)


def test_config_sizes_match_survey():
    assert len(flatten(scenegen.build_scene("c2"))["tri_mat"]) == 6436
    # open stage for the orbit-camera configs: floor (2) + boxes (24) + light (2)
    assert len(flatten(scenegen.build_scene("c3"))["tri_mat"]) == 256000 + 2000 + 28


def test_scene_validation():
    doc = scenegen.scene_doc(scenegen.build_scene("c1", resolution=(8, 8)))
    bad = json.loads(json.dumps(doc))
    bad["camera"]["fov"] = 200
    with pytest.raises(SceneValidationError):
        scene_from_doc(bad)
    bad = json.loads(json.dumps(doc))
    bad["shapes"][0]["material"] = "nope"
    with pytest.raises(SceneValidationError):
        scene_from_doc(bad)
    parse_scene(json.dumps(doc))


def test_render_config_validation():
    with pytest.raises(ConfigError):
        render.RenderConfig(r0=12)
    with pytest.raises(ConfigError):
        render.RenderConfig(mis_samples=1)
    with pytest.raises(ConfigError):
        render.RenderConfig(precision=16)
