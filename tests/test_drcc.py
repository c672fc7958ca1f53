"""The frame's entry pool (DrcState.entries) and the DRCC cache dump
(cache.py:476-507) against the reference's golden (tests/golden/drcc.npz)."""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_1910_02480_b200 import render
from paper_1910_02480_b200.errors import FormatError


@pytest.fixture(scope="module")
def g():
    return load_golden("drcc.npz")


def test_dump_reader_writer_round_trip(g, tmp_path):
    p = tmp_path / "ref.drcc"
    p.write_bytes(g["drcc"].tobytes())
    ents = render.read_cache_dump(str(p))
    assert [e.pixel for e in ents] == list(zip(g["e_px"].tolist(), g["e_py"].tolist()))
    q = tmp_path / "ours.drcc"
    render.write_cache_dump(ents, str(q))
    assert q.read_bytes() == g["drcc"].tobytes()
    raw = g["drcc"].tobytes()
    for bad, msg in ((b"XXXX" + raw[4:], "bad magic"), (raw[:-3], "truncated"),
                     (raw[:4] + (9).to_bytes(4, "little") + raw[8:], "unsupported DRCC version")):
        p.write_bytes(bad)
        with pytest.raises(FormatError, match=msg):
            render.read_cache_dump(str(p))


@pytest.mark.gpu
def test_entry_pool_and_dump_match_reference(g, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_02480_b200 import cnn, scene as scn

    sc = scn.parse_scene(json.dumps(g["doc"]))
    cfg = render.RenderConfig(direct_spp=2, indirect_tasks=5, mis_samples=16, precision=64)
    _, tel = render.render_drc(sc, cfg, cnn.random_network(8, 0))
    ents = tel["state"].entries()
    assert [e.pixel for e in ents] == list(zip(g["e_px"].tolist(), g["e_py"].tolist()))
    for field, key, tol in (("position", "e_pos", 1e-12), ("normal", "e_normal", 1e-12),
                            ("specular_throughput", "e_thr", 1e-12),
                            ("indirect_radiance", "e_rad", 1e-4)):
        got = np.stack([getattr(e, field) for e in ents])
        ref = g[key]
        assert np.abs(got - ref).max() <= tol * max(1.0, np.abs(ref).max()), field
    p = tmp_path / "ours.drcc"
    render.write_cache_dump(ents, str(p))
    back = render.read_cache_dump(str(p))
    assert len(back) == len(ents)
