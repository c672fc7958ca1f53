"""shim.install() over the unmodified reference (importable only in the build
container, where /root/reference exists; skipped elsewhere): the hot-path
surfaces are rebound, uninstall() restores them, and — with no GPU here — a
rebound call raises instead of falling back to the reference's CPU code."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg"
if not os.path.isdir(REF):  # pragma: no cover - the GPU box has no reference checkout
    pytest.skip("reference checkout not present", allow_module_level=True)
for p in (os.path.join(REF, "src"), os.path.join(REF, "trainer", "src")):
    if p not in sys.path:
        sys.path.insert(0, p)

import drc.cache  # noqa: E402
import drc.cnn  # noqa: E402
import drc.integrators  # noqa: E402

from paper_1910_02480_b200 import errors, shim  # noqa: E402

SURFACES = [(drc.cache, "render_drc"), (drc.integrators, "render"), (drc.cnn, "forward")]


def test_install_rebinds_and_uninstall_restores():
    before = [getattr(m, n) for m, n in SURFACES]
    shim.install()
    try:
        after = [getattr(m, n) for m, n in SURFACES]
        assert all(a is not b for a, b in zip(after, before))
        assert all("paper_1910_02480_b200" in a.__module__ for a in after)
        shim.install()  # idempotent: the saved originals stay the reference's
        assert shim._INSTALLED["drc.cnn.forward"] is before[2]
        import drc_trainer.model as model
        assert "paper_1910_02480_b200" in model.forward_reference.__module__
    finally:
        shim.uninstall()
    assert [getattr(m, n) for m, n in SURFACES] == before


def test_rebound_call_never_falls_back_to_cpu():
    net = drc.cnn.random_network(8, 0)
    x = np.zeros((7, 32, 32), np.float32)
    cpu = drc.cnn.forward(net, x)  # the reference itself (CPU)
    assert cpu.shape == (3, 32, 32)
    shim.install()
    try:
        import torch

        if torch.cuda.is_available():  # pragma: no cover - GPU box: the device path runs
            y = drc.cnn.forward(net, x)
            assert np.allclose(y, cpu, atol=1e-4)
        else:
            with pytest.raises((errors.DrcError, RuntimeError)):
                drc.cnn.forward(net, x)
    finally:
        shim.uninstall()
