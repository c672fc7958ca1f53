"""The training step's weight gradient on the tensor cores (k_wgrad:
MN-major UMMA operands read straight from NHWC activations, tap shifts by
TMA coordinates, deterministic split-K) against an fp64 restatement of
dW[co][ci][ky][kx] = sum_p dz[p][co] * x[p + (ky-1, kx-1)][ci] on the same
bf16-rounded operands, for every layer shape of MapAutoencoder k = 64."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1910_02480_b200 import _lib  # noqa: E402


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _wgrad_ref(x, dz):
    n, hw, _, cin = x.shape
    xp = np.zeros((n, hw + 2, hw + 2, cin))
    xp[:, 1:-1, 1:-1] = x
    dw = np.zeros((dz.shape[-1], cin, 3, 3))
    for ky in range(3):
        for kx in range(3):
            dw[:, :, ky, kx] = np.einsum("nyxo,nyxc->oc", dz, xp[:, ky:ky + hw, kx:kx + hw])
    return dw


@pytest.mark.parametrize("shape", [(64, 64, 32, 2), (8, 64, 32, 2), (64, 128, 16, 2),
                                   (128, 128, 16, 2), (128, 256, 8, 4), (256, 256, 8, 2),
                                   (256, 512, 4, 8), (512, 512, 4, 8), (768, 256, 8, 2),
                                   (384, 128, 16, 2), (192, 64, 32, 2), (64, 32, 32, 2),
                                   (32, 16, 32, 2), (64, 16, 16, 2), (128, 32, 16, 2)])
def test_wgrad_matches_fp64(shape):
    cin, cout, hw, n = shape
    rng = np.random.default_rng(sum(shape))
    x = rng.normal(size=(n, hw, hw, cin)).astype(np.float32)
    dz = rng.normal(size=(n, hw, hw, cout)).astype(np.float32)
    dw = np.zeros((cout, cin, 3, 3), np.float32)
    _lib.call("drcb_debug_wgrad", cin, cout, hw, n, x.ctypes.data_as(C.c_void_p),
              dz.ctypes.data_as(C.c_void_p), dw.ctypes.data_as(C.c_void_p))
    ref = _wgrad_ref(_bf16(x).astype(np.float64), _bf16(dz).astype(np.float64))
    err = np.abs(dw - ref).max() / np.abs(ref).max()
    assert err <= 2e-5, err


def test_wgrad_deterministic():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(8, 32, 32, 64)).astype(np.float32)
    dz = rng.normal(size=(8, 32, 32, 64)).astype(np.float32)
    outs = []
    for _ in range(2):
        dw = np.zeros((64, 64, 3, 3), np.float32)
        _lib.call("drcb_debug_wgrad", 64, 64, 32, 8, x.ctypes.data_as(C.c_void_p),
                  dz.ctypes.data_as(C.c_void_p), dw.ctypes.data_as(C.c_void_p))
        outs.append(dw)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("shape", [(64, 64, 32, 2), (192, 64, 32, 2), (64, 128, 16, 2)])
def test_wgrad_box_per_tap_variant_agrees(shape, monkeypatch):
    """The 32x32 / 16x16 layers run the dx-in-N variant (one X box with the dy
    shift as a row offset, three dx-shifted dZ boxes, N = 192);
    DRCB_WGRAD_TAPS forces one X box per tap."""
    cin, cout, hw, n = shape
    rng = np.random.default_rng(7)
    x = rng.normal(size=(n, hw, hw, cin)).astype(np.float32)
    dz = rng.normal(size=(n, hw, hw, cout)).astype(np.float32)
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("DRCB_WGRAD_TAPS", env)
        dw = np.zeros((cout, cin, 3, 3), np.float32)
        _lib.call("drcb_debug_wgrad", cin, cout, hw, n, x.ctypes.data_as(C.c_void_p),
                  dz.ctypes.data_as(C.c_void_p), dw.ctypes.data_as(C.c_void_p))
        out.append(dw)
    assert np.abs(out[0] - out[1]).max() <= 1e-5 * np.abs(out[1]).max()
