"""The tensor-core training step's backward pass against torch autograd
(fp32, on the GPU) on the SAME forward.

A 16-bit forward makes train-mode-BN gradients chaotic: a 1e-6 relative
perturbation before the bf16 rounding moves per-tensor gradients by ~35 %
(CPU emulation), so per-tensor gradients of any 16-bit
engine cannot be compared with an fp32 reference directly. Here torch's conv
outputs are pinned to the engine's stored bf16 Z (straight-through: values
from the engine, gradients through torch's convs), and torch rounds to bf16
exactly where the engine stores 16-bit tensors (input, weights, activations,
upsampled tensors, and the stored gradients dA / dZ). What remains is every
backward operation of the engine — L1 + head, LeakyReLU/BN backward, dgrad,
wgrad (the tcgen05 kernels), max-pool and upsample backward, the skip sums —
checked per parameter tensor (MapAutoencoder, model.py:20-88; train.py:97-103)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.nn.functional as F  # noqa: E402

from paper_1910_02480_b200 import cnn  # noqa: E402
from paper_1910_02480_b200.trainer import DeviceTrainer  # noqa: E402

LAYERS = [("enc1.conv1", "enc1.bn1", False), ("enc1.conv2", "enc1.bn2", False),
          ("enc2.conv1", "enc2.bn1", False), ("enc2.conv2", "enc2.bn2", False),
          ("enc3.conv1", "enc3.bn1", False), ("enc3.conv2", "enc3.bn2", False),
          ("bott.conv1", "bott.bn1", False), ("bott.conv2", "bott.bn2", False),
          ("dec3.deconv1", "dec3.bn1", True), ("dec3.deconv2", "dec3.bn2", True),
          ("dec2.deconv1", "dec2.bn1", True), ("dec2.deconv2", "dec2.bn2", True),
          ("dec1.deconv1", "dec1.bn1", True), ("dec1.deconv2", "dec1.bn2", True),
          ("head.deconv1", "head.bn1", True), ("head.deconv2", "head.bn2", True)]


def _bf(t):
    return t.to(torch.bfloat16).to(t.dtype)


def _st(t, value):  # forward value `value`, gradient of t
    return t + (value - t).detach()


def _round_grad(t):
    if t.requires_grad:
        t.register_hook(lambda g: _bf(g))
    return t


def test_backward_matches_torch_on_pinned_forward():
    n = 16
    net = cnn.random_network(64, 4)
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 1, (n, 7, 32, 32)).astype(np.float32)
    x[:, :3] *= 3
    y = np.exp(rng.normal(-1, 1, (n, 3, 32, 32))).astype(np.float32)
    tr = DeviceTrainer(net, lr=1e-4, mode="bf16")
    tr.step(x, y, apply=False)
    got = tr.grads()
    cout = [net.tensors[f"{name}.bias"].shape[0] for name, _, _ in LAYERS]
    Z = [tr.debug_z(l)[:n, :, :, :cout[l]].permute(0, 3, 1, 2).contiguous() for l in range(16)]

    def torch_grads(double):
        dt = torch.float64 if double else torch.float32
        P = {}
        for name, bn, _ in LAYERS:
            P[f"{name}.weight"] = torch.tensor(net.tensors[f"{name}.weight"], device="cuda", dtype=dt, requires_grad=True)
            P[f"{name}.bias"] = torch.tensor(net.tensors[f"{name}.bias"], device="cuda", dtype=dt, requires_grad=True)
            P[f"{bn}.weight"] = torch.tensor(net.tensors[f"{bn}.gamma"], device="cuda", dtype=dt, requires_grad=True)
            P[f"{bn}.bias"] = torch.tensor(net.tensors[f"{bn}.beta"], device="cuda", dtype=dt, requires_grad=True)
        for s in ("weight", "bias"):
            P[f"head.conv_out.{s}"] = torch.tensor(net.tensors[f"head.conv_out.{s}"], device="cuda",
                                                    dtype=dt, requires_grad=True)
        slope = float(net.slope)

        def layer(l, a_in):
            name, bn, de = LAYERS[l]
            w = P[f"{name}.weight"]
            zq = (F.conv_transpose2d if de else F.conv2d)(a_in, _st(w, _bf(w)), P[f"{name}.bias"],
                                                            padding=1)
            _round_grad(zq)                       # dZ is stored in bf16
            z = _st(zq, Z[l].to(dt))              # the engine's forward values
            a = F.leaky_relu(F.batch_norm(z, None, None, P[f"{bn}.weight"], P[f"{bn}.bias"],
                                          training=True, eps=1e-5), slope)
            a = _st(a, _bf(a))                    # activations stored in bf16
            return _round_grad(a)                 # dA stored in bf16

        def up(t):
            u = F.interpolate(t, scale_factor=2, mode="bilinear", align_corners=False)
            return _st(u, _bf(u))

        def cat(u, s):
            return _round_grad(torch.cat([u, s], 1))  # the concat gradient buffers are bf16

        def pool(t):
            return _round_grad(F.max_pool2d(t, 2))

        x0 = _bf(torch.from_numpy(x).cuda().to(dt))
        a0 = layer(0, x0)
        s1 = layer(1, a0)
        a2 = layer(2, pool(s1))
        s2 = layer(3, a2)
        a4 = layer(4, pool(s2))
        s3 = layer(5, a4)
        a6 = layer(6, pool(s3))
        a7 = layer(7, a6)
        a8 = layer(8, cat(up(a7), s3))
        a9 = layer(9, a8)
        a10 = layer(10, cat(up(a9), s2))
        a11 = layer(11, a10)
        a12 = layer(12, cat(up(a11), s1))
        a13 = layer(13, a12)
        a14 = layer(14, a13)
        a15 = layer(15, a14)
        # the head's input pinned too: L1's sign(pred - y) is the one chaotic spot
        # left (an ulp of a15 can flip a sign); the LeakyReLU gates are pinned by Z
        A15 = tr.debug_z(16)[:n, :, :, :cout[15]].permute(0, 3, 1, 2).contiguous()
        a15 = _round_grad(_st(a15, A15.to(dt)))
        pred = F.relu(F.conv2d(a15, P["head.conv_out.weight"], P["head.conv_out.bias"]))
        F.l1_loss(pred, torch.from_numpy(y).cuda().to(dt)).backward()


        return {k: v.grad.double().cpu().numpy() for k, v in P.items()}

    ref32, ref64 = torch_grads(False), torch_grads(True)
    worst, errs, spread = 0.0, {}, {}
    for name in ref32:
        g = got[name].astype(np.float64)
        conv_bias = name.endswith(".bias") and ("conv" in name) and "conv_out" not in name
        if conv_bias:
            # the bias in front of train-mode BN has a zero true gradient:
            # both sides hold rounding noise, small against the weights'
            scale = np.abs(got[name.replace(".bias", ".weight")]).max()
            assert np.abs(g).max() <= 1e-2 * scale, name
            continue
        den = max(np.linalg.norm(ref32[name]), 1e-30)
        errs[name] = float(np.linalg.norm(g - ref32[name]) / den)
        spread[name] = float(np.linalg.norm(ref64[name] - ref32[name]) / den)
    ratio = {k: errs[k] / max(spread[k], 2e-3) for k in errs}
    print("pinned forward, per-tensor gradient rel L2 vs torch: median %.2e max %.2e; "
          "torch's own fp32-vs-fp64 spread: median %.2e max %.2e; worst ratio %.2f (%s)" % (
              np.median(list(errs.values())), max(errs.values()), np.median(list(spread.values())),
              max(spread.values()), max(ratio.values()), max(ratio, key=ratio.get)))
    # the engine sits within the spread that torch's own change of arithmetic
    # (fp32 vs fp64, same bf16 storage points) produces: the bf16-stored
    # gradients amplify every last-bit difference through the BN-backward
    # cancellation; a missing or wrong term is an O(1) error
    assert max(ratio.values()) <= 2.0, sorted(ratio.items(), key=lambda kv: -kv[1])[:5]
    assert max(errs.values()) <= 0.1, sorted(errs.items(), key=lambda kv: -kv[1])[:5]


def _torch_model_grads(net, x, y, dt):
    """Plain MapAutoencoder step gradients in torch (train-mode BN, L1)."""
    P = {}
    for name, bn, _ in LAYERS:
        for s_, key in (("weight", f"{name}.weight"), ("bias", f"{name}.bias")):
            P[key] = torch.tensor(net.tensors[key], device="cuda", dtype=dt, requires_grad=True)
        P[f"{bn}.weight"] = torch.tensor(net.tensors[f"{bn}.gamma"], device="cuda", dtype=dt, requires_grad=True)
        P[f"{bn}.bias"] = torch.tensor(net.tensors[f"{bn}.beta"], device="cuda", dtype=dt, requires_grad=True)
    for s_ in ("weight", "bias"):
        P[f"head.conv_out.{s_}"] = torch.tensor(net.tensors[f"head.conv_out.{s_}"], device="cuda", dtype=dt,
                                                 requires_grad=True)
    slope = float(net.slope)

    def layer(l, a):
        name, bn, de = LAYERS[l]
        z = (F.conv_transpose2d if de else F.conv2d)(a, P[f"{name}.weight"], P[f"{name}.bias"], padding=1)
        return F.leaky_relu(F.batch_norm(z, None, None, P[f"{bn}.weight"], P[f"{bn}.bias"], training=True,
                                         eps=1e-5), slope)

    up = lambda t: F.interpolate(t, scale_factor=2, mode="bilinear", align_corners=False)  # noqa: E731
    x0 = torch.from_numpy(x).cuda().to(dt)
    s1 = layer(1, layer(0, x0))
    s2 = layer(3, layer(2, F.max_pool2d(s1, 2)))
    s3 = layer(5, layer(4, F.max_pool2d(s2, 2)))
    b = layer(7, layer(6, F.max_pool2d(s3, 2)))
    d3 = layer(9, layer(8, torch.cat([up(b), s3], 1)))
    d2 = layer(11, layer(10, torch.cat([up(d3), s2], 1)))
    d1 = layer(13, layer(12, torch.cat([up(d2), s1], 1)))
    h = layer(15, layer(14, d1))
    pred = F.relu(F.conv2d(h, P["head.conv_out.weight"], P["head.conv_out.bias"]))
    loss = F.l1_loss(pred, torch.from_numpy(y).cuda().to(dt))
    loss.backward()
    return float(loss), {k: v.grad.double().cpu().numpy() for k, v in P.items()}


def test_fp32_engine_at_k64_b64_within_torchs_own_precision_spread():
    """The fp32 (parity) engine at the BASELINE config-5 parity shape (k = 64,
    batch 64) against torch's own step: a 1e-4 per-tensor bar is below what
    fp32 itself resolves here (torch fp32 vs fp64 differ by ~4e-3 through the
    train-mode BN backward), so the engine must sit within that spread; the
    k = 8 golden (test_gpu_train.py) keeps the 1e-4 bar where it is met."""
    n = 64
    net = cnn.random_network(64, 3)
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (n, 7, 32, 32)).astype(np.float32)
    x[:, :3] *= 4
    y = np.exp(rng.normal(-1, 1, (n, 3, 32, 32))).astype(np.float32)
    tr = DeviceTrainer(net, lr=1e-4)
    loss = tr.step(x, y, apply=False)
    got = tr.grads()
    tf32 = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False  # a true fp32 reference (cuDNN defaults to TF32)
    try:
        l32, g32 = _torch_model_grads(net, x, y, torch.float32)
        l64, g64 = _torch_model_grads(net, x, y, torch.float64)
    finally:
        torch.backends.cudnn.allow_tf32 = tf32
    assert abs(loss - l64) <= 1e-5 * l64
    errs, spread = {}, {}
    for name in g64:
        if name.endswith(".bias") and "conv" in name and "conv_out" not in name:
            continue  # zero true gradient (bias before train-mode BN)
        den = np.linalg.norm(g64[name])
        errs[name] = float(np.linalg.norm(got[name] - g64[name]) / den)
        spread[name] = float(np.linalg.norm(g32[name] - g64[name]) / den)
    print("fp32 engine vs torch fp64: median %.2e max %.2e; torch fp32 vs fp64: median %.2e max %.2e" % (
        np.median(list(errs.values())), max(errs.values()), np.median(list(spread.values())),
        max(spread.values())))
    assert max(errs.values()) <= 2.0 * max(max(spread.values()), 1e-4), \
        sorted(errs.items(), key=lambda kv: -kv[1])[:5]
