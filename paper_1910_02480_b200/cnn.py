"""The map-upgrading autoencoder behind the reference's `drc.cnn` surface.

Weights travel in the reference's DRCW container (cnn.py:221-281); the
forward pass runs on the B200 through libdrcb (drcb_net_forward):

  mode "fp32"  SIMT fp32 engine, parity with cnn.forward within 1e-4;
  mode "tf32"  tcgen05 kind::tf32 implicit-GEMM engine;
  mode "bf16"  tcgen05 kind::f16 (bf16 operands, fp32 accumulate) engine.

`forward(net, x)` keeps the reference signature: (7,32,32) -> (3,32,32)
float32. `forward_batch` takes (N,7,32,32) numpy or CUDA tensors.
"""

from __future__ import annotations

import ctypes as C
import io
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import FormatError

DRCW_MAGIC = b"DRCW"
DRCW_VERSION = 1
DEFAULT_LEAKY_SLOPE = 0.01
BN_EPS = 1e-5
IN_CHANNELS = 7
OUT_CHANNELS = 3
MODES = {"fp32": 0, "tf32": 1, "bf16": 2, "fp16": 3}


def architecture(k):
    """Tensor table {name: shape} for base width k, in the reference's
    insertion order (cnn.py:39-78; random_network draws in this order)."""
    if k < 4 or k % 4 != 0:
        raise FormatError(f"base width must be a positive multiple of 4, got {k}")
    table = {}

    def conv(name, cin, cout, ks=3):
        table[f"{name}.weight"] = (cout, cin, ks, ks)
        table[f"{name}.bias"] = (cout,)

    def deconv(name, cin, cout):
        table[f"{name}.weight"] = (cin, cout, 3, 3)
        table[f"{name}.bias"] = (cout,)

    def bn(name, c):
        for t in ("gamma", "beta", "running_mean", "running_var"):
            table[f"{name}.{t}"] = (c,)

    for i, (cin, cout) in enumerate([(IN_CHANNELS, k), (k, 2 * k), (2 * k, 4 * k)], start=1):
        conv(f"enc{i}.conv1", cin, cout)
        bn(f"enc{i}.bn1", cout)
        conv(f"enc{i}.conv2", cout, cout)
        bn(f"enc{i}.bn2", cout)
    conv("bott.conv1", 4 * k, 8 * k)
    bn("bott.bn1", 8 * k)
    conv("bott.conv2", 8 * k, 8 * k)
    bn("bott.bn2", 8 * k)
    for i, (up, out) in zip((3, 2, 1), [(8 * k, 4 * k), (4 * k, 2 * k), (2 * k, k)]):
        deconv(f"dec{i}.deconv1", up + out, out)
        bn(f"dec{i}.bn1", out)
        deconv(f"dec{i}.deconv2", out, out)
        bn(f"dec{i}.bn2", out)
    deconv("head.deconv1", k, k // 2)
    bn("head.bn1", k // 2)
    deconv("head.deconv2", k // 2, k // 4)
    bn("head.bn2", k // 4)
    conv("head.conv_out", k // 4, OUT_CHANNELS, ks=1)
    return table


def flops_per_map(k=64):
    """Multiply-add FLOPs of one 32x32 forward (2*M*N*K per conv layer)."""
    total = 0
    hw = {"enc1": 32, "enc2": 16, "enc3": 8, "bott": 4, "dec3": 8, "dec2": 16, "dec1": 32,
          "head": 32}
    for name, shape in architecture(k).items():
        if not name.endswith(".weight"):
            continue
        s = hw[name.split(".")[0]]
        if "deconv" in name:
            cin, cout, kh, kw = shape
        else:
            cout, cin, kh, kw = shape
        total += 2 * s * s * cout * cin * kh * kw
    return total


@dataclass
class Network:
    tensors: dict
    k: int
    slope: float = DEFAULT_LEAKY_SLOPE
    version: int = DRCW_VERSION

    def __post_init__(self):
        expected = architecture(self.k)
        missing = set(expected) - set(self.tensors)
        if missing:
            raise FormatError(f"missing tensor {sorted(missing)[0]!r}")
        extra = set(self.tensors) - set(expected)
        if extra:
            raise FormatError(f"unexpected tensor {sorted(extra)[0]!r}")
        for name, shape in expected.items():
            if tuple(self.tensors[name].shape) != shape:
                raise FormatError(f"shape mismatch for {name!r}: expected {shape}, "
                                  f"got {tuple(self.tensors[name].shape)}")


def save_weights(net, path=None):
    buf = io.BytesIO()
    buf.write(DRCW_MAGIC)
    buf.write(struct.pack("<II", net.version, struct.unpack("<I", struct.pack("<f", net.slope))[0]))
    names = sorted(net.tensors)
    buf.write(struct.pack("<I", len(names)))
    for name in names:
        data = np.ascontiguousarray(net.tensors[name], dtype="<f4")
        enc = name.encode("utf-8")
        buf.write(struct.pack("<H", len(enc)) + enc + struct.pack("<B", data.ndim))
        buf.write(struct.pack(f"<{data.ndim}I", *data.shape))
        buf.write(data.tobytes())
    raw = buf.getvalue()
    if path is None:
        return raw
    with open(path, "wb") as f:
        f.write(raw)
    return None


def load_weights(src):
    """DRCW bytes or path -> Network (host-side parse; the device handle is
    built lazily by DeviceNet, which re-validates in C++)."""
    raw = src
    if isinstance(src, str):
        with open(src, "rb") as f:
            raw = f.read()
    mv = memoryview(raw)
    off = 0

    def take(n, what):
        nonlocal off
        if off + n > len(mv):
            raise FormatError(f"truncated while reading {what}", offset=len(mv))
        b = bytes(mv[off:off + n])
        off += n
        return b

    if take(4, "magic") != DRCW_MAGIC:
        raise FormatError("bad magic, not a DRCW file", offset=0)
    version, slope_bits = struct.unpack("<II", take(8, "header"))
    if version != DRCW_VERSION:
        raise FormatError(f"unsupported DRCW version {version}", offset=4)
    slope = struct.unpack("<f", struct.pack("<I", slope_bits))[0]
    (count,) = struct.unpack("<I", take(4, "tensor count"))
    tensors = {}
    for _ in range(count):
        (nlen,) = struct.unpack("<H", take(2, "name length"))
        name = take(nlen, "tensor name").decode("utf-8")
        (rank,) = struct.unpack("<B", take(1, "rank"))
        dims = struct.unpack(f"<{rank}I", take(4 * rank, f"{name} dims"))
        n = int(np.prod(dims)) if rank else 1
        tensors[name] = np.frombuffer(take(4 * n, f"{name} data"), dtype="<f4").reshape(dims).astype(np.float32)
    if off != len(mv):
        raise FormatError("trailing bytes after last tensor", offset=off)
    if "enc1.conv1.weight" not in tensors:
        raise FormatError("missing tensor 'enc1.conv1.weight'")
    k = int(tensors["enc1.conv1.weight"].shape[0])
    return Network(tensors=tensors, k=k, slope=float(slope), version=version)


def zero_network(k=64, slope=DEFAULT_LEAKY_SLOPE):
    tensors = {}
    for name, shape in architecture(k).items():
        fill = 1.0 if name.endswith(("gamma", "running_var")) else 0.0
        tensors[name] = np.full(shape, fill, dtype=np.float32)
    return Network(tensors=tensors, k=k, slope=slope)


def random_network(k=64, seed=0, slope=DEFAULT_LEAKY_SLOPE):
    """He-normal weights + random BN statistics, drawn in architecture order
    from numpy default_rng(seed) exactly as cnn.py:300-319 specifies."""
    rng = np.random.default_rng(seed)
    tensors = {}
    for name, shape in architecture(k).items():
        if name.endswith("gamma"):
            t = rng.uniform(0.8, 1.2, shape)
        elif name.endswith("beta"):
            t = rng.normal(0.0, 0.05, shape)
        elif name.endswith("running_mean"):
            t = rng.normal(0.0, 0.1, shape)
        elif name.endswith("running_var"):
            t = rng.uniform(0.5, 1.5, shape)
        elif name.endswith("bias"):
            t = rng.normal(0.0, 0.02, shape)
        else:
            t = rng.normal(0.0, np.sqrt(2.0 / int(np.prod(shape[1:]))), shape)
        tensors[name] = t.astype(np.float32)
    return Network(tensors=tensors, k=k, slope=slope)


def make_blur_network(k=16, slope=DEFAULT_LEAKY_SLOPE):
    """Deterministic stub network (cnn.py:322-346): prediction = the input
    radiance smoothed by two stacked 3x3 Gaussian taps."""
    if k < 12:
        raise FormatError("blur network needs k >= 12 (head width k//4 >= 3)")
    net = zero_network(k, slope)
    t = net.tensors
    g1 = np.exp(-0.5 * np.arange(-1, 2) ** 2)
    g1 /= g1.sum()
    g3 = np.outer(g1, g1).astype(np.float32)
    for c in range(3):
        t["enc1.conv1.weight"][c, c, 1, 1] = 1.0
        t["enc1.conv2.weight"][c, c, 1, 1] = 1.0
        t["dec1.deconv1.weight"][2 * k + c, c, 1, 1] = 1.0
        t["dec1.deconv2.weight"][c, c] = g3
        t["head.deconv1.weight"][c, c, 1, 1] = 1.0
        t["head.deconv2.weight"][c, c] = g3
        t["head.conv_out.weight"][c, c, 0, 0] = 1.0
    return net


class DeviceNet:
    """A Network resident in HBM (drcb_net_create): conv-form fp32 weights,
    folded batch norm and packed tensor-core operands."""

    def __init__(self, net_or_bytes):
        lib = _lib.load()
        raw = net_or_bytes if isinstance(net_or_bytes, (bytes, bytearray)) else save_weights(net_or_bytes)
        h = C.c_void_p()
        _lib.check(lib.drcb_net_create(bytes(raw), len(raw), C.byref(h)), "drcb_net_create")
        self.handle = h
        info = (C.c_int64 * 4)()
        _lib.call("drcb_net_info", h, info)
        self.k = int(info[0])
        self.n_params = int(info[1])

    def forward_device(self, x, y=None, mode="fp32"):
        """x: CUDA float32 tensor (N,7,32,32) -> (N,3,32,32) CUDA tensor."""
        import torch

        if x.dtype != torch.float32 or not x.is_cuda or x.dim() != 4 or tuple(x.shape[1:]) != (7, 32, 32):
            raise FormatError(f"forward expects a CUDA float32 (N,7,32,32) tensor, got {tuple(x.shape)}")
        x = x.contiguous()
        if y is None:
            y = torch.empty((x.shape[0], 3, 32, 32), dtype=torch.float32, device=x.device)
        _lib.call("drcb_net_forward", self.handle, _lib.ptr(x), _lib.ptr(y), int(x.shape[0]),
                  MODES[mode], _lib.stream_ptr())
        return y

    def close(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.drcb_net_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_net(net):
    dn = getattr(net, "_drcb_device_net", None)
    if dn is None:
        dn = DeviceNet(net)
        try:
            object.__setattr__(net, "_drcb_device_net", dn)
        except Exception:
            pass
    return dn


def forward_batch(net, x, mode="fp32"):
    """(N,7,32,32) float32 numpy -> (N,3,32,32) float32 numpy, on the GPU."""
    import torch

    x = np.asarray(x, dtype=np.float32)
    if x.ndim != 4 or x.shape[1:] != (IN_CHANNELS, 32, 32):
        raise FormatError(f"forward_batch expects (N,7,32,32) input, got {x.shape}")
    dn = device_net(net)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    y = dn.forward_device(xd, mode=mode)
    return y.cpu().numpy()


def forward(net, x, mode="fp32"):
    """Map stack (7,32,32) -> predicted radiance (3,32,32), nonnegative
    (the drc.cnn.forward contract, cnn.py:193-198)."""
    x = np.asarray(x, dtype=np.float32)
    if x.shape != (IN_CHANNELS, 32, 32):
        raise FormatError(f"forward expects (7,32,32) input, got {x.shape}")
    return forward_batch(net, x[None], mode=mode)[0]
