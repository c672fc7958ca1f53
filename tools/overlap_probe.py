"""Can a SIMT kernel (the map-path stacks) and the tensor-core U-Net run
concurrently on one B200? Times each alone and both on two streams.

  python tools/overlap_probe.py [--points 4096] [--maps 4096] [--iters 5]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=4096)
    ap.add_argument("--maps", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_1910_02480_b200 import _lib, cnn, render, scenegen
    from paper_1910_02480_b200.scene import device_scene

    scene = scenegen.build_scene("c3")
    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=1, mis_samples=16, max_path_depth=8,
                              rr_start=5, seed=0, precision=32, net_mode="fp16")
    rng = np.random.default_rng(0)
    n = args.points
    P = np.stack([rng.uniform(-1.5, 1.5, n), np.full(n, 1e-3), rng.uniform(-1.5, 1.5, n)], 1)
    N = np.tile([0.0, 1.0, 0.0], (n, 1))
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
    pos, nrm = dev(P, torch.float32), dev(N, torch.float32)
    keys = dev(np.arange(n, dtype=np.int64) * 7919 + 1, torch.int64)
    stacks = torch.zeros((n, 7, 32, 32), device="cuda")
    s_r = torch.zeros(n, device="cuda")
    s_d = torch.zeros(n, device="cuda")
    frames = torch.zeros((n, 9), device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cs = render._cfg_struct(cfg, 32)
    ds = device_scene(scene)
    net = cnn.device_net(cnn.random_network(64, seed=2))
    x = torch.rand((args.maps, 7, 32, 32), device="cuda")
    y = torch.empty((args.maps, 3, 32, 32), device="cuda")

    def maps():
        _lib.call("drcb_render_stacks", ds.handle, C.byref(cs), _lib.ptr(pos), _lib.ptr(nrm),
                  _lib.ptr(keys), n, _lib.ptr(stacks), _lib.ptr(s_r), _lib.ptr(s_d),
                  _lib.ptr(frames), _lib.ptr(nf), _lib.stream_ptr())

    def unet():
        net.forward_device(x, y, mode="fp16")

    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.iters

    def both():
        cur = torch.cuda.current_stream()
        ev = cur.record_event()
        sa.wait_event(ev)
        sb.wait_event(ev)
        with torch.cuda.stream(sa):
            unet()
        with torch.cuda.stream(sb):
            maps()
        cur.wait_stream(sa)
        cur.wait_stream(sb)

    t_maps, t_net, t_both = timed(maps), timed(unet), timed(both)
    print(json.dumps({"maps_ms": t_maps, "unet_ms": t_net, "both_ms": t_both,
                      "sum_ms": t_maps + t_net, "overlap_ms": t_maps + t_net - t_both,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("DRCB_")}}))


if __name__ == "__main__":
    main()
