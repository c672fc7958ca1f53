"""Board power and SM clock while one stage of the frame runs back to back:
the map-path stacks (the cache points of config 3's first frame), the fp16
U-Net forward (4,096 maps) and whole DRC frames. Each
workload runs for ~`--seconds` while nvidia-smi samples power.draw and
clocks.sm every 50 ms; reports mean power, median clock and the energy of one
invocation (mean power x its time). The frame pipeline runs at the board's
power limit: this shows which stage's energy sets the rate.

  python tools/power_probe.py [--seconds 4]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class Sampler:
    def __init__(self, period_ms=50):
        self.rows, self.stop_ev = [], threading.Event()
        self.p = subprocess.Popen(
            ["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
             f"-lms={period_ms}", "-i", "0"], stdout=subprocess.PIPE, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.p.stdout:
            try:
                w, mhz = (float(v) for v in line.strip().split(","))
                self.rows.append((time.time(), w, mhz))
            except ValueError:
                pass

    def window(self, t0, t1):
        r = [x for x in self.rows if t0 <= x[0] <= t1]
        if not r:
            return None, None
        return statistics.mean(x[1] for x in r), statistics.median(x[2] for x in r)

    def close(self):
        self.p.terminate()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    args = ap.parse_args()
    import torch

    from paper_1910_02480_b200 import _lib, cnn, render, scenegen
    from paper_1910_02480_b200.scene import device_scene

    res, _, _, _, _, wseed = scenegen.CONFIGS["c3"]
    scene = scenegen.build_scene("c3")
    cfg = render.RenderConfig(direct_spp=1, indirect_tasks=1, mis_samples=16, max_path_depth=8,
                              rr_start=5, seed=0, precision=32, net_mode="fp16")
    cams = scenegen.orbit_cameras(8, res, seed=2)
    hostnet = cnn.random_network(64, seed=wseed)
    plan = render.plan_points(res, cfg)
    # the map-path stage on points of a real frame: the G-buffer hits of
    # frame 0's planned cache points
    gb, _ = render.gbuffer_direct(scene, cfg, camera=cams[0])
    idx = plan[1].astype(np.int64) * res[0] + plan[0]
    found = gb["found"][idx]
    P = gb["position"][idx][found]
    N = gb["normal"][idx][found]
    n = len(P)
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
    pos, nrm = dev(P, torch.float32), dev(N, torch.float32)
    keys = dev(plan[2][found].view(np.int64), torch.int64)
    stacks = torch.zeros((n, 7, 32, 32), device="cuda")
    s_r = torch.zeros(n, device="cuda")
    s_d = torch.zeros(n, device="cuda")
    frames = torch.zeros((n, 9), device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    cs = render._cfg_struct(cfg, 32)
    ds = device_scene(scene)
    net = cnn.device_net(hostnet)
    x = torch.rand((4096, 7, 32, 32), device="cuda")
    y = torch.empty((4096, 3, 32, 32), device="cuda")
    h, w = res[1], res[0]
    img = torch.empty((h, w, 3), device="cuda")

    def maps():
        _lib.call("drcb_render_stacks", ds.handle, C.byref(cs), _lib.ptr(pos), _lib.ptr(nrm),
                  _lib.ptr(keys), n, _lib.ptr(stacks), _lib.ptr(s_r), _lib.ptr(s_d),
                  _lib.ptr(frames), _lib.ptr(nf), _lib.stream_ptr())

    def unet():
        net.forward_device(x, y, mode="fp16")

    def frame():
        render.render_drc_device(scene, cfg, hostnet, camera=cams[0], out=img, plan=plan,
                                 telemetry=False)

    smp = Sampler()
    time.sleep(0.5)
    out = {"points": n}
    for name, fn in (("map_stacks_4096_points", maps), ("unet_fp16_4096_maps", unet),
                     ("drc_frame_1024", frame)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        k = 0
        while time.time() - t0 < args.seconds:
            for _ in range(4):
                fn()
            k += 4
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.time()
        ms = e0.elapsed_time(e1) / k
        wmean, mhz = smp.window(t0 + 0.5, t1)
        out[name] = {"ms": ms, "watts": wmean, "sm_mhz": mhz,
                     "joules": None if wmean is None else wmean * ms * 1e-3}
        time.sleep(1.0)
    smp.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
