"""Benchmark: predicted-radiance DRC frames/s at 1024^2 (BASELINE.json config 3).

One step = one batch of 8 complete DRC frames (G-buffer + direct, cache-point
map path tracing, U-Net, MIS shading, interpolation, composite) over the
258,028-triangle config-3 scene, each frame from its own orbit camera.
BASELINE config 3 shards that 8-frame batch across the ranks with the scene
replicated and no collective (strong scaling: 8 / N frames per rank, one
frame per GPU at N = 8; value = 8 frames x steps / max-over-ranks time);
--weak gives every rank its own 8 frames instead.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

--impl reference times the CPU restatement of the reference path (the C
oracle; the reference itself is pure Python and cannot run whole frames at
this size) on the host cores over a bounded sample and
extrapolates frames/s.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FRAMES_PER_RANK = 8
METRIC = "frames/sec at 1024^2 (DRC frame: G-buffer+direct, map path tracing, U-Net, shade, interp)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--tasks", type=int, default=1)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--net", default=os.environ.get("DRCB_BENCH_NET", "fp16"))
    ap.add_argument("--frames", type=int, default=FRAMES_PER_RANK,
                    help="frames per step (the whole job's; per rank with --weak)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank renders --frames frames per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-points", type=int, default=256,
                    help="cache points of the CPU baseline's sample (~10 s of oracle work)")
    ap.add_argument("--cpu-pixels", type=int, default=65536)
    ap.add_argument("--ref-points", type=int, default=64,
                    help="cache points per --impl reference step (~3 s each)")
    ap.add_argument("--ref-pixels", type=int, default=16384)
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--direct-spp", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager steps instead of CUDA-graph replays")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary c4 (1080p) and tasks=16 frame rates")
    ap.add_argument("--no-train", action="store_true",
                    help="skip the secondary training-step measurement")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        """Spawn the sampler and wait for its first row: nvidia-smi's start-up
        stalls the GPU for ~0.1 s, which must not land in the timed region
        (measured: a 200 ms first step when it did)."""
        self.t_from = None
        if os.environ.get("BENCH_NO_SMI"):  # A/B switch for the sampler's own cost
            self.proc = None
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while len(self.rows) < 2 and time.time() - t0 < 10:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def mark(self):
        """Only rows read after this call count (the timed region)."""
        self.t_from = time.time()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for t, r in self.rows if len(r) >= 8 and (self.t_from is None or t >= self.t_from)]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------

def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def cpu_baseline(scene, cams, cfg, net_host, npts_total, n_pixels, n_points, rank):
    """Oracle (CPU restatement of the reference path) on a bounded sample of
    the same workload; returns per-frame extrapolation."""
    from oracle import oracle as O

    nthreads = os.cpu_count() or 1
    O.set_threads(nthreads)
    from paper_1910_02480_b200 import cnn
    from paper_1910_02480_b200.render import plan_points

    osc = O.OracleScene(scene)
    onet = O.OracleNet(cnn.save_weights(net_host))
    cam = cams[0]
    w, h = cam.resolution
    p0 = (h // 2) * w
    t0 = time.perf_counter()
    geo, _ = O.gbuffer_direct(osc, cam, cfg, p0, p0 + n_pixels)
    t_px = (time.perf_counter() - t0) / n_pixels
    px, py, keys, _, _ = plan_points((w, h), cfg)
    idx = py.astype(np.int64) * w + px
    # G-buffer rows for the sampled cache points (pixel rows outside the
    # sample are filled from a second bounded call on just those pixels)
    sel = np.linspace(0, len(px) - 1, n_points).astype(np.int64)
    pos, nrm, ks, dirs, mats = [], [], [], [], []
    for j in sel:
        g, _ = O.gbuffer_direct(osc, cam, cfg, int(idx[j]), int(idx[j]) + 1)
        q = int(idx[j])
        if g["found"][q]:
            pos.append(g["position"][q]); nrm.append(g["normal"][q]); ks.append(keys[j])
            dirs.append(g["direction"][q]); mats.append(g["mat"][q])
    t1 = time.perf_counter()
    st, s_r, _, frames = O.render_stacks(osc, np.array(pos), np.array(nrm), np.array(ks, np.uint64), cfg)
    pred = onet.forward(st)
    O.shade(osc, pred, s_r, frames, -np.array(dirs), np.array(mats), np.array(ks, np.uint64), cfg)
    t_pt = (time.perf_counter() - t1) / max(1, len(pos))
    frame_s = w * h * t_px + npts_total * t_pt
    return {"value": 1.0 / frame_s, "unit": "frames/s", "cores": nthreads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"oracle on {n_pixels} px (G-buffer+direct) + {len(pos)} cache points "
                      f"(maps+U-Net fp32+shade) of config {cfg_name()} frame 0; frame time "
                      f"extrapolated = {w}x{h}*{t_px*1e6:.1f}us + {npts_total}*{t_pt*1e3:.1f}ms",
            "seconds_per_frame": frame_s}


def cpu_model():
    """The host CPU the baseline ran on (SURVEY §8(d) asks for it)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or platform.machine()


_CFG_NAME = ["c3"]


def cfg_name():
    return _CFG_NAME[0]


def train_throughput(cnn, world=1, batches=(64, 256, 1024), global_batch=4096, steps=5, warmup=2):
    """Secondary figure (BASELINE config 5 is not the metric's config): the
    autoencoder's training step (train-mode BN, L1, Adam, fp32 master
    weights) on synthetic (B,7,32,32) batches, CUDA-event timed on
    device-resident batches. Every rank runs it: with world > 1 the trainer
    gets a libdrcb NCCL communicator (SyncBN statistics + the 7.8M-float
    gradient all-reduce inside the step), the per-rank batch is
    fixed (weak scaling; `global_batch` is split over the ranks: strong) and
    the step time is the max over ranks. The fp32 parity engine is timed on a
    single rank only."""
    import torch
    import torch.distributed as dist

    from paper_1910_02480_b200.dist import attach_nccl
    from paper_1910_02480_b200.trainer import DeviceTrainer

    net = cnn.random_network(64, seed=3)
    out = {"model": "MapAutoencoder k=64 (7,32,32)->(3,32,32)", "unit": "samples/s",
           "world": world, "allreduce": "libdrcb NCCL (grads + SyncBN)" if world > 1 else None}
    # one process: the bf16 step is replayed from a captured CUDA graph
    # (DeviceTrainer.step_graph, bit-identical to the eager step); the eager
    # launch sequence is timed beside it at the smallest batch
    graphs = world == 1
    runs = [("bf16", b, f"bf16_b{b}", graphs) for b in batches]
    if graphs:
        runs.append(("bf16", batches[0], f"bf16_b{batches[0]}_eager", False))
    if global_batch and global_batch % world == 0:
        runs.append(("bf16", global_batch // world, f"bf16_global{global_batch}", graphs))
    if world == 1:
        runs.append(("fp32", batches[0], f"fp32_b{batches[0]}", False))
    out["graph_replay"] = graphs
    trainers = {}
    for mode, b, key, graph in runs:
        if (mode, graph) not in trainers:
            tr = DeviceTrainer(net, lr=1e-4, mode=mode)
            if world > 1:
                attach_nccl(tr)
            trainers[(mode, graph)] = tr
        tr = trainers[(mode, graph)]
        g = torch.Generator(device="cuda").manual_seed(3)
        x = torch.rand((b, 7, 32, 32), device="cuda", generator=g)
        y = torch.rand((b, 3, 32, 32), device="cuda", generator=g)
        step = (lambda: tr.step_graph(x, y)) if graph else (lambda: tr.step(x, y, want_loss=False))
        for _ in range(warmup):
            step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        out[key] = {"samples_per_s": b * world / (ms / 1e3), "ms_per_step": ms,
                    "batch_per_rank": b, "global_batch": b * world}
        if mode == "bf16":
            # forward + dgrad + wgrad = 3x the forward's multiply-adds per sample,
            # against the measured dense bf16 peaks (burst, and sustained: the
            # step runs back to back under the power cap)
            tf = 3 * cnn.flops_per_map(64) * b / (ms * 1e-3) / 1e12
            pk = measured_peaks()[0]
            out[key]["tflops_per_gpu"] = tf
            out[key]["frac_bf16_peak"] = tf / pk["bf16_tflops"]
            if pk.get("bf16_tflops_sustained"):
                out[key]["frac_bf16_peak_sustained"] = tf / pk["bf16_tflops_sustained"]
        del x, y
    for tr in trainers.values():
        comm = getattr(tr, "_comm", None)
        tr.close()
        if comm is not None:
            comm.close()
    return out


class _Sampler:  # the oracle's sampler argument (kind, spp, seed)
    def __init__(self, kind="independent", spp=1, seed=0):
        self.kind, self.spp, self.seed = kind, spp, seed


def next_rows(scene, cam, cpu=True, spp=4, grid=(8, 8), ref_spp=256):
    """SURVEY §8(f) rows beside the headline (rank 0, one GPU): f2 render(mode="pt")
    frames/s at config 3's scene and camera (fp32 rays, `spp` paths per pixel,
    depth 8, RR from 5; CUDA events around drcb_render_pt), and f1 reference-mode
    dataset generation (dataset.generate_examples, `grid` points at `ref_spp`,
    wall clock through the public API). With `cpu`, the oracle's path tracer on
    the host cores over a bounded sample (camera paths; one reference map)."""
    import ctypes as C
    import math

    import torch

    from paper_1910_02480_b200 import _lib, dataset, render
    from paper_1910_02480_b200.scene import device_scene

    out = {}
    w, h = cam.resolution
    rc = render.RenderConfig(spp=spp, max_path_depth=8, rr_start=5, seed=0, precision=32)
    cs = render._cfg_struct(rc, 32)
    cs.direct_spp = spp
    ds = device_scene(scene)
    img = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    camst = render.camera_struct(cam)

    def pt():
        _lib.call("drcb_render_pt", ds.handle, C.byref(camst), C.byref(cs), _lib.ptr(img),
                  _lib.ptr(nf), _lib.stream_ptr())

    pt()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        pt()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    paths = w * h * spp
    out["pt"] = {"what": f"render(mode='pt') {w}x{h}, {spp} spp, depth 8 (f2)", "ms_per_frame": ms,
                 "frames_per_s": 1e3 / ms, "mpaths_per_s": paths / ms / 1e3}
    sc = dataclasses.replace(scene, camera=cam) if dataclasses.is_dataclass(scene) else scene
    dataset.generate_examples(sc, (1, 1), ref_spp, seed=0, precision=32)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ex = dataset.generate_examples(sc, grid, ref_spp, seed=0, precision=32)
    dt = time.perf_counter() - t0
    out["dataset"] = {"what": f"generate_examples grid {grid[0]}x{grid[1]}, ref_spp {ref_spp}, "
                              f"fp32 (f1; through the public API, one read-back per call)",
                      "examples": len(ex), "seconds": dt, "examples_per_s": len(ex) / dt,
                      "mpaths_per_s": len(ex) * 1024 * ref_spp / dt / 1e6}
    if cpu:
        from oracle import oracle as O

        O.set_threads(os.cpu_count() or 1)
        osc = O.OracleScene(scene)
        f, r, u = cam.basis()
        th = math.tan(math.radians(cam.fov) * 0.5)
        n = 8192
        ys = np.full(n, h // 2, dtype=np.int64)
        xs = np.arange(n, dtype=np.int64) % w
        ndc_x = ((xs + 0.5) / w * 2.0 - 1.0) * th * (w / h)
        ndc_y = (1.0 - (ys + 0.5) / h * 2.0) * th
        d = np.asarray(f) + ndc_x[:, None] * np.asarray(r) + ndc_y[:, None] * np.asarray(u)
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        o = np.broadcast_to(np.asarray(cam.position, dtype=np.float64), d.shape)
        t0 = time.perf_counter()
        O.trace_radiance_batch(osc, o, d, (ys * w + xs).astype(np.uint64), np.zeros(n, np.uint64),
                               _Sampler(), 8, False, 5)
        cpu_pps = n / (time.perf_counter() - t0)
        out["pt"]["cpu_oracle"] = {"paths_per_s": cpu_pps, "cores": os.cpu_count() or 1,
                                   "frames_per_s": cpu_pps / paths,
                                   "sample": f"{n} camera paths of the frame's middle rows"}
        out["pt"]["vs_cpu_oracle"] = out["pt"]["frames_per_s"] / (cpu_pps / paths)
        # one reference map (1,024 texels x ref_spp paths) on the oracle
        geo = render.primary_chain_batch(scene, np.asarray(cam.position, np.float64)[None],
                                         d[w // 2][None], precision=64)
        if geo["found"][0]:
            pos, nrm = geo["position"][0], geo["normal"][0]
            tex = np.arange(1024)
            phi = 2 * np.pi * ((tex % 32) + 0.5) / 32
            theta = 0.5 * np.pi * ((tex // 32) + 0.5) / 32
            loc = np.stack([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), np.cos(theta)], 1)
            a = np.array([0.0, 1.0, 0.0]) if abs(nrm[1]) < 0.9 else np.array([1.0, 0.0, 0.0])
            t_ = np.cross(a, nrm)
            t_ /= np.linalg.norm(t_)
            b_ = np.cross(nrm, t_)
            dirs = loc[:, :1] * t_ + loc[:, 1:2] * b_ + loc[:, 2:] * nrm
            k = 64  # a bounded share of the ref_spp paths per texel, scaled below
            oo = np.repeat(pos[None] + 1e-4 * nrm, 1024 * k, 0)
            dd = np.repeat(dirs, k, 0)
            t0 = time.perf_counter()
            O.trace_radiance_batch(osc, oo, dd, np.repeat(tex, k).astype(np.uint64),
                                   np.tile(np.arange(k), 1024).astype(np.uint64),
                                   _Sampler(spp=k), 8, True, 5)
            per_ex = (time.perf_counter() - t0) * ref_spp / k
            out["dataset"]["cpu_oracle"] = {"seconds_per_example": per_ex,
                                            "examples_per_s": 1.0 / per_ex,
                                            "cores": os.cpu_count() or 1,
                                            "sample": f"1024 texels x {k} of {ref_spp} paths of one "
                                                      f"reference map, scaled"}
            out["dataset"]["vs_cpu_oracle"] = out["dataset"]["examples_per_s"] * per_ex
    return out


def secondary_frames(config, tasks, frames, rank, world, steps=2, warmup=1, streams=2):
    """Secondary frames/s figure for another BASELINE configuration (eager
    multi-stream steps, CUDA-event timed, max over ranks, weak scaling: every
    rank renders `frames` frames of its own). c4 = 1920x1080 with the 1.04M-
    triangle scene, two lights and 4 jittered direct samples per pixel; c3
    with tasks=16 = the paper's operating point (65,536 cache points/frame)."""
    import torch
    import torch.distributed as dist

    from paper_1910_02480_b200 import cnn, render, scenegen
    from paper_1910_02480_b200.dist import frame_shard
    from paper_1910_02480_b200.scene import device_scene, flatten

    res, _, _, _, _, wseed = scenegen.CONFIGS[config]
    spp = 4 if config == "c4" else 1
    cfg = render.RenderConfig(direct_spp=spp, indirect_tasks=tasks, mis_samples=16,
                              max_path_depth=8, rr_start=5, seed=0, precision=32, net_mode="bf16")
    scene = scenegen.build_scene(config)
    cams = scenegen.orbit_cameras(frames * world, res, seed=2)
    mine = [cams[i] for i in frame_shard(len(cams), rank, world)]
    net = cnn.random_network(64, seed=wseed)
    t_build = time.perf_counter()
    ds = device_scene(scene)
    t_build = time.perf_counter() - t_build
    plan = render.plan_points(res, cfg)
    w, h = res
    outs = [torch.empty((h, w, 3), dtype=torch.float32, device="cuda") for _ in mine]
    sts = [torch.cuda.Stream() for _ in range(streams)]
    cur = torch.cuda.current_stream()

    def step():
        ev = cur.record_event()
        for s_ in sts:
            s_.wait_event(ev)
        for i, cam in enumerate(mine):
            with torch.cuda.stream(sts[i % streams]):
                render.render_drc_device(scene, cfg, net, camera=cam, out=outs[i], plan=plan,
                                         telemetry=False)
        for s_ in sts:
            cur.wait_stream(s_)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    _, tel = render.render_drc_device(scene, cfg, net, camera=mine[0], out=outs[0], plan=plan)
    st = ds.stats()
    return {"workload": f"{config}: {w}x{h}, {len(mine)} frames/rank/step, indirect_tasks={tasks}, "
                        f"direct_spp={spp}, bf16 U-Net, fp32 rays",
            "frames_per_s": steps * len(mine) * world / (ms / 1e3), "ms_per_frame_per_rank":
            ms / (steps * len(mine)), "cache_points_per_frame": int(len(plan[0])),
            "scene_tris": int(len(flatten(scene)["tri_mat"])), "bvh_refs": st.get("n_refs"),
            "scene_build_s": t_build,
            "stage_ms_per_frame": {k: v / 1e3 for k, v in tel["stage_us"].items()}}


def traversal_traffic():
    """Per-launch memory traffic of the casting kernels from the committed ncu
    capture (profiles/*_traversal_traffic.json), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(REPO, "profiles", "*_traversal_traffic.json")))
    if not files:
        return None
    return json.load(open(files[-1])).get("kernels")


def l2_read_peak(mb=48, iters=100):
    """Measured L2 -> SM read bandwidth (GB/s): libdrcb's probe kernel
    streams an L2-resident buffer (48 MB of the 126 MB L2) with 16-B
    ld.global.cg loads, CUDA-event timed after a warm-up pass; best of 3."""
    import torch

    from paper_1910_02480_b200 import _lib

    buf = torch.ones(mb * (1 << 20) // 4, dtype=torch.int32, device="cuda")
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    nbytes = buf.numel() * 4

    def run(k):
        _lib.call("drcb_l2_read_probe", _lib.ptr(buf), nbytes, k, _lib.ptr(sink), _lib.stream_ptr())

    run(2)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(iters)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def network_modes(cnn, net, n_maps=4096, iters=10):
    """Secondary: one U-Net forward of n_maps through each tensor-core operand
    mode (CUDA-event timed, device-resident input), TFLOP/s against the
    measured dense bf16 peak (fp16 runs at the bf16 tensor rate; tf32 at half
    of it). bf16 = the BASELINE precision; fp16 = the 16-bit mode that meets
    the 1e-2 bar on every BASELINE weight set (tests/test_gpu_tc.py)."""
    import torch

    peaks, _ = measured_peaks()
    dn = cnn.device_net(net)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((n_maps, 7, 32, 32), device="cuda", generator=g)
    x[:, :3] *= 10.0
    y = torch.empty((n_maps, 3, 32, 32), device="cuda")
    out = {}
    for mode, peak in (("bf16", peaks.get("bf16_tflops", 1590.0)),
                       ("fp16", peaks.get("bf16_tflops", 1590.0)),
                       ("tf32", peaks.get("bf16_tflops", 1590.0) / 2)):
        for _ in range(2):
            dn.forward_device(x, y, mode=mode)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            dn.forward_device(x, y, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        tf = n_maps * cnn.flops_per_map(64) / (ms * 1e-3) / 1e12
        out[mode] = {"ms": ms, "tflops": tf, "frac_of_mode_peak": tf / peak, "mode_peak": peak}
    return out


def network_traffic(n_maps):
    """DRAM bytes (read + write) of one U-Net forward over n_maps, scaled from
    the committed ncu capture (profiles/*_network_traffic.json, 4,096 maps);
    None when no capture is committed."""
    import glob

    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                          "profiles", "*_network_traffic.json")))
    if not files:
        return None
    d = json.load(open(files[-1]))
    return int(d["dram_bytes_total"] * n_maps / d["maps"])


def main():
    args = parse()
    _CFG_NAME[0] = args.config
    rank, world, local = dist_env()
    from paper_1910_02480_b200 import cnn, render, scenegen

    res, _, _, _, _, wseed = scenegen.CONFIGS[args.config]
    direct_spp = args.direct_spp or (4 if args.config == "c4" else 1)  # BASELINE config 4: 4 spp
    cfg = render.RenderConfig(direct_spp=direct_spp, indirect_tasks=args.tasks, mis_samples=16,
                              max_path_depth=8, rr_start=5, seed=0, precision=args.precision,
                              net_mode=args.net if args.net in ("fp32", "tf32", "bf16", "fp16") else "fp32")
    workload = {"workload": f"{args.config}: DRC frames {res[0]}x{res[1]}, "
                            f"{args.frames} frames/{'rank/' if args.weak else ''}step, "
                            f"indirect_tasks={args.tasks}, "
                            f"direct_spp={direct_spp}, orbit cameras r=3 (seed 2)",
                "scene_tris": None, "cache_points_per_frame": None,
                "precision": f"rays fp{args.precision}, U-Net {cfg.net_mode}",
                "l2": "flushed between steps (256 MB write)"}
    scene = scenegen.build_scene(args.config)
    from paper_1910_02480_b200.dist import frame_shard

    n_frames = args.frames * max(world, 1) if args.weak else args.frames
    cams = scenegen.orbit_cameras(n_frames, res, seed=2)
    my_cams = [cams[i] for i in frame_shard(len(cams), rank, max(world, 1))]
    scaling = "weak" if args.weak else "strong"
    net = cnn.random_network(64, seed=wseed)
    plan = render.plan_points(res, cfg)
    n_pts = len(plan[0])
    workload["cache_points_per_frame"] = n_pts
    from paper_1910_02480_b200.scene import flatten

    workload["scene_tris"] = int(len(flatten(scene)["tri_mat"]))

    if args.impl == "reference":
        if rank != 0:
            return
        vals, walls = [], []
        cb = None
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            cb = cpu_baseline(scene, cams, cfg, net, n_pts, args.ref_pixels, args.ref_points, rank)
            if i >= args.warmup:
                vals.append(cb["value"])
                walls.append(time.perf_counter() - t0)
        v = float(np.mean(vals))
        cb["value"] = v
        # a step is the bounded sample (wall time on the host cores); the
        # frame rate is that sample's throughput scaled to whole frames
        cb["ms_per_frame_extrapolated"] = 1e3 / v
        line = {"metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * float(np.mean(walls)),
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded procedural scene, SURVEY §8d)", "config": workload,
                "impl": "reference", "cpu_baseline": cb,
                "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1910_02480_b200 import _lib
    from paper_1910_02480_b200.scene import device_scene

    ds = device_scene(scene)
    st = ds.stats()
    dn = cnn.device_net(net)
    dtype = torch.float32 if args.precision == 32 else torch.float64
    w, h = res
    outs = [torch.empty((h, w, 3), dtype=dtype, device="cuda") for _ in my_cams]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # frames alternate over NSTREAMS streams: one frame's path tracing (SIMT
    # units) overlaps another frame's U-Net (tensor cores)
    streams = [torch.cuda.Stream() for _ in range(args.streams)]
    main = torch.cuda.current_stream()

    def frame(i, tel=False):
        return render.render_drc_device(scene, cfg, net, camera=my_cams[i], out=outs[i], plan=plan,
                                        telemetry=tel)

    frame_cpu = []

    def step(tel=False):
        stages = []
        cur = torch.cuda.current_stream()  # the capture stream while a graph is recorded
        ev = cur.record_event()
        for s_ in streams:
            s_.wait_event(ev)
        for i in range(len(my_cams)):
            t0 = time.time()
            with torch.cuda.stream(streams[i % len(streams)]):
                _, t = frame(i, tel)
            if os.environ.get("BENCH_DEBUG"):
                frame_cpu.append(round(1e3 * (time.time() - t0), 1))
            if t:
                stages.append(t["stage_us"])
        for s_ in streams:
            cur.wait_stream(s_)
        return stages

    clocks = ClockSampler(local)
    clocks.start()  # before the warm-up: its start-up stall stays out of the timed region
    # host-side housekeeping before the warm-up: the GPU must not sit idle
    # between the warm-up and the timed steps (an idle gap lets the clocks
    # drop and the first timed step ran up to 0.5 s instead of 80 ms)
    import gc

    gc.collect()
    gc.disable()
    for _ in range(args.warmup):
        step()

    # One step (8 frames, 2 streams, ~1,000 kernels + stream-ordered
    # allocations) captured as a CUDA graph and replayed: the GPU no longer
    # depends on the launching thread keeping ahead of it (a stalled host
    # thread starved the first timed step by up to 0.5 s). Every replay
    # re-executes every kernel of the step.
    graph, per_step_launches = None, None
    if not args.no_graph:
        try:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            la = _lib.load().drcb_kernel_launches()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                step()
            per_step_launches = int(_lib.load().drcb_kernel_launches() - la)
            for _ in range(max(1, args.warmup)):
                g.replay()
            graph = g
        except Exception as e:  # eager steps remain the fallback
            print(f"bench: CUDA graph capture failed ({e!r}); timing eager steps", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()

    def timed_step():
        if graph is not None:
            graph.replay()
        else:
            step()

    # ---- timed region (device-resident inputs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.load().drcb_kernel_launches()
    ev0.record()
    stage_rows = []
    dbg = os.environ.get("BENCH_DEBUG")
    step_ev = []
    cpu_t = []
    for _ in range(args.steps):
        if dbg:
            step_ev.append(torch.cuda.Event(enable_timing=True))
            step_ev[-1].record()
            cpu_t.append(time.time())
        timed_step()
        flush.fill_(1.0)
    ev1.record()
    if dbg:
        cpu_t.append(time.time())
        torch.cuda.synchronize()
        step_ev.append(ev1)
        print("per-step ms", [round(a.elapsed_time(b), 1) for a, b in zip(step_ev, step_ev[1:])],
              "cpu enqueue ms", [round(1e3 * (b - a), 1) for a, b in zip(cpu_t, cpu_t[1:])],
              "frame cpu ms (last 48)", frame_cpu[-48:], file=sys.stderr)
    launches_timed = int(_lib.load().drcb_kernel_launches() - l0)
    if graph is not None:
        launches_timed = per_step_launches * args.steps
    torch.cuda.synchronize()
    gc.enable()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    # stage split from an untimed single-stream pass (CUDA events per stage),
    # after one eager frame (the graph replays used the graph's own memory
    # pool; the first eager frame refills the stream-ordered pool)
    frame(0, False)
    torch.cuda.synchronize()
    sub_rows = []
    for i in range(len(my_cams)):
        _, tl = frame(i, True)
        stage_rows.append(tl["stage_us"])
        sub_rows.append(tl["substage_us"])
    # traversal counters of one frame (untimed; drcb_trav_stats adds atomics)
    trav = None
    try:
        import ctypes as C

        buf = torch.zeros(12, dtype=torch.int64, device="cuda")
        _lib.call("drcb_trav_stats", C.c_void_p(buf.data_ptr()))
        frame(0, False)
        torch.cuda.synchronize()
        _lib.call("drcb_trav_stats", None)
        c = buf.cpu().tolist()
        trav = {"casts_per_frame": c[2], "shadow_casts_per_frame": c[11],
                "nodes_per_cast": c[0] / max(c[2], 1), "prims_per_cast": c[1] / max(c[2], 1)}
    except Exception as e:  # secondary figure
        trav = {"error": repr(e)}
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    frames_total = args.steps * n_frames
    value = frames_total / (ms / 1e3)

    # ---- e2e: public API with host buffers (plan H2D inside the call, image D2H)
    pinned = [torch.empty((h, w, 3), dtype=dtype, pin_memory=True) for _ in my_cams]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ev = main.record_event()
        for s_ in streams:
            s_.wait_event(ev)
        for i in range(len(my_cams)):
            with torch.cuda.stream(streams[i % len(streams)]):
                img, _ = render.render_drc_device(scene, cfg, net, camera=my_cams[i], out=outs[i],
                                                  telemetry=False)
                pinned[i].copy_(img, non_blocking=True)
        for s_ in streams:
            main.wait_stream(s_)
        flush.fill_(1.0)
    e1.record()
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    te = torch.tensor([ems], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = frames_total / (float(te.item()) / 1e3)
    h2d = n_frames * n_pts * (4 + 4 + 8)  # the whole job's plan uploads
    d2h = n_frames * h * w * 3 * (4 if args.precision == 32 else 8)

    # ---- roofline of the dominant stage (live CUDA-event stage times)
    peaks, src = measured_peaks()
    avg = {k: float(np.mean([r[k] for r in stage_rows])) for k in stage_rows[0]}
    dom = max(avg, key=avg.get)
    flop_map = cnn.flops_per_map(64)
    if dom == "network":
        achieved = n_pts * flop_map / (avg["network"] * 1e-6) / 1e12
        peak = peaks.get("bf16_tflops", 1590.0)
        peak_s = peaks.get("bf16_tflops_sustained")
        roof = {"bound": "tensor", "kernel": "U-Net forward (all conv layers)", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                # the stage runs inside a long step: the sustained cuBLAS figure
                # is the rule's other denominator (frac stays on the burst one)
                "peak_sustained": peak_s, "frac_sustained": achieved / peak_s if peak_s else None,
                "traffic": network_traffic(n_pts),
                "algorithmic": f"{flop_map/1e9:.5f} GFLOP/map x {n_pts} maps"}
    else:
        # traversal-bound stages: algorithmic bytes = scene bytes read once
        # per launch lower bound is meaningless; report counted casts instead
        casts = None
        roof = {"bound": "hbm", "kernel": dom, "achieved": None, "peak": peaks.get("hbm_gbs"),
                "unit": "GB/s", "frac": None, "traffic": None}
    roof["peak_source"] = src
    roof["stage_ms_per_frame"] = {k: v / 1e3 for k, v in avg.items()}
    # the elementwise stages against the measured HBM peak (their bound is
    # issue, see "bound"):
    # algorithmic bytes = every distinct tensor read once + written once
    sub = {k: float(np.mean([r[k] for r in sub_rows])) for k in sub_rows[0]}
    rb = 4 if args.precision == 32 else 8
    hbm = peaks.get("hbm_gbs", 6650.0)
    px_bytes = w * h * (2 + 4 * 3 * rb)  # found+escaped, throughput, normal, direct, image
    pt_bytes = n_pts * (3 * 1024 * 4 + 13 * rb + 4 + 8 + 1)  # pred map, s_r, frame, wo, L; mat, key, live
    roof["elementwise"] = {
        "interp_composite": {"bytes_per_frame": px_bytes, "us": sub["interp"],
                             "achieved_gbs": px_bytes / (sub["interp"] * 1e3),
                             "frac_hbm": px_bytes / (sub["interp"] * 1e3) / hbm},
        "shade": {"bytes_per_frame": pt_bytes, "us": sub["shade"],
                  "achieved_gbs": pt_bytes / (sub["shade"] * 1e3),
                  "frac_hbm": pt_bytes / (sub["shade"] * 1e3) / hbm},
        "bound": ("issue, not HBM: per-pixel scans of the nearby cache entries (k_interp, ncu "
                  "72 % issue-active, 26.8 active threads per warp instruction) and per-map CDF "
                  "chains (k_shade, one warp per map, 57 % issue-active); "
                  "profiles/r02_ncu_full_summary.md"),
    }
    if trav and "casts_per_frame" in trav:
        # every cast of a frame is made by the G-buffer/direct and map stages
        tr_ms = (avg["gbuffer_direct"] + avg["maps"]) / 1e3
        trav["mrays_per_s"] = trav["casts_per_frame"] / (tr_ms * 1e-3) / 1e6
        trav["note"] = ("BVH + triangles (76 MB) stay L2/L1-resident: the casting kernels are bound "
                        "by SIMT issue and divergence, not HBM (profiles/*_ncu_full_summary.md)")
        # achieved memory bandwidth of the map-path stage: bytes per launch from
        # the committed full capture (profiles/*_traversal_traffic.json) over the
        # live stage time
        tt = traversal_traffic()
        if tt and "map_paths" in tt:
            mp = tt["map_paths"]
            sec = avg["maps"] * 1e-6
            trav["maps_stage"] = {
                "l2_to_l1_gbs": mp["l2_to_l1_bytes"] / sec / 1e9,
                "l1_to_l2_write_gbs": mp["l1_to_l2_write_bytes"] / sec / 1e9,
                "dram_gbs": (mp["dram_read_bytes"] + mp["dram_write_bytes"]) / sec / 1e9,
                "frac_hbm": (mp["dram_read_bytes"] + mp["dram_write_bytes"]) / sec / 1e9 /
                            peaks.get("hbm_gbs", 6650.0),
                "l1_hit_pct": mp.get("l1_hit_pct"), "l2_hit_pct": mp.get("l2_hit_pct"),
                "source": "bytes per launch: ncu full capture; time: live CUDA events"}
            try:  # the L2 side of the roofline (SIMT-issue-bound, not L2-bound)
                l2 = l2_read_peak()
                ms_ = trav["maps_stage"]
                ms_["l2_read_peak_gbs"] = l2
                ms_["frac_l2_read"] = ms_["l2_to_l1_gbs"] / l2
                ms_["frac_l2_total"] = (ms_["l2_to_l1_gbs"] + ms_["l1_to_l2_write_gbs"]) / l2
                ms_["l2_peak_source"] = "measured live: drcb_l2_read_probe (48 MB, 16-B ld.global.cg)"
            except Exception as e:  # secondary figure
                trav["maps_stage"]["l2_read_peak_error"] = repr(e)

    cb = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(scene, cams, cfg, net, n_pts, args.cpu_pixels, args.cpu_points, rank)
        except Exception as e:  # the baseline must never break the GPU line
            cb = {"value": None, "error": repr(e)}
    launches = launches_timed
    train = None
    if not args.no_train:
        try:
            train = train_throughput(cnn, world=max(world, 1))
        except Exception as e:  # secondary figure; never breaks the GPU line
            train = {"error": repr(e)}
    secondary = {}
    try:
        secondary["network_modes_4096_maps"] = network_modes(cnn, net)
    except Exception as e:  # secondary figure; never breaks the GPU line
        secondary["network_modes_4096_maps"] = {"error": repr(e)}
    if not args.no_secondary:
        if world <= 1:
            try:
                secondary["next_rows_c3"] = next_rows(scene, cams[0], cpu=not args.no_cpu_baseline)
            except Exception as e:  # secondary figure; never breaks the GPU line
                secondary["next_rows_c3"] = {"error": repr(e)}
        for key, c_, tk in (("c4_1080p", "c4", 1), ("c3_tasks16", "c3", 16)):
            try:
                secondary[key] = secondary_frames(c_, tk, 8 if c_ == "c4" else 1, rank,
                                                  max(world, 1))
            except Exception as e:  # secondary figure; never breaks the GPU line
                secondary[key] = {"error": repr(e)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": f"f{args.precision} rays / {cfg.net_mode} U-Net",
            "data": "synthetic (seeded procedural scene + random-init U-Net, SURVEY §8d)",
            "config": workload, "clocks": clk, "roofline": roof, "cpu_baseline": cb,
            "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "scene_stats": st,
            "train": train,
            "traversal": trav,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
