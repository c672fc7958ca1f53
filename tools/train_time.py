"""Time the tensor-core training step (bf16 NHWC engine) with CUDA events,
for A/B runs and ncu launch lists:

  python tools/train_time.py [--batch 4096] [--iters 5] [--mode bf16]
  ncu --metrics gpu__time_duration.sum --csv python tools/train_time.py --iters 1
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--graph", action="store_true", help="replay a captured step graph")
    args = ap.parse_args()
    import torch

    from paper_1910_02480_b200 import cnn
    from paper_1910_02480_b200.trainer import DeviceTrainer

    tr = DeviceTrainer(cnn.random_network(64, seed=3), lr=1e-4, mode=args.mode)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((args.batch, 7, 32, 32), device="cuda", generator=g)
    y = torch.rand((args.batch, 3, 32, 32), device="cuda", generator=g)
    step = (lambda: tr.step_graph(x, y)) if args.graph else (lambda: tr.step(x, y, want_loss=False))
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    tf = args.batch * 3 * cnn.flops_per_map(64) / (ms * 1e-3) / 1e12
    print(json.dumps({"batch": args.batch, "mode": args.mode, "graph": args.graph, "ms": ms,
                      "samples_per_s": args.batch / ms * 1e3, "tflops": tf}))


if __name__ == "__main__":
    main()
