"""Time one tensor-core U-Net forward (bf16, 4,096 maps by default) with CUDA
events, for A/B runs of the DRCB_* switches and for ncu launch
lists of the per-layer kernels:

  python tools/net_time.py [--maps 4096] [--iters 20] [--mode bf16]
  DRCB_NO_FUSED_POOL=1 python tools/net_time.py
  ncu --metrics gpu__time_duration.sum --csv python tools/net_time.py --iters 1
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--maps", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--mode", default="fp16")
    args = ap.parse_args()
    import torch

    from paper_1910_02480_b200 import cnn

    net = cnn.random_network(64, seed=2)
    dn = cnn.device_net(net)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((args.maps, 7, 32, 32), device="cuda", generator=g)
    y = torch.empty((args.maps, 3, 32, 32), device="cuda")
    for _ in range(3):
        dn.forward_device(x, y, mode=args.mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        dn.forward_device(x, y, mode=args.mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    tf = args.maps * cnn.flops_per_map(64) / (ms * 1e-3) / 1e12
    env = {k: v for k, v in os.environ.items() if k.startswith("DRCB_")}
    print(json.dumps({"maps": args.maps, "mode": args.mode, "ms": ms, "tflops": tf,
                      "checksum": float(y.double().sum()), "env": env}))


if __name__ == "__main__":
    main()
