"""A/B of render-kernel variants: render frames of a bench config, print the
SHA-256 of every output image (bit-identity across variants) and the maps
stage time from the frame telemetry.

  python tools/maps_ab.py --config c3 --frames 4      # (per build / env variant)
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_1910_02480_b200 import cnn, render, scenegen

    res, _, _, _, _, wseed = scenegen.CONFIGS[args.config]
    cfg = render.RenderConfig(direct_spp=4 if args.config == "c4" else 1, indirect_tasks=1,
                              mis_samples=16, max_path_depth=8, rr_start=5, seed=0,
                              precision=args.precision, net_mode="fp16")
    scene = scenegen.build_scene(args.config)
    cams = scenegen.orbit_cameras(args.frames, res, seed=2)
    net = cnn.random_network(64, seed=wseed)
    plan = render.plan_points(res, cfg)
    hashes, maps, gbuf = [], [], []
    for rep in range(args.reps):
        for i, cam in enumerate(cams):
            img, tel = render.render_drc_device(scene, cfg, net, camera=cam, plan=plan, telemetry=True)
            torch.cuda.synchronize()
            if rep == 0:
                hashes.append(hashlib.sha256(img.cpu().numpy().tobytes()).hexdigest()[:16])
            elif tel and "stage_us" in tel:
                maps.append(tel["stage_us"]["maps"])
                gbuf.append(tel["stage_us"]["gbuffer_direct"])
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("DRCB_")},
                      "maps_ms": sum(maps) / max(len(maps), 1) / 1e3,
                      "gbuffer_direct_ms": sum(gbuf) / max(len(gbuf), 1) / 1e3, "hashes": hashes}))


if __name__ == "__main__":
    main()
