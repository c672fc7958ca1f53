"""Generate golden vectors by running the UNMODIFIED reference
(/root/reference/pkg, imported read-only via sys.path) in the build container.

The GPU box has no reference checkout, so the outputs are committed as small
.npz fixtures next to this script; tests/ compare libdrcb and the C oracle
against them. Re-run with:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "trainer", "src"))
sys.path.insert(0, REPO)

from drc import cnn as rcnn  # noqa: E402
from drc import geometry as rgeo  # noqa: E402
from drc import hemimap as rhemi  # noqa: E402
from drc import integrators as rint  # noqa: E402
from drc.cache import DrcState, plan_pass, render_drc  # noqa: E402
from drc.integrators import RenderConfig  # noqa: E402
from drc.sampler import Sampler  # noqa: E402
from drc.scene import parse_scene  # noqa: E402

from paper_1910_02480_b200 import scenegen  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path)} bytes")


def doc_array(doc):
    return np.frombuffer(json.dumps(doc).encode("utf-8"), dtype=np.uint8)


def ref_scene_doc(name, res):
    with open(os.path.join(REF, "scenes", f"{name}.json")) as f:
        doc = json.load(f)
    doc["camera"]["resolution"] = [res, res]
    return doc


def random_shape_doc(rng, n_spheres, n_quads, n_tris):
    # the shape mix of tests/test_geometry.py:39-57
    shapes = []
    for _ in range(n_spheres):
        shapes.append({"type": "sphere", "center": list(rng.uniform(-5, 5, 3)),
                       "radius": float(rng.uniform(0.1, 1.2)), "material": "gray"})
    for _ in range(n_quads):
        shapes.append({"type": "quad", "corner": list(rng.uniform(-5, 5, 3)),
                       "edge_u": list(rng.uniform(-2, 2, 3)), "edge_v": list(rng.uniform(-2, 2, 3)),
                       "material": "gray"})
    verts = rng.uniform(-5, 5, (3 * n_tris, 3))
    shapes.append({"type": "mesh", "vertices": verts.tolist(),
                   "triangles": np.arange(3 * n_tris).reshape(-1, 3).tolist(), "material": "gray"})
    return {"camera": {"position": [0, 0, -5], "look_at": [0, 0, 0], "up": [0, 1, 0], "fov": 40.0,
                       "resolution": [64, 64]},
            "global_up": [0, 1, 0],
            "materials": {"gray": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5]},
                          "lamp": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5],
                                   "emission": [4.0, 4.0, 4.0]}},
            "shapes": shapes, "point_lights": []}


def geometry_fixture():
    rng = np.random.default_rng(2024)
    doc = random_shape_doc(rng, 40, 40, 20)
    # make a few prims emissive so light tables are exercised
    doc["shapes"][3]["material"] = "lamp"
    doc["shapes"][45]["material"] = "lamp"
    scene = parse_scene(json.dumps(doc))
    n = 4000
    O = rng.uniform(-8, 8, (n, 3))
    D = rng.normal(size=(n, 3))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    r = rgeo.intersect_batch(scene.geometry, O, D)
    tmax = rng.uniform(0.5, 12.0, n)
    s = rgeo.intersect_batch(scene.geometry, O, D, t_max=tmax, record=False)
    save("geometry_mixed.npz", doc=doc_array(doc), O=O, D=D, hit=r["hit"], t=r["t"],
         prim=r["prim"], mat=r["mat"], position=r["position"], normal=r["normal"], tmax=tmax,
         shadow_hit=s["hit"])


def frame_fixture(name, doc, k, seed_w, cfg_kw, n_points=6, net=None):
    """Stage-level and whole-frame outputs of one small scene."""
    scene = parse_scene(json.dumps(doc))
    cfg = RenderConfig(threads=1, **cfg_kw)
    w, h = scene.camera.resolution
    state = DrcState(scene, cfg)
    geo = state.geo
    direct, _ = rint.render(scene, cfg, "direct")
    if net is None:
        net = rcnn.random_network(k, seed_w)
    # cache points: the first pass-0 grid points that are found
    plan = plan_pass((w, h), 0, cfg.r0, jitter_seed=cfg.seed)
    xs, ys = plan.task_points(0)
    gx, gy = np.meshgrid(xs, ys)
    pts = [(x, y) for x, y in zip(gx.ravel(), gy.ravel()) if geo["found"][y * w + x]][:n_points]
    keys = [(1 << 40) + y * w + x for x, y in pts]
    hits = []
    for x, y in pts:
        i = y * w + x
        hits.append(rgeo.Hit(position=geo["position"][i], normal=geo["normal"][i],
                             distance=float(geo["t_total"][i]), material_id=int(geo["mat"][i]),
                             is_emitter=False, emitted=np.zeros(3)))
    msampler = Sampler(cfg.sampler_kind, cfg.seed, 1)
    stacks = rhemi.render_input_stacks_batch(scene, hits, msampler, cfg, keys) if hits else []
    st = np.stack([s.as_tensor() for s in stacks]) if stacks else np.zeros((0, 7, 32, 32), np.float32)
    preds = np.stack([rcnn.forward(net, s) for s in st]) if stacks else np.zeros((0, 3, 32, 32), np.float32)
    shade = []
    for (x, y), hit, stk, key, pred in zip(pts, hits, stacks, keys, preds):
        i = y * w + x
        radmap = rhemi.HemiMap(np.moveaxis(pred, 0, -1), stk.radiance.frame, scale=stk.s_r)
        shade.append(rint.shade_indirect(scene, hit, radmap, stk.radiance.frame,
                                         -geo["direction"][i], msampler, cfg.mis_samples, key=key))
    frames = np.stack([np.stack([s.radiance.frame.t, s.radiance.frame.b, s.radiance.frame.n])
                       for s in stacks]) if stacks else np.zeros((0, 3, 3))
    img, tel = render_drc(scene, cfg, net)
    out = dict(doc=doc_array(doc), k=k, seed_w=seed_w, cfg=doc_array(cfg_kw),
               found=geo["found"], escaped=geo["escaped"], position=geo["position"],
               normal=geo["normal"], mat=geo["mat"], throughput=geo["throughput"],
               direction=geo["direction"], t_total=geo["t_total"], direct=direct,
               pts=np.array(pts, dtype=np.int64).reshape(-1, 2),
               keys=np.array(keys, dtype=np.uint64), stacks=st,
               s_r=np.array([s.s_r for s in stacks]), s_d=np.array([s.s_d for s in stacks]),
               frames=frames, preds=preds, shade=np.array(shade).reshape(-1, 3), image=img,
               entries=tel["entries"], tasks=tel["tasks"])
    save(name, **out)


def trace_fixture():
    scene = scenegen.build_scene("c1", resolution=(32, 32))
    doc = scenegen.scene_doc(scene)
    rscene = parse_scene(json.dumps(doc))
    rng = np.random.default_rng(7)
    n = 1024
    O = rng.uniform(-0.9, 0.9, (n, 3))
    D = rng.normal(size=(n, 3))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    pix = rng.integers(0, 1 << 40, n).astype(np.uint64)
    smp = rng.integers(0, 1024, n).astype(np.uint64)
    s = Sampler("independent", 3, 1)
    L0 = rint.trace_radiance_batch(rscene, O, D, pix, smp, s, 8, skip_first_emission=False, rr_start=5)
    L1 = rint.trace_radiance_batch(rscene, O, D, pix, smp, s, 8, skip_first_emission=True, rr_start=5)
    s4 = Sampler("stratified", 5, 4)
    Ld = rint.li_direct_batch(rscene, O, D, pix, smp % np.uint64(4), s4, include_background=True)
    ch = rint.primary_chain_batch(rscene, O, D)
    save("trace_c1.npz", doc=doc_array(doc), O=O, D=D, pix=pix, smp=smp, L_full=L0, L_skip=L1,
         L_direct_strat=Ld, chain_found=ch["found"], chain_position=ch["position"])


def cnn_fixture():
    rng = np.random.default_rng(11)
    out = {}
    for k, seed, n in ((8, 5, 4), (64, 1, 2)):
        net = rcnn.random_network(k, seed)
        raw = rcnn.save_weights(net)
        x = rng.uniform(0, 1, (n, 7, 32, 32)).astype(np.float32)
        x[:, :3] *= rng.uniform(0.5, 20.0)  # radiance channels span a wide range
        y = np.stack([rcnn.forward(net, xi) for xi in x])
        out[f"x_k{k}"] = x
        out[f"y_k{k}"] = y
        out[f"sha_k{k}"] = np.frombuffer(hashlib.sha256(raw).digest(), dtype=np.uint8)
    # hand-checkable primitives (test_cnn.py KAT style)
    xb = rng.normal(size=(3, 8, 8)).astype(np.float32)
    out["up_in"] = xb
    out["up_out"] = rcnn.upsample_bilinear2x2(xb)
    blur = rcnn.make_blur_network(16)
    xs = rng.uniform(0, 1, (2, 7, 32, 32)).astype(np.float32)
    out["blur_x"] = xs
    out["blur_y"] = np.stack([rcnn.forward(blur, v) for v in xs])
    save("cnn.npz", **out)


def glass_fixtures():
    """Transmission (dielectric) materials: the reference's cornell box with
    two glass spheres as a whole frame, and the lens scene of the reference's
    refraction test (pkg/tests/test_integrators.py:132-170) with a lamp, for
    chains / paths / direct estimates through glass (bsdf.py:198-215, 257-319;
    integrators.py:427-518)."""
    doc = ref_scene_doc("cornell", 32)
    doc["materials"]["glass"] = {"kind": "transmission", "albedo": [0.95, 0.95, 0.95], "ior": 1.5}
    doc["materials"]["tint"] = {"kind": "transmission", "albedo": [0.9, 0.7, 0.5], "ior": 1.33}
    doc["shapes"].append({"type": "sphere", "center": [1.9, 1.2, 2.2], "radius": 1.0,
                          "material": "glass"})
    doc["shapes"].append({"type": "sphere", "center": [3.9, 0.8, 1.5], "radius": 0.7,
                          "material": "tint"})
    frame_fixture("frame_glass.npz", doc, 8, 6, dict(direct_spp=2, indirect_tasks=2, mis_samples=8),
                  n_points=8)
    lens = {"camera": {"position": [0, 0, -5], "look_at": [0, 0, 0], "up": [0, 1, 0], "fov": 40.0,
                       "resolution": [16, 16]},
            "global_up": [0, 1, 0],
            "materials": {"glass": {"kind": "transmission", "albedo": [0.95, 0.95, 0.95], "ior": 1.5},
                          "gray": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5]},
                          "lamp": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5],
                                   "emission": [6.0, 6.0, 6.0]}},
            "shapes": [{"type": "sphere", "center": [0, 0, 0], "radius": 1.0, "material": "glass"},
                       {"type": "quad", "corner": [-50, -3, -50], "edge_u": [100, 0, 0],
                        "edge_v": [0, 0, 100], "material": "gray"},
                       {"type": "quad", "corner": [-1, 4, -1], "edge_u": [2, 0, 0],
                        "edge_v": [0, 0, 2], "material": "lamp"}],
            "point_lights": []}
    rscene = parse_scene(json.dumps(lens))
    rng = np.random.default_rng(17)
    n = 2048
    gx, gy = np.meshgrid(np.linspace(-0.95, 0.95, 32), np.linspace(-0.95, 0.95, 32))
    O = np.concatenate([np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, -5.0)], axis=1),
                        rng.uniform(-2.5, 2.5, (n - gx.size, 3)) + np.array([0, 0, -4.0])])
    D = np.concatenate([np.tile([0.0, 0.0, 1.0], (gx.size, 1)),
                        rng.normal(size=(n - gx.size, 3)) * 0.3 + np.array([0, 0, 1.0])])
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    pix = rng.integers(0, 1 << 40, n).astype(np.uint64)
    smp = rng.integers(0, 1024, n).astype(np.uint64)
    ch = rint.primary_chain_batch(rscene, O, D)
    s = Sampler("independent", 3, 1)
    L = rint.trace_radiance_batch(rscene, O, D, pix, smp, s, 8, skip_first_emission=False, rr_start=5)
    Ld = rint.li_direct_batch(rscene, O, D, pix, smp, s, include_background=True)
    save("glass_chain.npz", doc=doc_array(lens), O=O, D=D, pix=pix, smp=smp,
         **{f"chain_{k}": np.asarray(v) for k, v in ch.items()}, L=L, L_direct=Ld)


def progressive_fixture():
    """The progressive control plane of render_drc (cache.py:426-469): per-pass
    telemetry (index, r, tasks, cumulative entries), mid-run snapshots at task
    budgets, and an interrupt that fires at its second poll (after pass 1),
    against which libdrcb's host pass loop is checked."""
    doc = scenegen.scene_doc(scenegen.build_scene("c1", resolution=(40, 40)))
    scene = parse_scene(json.dumps(doc))
    net = rcnn.random_network(8, 2)
    kw = dict(direct_spp=1, mis_samples=8, seed=3, threads=1)
    img, tel = render_drc(scene, RenderConfig(passes=3, **kw), net, snapshots=[2, 5, 9])
    polls = []

    def interrupt():
        polls.append(1)
        return len(polls) >= 2

    img_i, tel_i = render_drc(scene, RenderConfig(passes=3, **kw), net, interrupt=interrupt)
    pas = np.array([[p["index"], p["r"], p["tasks"], p["entries"]] for p in tel["passes"]])
    pas_i = np.array([[p["index"], p["r"], p["tasks"], p["entries"]] for p in tel_i["passes"]])
    snaps = tel["snapshots"]
    save("drc_progressive.npz", doc=doc_array(doc), cfg=doc_array(dict(passes=3, direct_spp=1,
                                                                        mis_samples=8, seed=3)),
         k=8, seed_w=2, image=img, passes=pas, tasks=tel["tasks"], entries=tel["entries"],
         snap_budgets=np.array(sorted(snaps)), snaps=np.stack([snaps[b] for b in sorted(snaps)]),
         image_interrupted=img_i, passes_interrupted=pas_i, tasks_interrupted=tel_i["tasks"])


def main():
    geometry_fixture()
    trace_fixture()
    cnn_fixture()
    c1 = scenegen.scene_doc(scenegen.build_scene("c1", resolution=(48, 48)))
    frame_fixture("frame_c1.npz", c1, 8, 0, dict(direct_spp=2, indirect_tasks=5, mis_samples=16))
    frame_fixture("frame_cornell.npz", ref_scene_doc("cornell", 32), 8, 3,
                  dict(direct_spp=2, indirect_tasks=2, mis_samples=8))
    frame_fixture("frame_glossybox.npz", ref_scene_doc("glossybox", 32), 8, 4,
                  dict(direct_spp=3, indirect_tasks=1, mis_samples=16, sampler_kind="stratified"))
    frame_fixture("frame_room.npz", ref_scene_doc("room", 32), 16, 0,
                  dict(direct_spp=2, indirect_tasks=3, mis_samples=8, seed=9),
                  net=rcnn.make_blur_network(16))
    env = {"camera": {"position": [0, 0, -5], "look_at": [0, 0, 0], "up": [0, 1, 0], "fov": 40.0,
                      "resolution": [16, 16]},
           "global_up": [0, 1, 0], "materials": {"gray": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5]}},
           "shapes": [{"type": "sphere", "center": [0, 0, 0], "radius": 1.0, "material": "gray"}],
           "point_lights": [], "environment": [1.0, 1.0, 1.0]}
    frame_fixture("frame_furnace.npz", env, 8, 1, dict(direct_spp=2, indirect_tasks=1, mis_samples=8))


if __name__ == "__main__" and not ({"--train", "--pt", "--data", "--drcc", "--glass", "--progressive"}
                                   & set(sys.argv)):
    main()
    glass_fixtures()
    progressive_fixture()
if __name__ == "__main__" and "--glass" in sys.argv:
    glass_fixtures()
if __name__ == "__main__" and "--progressive" in sys.argv:
    progressive_fixture()


def train_fixture():
    """Two optimisation steps of the reference trainer (train.py:85-103):
    MapAutoencoder in train mode, L1Loss, Adam(lr, betas), from DRCW weights."""
    import torch

    from drc_trainer.model import export_drcw, import_drcw

    torch.manual_seed(0)
    out = {}
    for k, seed, n in ((8, 7, 4),):
        net = rcnn.random_network(k, seed)
        raw = rcnn.save_weights(net)
        model = import_drcw(raw)
        model.train()
        opt = torch.optim.Adam(model.parameters(), lr=1e-4, betas=(0.9, 0.999))
        loss_fn = torch.nn.L1Loss()
        rng = np.random.default_rng(seed)
        xs, ys, losses = [], [], []
        for step in range(2):
            x = rng.uniform(0, 1, (n, 7, 32, 32)).astype(np.float32)
            x[:, :3] *= 4.0
            y = np.exp(rng.normal(-1.0, 1.0, (n, 3, 32, 32))).astype(np.float32)
            xs.append(x)
            ys.append(y)
            opt.zero_grad()
            loss = loss_fn(model(torch.from_numpy(x)), torch.from_numpy(y))
            loss.backward()
            if step == 0:
                for name, p in model.named_parameters():
                    out[f"k{k}_grad0/{name}"] = p.grad.detach().numpy().copy()
            opt.step()
            losses.append(float(loss))
        out[f"k{k}_x"] = np.stack(xs)
        out[f"k{k}_y"] = np.stack(ys)
        out[f"k{k}_loss"] = np.array(losses)
        out[f"k{k}_weights_in"] = np.frombuffer(raw, dtype=np.uint8)
        out[f"k{k}_weights_out"] = np.frombuffer(export_drcw(model), dtype=np.uint8)
    save("train.npz", **out)


if __name__ == "__main__" and "--train" in sys.argv:
    train_fixture()


def pt_dataset_fixture():
    """render(mode="pt") and reference-mode examples (dataset.py:53-127)."""
    from drc.dataset import generate_examples

    doc = ref_scene_doc("cornell", 24)
    scene = parse_scene(json.dumps(doc))
    cfg = RenderConfig(threads=1, spp=3, max_path_depth=5, rr_start=3, seed=4)
    img, _ = rint.render(scene, cfg, "pt")
    doc2 = ref_scene_doc("glossybox", 16)
    scene2 = parse_scene(json.dumps(doc2))
    cfg2 = RenderConfig(threads=1, max_path_depth=4, rr_start=3)
    ex = generate_examples(scene2, (2, 2), 256, seed=5, config=cfg2)
    save("pt_dataset.npz", doc=doc_array(doc), pt=img, doc2=doc_array(doc2),
         ex_input=np.stack([e.input for e in ex]), ex_target=np.stack([e.target for e in ex]),
         ex_sr=np.array([e.s_r for e in ex]), ex_sd=np.array([e.s_d for e in ex]),
         ex_pixel=np.array([e.pixel for e in ex]))


if __name__ == "__main__" and "--pt" in sys.argv:
    pt_dataset_fixture()


def data_fixture():
    """The trainer's input pipeline and loop (trainer/src/drc_trainer/data.py,
    train.py:65-116): augment/ablate variants, split_by_scene, DRCD bytes and a
    short train() run (k = 8) with its initial/final weights and history."""
    import torch

    from drc.dataset import TrainingExample, write_dataset
    from drc_trainer import data as rdata
    from drc_trainer import train as rtrain
    from drc_trainer.model import export_drcw

    rng = np.random.default_rng(11)
    scenes = ["alpha", "beta", "gamma", "delta", "eps"]
    exs = []
    for i in range(15):
        x = rng.uniform(0, 1, (7, 32, 32)).astype(np.float32)
        x[:3] *= 3.0
        nv = rng.normal(size=(3, 32, 32))
        nv /= np.linalg.norm(nv, axis=0, keepdims=True)
        x[3:6] = nv.astype(np.float32)
        x[3:5, 5, 7] = 0.0  # exact zeros in the normal pair
        y = np.exp(rng.normal(-1.0, 1.0, (3, 32, 32))).astype(np.float32)
        exs.append(TrainingExample(input=x, target=y, s_r=float(rng.uniform(0.1, 2)),
                                   s_d=float(rng.uniform(0.5, 3)), scene_id=scenes[i % 5],
                                   pixel=(i, 2 * i)))
    raw = write_dataset(exs)
    rex = rdata.read_drcd(raw)
    aug = [v for e in rex[:2] for v in rdata.augment(e)]
    abl_n = rdata.ablate(rex[0], ("normals",))
    abl_nd = [rdata.transform_example(rdata.ablate(rex[1], ("normals", "distance")), s, f)
              for s in (8, 24) for f in (False, True)]
    splits = {}
    for seed in (0, 1, 5):
        tr, va = rdata.split_by_scene(rex, 0.2, seed)
        splits[f"split{seed}_val"] = np.array([i for i, e in enumerate(rex) if any(e is v for v in va)])
    cfg = rtrain.TrainConfig(learning_rate=1e-3, batch_size=8, epochs=2, k=8, seed=3,
                             val_fraction=0.2, ablation=("distance",))
    model, hist = rtrain.train(rex, cfg, None, log=lambda *a: None)
    torch.manual_seed(cfg.seed)
    from drc_trainer.model import MapAutoencoder
    init = MapAutoencoder(k=8)
    save("data.npz", drcd=np.frombuffer(raw, dtype=np.uint8),
         aug_input=np.stack([e.input for e in aug]), aug_target=np.stack([e.target for e in aug]),
         abl_n=abl_n.input, abl_nd_input=np.stack([e.input for e in abl_nd]),
         **splits,
         hist_step=np.array([h[0] for h in hist]),
         hist_split=np.array([0 if h[1] == "train" else 1 for h in hist]),
         hist_loss=np.array([h[2] for h in hist]),
         init_weights=np.frombuffer(export_drcw(init), dtype=np.uint8),
         final_weights=np.frombuffer(export_drcw(model), dtype=np.uint8))


if __name__ == "__main__" and "--data" in sys.argv:
    data_fixture()


def drcc_fixture():
    """The entry pool of the frame_c1 frame (DrcState.entries, cache.py:196-201)
    and its DRCC dump bytes (write_cache_dump, cache.py:476-485)."""
    import tempfile

    from drc.cache import write_cache_dump

    c1 = scenegen.scene_doc(scenegen.build_scene("c1", resolution=(48, 48)))
    scene = parse_scene(json.dumps(c1))
    cfg = RenderConfig(threads=1, direct_spp=2, indirect_tasks=5, mis_samples=16)
    net = rcnn.random_network(8, 0)
    _, tel = render_drc(scene, cfg, net)
    ents = tel["state"].entries()
    with tempfile.NamedTemporaryFile(suffix=".drcc") as f:
        write_cache_dump(ents, f.name)
        raw = open(f.name, "rb").read()
    save("drcc.npz", doc=doc_array(c1), drcc=np.frombuffer(raw, dtype=np.uint8),
         e_px=np.array([e.pixel[0] for e in ents]), e_py=np.array([e.pixel[1] for e in ents]),
         e_pos=np.stack([e.position for e in ents]), e_normal=np.stack([e.normal for e in ents]),
         e_rad=np.stack([e.indirect_radiance for e in ents]),
         e_thr=np.stack([e.specular_throughput for e in ents]))


if __name__ == "__main__" and "--drcc" in sys.argv:
    drcc_fixture()
