"""Drop-in installation over the reference package (drc / drc_trainer).

    import paper_1910_02480_b200.shim as shim
    shim.install()          # rebinding only; idempotent

rebinds the reference's hot-path surfaces to the B200 implementation:

  drc.cache.render_drc                      -> render.render_drc
  drc.integrators.render (drc/direct/pt)    -> render.render
  drc.cnn.forward                           -> cnn.forward
  drc_trainer.model.forward_reference       -> batched device forward
  drc_trainer.data.{read_drcd, augment, transform_example, ablate,
                    split_by_scene}         -> data (device augmentation)
  drc_trainer.train.train                   -> trainer.train (device loop)

The reference objects (Scene, RenderConfig, Network) are accepted as-is
(duck typing). Nothing falls back to the CPU: if libdrcb.so or the GPU is
missing the rebound calls raise.
"""

from __future__ import annotations

import importlib

_INSTALLED = {}


def _with_b200_fields(config, net_mode, precision):
    if hasattr(config, "precision") and hasattr(config, "net_mode"):
        return config
    from .render import RenderConfig

    fields = {k: getattr(config, k) for k in RenderConfig.__dataclass_fields__
              if hasattr(config, k)}
    fields.setdefault("precision", precision)
    fields.setdefault("net_mode", net_mode)
    return RenderConfig(**fields)


def install(net_mode="fp32", precision=64):
    from . import cnn, render

    def render_drc(scene, config, net, interrupt=None, snapshots=None):
        cfg = _with_b200_fields(config, net_mode, precision)
        return render.render_drc(scene, cfg, net, interrupt=interrupt, snapshots=snapshots)

    def render_any(scene, config, mode="pt", weights=None, interrupt=None):
        if mode in ("drc", "direct", "pt"):
            return render.render(scene, _with_b200_fields(config, net_mode, precision), mode,
                                 weights, interrupt)
        return _INSTALLED["drc.integrators.render"](scene, config, mode, weights, interrupt)

    def forward(net, x):
        return cnn.forward(net, x, mode=net_mode)

    targets = {
        "drc.cache": {"render_drc": render_drc},
        "drc.integrators": {"render": render_any},
        "drc.cnn": {"forward": forward},
    }
    for modname, attrs in targets.items():
        mod = importlib.import_module(modname)
        for name, fn in attrs.items():
            key = f"{modname}.{name}"
            if key not in _INSTALLED:
                _INSTALLED[key] = getattr(mod, name)
            setattr(mod, name, fn)
    try:
        model = importlib.import_module("drc_trainer.model")
    except ImportError:
        return
    import numpy as np

    def forward_reference(model_or_weights, x):
        w = model_or_weights
        raw = model.export_drcw(w) if hasattr(w, "state_dict") else w
        net = cnn.load_weights(raw)
        arr = np.asarray(x, dtype=np.float32)
        single = arr.ndim == 3
        out = cnn.forward_batch(net, arr[None] if single else arr, mode=net_mode)
        return out[0] if single else out

    if "drc_trainer.model.forward_reference" not in _INSTALLED:
        _INSTALLED["drc_trainer.model.forward_reference"] = model.forward_reference
    model.forward_reference = forward_reference

    # the trainer's input pipeline and loop (data.py, train.py:65-116)
    from . import data as bdata
    from . import trainer as btrainer

    def train(examples, config, weights_out, curves_out=None, log=print):
        trainer, history = btrainer.train(examples, config, weights_out, curves_out, log)
        m = model.import_drcw(trainer.export())
        m.eval()
        return m, history

    tmods = {
        "drc_trainer.data": {"read_drcd": bdata.read_drcd, "augment": bdata.augment,
                             "transform_example": bdata.transform_example,
                             "ablate": bdata.ablate, "split_by_scene": bdata.split_by_scene},
        "drc_trainer.train": {"train": train},
    }
    for modname, attrs in tmods.items():
        mod = importlib.import_module(modname)
        for name, fn in attrs.items():
            key = f"{modname}.{name}"
            if key not in _INSTALLED:
                _INSTALLED[key] = getattr(mod, name)
            setattr(mod, name, fn)


def uninstall():
    for key, fn in list(_INSTALLED.items()):
        modname, name = key.rsplit(".", 1)
        setattr(importlib.import_module(modname), name, fn)
        del _INSTALLED[key]
