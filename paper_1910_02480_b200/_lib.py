"""ctypes binding of libdrcb.so (include/drcb.h).

This is the only place Python touches the native library. There is no
fallback: if the library (or a GPU) is missing, calls raise. Device buffers
are torch CUDA tensors passed by data_ptr(); torch is plumbing only.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import STATUS_TO_ERROR, CudaError, DrcError

_HERE = os.path.dirname(os.path.abspath(__file__))
# DRCB_LIB: another build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("DRCB_LIB") or os.path.join(_HERE, "libdrcb.so")

c_dp = C.POINTER(C.c_double)
c_ip = C.POINTER(C.c_int32)
vp = C.c_void_p


class SceneDesc(C.Structure):
    _fields_ = [
        ("n_spheres", C.c_int32), ("n_quads", C.c_int32), ("n_tris", C.c_int32),
        ("n_materials", C.c_int32), ("n_point_lights", C.c_int32),
        ("sph_center", vp), ("sph_radius", vp), ("sph_mat", vp),
        ("quad_corner", vp), ("quad_eu", vp), ("quad_ev", vp), ("quad_mat", vp),
        ("tri_v0", vp), ("tri_v1", vp), ("tri_v2", vp), ("tri_mat", vp),
        ("mat_kind", vp), ("mat_albedo", vp), ("mat_exponent", vp), ("mat_ior", vp),
        ("mat_emission", vp),
        ("point_pos", vp), ("point_intensity", vp),
        ("global_up", C.c_double * 3), ("rotated_up", C.c_double * 3),
        ("environment", C.c_double * 3),
    ]


class Camera(C.Structure):
    _fields_ = [
        ("position", C.c_double * 3), ("forward", C.c_double * 3),
        ("right", C.c_double * 3), ("up", C.c_double * 3),
        ("tan_half", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
    ]


class RenderCfg(C.Structure):
    _fields_ = [
        ("direct_spp", C.c_int32), ("max_path_depth", C.c_int32),
        ("mis_samples", C.c_int32), ("rr_start", C.c_int32),
        ("sampler_kind", C.c_int32), ("precision", C.c_int32),
        ("tile", C.c_int32), ("include_background", C.c_int32),
        ("map_spp", C.c_int32), ("reserved", C.c_int32), ("seed", C.c_uint64),
    ]


class Entries(C.Structure):
    _fields_ = [("px", C.c_void_p), ("py", C.c_void_p), ("position", C.c_void_p),
                ("normal", C.c_void_p), ("radiance", C.c_void_p), ("throughput", C.c_void_p)]


class AugmentTrig(C.Structure):
    _fields_ = [("cos_a", C.c_double * 4), ("sin_a", C.c_double * 4)]


class GBuffer(C.Structure):
    _fields_ = [
        ("found", vp), ("escaped", vp), ("position", vp), ("normal", vp),
        ("throughput", vp), ("direction", vp), ("t_total", vp), ("mat", vp),
    ]


# (name, restype, argtypes)
_SIGS = [
    ("drcb_scene_create", C.c_int, [C.POINTER(SceneDesc), C.POINTER(vp)]),
    ("drcb_scene_destroy", None, [vp]),
    ("drcb_scene_stats", C.c_int, [vp, C.POINTER(C.c_int64)]),
    ("drcb_intersect", C.c_int, [vp, C.c_int32, vp, vp, C.c_int64, vp, vp, C.c_int32,
                                 vp, vp, vp, vp, vp, vp, vp]),
    ("drcb_primary_chain", C.c_int, [vp, C.c_int32, vp, vp, C.c_int64, C.POINTER(GBuffer), vp]),
    ("drcb_li_direct", C.c_int, [vp, C.POINTER(RenderCfg), vp, vp, vp, vp, C.c_int64,
                                 C.c_int32, vp, vp, vp]),
    ("drcb_trace_radiance", C.c_int, [vp, C.POINTER(RenderCfg), vp, vp, vp, vp, C.c_int64,
                                      C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]),
    ("drcb_gbuffer_direct", C.c_int, [vp, C.POINTER(Camera), C.POINTER(RenderCfg),
                                      C.POINTER(GBuffer), vp, vp, vp]),
    ("drcb_render_stacks", C.c_int, [vp, C.POINTER(RenderCfg), vp, vp, vp, C.c_int64, vp, vp,
                                     vp, vp, vp, vp]),
    ("drcb_shade", C.c_int, [vp, C.POINTER(RenderCfg), vp, vp, vp, vp, vp, vp, C.c_int64, vp,
                             vp]),
    ("drcb_interp_composite", C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(GBuffer),
                                        vp, vp, vp, vp, C.c_int64, C.c_int32, vp, vp, vp]),
    ("drcb_render_drc", C.c_int, [vp, vp, C.POINTER(Camera), C.POINTER(RenderCfg), vp, vp, vp,
                                  C.c_int64, C.c_int32, C.c_int32, vp, vp, vp]),
    ("drcb_frame_begin", C.c_int, [vp, vp, C.POINTER(Camera), C.POINTER(RenderCfg), C.c_int32,
                                   C.c_int64, C.POINTER(vp), vp]),
    ("drcb_frame_add_points", C.c_int, [vp, vp, vp, vp, C.c_int64, vp]),
    ("drcb_frame_composite", C.c_int, [vp, C.c_int32, vp, vp]),
    ("drcb_frame_info", C.c_int, [vp, C.POINTER(C.c_int64), vp]),
    ("drcb_frame_entries", C.c_int, [vp, C.POINTER(Entries), vp]),
    ("drcb_frame_end", C.c_int, [vp, vp]),
    ("drcb_render_pt", C.c_int, [vp, C.POINTER(Camera), C.POINTER(RenderCfg), vp, vp, vp]),
    ("drcb_reference_map", C.c_int, [vp, C.POINTER(RenderCfg), vp, vp, C.c_uint64, C.c_int32, vp,
                                     vp, vp]),
    ("drcb_net_create", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(vp)]),
    ("drcb_net_destroy", None, [vp]),
    ("drcb_net_info", C.c_int, [vp, C.POINTER(C.c_int64)]),
    ("drcb_net_forward", C.c_int, [vp, vp, vp, C.c_int64, C.c_int32, vp]),
    ("drcb_kernel_launches", C.c_int64, []),
    ("drcb_l2_read_probe", C.c_int, [vp, C.c_int64, C.c_int32, vp, vp]),
    ("drcb_trav_stats", C.c_int, [vp]),
    ("drcb_debug_conv", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, vp, vp,
                                  vp]),
    ("drcb_debug_wgrad", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, vp, vp, vp]),
    ("drcb_trainer_create", C.c_int, [C.c_char_p, C.c_size_t, C.c_float, C.c_float, C.c_float,
                                      C.c_float, C.POINTER(vp)]),
    ("drcb_trainer_destroy", None, [vp]),
    ("drcb_trainer_info", C.c_int, [vp, C.POINTER(C.c_int64)]),
    ("drcb_trainer_buffers", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    ("drcb_trainer_step", C.c_int, [vp, vp, vp, C.c_int64, C.POINTER(C.c_double), C.c_int32, vp]),
    ("drcb_render_drc_entries", C.c_int, [vp, vp, C.POINTER(Camera), C.POINTER(RenderCfg), vp, vp,
                                          vp, C.c_int64, C.c_int32, C.c_int32, vp, vp,
                                          C.POINTER(Entries), vp]),
    ("drcb_trainer_set_mode", C.c_int, [vp, C.c_int32]),
    ("drcb_augment_gather", C.c_int, [vp, vp, vp, vp, C.c_int64, vp, C.c_int32, vp, vp, vp]),
    ("drcb_trainer_apply", C.c_int, [vp, C.c_float, vp]),
    ("drcb_trainer_export", C.c_int64, [vp, vp, C.c_int64]),
    ("drcb_trainer_set_comm", C.c_int, [vp, vp, C.c_int32]),
    ("drcb_trainer_debug_z", C.c_int, [vp, C.c_int32, vp, vp]),
    ("drcb_trainer_last_loss", C.c_int, [vp, C.POINTER(C.c_double), vp]),
    ("drcb_trainer_set_reducer", C.c_int, [vp, vp, vp, C.c_int32]),
    ("drcb_loopback_create", C.c_int, [C.c_int32, C.POINTER(vp)]),
    ("drcb_loopback_rank", C.c_int, [vp, C.c_int32, C.POINTER(vp)]),
    ("drcb_loopback_reduce", C.c_int, [vp, vp, C.c_int64, C.c_int32, vp]),
    ("drcb_loopback_destroy", None, [vp, C.POINTER(vp), C.c_int32]),
    ("drcb_copy_sync", C.c_int, [vp, vp, C.c_int64, vp]),
    ("drcb_nccl_unique_id", C.c_int, [vp]),
    ("drcb_nccl_comm_create", C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(vp)]),
    ("drcb_nccl_comm_destroy", C.c_int, [vp]),
    ("drcb_allreduce_sum_f32", C.c_int, [vp, vp, C.c_int64, vp]),
    ("drcb_last_error", C.c_char_p, []),
    ("drcb_version", C.c_int, []),
]

EXPORTED = [name for name, _, _ in _SIGS]

_lib = None


def load():
    """Load libdrcb.so once; raise loudly if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DrcError(
            f"libdrcb.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status, what=""):
    if status == 0:
        return
    lib = load()
    msg = lib.drcb_last_error().decode("utf-8", "replace")
    cls = STATUS_TO_ERROR.get(int(status), CudaError)
    raise cls(f"{what}: {msg}" if what else msg)


def call(name, *args):
    lib = load()
    check(getattr(lib, name)(*args), name)


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
