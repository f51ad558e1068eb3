"""ctypes binding of the C ABI in include/psdf.h (libpsdf.so).

This is the Python face of the drop-in boundary: the same entry points a
C / C++ / cgo / JNI caller binds.  There is no fallback — if libpsdf.so is
missing or no GPU is visible the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PSDF_LIB selects a diagnostics build (e.g. lib/libpsdf_stats.so) by name
LIB_PATH = os.path.join(HERE, "lib", os.environ.get("PSDF_LIB", "libpsdf.so"))

PSDF_OK = 0
ERRORS = {1: "invalid_argument", 2: "out_of_range", 3: "runtime_error", 4: "cuda", 5: "nccl"}


class PsdfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"psdf error {code} ({ERRORS.get(code, '?')}): {msg}")
        self.code = code


class PsdfInvalidArgument(PsdfError, ValueError):
    """std::invalid_argument in the reference."""


class PsdfOutOfRange(PsdfError, IndexError):
    """std::out_of_range in the reference."""


class psdf_camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("rot", C.c_double * 9),
                ("pos", C.c_double * 3), ("id", C.c_int32), ("pad_", C.c_int32)]


class psdf_render_opts(C.Structure):
    _fields_ = [("tau", C.c_double), ("early_stop", C.c_double), ("bg", C.c_double * 3),
                ("n_max", C.c_int32), ("camera_id", C.c_int32), ("no_spatial", C.c_int32),
                ("no_angular", C.c_int32), ("no_fresnel", C.c_int32),
                ("sh_order_override", C.c_int32), ("need_colors", C.c_int32)]


class psdf_step_params(C.Structure):
    _fields_ = [("tau", C.c_double), ("lr_vox", C.c_double), ("lr_mlp", C.c_double),
                ("l_sdf", C.c_double), ("l_eik", C.c_double), ("l_norm", C.c_double),
                ("l_feat", C.c_double), ("l_probe", C.c_double), ("photo_scale", C.c_double),
                ("use_camera_bias", C.c_int32), ("pad_", C.c_int32)]


class psdf_grid_desc(C.Structure):
    _fields_ = [("T", C.c_int32), ("P", C.c_int32), ("n_s", C.c_int32), ("n_a", C.c_int32),
                ("sh_order", C.c_int32), ("res", C.c_int32 * 3), ("voxel_size", C.c_double),
                ("origin", C.c_double * 3), ("far_field_voxels", C.c_double), ("ncam", C.c_int32),
                ("pad_", C.c_int32)]


class psdf_counts(C.Structure):
    _fields_ = [("n_rays", C.c_int64), ("n_marched", C.c_int64), ("n_extra", C.c_int64),
                ("n_shaded", C.c_int64), ("n_alpha", C.c_int64), ("n_bwd_rays", C.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class psdf_losses(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("photo", "sdf", "eik", "normal", "features", "probes",
                                          "total", "psnr", "sq_err", "mask_px")]

    def as_dict(self):
        return {k: float(getattr(self, k)) for k, _ in self._fields_}


# Every symbol include/psdf.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "psdf_abi_version", "psdf_create", "psdf_destroy", "psdf_last_error", "psdf_upload_grid",
    "psdf_upload_mlp", "psdf_mlp_size", "psdf_download_params", "psdf_set_keep_raypass_grads",
    "psdf_download_grads", "psdf_smooth_all", "psdf_render", "psdf_render_device",
    "psdf_train_reset", "psdf_train_step", "psdf_upload_views", "psdf_train_step_views",
    "psdf_comm_unique_id", "psdf_comm_init", "psdf_last_timing", "psdf_stream",
    "psdf_host_alloc", "psdf_host_free", "psdf_march_rays", "psdf_pixel_dirs",
    "psdf_last_k2_breakdown", "psdf_grid_info", "psdf_download_structure", "psdf_subdivide",
    "psdf_raise_sh_order", "psdf_last_h2d_bytes", "psdf_init_visual_hull", "psdf_save_checkpoint",
    "psdf_load_checkpoint", "psdf_eval_psnr", "psdf_point_mesh_distance", "psdf_chamfer",
    "psdf_debug_set_shard", "psdf_marching_cubes", "psdf_download_mesh",
    "psdf_last_wave_counts", "psdf_debug_wave", "psdf_set_grad_exchange",
]

_lib = None
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)


def load():
    """Loads libpsdf.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} is missing — run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.psdf_abi_version.restype = C.c_int
    L.psdf_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.psdf_destroy.argtypes = [vp]
    L.psdf_last_error.restype = C.c_char_p
    L.psdf_last_error.argtypes = [vp]
    L.psdf_upload_grid.argtypes = [vp, C.POINTER(psdf_grid_desc), _ip, _ip, _ip, _fp, _fp, _fp, _fp]
    L.psdf_upload_mlp.argtypes = [vp, _fp, C.c_int64]
    L.psdf_mlp_size.restype = C.c_int64
    L.psdf_mlp_size.argtypes = [C.c_int, C.c_int, C.c_int]
    L.psdf_download_params.argtypes = [vp, _fp, _fp, _fp, _fp, _fp]
    L.psdf_set_keep_raypass_grads.argtypes = [vp, C.c_int]
    L.psdf_download_grads.argtypes = [vp, C.c_int, _fp, _fp, _fp, _fp, _fp]
    L.psdf_smooth_all.argtypes = [vp]
    L.psdf_render.argtypes = [vp, C.POINTER(psdf_camera), C.POINTER(psdf_render_opts), _fp, _fp, _fp,
                              C.POINTER(psdf_counts)]
    L.psdf_render_device.argtypes = [vp, C.POINTER(psdf_camera), C.POINTER(psdf_render_opts), vp, vp,
                                     vp, C.POINTER(psdf_counts)]
    L.psdf_eval_psnr.argtypes = [vp, C.POINTER(psdf_camera), C.POINTER(psdf_render_opts), _fp,
                                 C.POINTER(C.c_uint8), C.POINTER(C.c_double), C.POINTER(psdf_counts)]
    _dp, _i32 = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    L.psdf_point_mesh_distance.argtypes = [vp, _dp, C.c_int64, _dp, C.c_int64, _i32, C.c_int64, _dp]
    L.psdf_chamfer.argtypes = [vp, _dp, C.c_int64, _dp, C.c_int64, _i32, C.c_int64, _dp, C.c_int64, _dp,
                               C.c_int64, _i32, C.c_int64, C.c_double, _dp]
    L.psdf_marching_cubes.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.psdf_download_mesh.argtypes = [vp, _dp, _i32]
    L.psdf_train_reset.argtypes = [vp]
    L.psdf_train_step.argtypes = [vp, C.c_int, C.POINTER(psdf_camera), C.POINTER(_fp),
                                  C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(psdf_step_params),
                                  C.POINTER(psdf_losses), C.POINTER(psdf_counts)]
    L.psdf_upload_views.argtypes = [vp, C.c_int, C.POINTER(psdf_camera), C.POINTER(_fp),
                                    C.POINTER(C.POINTER(C.c_uint8))]
    L.psdf_train_step_views.argtypes = [vp, C.c_int, _ip, C.POINTER(psdf_step_params),
                                        C.POINTER(psdf_losses), C.POINTER(psdf_counts)]
    L.psdf_comm_unique_id.argtypes = [vp]
    L.psdf_comm_init.argtypes = [vp, vp, C.c_int, C.c_int]
    L.psdf_debug_set_shard.argtypes = [vp, C.c_int, C.c_int]
    L.psdf_last_timing.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_int)]
    L.psdf_stream.restype = vp
    L.psdf_stream.argtypes = [vp]
    L.psdf_host_alloc.restype = vp
    L.psdf_host_alloc.argtypes = [C.c_size_t]
    L.psdf_host_free.argtypes = [vp]
    _dp = C.POINTER(C.c_double)
    L.psdf_march_rays.argtypes = [vp, C.c_int, _dp, _dp, C.c_int, _dp, _ip]
    L.psdf_pixel_dirs.argtypes = [C.POINTER(psdf_camera), _dp]
    L.psdf_last_k2_breakdown.argtypes = [vp, _dp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.psdf_last_wave_counts.argtypes = [vp, C.POINTER(C.c_int64)]
    L.psdf_debug_wave.argtypes = [vp, C.c_int, vp, C.c_int64]
    L.psdf_set_grad_exchange.argtypes = [vp, C.c_int]
    L.psdf_grid_info.argtypes = [vp, C.POINTER(psdf_grid_desc)]
    L.psdf_download_structure.argtypes = [vp, _ip, _ip, _ip]
    L.psdf_subdivide.argtypes = [vp, C.c_double, _ip, _ip]
    L.psdf_raise_sh_order.argtypes = [vp, C.c_int]
    L.psdf_last_h2d_bytes.restype = C.c_int64
    L.psdf_save_checkpoint.argtypes = [vp, C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_uint64]
    L.psdf_load_checkpoint.argtypes = [vp, C.c_char_p, _ip, _ip, _ip, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_uint64)]
    L.psdf_init_visual_hull.argtypes = [vp, C.POINTER(psdf_grid_desc), C.c_int, C.c_int, C.POINTER(psdf_camera),
                                        C.POINTER(C.POINTER(C.c_uint8)), _ip, _ip]
    L.psdf_last_h2d_bytes.argtypes = [vp]
    _lib = L
    return L


def check(rc, ctx=None):
    if rc != PSDF_OK:
        msg = load().psdf_last_error(ctx).decode(errors="replace")
        if rc == 1:
            raise PsdfInvalidArgument(rc, msg)
        if rc == 2:
            raise PsdfOutOfRange(rc, msg)
        raise PsdfError(rc, msg)
