"""TEST INFRASTRUCTURE — ctypes bindings for the checkers under oracle/.

Two libraries, both CPU-only and never used by the product path:

* ``_ref/libsdfrecon_ref.so`` — the UNMODIFIED reference (``/root/reference/
  proj/src``) plus ``ref_harness.cpp``; see ``oracle/Makefile``.
* ``_build/libpsdf_oracle.so`` — ``psdf_oracle.c``, our C restatement of the
  reference's hot path, pinned against the reference in ``tests/``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsdfrecon_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libpsdf_oracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class RefCamera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("rot", C.c_double * 9),
                ("pos", C.c_double * 3), ("id", C.c_int32), ("pad_", C.c_int32)]


class RefRenderOpts(C.Structure):
    _fields_ = [("tau", C.c_double), ("early_stop", C.c_double), ("bg", C.c_double * 3),
                ("n_max", C.c_int32), ("camera_id", C.c_int32), ("no_spatial", C.c_int32),
                ("no_angular", C.c_int32), ("no_fresnel", C.c_int32),
                ("sh_order_override", C.c_int32), ("need_colors", C.c_int32)]


class RefStepParams(C.Structure):
    _fields_ = [("tau", C.c_double), ("lr_vox", C.c_double), ("lr_mlp", C.c_double),
                ("l_sdf", C.c_double), ("l_eik", C.c_double), ("l_norm", C.c_double),
                ("l_feat", C.c_double), ("l_probe", C.c_double), ("photo_scale", C.c_double),
                ("use_camera_bias", C.c_int32), ("pad_", C.c_int32)]


def ptr(a, t=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def render_opts(tau=100.0, n_max=512, early_stop=1e-4, bg=(0.0, 0.0, 0.0), camera_id=-1,
                no_spatial=False, no_angular=False, no_fresnel=False, sh_order_override=-1,
                need_colors=True):
    """renderer.hpp:13-27 defaults."""
    o = RefRenderOpts()
    o.tau = tau
    o.n_max = n_max
    o.early_stop = early_stop
    o.bg[:] = list(bg)
    o.camera_id = camera_id
    o.no_spatial = int(no_spatial)
    o.no_angular = int(no_angular)
    o.no_fresnel = int(no_fresnel)
    o.sh_order_override = sh_order_override
    o.need_colors = int(need_colors)
    return o


def camera_dict(c: RefCamera) -> dict:
    return dict(fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy, width=c.width, height=c.height,
                rot=list(c.rot), pos=list(c.pos), id=c.id)


def camera_from_dict(d: dict) -> RefCamera:
    c = RefCamera()
    c.fx, c.fy, c.cx, c.cy = d["fx"], d["fy"], d["cx"], d["cy"]
    c.width, c.height = d["width"], d["height"]
    c.rot[:] = list(d["rot"])
    c.pos[:] = list(d["pos"])
    c.id = d.get("id", 0)
    return c


_ref = None


def reflib():
    global _ref
    if _ref is not None:
        return _ref
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_scene_sphere.restype = C.c_void_p
    L.ref_scene_sphere.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_int, C.c_uint64]
    L.ref_scene_analytic.restype = C.c_void_p
    L.ref_scene_analytic.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _ip,
                                     _dp, _dp, C.c_int, C.c_uint64]
    L.ref_scene_free.argtypes = [C.c_void_p]
    L.ref_subdivide.argtypes = [C.c_void_p]
    L.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int64, C.c_uint64]
    L.ref_load_checkpoint.restype = C.c_void_p
    L.ref_load_checkpoint.argtypes = [C.c_char_p, C.c_void_p]
    L.ref_scene_hull.restype = C.c_void_p
    L.ref_scene_hull.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_uint64]
    L.ref_raise_sh_order.argtypes = [C.c_void_p, C.c_int]
    L.ref_scene_randomize.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                      C.c_double]
    L.ref_scene_info.argtypes = [C.c_void_p, _lp, _dp]
    L.ref_scene_export.argtypes = [C.c_void_p, _ip, _ip, _ip, _dp, _dp, _dp, _dp]
    L.ref_scene_import.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
    L.ref_smooth_all.argtypes = [C.c_void_p]
    L.ref_mlp_export.argtypes = [C.c_void_p, _dp]
    L.ref_mlp_import.argtypes = [C.c_void_p, _dp]
    L.ref_make_lookat_camera.argtypes = [C.c_int, _dp, _dp, _dp, C.c_double, C.c_double, C.c_int,
                                         C.c_int, C.POINTER(RefCamera)]
    L.ref_make_ring_cameras.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                        C.POINTER(RefCamera)]
    L.ref_march_ray.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp]
    L.ref_pixel_dir.argtypes = [C.POINTER(RefCamera), C.c_double, C.c_double, _dp]
    L.ref_render_ray.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(RefRenderOpts), C.c_int, _dp, _dp,
                                 _dp]
    L.ref_render_image.argtypes = [C.c_void_p, C.POINTER(RefCamera), C.POINTER(RefRenderOpts), _dp,
                                   _dp, _dp, _lp, C.c_int]
    L.ref_render_image_api.argtypes = [C.c_void_p, C.POINTER(RefCamera), C.POINTER(RefRenderOpts),
                                       _dp, _dp, C.c_int]
    L.ref_ray_backward.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(RefRenderOpts), _dp, C.c_double,
                                   C.c_int, _dp, _dp, _dp, _dp, _dp]
    L.ref_photo_pixel.argtypes = [_dp, _dp, C.c_int, C.c_double, C.c_double, _dp]
    L.ref_regularizer.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _dp]
    L.ref_gt_fold.argtypes = [C.c_void_p, _dp, _dp, _dp]
    L.ref_train_reset.argtypes = [C.c_void_p]
    L.ref_set_keep_grads.argtypes = [C.c_void_p, C.c_int]
    L.ref_last_phase_ms.argtypes = [C.c_void_p, _dp]
    L.ref_train_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(RefCamera), C.POINTER(_dp),
                                 C.POINTER(_dp), C.POINTER(RefStepParams), C.c_int, _dp, _lp]
    L.ref_grads_export.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp]
    L.ref_train_full.argtypes = [C.c_void_p, C.c_int, C.POINTER(RefCamera), C.POINTER(_dp),
                                 C.POINTER(_dp), C.c_int, C.c_int, _dp, C.c_double, C.c_int,
                                 C.c_uint64, C.c_int, _dp]
    L.ref_raytrace.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp, _dp, C.c_int, _dp, _dp,
                               C.POINTER(RefCamera), _dp, _dp]
    L.ref_gradcheck.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int, _dp, C.POINTER(C.c_int)]
    L.ref_alpha_from_sdf.restype = C.c_double
    L.ref_alpha_from_sdf.argtypes = [C.c_double, C.c_double, C.c_double]
    L.ref_eval_sh_basis.argtypes = [_dp, C.c_int, _dp]
    L.ref_fresnel_powers.argtypes = [C.c_double, _dp]
    L.ref_gaussian_kernel.argtypes = [_dp]
    L.ref_adam_steps.argtypes = [C.c_int, _dp, _dp, C.c_int, _dp]
    L.ref_psnr_masked.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, _dp]
    _i32p, _i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    L.ref_marching_cubes.argtypes = [C.c_void_p, _dp, C.c_int64, _i32p, C.c_int64, _i64p, _i64p]
    L.ref_marching_cubes_field.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_double, _dp, C.c_int64,
                                           _i32p, C.c_int64, _i64p, _i64p]
    L.ref_point_mesh_distance.argtypes = [_dp, C.c_int64, _dp, C.c_int64, _i32p, C.c_int64, _dp]
    L.ref_sample_mesh_points.argtypes = [_dp, C.c_int64, _i32p, C.c_int64, C.c_int, C.c_uint64, _dp]
    L.ref_chamfer.argtypes = [_dp, C.c_int64, _dp, C.c_int64, _i32p, C.c_int64, _dp, C.c_int64, _dp,
                              C.c_int64, _i32p, C.c_int64, C.c_double, _dp]
    _ref = L
    return L


def _check(rc, L):
    if rc < 0:
        raise RuntimeError(L.ref_last_error().decode())


# --------------------------------------------------------------------------
# Scene description used by both checkers and by the GPU path's parity tests.
# --------------------------------------------------------------------------
class GridArrays:
    """Flat arrays describing a grid + MLP, in the upload layout of include/psdf.h."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    def copy(self):
        d = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.__dict__.items()}
        return GridArrays(**d)


class RefScene:
    """A scene owned by the reference library (sdfrecon::SparseGrid + DecoderMlp)."""

    def __init__(self, handle):
        self.L = reflib()
        self.h = C.c_void_p(handle)

    @classmethod
    def sphere(cls, res=32, n_s=2, n_a=2, sh_order=2, band_voxels=32, radius=0.3, center=(0, 0, 0),
               far_field_voxels=4.0, ncam=1, mlp_seed=1, origin=(-0.5, -0.5, -0.5)):
        L = reflib()
        h = L.ref_scene_sphere(res, 1.0 / res, origin[0], origin[1], origin[2], n_s, n_a, sh_order,
                               band_voxels, far_field_voxels, center[0], center[1], center[2], radius,
                               ncam, mlp_seed)
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        return cls(h)

    @classmethod
    def hull(cls, cams, masks, res=32, n_s=2, n_a=2, sh_order=2, band_voxels=6, far_field_voxels=4.0,
             ncam=0, mlp_seed=1, origin=(-0.5, -0.5, -0.5)):
        """init_grid_visual_hull (grid.cpp:470-504): masks are uint8 images (> 127 = foreground)."""
        L = reflib()
        n = len(cams)
        carr = (RefCamera * n)(*cams)
        ms = [np.ascontiguousarray(m, np.uint8) for m in masks]
        mp = (C.c_void_p * n)(*[m.ctypes.data for m in ms])
        h = L.ref_scene_hull(res, 1.0 / res, origin[0], origin[1], origin[2], n_s, n_a, sh_order, band_voxels,
                             far_field_voxels, n, C.cast(carr, C.c_void_p), C.cast(mp, C.c_void_p), ncam, mlp_seed)
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        return cls(h)

    @classmethod
    def analytic(cls, prims, res=32, n_s=2, n_a=2, sh_order=2, band_voxels=6, far_field_voxels=4.0,
                 ncam=1, mlp_seed=1):
        """prims: list of (kind, center, extent), kind 0 sphere / 1 box / 2 torus."""
        L = reflib()
        kinds = np.array([p[0] for p in prims], dtype=np.int32)
        cen = np.array([p[1] for p in prims], dtype=np.float64).ravel()
        ext = np.array([p[2] for p in prims], dtype=np.float64).ravel()
        h = L.ref_scene_analytic(res, 1.0 / res, -0.5, -0.5, -0.5, n_s, n_a, sh_order, band_voxels,
                                 far_field_voxels, len(prims), ptr(kinds, _ip), ptr(cen), ptr(ext),
                                 ncam, mlp_seed)
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        return cls(h)

    def __del__(self):
        try:
            if self.h:
                self.L.ref_scene_free(self.h)
                self.h = None
        except Exception:
            pass

    def randomize(self, seed, sdf_jitter=0.0, plane_amp=0.2, probe_amp=0.3, bias_amp=0.1):
        self.L.ref_scene_randomize(self.h, seed, sdf_jitter, plane_amp, probe_amp, bias_amp)

    def info(self):
        info = np.zeros(10, np.int64)
        geom = np.zeros(5, np.float64)
        self.L.ref_scene_info(self.h, ptr(info, _lp), ptr(geom))
        return info, geom

    def export(self) -> GridArrays:
        info, geom = self.info()
        T, P, n_s, n_a, order = (int(x) for x in info[:5])
        res = tuple(int(x) for x in info[5:8])
        nc = order * order
        a = GridArrays(
            T=T, P=P, n_s=n_s, n_a=n_a, sh_order=order, res=res, voxel_size=float(geom[0]),
            origin=tuple(float(x) for x in geom[1:4]), far_field_voxels=float(geom[4]),
            tile_coords=np.zeros((T, 3), np.int32), probe_ids=np.zeros((T, 8), np.int32),
            probe_coords=np.zeros((P, 3), np.int32), raw=np.zeros((T, 4096)),
            smooth=np.zeros((T, 4096)), planes=np.zeros((T, 3, 256, n_s)),
            probes=np.zeros((P, nc, n_a)), mlp=np.zeros(int(info[8])), ncam=int(info[9]))
        self.L.ref_scene_export(self.h, ptr(a.tile_coords, _ip), ptr(a.probe_ids, _ip),
                                ptr(a.probe_coords, _ip), ptr(a.raw), ptr(a.smooth), ptr(a.planes),
                                ptr(a.probes))
        self.L.ref_mlp_export(self.h, ptr(a.mlp))
        return a

    def save_checkpoint(self, path, lod_cursor=0, iteration=0, seed=0):
        """save_checkpoint (checkpoint.cpp:54-104), the reference's own writer."""
        _check(self.L.ref_save_checkpoint(self.h, str(path).encode(), lod_cursor, iteration, seed), self.L)

    @classmethod
    def load_checkpoint(cls, path):
        """load_checkpoint (checkpoint.cpp:106-181); returns (scene, (lod_cursor, iteration, seed))."""
        L = reflib()
        out = (C.c_int64 * 3)()
        h = L.ref_load_checkpoint(str(path).encode(), out)
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        return cls(h), (int(out[0]), int(out[1]), int(out[2]) & 0xFFFFFFFFFFFFFFFF)

    def subdivide(self):
        """grid = grid.subdivide() (grid.cpp:271-345), the reference's own member."""
        _check(self.L.ref_subdivide(self.h), self.L)

    def raise_sh_order(self, order):
        """SparseGrid::raise_sh_order (grid.cpp:252-262); ValueError when the reference throws."""
        if self.L.ref_raise_sh_order(self.h, int(order)) != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def import_(self, raw=None, smooth=None, planes=None, probes=None, mlp=None):
        c = lambda x: None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        raw, smooth, planes, probes, mlp = c(raw), c(smooth), c(planes), c(probes), c(mlp)
        self.L.ref_scene_import(self.h, ptr(raw), ptr(smooth), ptr(planes), ptr(probes))
        if mlp is not None:
            self.L.ref_mlp_import(self.h, ptr(mlp))

    def round_to_f32(self):
        """Make every parameter (raw, smooth, planes, probes, MLP) fp32-representable,
        installing the rounded smoothed SDF verbatim (SURVEY.md hard part 2)."""
        a = self.export()
        f = lambda x: x.astype(np.float32).astype(np.float64)
        self.import_(raw=f(a.raw), smooth=f(a.smooth), planes=f(a.planes), probes=f(a.probes),
                     mlp=f(a.mlp))

    def render_image(self, cam: RefCamera, opts: RefRenderOpts, threads=0):
        w, h = cam.width, cam.height
        rgb = np.zeros((h, w, 3))
        alpha = np.zeros((h, w))
        depth = np.zeros((h, w))
        counts = np.zeros(5, np.int64)
        _check(self.L.ref_render_image(self.h, C.byref(cam), C.byref(opts), ptr(rgb), ptr(alpha),
                                       ptr(depth), ptr(counts, _lp), threads), self.L)
        return rgb, alpha, depth, counts

    def render_image_api(self, cam: RefCamera, opts: RefRenderOpts, threads=0):
        w, h = cam.width, cam.height
        rgb = np.zeros((h, w, 3))
        alpha = np.zeros((h, w))
        _check(self.L.ref_render_image_api(self.h, C.byref(cam), C.byref(opts), ptr(rgb), ptr(alpha),
                                           threads), self.L)
        return rgb, alpha

    def marching_cubes(self):
        """mesh.cpp:363 marching_cubes(grid) -> (verts (nv, 3) f64, tris (nt, 3) i32)."""
        nv, nt = C.c_int64(), C.c_int64()
        i32 = C.POINTER(C.c_int32)
        _check(self.L.ref_marching_cubes(self.h, None, 0, None, 0, C.byref(nv), C.byref(nt)), self.L)
        v = np.zeros((nv.value, 3))
        t = np.zeros((nt.value, 3), np.int32)
        _check(self.L.ref_marching_cubes(self.h, ptr(v), nv.value, t.ctypes.data_as(i32), nt.value,
                                         C.byref(nv), C.byref(nt)), self.L)
        return v, t

    def march_ray(self, o, d, n_max=512):
        ts = np.zeros(max(n_max, 1))
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        n = self.L.ref_march_ray(self.h, ptr(o), ptr(d), n_max, ptr(ts))
        return ts[:n].copy()

    def render_ray(self, o, d, opts, max_n=512):
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        s = np.zeros((max_n, 8))
        col = np.zeros((max_n, 3))
        res = np.zeros(6)
        n = self.L.ref_render_ray(self.h, ptr(o), ptr(d), C.byref(opts), max_n, ptr(s), ptr(col),
                                  ptr(res))
        _check(n, self.L)
        return s[:n].copy(), col[:n].copy(), res

    def grad_like(self):
        a = self.export()
        return dict(raw=np.zeros_like(a.raw), smooth=np.zeros_like(a.smooth),
                    planes=np.zeros_like(a.planes), probes=np.zeros_like(a.probes),
                    mlp=np.zeros_like(a.mlp))

    def ray_backward(self, o, d, opts, up_color, up_alpha, fold=True):
        g = self.grad_like()
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        uc = np.asarray(up_color, np.float64)
        _check(self.L.ref_ray_backward(self.h, ptr(o), ptr(d), C.byref(opts), ptr(uc), up_alpha,
                                       int(fold), ptr(g["raw"]), ptr(g["smooth"]), ptr(g["planes"]),
                                       ptr(g["probes"]), ptr(g["mlp"])), self.L)
        return g

    def regularizer(self, which, lam):
        g = self.grad_like()
        out = np.zeros(2)
        _check(self.L.ref_regularizer(self.h, which, lam, ptr(out), ptr(g["raw"]), ptr(g["smooth"]),
                                      ptr(g["planes"]), ptr(g["probes"])), self.L)
        return out, g

    def gt_fold(self, staged, raw_in=None):
        out = np.zeros_like(np.asarray(staged))
        staged = np.ascontiguousarray(staged, np.float64)
        raw_in = None if raw_in is None else np.ascontiguousarray(raw_in, np.float64)
        self.L.ref_gt_fold(self.h, ptr(staged), ptr(raw_in), ptr(out))
        return out

    def train_reset(self):
        self.L.ref_train_reset(self.h)

    def train_step(self, cams, gts, masks, hp: RefStepParams, threads=0):
        n = len(cams)
        arr = (RefCamera * n)(*cams)
        gts = [np.ascontiguousarray(g, np.float64) for g in gts]
        masks = [np.ascontiguousarray(m, np.float64) for m in masks]
        gp = (_dp * n)(*[ptr(g) for g in gts])
        mp = (_dp * n)(*[ptr(m) for m in masks])
        losses = np.zeros(10)
        counts = np.zeros(6, np.int64)
        _check(self.L.ref_train_step(self.h, n, arr, gp, mp, C.byref(hp), threads, ptr(losses),
                                     ptr(counts, _lp)), self.L)
        return losses, counts

    def keep_grads(self, keep):
        self.L.ref_set_keep_grads(self.h, int(keep))

    def last_phase_ms(self):
        out = np.zeros(3)
        self.L.ref_last_phase_ms(self.h, ptr(out))
        return out

    def grads(self, stage):
        g = self.grad_like()
        self.L.ref_grads_export(self.h, stage, ptr(g["raw"]), ptr(g["smooth"]), ptr(g["planes"]),
                                ptr(g["probes"]), ptr(g["mlp"]))
        return g

    def train_full(self, cams, gts, masks, iterations, images_per_batch, brackets, lambda_photo=40.0,
                   camera_bias=False, seed=0, threads=0):
        n = len(cams)
        arr = (RefCamera * n)(*cams)
        gts = [np.ascontiguousarray(g, np.float64) for g in gts]
        masks = [np.ascontiguousarray(m, np.float64) for m in masks]
        gp = (_dp * n)(*[ptr(g) for g in gts])
        mp = (_dp * n)(*[ptr(m) for m in masks])
        br = np.ascontiguousarray(brackets, np.float64)
        psnr = np.zeros(1)
        _check(self.L.ref_train_full(self.h, n, arr, gp, mp, iterations, images_per_batch, ptr(br),
                                     lambda_photo, int(camera_bias), seed, threads, ptr(psnr)), self.L)
        return float(psnr[0])


def lookat_camera(id, eye, target, up, fx, fy, width, height) -> RefCamera:
    L = reflib()
    c = RefCamera()
    e = np.asarray(eye, np.float64)
    t = np.asarray(target, np.float64)
    u = np.asarray(up, np.float64)
    L.ref_make_lookat_camera(id, ptr(e), ptr(t), ptr(u), fx, fy, width, height, C.byref(c))
    return c


def ring_cameras(n_views, resolution, radius=2.0, elevation=0.35, seed=0):
    L = reflib()
    arr = (RefCamera * n_views)()
    L.ref_make_ring_cameras(n_views, resolution, radius, elevation, seed, arr)
    return [arr[i] for i in range(n_views)]


# acceptance.cpp:54-74 (glossy sphere scene) lights, used for synthetic GT.
ACCEPT_LIGHTS = dict(pos=[[1.5, 2.0, 1.0], [-1.8, 1.2, -1.4]], intensity=[[6.0, 6.0, 5.5],
                                                                        [3.0, 3.2, 3.6]])


def raytrace(prims, cam: RefCamera, lights=ACCEPT_LIGHTS):
    """prims: list of (kind, center, extent, albedo, r0, spec_exp)."""
    L = reflib()
    kinds = np.array([p[0] for p in prims], np.int32)
    cen = np.array([p[1] for p in prims], np.float64).ravel()
    ext = np.array([p[2] for p in prims], np.float64).ravel()
    alb = np.array([p[3] for p in prims], np.float64).ravel()
    r0 = np.array([p[4] for p in prims], np.float64)
    se = np.array([p[5] for p in prims], np.float64)
    lp = np.array(lights["pos"], np.float64).ravel()
    li = np.array(lights["intensity"], np.float64).ravel()
    rgb = np.zeros((cam.height, cam.width, 3))
    mask = np.zeros((cam.height, cam.width))
    _check(L.ref_raytrace(len(prims), ptr(kinds, _ip), ptr(cen), ptr(ext), ptr(alb), ptr(r0),
                          ptr(se), len(lights["pos"]), ptr(lp), ptr(li), C.byref(cam), ptr(rgb),
                          ptr(mask)), L)
    return rgb, mask


GLOSSY_SPHERE = [(0, (0.0, 0.0, 0.0), (0.3, 0.3, 0.3), (0.55, 0.3, 0.2), 0.08, 32.0)]


def _mesh_args(verts, tris):
    v = np.ascontiguousarray(verts, np.float64)
    t = np.ascontiguousarray(tris, np.int32)
    return v, t, t.ctypes.data_as(C.POINTER(C.c_int32))


def ref_point_mesh_distance(points, verts, tris):
    """metrics.cpp:131-135 through the reference library."""
    L = reflib()
    p = np.ascontiguousarray(points, np.float64)
    v, t, tp = _mesh_args(verts, tris)
    out = np.zeros(len(p))
    _check(L.ref_point_mesh_distance(ptr(p), len(p), ptr(v), len(v), tp, len(t), ptr(out)), L)
    return out


def ref_sample_mesh_points(verts, tris, n, seed):
    """metrics.cpp:137-166 through the reference library."""
    L = reflib()
    v, t, tp = _mesh_args(verts, tris)
    out = np.zeros((n, 3))
    _check(L.ref_sample_mesh_points(ptr(v), len(v), tp, len(t), n, seed, ptr(out)), L)
    return out


def ref_chamfer(pred_pts, pred_verts, pred_tris, gt_pts, gt_verts, gt_tris, max_dist):
    """metrics.cpp:182-194 through the reference library."""
    L = reflib()
    pp = np.ascontiguousarray(pred_pts, np.float64)
    gp = np.ascontiguousarray(gt_pts, np.float64)
    pv, pt, ptp = _mesh_args(pred_verts, pred_tris)
    gv, gt, gtp = _mesh_args(gt_verts, gt_tris)
    out = np.zeros(3)
    _check(L.ref_chamfer(ptr(pp), len(pp), ptr(pv), len(pv), ptp, len(pt), ptr(gp), len(gp), ptr(gv), len(gv),
                         gtp, len(gt), max_dist, ptr(out)), L)
    return out


def ref_marching_cubes_field(values, origin=(0.0, 0.0, 0.0), spacing=1.0):
    """mesh.cpp:396 marching_cubes_field(values[x][y][z]) through the reference library
    -> (verts (nv, 3) f64, tris (nt, 3) i32)."""
    L = reflib()
    f = np.ascontiguousarray(values, np.float64)
    nx, ny, nz = f.shape
    o = np.ascontiguousarray(origin, np.float64)
    nv, nt = C.c_int64(), C.c_int64()
    i32 = C.POINTER(C.c_int32)
    _check(L.ref_marching_cubes_field(ptr(f), nx, ny, nz, ptr(o), spacing, None, 0, None, 0,
                                      C.byref(nv), C.byref(nt)), L)
    v = np.zeros((nv.value, 3))
    t = np.zeros((nt.value, 3), np.int32)
    _check(L.ref_marching_cubes_field(ptr(f), nx, ny, nz, ptr(o), spacing, ptr(v), nv.value,
                                      t.ctypes.data_as(i32), nt.value, C.byref(nv), C.byref(nt)), L)
    return v, t
