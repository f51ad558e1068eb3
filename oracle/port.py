"""TEST INFRASTRUCTURE — ctypes bindings for the C restatement (psdf_oracle.c).

``OracleGrid`` holds a grid + MLP in f64 and exposes the restated hot path:
march, render, per-ray backward, regularizers, G^T fold and a full train step.
Used only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .refcore import ORACLE_SO, HERE, RefCamera, RefRenderOpts, RefStepParams, ptr, _dp, _ip, _lp

_lib = None


def build_oracle():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(ORACLE_SO):
        build_oracle()
    L = C.CDLL(ORACLE_SO)
    L.og_create.restype = C.c_void_p
    L.og_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, C.c_double, _dp,
                            C.c_double, _ip, _ip, _ip, _dp, _dp, _dp, _dp, _dp, C.c_int]
    L.og_free.argtypes = [C.c_void_p]
    L.og_mlp_size.restype = C.c_int64
    L.og_mlp_size.argtypes = [C.c_void_p]
    L.og_export.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
    L.og_smooth_all.argtypes = [C.c_void_p]
    L.og_march_ray.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp]
    L.og_pixel_dir.argtypes = [C.POINTER(RefCamera), C.c_double, C.c_double, _dp]
    L.og_pixel_dirs.argtypes = [C.POINTER(RefCamera), _dp]
    L.og_render_ray.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(RefRenderOpts), _dp]
    L.og_render_image.argtypes = [C.c_void_p, C.POINTER(RefCamera), C.POINTER(RefRenderOpts), _dp, _dp,
                                  _dp, _lp]
    L.og_grads_new.restype = C.c_void_p
    L.og_grads_new.argtypes = [C.c_void_p]
    L.og_grads_free.argtypes = [C.c_void_p]
    L.og_grads_clear.argtypes = [C.c_void_p, C.c_void_p]
    L.og_grads_export.argtypes = [C.c_void_p, C.c_void_p, _dp, _dp, _dp, _dp, _dp]
    L.og_ray_backward.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(RefRenderOpts), _dp, C.c_double,
                                  C.c_void_p]
    L.og_photo_pixel.argtypes = [_dp, _dp, C.c_int, C.c_double, C.c_double, _dp]
    L.og_regularizer.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p, _dp]
    L.og_gt_fold.argtypes = [C.c_void_p, C.c_void_p]
    L.og_train_reset.argtypes = [C.c_void_p]
    L.og_train_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(RefCamera), C.POINTER(_dp),
                                C.POINTER(_dp), C.POINTER(RefStepParams), _dp, _lp, C.c_void_p,
                                C.c_void_p]
    L.og_regularizer_range.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_void_p, _dp]
    L.og_raypass_tiles.argtypes = [C.c_void_p, C.c_int, C.POINTER(RefCamera), C.POINTER(_dp),
                                   C.POINTER(_dp), C.POINTER(RefStepParams), C.c_int64, C.c_int64,
                                   C.c_void_p, _dp]
    L.og_alpha_from_sdf.restype = C.c_double
    L.og_alpha_from_sdf.argtypes = [C.c_double, C.c_double, C.c_double]
    L.og_sh_basis.argtypes = [_dp, C.c_int, _dp]
    L.og_fresnel_powers.argtypes = [C.c_double, _dp]
    L.og_gaussian_taps.argtypes = [_dp]
    L.og_adam_steps.argtypes = [C.c_int, _dp, _dp, C.c_int, _dp]
    _lib = L
    return L


class OracleGrid:
    """The C restatement's grid, built from a GridArrays description."""

    def __init__(self, a, smooth=True):
        """a: GridArrays (see refcore.GridArrays). smooth=True installs a.smooth
        verbatim; False recomputes it from a.raw (grid.cpp:247-250)."""
        self.L = lib()
        self.a = a
        f = lambda x: np.ascontiguousarray(x, np.float64)
        i = lambda x: np.ascontiguousarray(x, np.int32)
        res = np.array(a.res, np.int32)
        org = np.array(a.origin, np.float64)
        self._keep = [f(a.raw), f(a.smooth), f(a.planes), f(a.probes), f(a.mlp), i(a.tile_coords),
                      i(a.probe_ids), i(a.probe_coords), res, org]
        raw, sm, pl, pr, mlp, tc, pid, pc, res, org = self._keep
        self.h = C.c_void_p(self.L.og_create(a.T, a.P, a.n_s, a.n_a, a.sh_order, ptr(res, _ip),
                                             a.voxel_size, ptr(org), a.far_field_voxels, ptr(tc, _ip),
                                             ptr(pid, _ip), ptr(pc, _ip), ptr(raw),
                                             ptr(sm) if smooth else None, ptr(pl), ptr(pr), ptr(mlp),
                                             a.ncam))

    def __del__(self):
        try:
            if self.h:
                self.L.og_free(self.h)
                self.h = None
        except Exception:
            pass

    def export(self):
        a = self.a
        out = dict(raw=np.zeros_like(a.raw, dtype=np.float64), smooth=np.zeros_like(a.smooth, dtype=np.float64),
                   planes=np.zeros_like(a.planes, dtype=np.float64),
                   probes=np.zeros_like(a.probes, dtype=np.float64), mlp=np.zeros_like(a.mlp, dtype=np.float64))
        self.L.og_export(self.h, ptr(out["raw"]), ptr(out["smooth"]), ptr(out["planes"]),
                         ptr(out["probes"]), ptr(out["mlp"]))
        return out

    def march_ray(self, o, d, n_max=512):
        ts = np.zeros(max(n_max, 1))
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        n = self.L.og_march_ray(self.h, ptr(o), ptr(d), n_max, ptr(ts))
        return ts[:n].copy()

    def render_image(self, cam, opts):
        w, h = cam.width, cam.height
        rgb = np.zeros((h, w, 3))
        alpha = np.zeros((h, w))
        depth = np.zeros((h, w))
        counts = np.zeros(5, np.int64)
        self.L.og_render_image(self.h, C.byref(cam), C.byref(opts), ptr(rgb), ptr(alpha), ptr(depth),
                               ptr(counts, _lp))
        return rgb, alpha, depth, counts

    def _grads(self, gb):
        a = self.a
        out = dict(raw=np.zeros(a.raw.shape), smooth=np.zeros(a.smooth.shape),
                   planes=np.zeros(a.planes.shape), probes=np.zeros(a.probes.shape),
                   mlp=np.zeros(a.mlp.shape))
        self.L.og_grads_export(self.h, gb, ptr(out["raw"]), ptr(out["smooth"]), ptr(out["planes"]),
                               ptr(out["probes"]), ptr(out["mlp"]))
        return out

    def ray_backward(self, o, d, opts, up_color, up_alpha, fold=True):
        gb = C.c_void_p(self.L.og_grads_new(self.h))
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        uc = np.asarray(up_color, np.float64)
        self.L.og_ray_backward(self.h, ptr(o), ptr(d), C.byref(opts), ptr(uc), up_alpha, gb)
        if fold:
            self.L.og_gt_fold(self.h, gb)
        g = self._grads(gb)
        self.L.og_grads_free(gb)
        return g

    def regularizer(self, which, lam):
        gb = C.c_void_p(self.L.og_grads_new(self.h))
        out = np.zeros(2)
        self.L.og_regularizer(self.h, which, lam, gb, ptr(out))
        g = self._grads(gb)
        self.L.og_grads_free(gb)
        return out, g

    def train_reset(self):
        self.L.og_train_reset(self.h)

    def new_grads(self):
        return C.c_void_p(self.L.og_grads_new(self.h))

    def free_grads(self, gb):
        self.L.og_grads_free(gb)

    def grads_of(self, gb):
        return self._grads(gb)

    def raypass_tiles(self, cams, gts, masks, hp, tile_begin, tile_end, gb):
        """Ray pass over work tiles [tile_begin, tile_end) into gb (data-parallel shard)."""
        n = len(cams)
        arr = (RefCamera * n)(*cams)
        gts = [np.ascontiguousarray(g, np.float64) for g in gts]
        masks = [np.ascontiguousarray(m, np.float64) for m in masks]
        gp = (_dp * n)(*[ptr(g) for g in gts])
        mp = (_dp * n)(*[ptr(m) for m in masks])
        out = np.zeros(3)
        self.L.og_raypass_tiles(self.h, n, arr, gp, mp, C.byref(hp), tile_begin, tile_end, gb, ptr(out))
        return out

    def regularizer_range(self, which, lam, begin, end, gb):
        out = np.zeros(2)
        self.L.og_regularizer_range(self.h, which, lam, begin, end, gb, ptr(out))
        return out

    def gt_fold_into(self, gb):
        self.L.og_gt_fold(self.h, gb)

    def train_step(self, cams, gts, masks, hp):
        n = len(cams)
        arr = (RefCamera * n)(*cams)
        gts = [np.ascontiguousarray(g, np.float64) for g in gts]
        masks = [np.ascontiguousarray(m, np.float64) for m in masks]
        gp = (_dp * n)(*[ptr(g) for g in gts])
        mp = (_dp * n)(*[ptr(m) for m in masks])
        losses = np.zeros(10)
        counts = np.zeros(6, np.int64)
        g0 = C.c_void_p(self.L.og_grads_new(self.h))
        g1 = C.c_void_p(self.L.og_grads_new(self.h))
        self.L.og_train_step(self.h, n, arr, gp, mp, C.byref(hp), ptr(losses), ptr(counts, _lp), g0, g1)
        self.last_grads = (self._grads(g0), self._grads(g1))
        self.L.og_grads_free(g0)
        self.L.og_grads_free(g1)
        return losses, counts


def pixel_dir(cam, u, v):
    d = np.zeros(3)
    lib().og_pixel_dir(C.byref(cam), u, v, ptr(d))
    return d


def pixel_dirs(cam):
    """og_pixel_dir at every pixel centre, [height][width][3]."""
    d = np.zeros((cam.height, cam.width, 3))
    lib().og_pixel_dirs(C.byref(cam), ptr(d))
    return d


def step_params(tau, lr_vox, lr_mlp, l_sdf=0.7, l_eik=0.3, l_norm=0.2, l_feat=0.15, l_probe=0.25,
                photo_scale=20.0, use_camera_bias=False):
    hp = RefStepParams()
    hp.tau, hp.lr_vox, hp.lr_mlp = tau, lr_vox, lr_mlp
    hp.l_sdf, hp.l_eik, hp.l_norm, hp.l_feat, hp.l_probe = l_sdf, l_eik, l_norm, l_feat, l_probe
    hp.photo_scale = photo_scale
    hp.use_camera_bias = int(use_camera_bias)
    return hp


def work_tiles(cams):
    """Number of 8x4-pixel work tiles of a batch (the CUDA path's ray partition)."""
    return sum(((c.width + 7) // 8) * ((c.height + 3) // 4) for c in cams)


def kat_alpha(si, sn, tau):
    return lib().og_alpha_from_sdf(si, sn, tau)


def kat_sh(direction, order):
    out = np.zeros(16)
    d = np.asarray(direction, np.float64)
    lib().og_sh_basis(ptr(d), order, ptr(out))
    return out[: order * order]


def kat_fresnel(ndv):
    out = np.zeros(6)
    lib().og_fresnel_powers(ndv, ptr(out))
    return out


def kat_gaussian():
    out = np.zeros(5)
    lib().og_gaussian_taps(ptr(out))
    return out


def kat_adam(params, grads_seq, lrs):
    p = np.ascontiguousarray(params, np.float64).copy()
    g = np.ascontiguousarray(grads_seq, np.float64)
    lr = np.ascontiguousarray(lrs, np.float64)
    lib().og_adam_steps(p.size, ptr(p), ptr(g), len(lr), ptr(lr))
    return p


def psnr_masked(img, gt, mask):
    """metrics.cpp:196-211 restated: squared error over the three channels of
    every pixel with mask > 0.5, summed in row-major pixel order in f64; 99 dB
    when no pixel is masked or the error is 0, capped at 99.  Pure Python loop
    (small images only) so the summation order is the reference's."""
    img = np.asarray(img, np.float64)
    gt = np.asarray(gt, np.float64)
    mask = np.asarray(mask, np.float64)
    if img.shape != gt.shape:
        raise ValueError("psnr_masked: image shape mismatch")
    h, w = mask.shape
    sq, n = 0.0, 0
    for v in range(h):
        for u in range(w):
            if mask[v, u] <= 0.5:
                continue
            dx = img[v, u, 0] - gt[v, u, 0]
            dy = img[v, u, 1] - gt[v, u, 1]
            dz = img[v, u, 2] - gt[v, u, 2]
            sq += (dx * dx + dy * dy) + dz * dz  # Vec3::norm2 (vec.hpp)
            n += 3
    if n == 0:
        return 99.0
    mse = sq / n
    if mse <= 0.0:
        return 99.0
    return min(99.0, 10.0 * np.log10(1.0 / mse))


def _dot(a, b):  # Vec3::dot (vec.hpp:26): (x*x' + y*y') + z*z'
    return (a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1]) + a[..., 2] * b[..., 2]


def _norm(a):
    return np.sqrt(_dot(a, a))


def point_triangle_distances(p, a, b, c):
    """metrics.cpp:11-47 (Ericson's closest point) restated over arrays of
    triangles for one point; every branch is evaluated in the reference's
    operation order and the first region that applies is selected, so each
    value is the reference's f64 result bit for bit."""
    with np.errstate(divide="ignore", invalid="ignore"):
        ab, ac, ap = b - a, c - a, p - a
        d1, d2 = _dot(ab, ap), _dot(ac, ap)
        bp = p - b
        d3, d4 = _dot(ab, bp), _dot(ac, bp)
        vc = d1 * d4 - d3 * d2
        cp = p - c
        d5, d6 = _dot(ab, cp), _dot(ac, cp)
        vb = d5 * d2 - d1 * d6
        va = d3 * d6 - d5 * d4
        v_ab = d1 / (d1 - d3)
        w_ac = d2 / (d2 - d6)
        w_bc = (d4 - d3) / ((d4 - d3) + (d5 - d6))
        denom = 1.0 / ((va + vb) + vc)
        v_in, w_in = vb * denom, vc * denom
        conds = [(d1 <= 0.0) & (d2 <= 0.0),
                 (d3 >= 0.0) & (d4 <= d3),
                 (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0),
                 (d6 >= 0.0) & (d5 <= d6),
                 (vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0),
                 (va <= 0.0) & ((d4 - d3) >= 0.0) & ((d5 - d6) >= 0.0)]
        vals = [_norm(p - a), _norm(p - b), _norm(p - (a + ab * v_ab[:, None])), _norm(p - c),
                _norm(p - (a + ac * w_ac[:, None])), _norm(p - (b + (c - b) * w_bc[:, None]))]
        inside = _norm(p - ((a + ab * v_in[:, None]) + ac * w_in[:, None]))
    return np.select(conds, vals, inside)


def point_mesh_distance(points, verts, tris):
    """MeshDistance::distance (metrics.cpp:131-135) as a brute-force minimum
    over the triangles (the BVH only prunes; test_geometry.cpp:212-226 checks
    it against this scan)."""
    v = np.asarray(verts, np.float64)
    t = np.asarray(tris, np.int64)
    if len(t) == 0:
        raise ValueError("MeshDistance: empty mesh")
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    # best = std::min(best, d) from numeric_limits<double>::max(): a NaN
    # distance (degenerate triangle) never replaces best, which fmin mirrors
    return np.array([np.fmin.reduce(point_triangle_distances(np.asarray(p, np.float64), a, b, c),
                                    initial=np.finfo(np.float64).max) for p in points])


def chamfer(pred_pts, pred_verts, pred_tris, gt_pts, gt_verts, gt_tris, max_dist):
    """metrics.cpp:168-194: two-way mean point-to-mesh distance x1000, points
    beyond max_dist (> 0) excluded, summed in point order."""
    if len(pred_pts) == 0 or len(gt_pts) == 0 or len(pred_tris) == 0 or len(gt_tris) == 0:
        raise ValueError("chamfer: empty input")

    def mean(d):
        s, n = 0.0, 0
        for x in d:
            if max_dist > 0.0 and x > max_dist:
                continue
            s += float(x)
            n += 1
        return s / n if n else 0.0
    acc = 1000.0 * mean(point_mesh_distance(pred_pts, gt_verts, gt_tris))
    comp = 1000.0 * mean(point_mesh_distance(gt_pts, pred_verts, pred_tris))
    return np.array([acc, comp, 0.5 * (acc + comp)])
