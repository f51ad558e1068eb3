"""Host-side mirror of the reference's hot-path API (include/sdfrecon/*.hpp),
driving the CUDA path through the C ABI (include/psdf.h).

Names follow the reference: ``GridConfig``, ``init_grid_sphere``,
``make_lookat_camera`` / ``make_ring_cameras``, ``RenderOptions``,
``render_image``, ``Bracket`` / ``warmup_scale`` and a ``Trainer`` whose
``step`` is one iteration of ``train()``'s loop body (trainer.cpp:125-209).
Errors map to the reference's exception types (ValueError for
std::invalid_argument, IndexError for std::out_of_range, RuntimeError for
std::runtime_error).

Host arrays use the flat layouts documented in include/psdf.h.  Grid
construction here is plain numpy (it runs once per LOD, outside the hot path).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (check, psdf_camera, psdf_counts, psdf_grid_desc, psdf_losses, psdf_render_opts,
                   psdf_step_params)

TILE = 16
HIDDEN = 32
FRESNEL_POWERS = 6


# ----------------------------------------------------------------- cameras
def make_lookat_camera(id, eye, target, up, fx, fy, width, height) -> psdf_camera:
    """camera.cpp:5-23."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd = fwd / math.sqrt((fwd[0] * fwd[0] + fwd[1] * fwd[1]) + fwd[2] * fwd[2])

    def cross(a, b):
        return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]])

    def normalized(v):
        n = math.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])
        return v / n if n > 0 else np.zeros(3)

    right = normalized(cross(fwd, np.asarray(up, np.float64)))
    if math.sqrt(float(right @ right)) < 1e-9:
        right = normalized(cross(fwd, np.array([1.0, 0, 0])))
    down = cross(fwd, right)
    c = psdf_camera()
    c.id = id
    c.fx, c.fy = fx, fy
    c.cx, c.cy = (width - 1) * 0.5, (height - 1) * 0.5
    c.width, c.height = width, height
    c.pos[:] = list(eye)
    c.rot[:] = [right[0], down[0], fwd[0], right[1], down[1], fwd[1], right[2], down[2], fwd[2]]
    return c


def make_ring_cameras(n_views, resolution, radius=2.0, elevation=0.35, seed=0, height=None):
    """synth.cpp:238-255 (ring of look-at cameras, f = 1.2 * H); ``height``
    allows non-square images for the 1600x1200 / 2048x1536 configs."""
    w = resolution
    h = resolution if height is None else height
    phase = (seed % 360) * math.pi / 180.0
    f = h * 1.2
    cams = []
    for i in range(n_views):
        az = phase + 2.0 * math.pi * i / n_views
        el = elevation * (1.0 if i % 2 == 0 else -1.0)
        eye = (radius * math.cos(el) * math.cos(az), radius * math.sin(el),
               radius * math.cos(el) * math.sin(az))
        cams.append(make_lookat_camera(i, eye, (0, 0, 0), (0, 1, 0), f, f, w, h))
    return cams


def camera_from(obj) -> psdf_camera:
    """Accepts a psdf_camera or any struct with the same fields (e.g. the oracle's)."""
    if isinstance(obj, psdf_camera):
        return obj
    c = psdf_camera()
    for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
        setattr(c, k, getattr(obj, k))
    c.rot[:] = list(obj.rot)
    c.pos[:] = list(obj.pos)
    return c


# ----------------------------------------------------------------- options
@dataclass
class RenderOptions:
    """renderer.hpp:13-27."""
    tau: float = 100.0
    n_max: int = 512
    early_stop_transmittance: float = 1e-4
    background: tuple = (0.0, 0.0, 0.0)
    camera_id: int = -1
    no_spatial: bool = False
    no_angular: bool = False
    no_fresnel: bool = False
    sh_order_override: int = -1
    need_colors: bool = True

    def to_c(self) -> psdf_render_opts:
        o = psdf_render_opts()
        o.tau = self.tau
        o.n_max = self.n_max
        o.early_stop = self.early_stop_transmittance
        o.bg[:] = list(self.background)
        o.camera_id = self.camera_id
        o.no_spatial, o.no_angular, o.no_fresnel = int(self.no_spatial), int(self.no_angular), int(self.no_fresnel)
        o.sh_order_override = self.sh_order_override
        o.need_colors = int(self.need_colors)
        return o


@dataclass
class Bracket:
    """schedule.hpp:11-30."""
    a: float
    b: float | None = None

    def __post_init__(self):
        if self.b is None:
            self.b = self.a

    def at(self, it, total):
        if total <= 1:
            return self.a
        t = it / (total - 1)
        return self.a + (self.b - self.a) * t

    def at_geometric(self, it, total):
        if total <= 1:
            return self.a
        t = it / (total - 1)
        return self.a * math.pow(self.b / self.a, t)


def warmup_scale(it):
    """schedule.hpp:58-60."""
    return (it + 1) / 50.0 if it < 50 else 1.0


@dataclass
class LodSchedule:
    """schedule.hpp:32-45 defaults."""
    iterations: int = 0
    images_per_batch: int = 1
    sh_order: int = 2
    image_divisor: int = 1
    lr_voxels: Bracket = field(default_factory=lambda: Bracket(1e-2))
    lr_mlp: Bracket = field(default_factory=lambda: Bracket(1e-3))
    lambda_eik: Bracket = field(default_factory=lambda: Bracket(0.1))
    lambda_sdf: Bracket = field(default_factory=lambda: Bracket(1.0))
    lambda_features: Bracket = field(default_factory=lambda: Bracket(0.01))
    lambda_normal: Bracket = field(default_factory=lambda: Bracket(0.01))
    lambda_probes: Bracket = field(default_factory=lambda: Bracket(0.01))
    tau: Bracket = field(default_factory=lambda: Bracket(30.0, 3000.0))

    def step_params(self, it, voxel_size, lambda_photo=40.0, camera_bias=False) -> psdf_step_params:
        """Per-iteration hyper-parameters exactly as trainer.cpp:126-134."""
        n = self.iterations
        hp = psdf_step_params()
        hp.lr_vox = self.lr_voxels.at(it, n) * warmup_scale(it)
        hp.lr_mlp = self.lr_mlp.at(it, n) * warmup_scale(it)
        hp.l_sdf = self.lambda_sdf.at(it, n)
        hp.l_eik = self.lambda_eik.at(it, n)
        hp.l_norm = self.lambda_normal.at(it, n)
        hp.l_feat = self.lambda_features.at(it, n)
        hp.l_probe = self.lambda_probes.at(it, n)
        hp.tau = self.tau.at_geometric(it, n) / voxel_size
        hp.photo_scale = lambda_photo / self.images_per_batch
        hp.use_camera_bias = int(camera_bias)
        return hp


def step_params(tau, lr_vox, lr_mlp, l_sdf=0.7, l_eik=0.3, l_norm=0.2, l_feat=0.15, l_probe=0.25,
                photo_scale=20.0, use_camera_bias=False) -> psdf_step_params:
    hp = psdf_step_params()
    hp.tau, hp.lr_vox, hp.lr_mlp = tau, lr_vox, lr_mlp
    hp.l_sdf, hp.l_eik, hp.l_norm, hp.l_feat, hp.l_probe = l_sdf, l_eik, l_norm, l_feat, l_probe
    hp.photo_scale = photo_scale
    hp.use_camera_bias = int(use_camera_bias)
    return hp


# ----------------------------------------------------------------- grid
@dataclass
class GridConfig:
    """grid.hpp:42-51."""
    voxel_size: float = 1.0 / 16.0
    origin: tuple = (-0.5, -0.5, -0.5)
    resolution: tuple = (16, 16, 16)
    n_s: int = 4
    n_a: int = 4
    sh_order: int = 2
    far_field_voxels: float = 4.0
    band_voxels: int = 6


class HostGrid:
    """A SparseGrid + DecoderMlp in the flat upload layout (fp32)."""

    def __init__(self, cfg: GridConfig, tile_coords, probe_ids, probe_coords, raw, planes, probes,
                 mlp, ncam=0, smooth=None):
        self.cfg = cfg
        self.tile_coords = np.ascontiguousarray(tile_coords, np.int32).reshape(-1, 3)
        self.probe_ids = np.ascontiguousarray(probe_ids, np.int32).reshape(-1, 8)
        self.probe_coords = np.ascontiguousarray(probe_coords, np.int32).reshape(-1, 3)
        self.raw = np.ascontiguousarray(raw, np.float32).reshape(-1, 4096)
        self.smooth = None if smooth is None else np.ascontiguousarray(smooth, np.float32).reshape(-1, 4096)
        self.planes = np.ascontiguousarray(planes, np.float32)
        self.probes = np.ascontiguousarray(probes, np.float32)
        self.mlp = np.ascontiguousarray(mlp, np.float32)
        self.ncam = ncam

    @property
    def T(self):
        return self.tile_coords.shape[0]

    @property
    def P(self):
        return self.probe_coords.shape[0]

    def desc(self) -> psdf_grid_desc:
        d = psdf_grid_desc()
        c = self.cfg
        d.T, d.P = self.T, self.P
        d.n_s, d.n_a, d.sh_order = c.n_s, c.n_a, c.sh_order
        d.res[:] = list(c.resolution)
        d.voxel_size = c.voxel_size
        d.origin[:] = list(c.origin)
        d.far_field_voxels = c.far_field_voxels
        d.ncam = self.ncam
        return d

    @classmethod
    def from_arrays(cls, a, ncam=None):
        """From an oracle/refcore GridArrays-like object (f64 arrays are rounded to fp32)."""
        cfg = GridConfig(voxel_size=a.voxel_size, origin=tuple(a.origin), resolution=tuple(a.res),
                         n_s=a.n_s, n_a=a.n_a, sh_order=a.sh_order,
                         far_field_voxels=a.far_field_voxels)
        return cls(cfg, a.tile_coords, a.probe_ids, a.probe_coords, a.raw, a.planes, a.probes, a.mlp,
                   ncam=a.ncam if ncam is None else ncam, smooth=getattr(a, "smooth", None))


def glorot_mlp(n_s, n_a, ncam, seed) -> np.ndarray:
    """Glorot-uniform MLP with the decoder.cpp:9-30 shapes and bounds (numpy RNG;
    the reference uses mt19937_64, so values differ but the distribution matches)."""
    rng = np.random.default_rng(seed)
    n_in = n_s + n_a + FRESNEL_POWERS

    def fill(fan_in, fan_out, count):
        b = math.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-b, b, count)

    parts = [fill(n_in, HIDDEN, HIDDEN * n_in), np.zeros(HIDDEN), fill(HIDDEN, HIDDEN, HIDDEN * HIDDEN),
             np.zeros(HIDDEN), fill(HIDDEN, 3, 3 * HIDDEN), np.zeros(3), np.zeros(ncam * HIDDEN)]
    return np.concatenate(parts).astype(np.float32)


def init_grid_sphere(cfg: GridConfig, center, radius, ncam=0, mlp_seed=0, sdf_fn=None) -> HostGrid:
    """init_grid_sphere / init_common (grid.cpp:359-398, 462-467), vectorised:
    tiles whose 16^3 block has |s| <= band somewhere or a sign change are
    allocated in (tx, ty, tz) order; corner probes are created in allocation
    order (grid.cpp:58-76).  ``sdf_fn(points[N,3]) -> s[N]`` overrides the
    sphere (used for union scenes)."""
    res = np.array(cfg.resolution)
    if np.any(res % TILE):
        raise ValueError("grid resolution must be a multiple of 16")
    nt = res // TILE
    center = np.asarray(center, np.float64)
    band = cfg.band_voxels * cfg.voxel_size
    org = np.asarray(cfg.origin, np.float64)
    loc = (np.arange(TILE) + 0.5)
    tiles, raws = [], []
    for tx in range(nt[0]):
        xs = org[0] + (tx * TILE + loc) * cfg.voxel_size
        for ty in range(nt[1]):
            ys = org[1] + (ty * TILE + loc) * cfg.voxel_size
            # all tz at once: [nt2, 16, 16, 16]
            zs = org[2] + (np.arange(nt[2])[:, None] * TILE + loc[None, :]) * cfg.voxel_size
            X = xs[None, :, None, None]
            Y = ys[None, None, :, None]
            Z = zs[:, None, None, :]
            if sdf_fn is None:
                s = np.sqrt((X - center[0]) ** 2 + (Y - center[1]) ** 2 + (Z - center[2]) ** 2) - radius
            else:
                P = np.stack(np.broadcast_arrays(X, Y, Z), -1).reshape(-1, 3)
                s = sdf_fn(P).reshape(nt[2], TILE, TILE, TILE)
            s = s.reshape(nt[2], -1)
            keep = (np.abs(s).min(1) <= band) | ((s >= 0).any(1) & (s < 0).any(1))
            for tz in np.nonzero(keep)[0]:
                tiles.append((tx, ty, int(tz)))
                raws.append(s[tz])
    T = len(tiles)
    probe_index = {}
    probe_coords = []
    probe_ids = np.zeros((T, 8), np.int32)
    for t, (tx, ty, tz) in enumerate(tiles):
        for i in range(8):
            key = (tx + (i & 1), ty + ((i >> 1) & 1), tz + ((i >> 2) & 1))
            if key not in probe_index:
                probe_index[key] = len(probe_coords)
                probe_coords.append(key)
            probe_ids[t, i] = probe_index[key]
    nc = cfg.sh_order * cfg.sh_order
    raw = np.array(raws, np.float64).reshape(T, 4096) if T else np.zeros((0, 4096))
    planes = np.full((T, 3, 256, cfg.n_s), 0.5, np.float32)
    probes = np.zeros((len(probe_coords), nc, cfg.n_a), np.float32)
    mlp = glorot_mlp(cfg.n_s, cfg.n_a, ncam, mlp_seed)
    return HostGrid(cfg, np.array(tiles, np.int32).reshape(-1, 3), probe_ids,
                    np.array(probe_coords, np.int32).reshape(-1, 3), raw, planes, probes, mlp, ncam=ncam)


def analytic_sdf(prims):
    """Union-of-primitives SDF (synth.cpp:17-35, 142-154); prims = [(kind, center, extent)],
    kind 0 sphere / 1 box / 2 torus."""
    def f(P):
        best = np.full(P.shape[0], np.inf)
        for kind, c, e in prims:
            q = P - np.asarray(c, np.float64)
            if kind == 0:
                d = np.sqrt((q * q).sum(1)) - e[0]
            elif kind == 1:
                dd = np.abs(q) - np.asarray(e, np.float64)
                out = np.maximum(dd, 0.0)
                d = np.sqrt((out * out).sum(1)) + np.minimum(dd.max(1), 0.0)
            else:
                qx = np.sqrt(q[:, 0] ** 2 + q[:, 2] ** 2) - e[0]
                d = np.sqrt(qx * qx + q[:, 1] ** 2) - e[1]
            best = np.minimum(best, d)
        return best
    return f


# The named synthetic shapes of BASELINE.json's configs, as primitive unions
# for analytic_sdf / init_grid_analytic ((kind, center, extent); kind 0 sphere
# radius extent[0], 1 box half-extents, 2 torus (major, minor) in the xz plane
# about +y, synth.cpp:17-35).
#   sphere: the acceptance scene's sphere (acceptance.cpp:54-74, r = 0.3)
#   torus:  configs[0]'s torus (major 0.25, minor 0.1)
#   human:  configs[2]'s MVMannequins-like figure (a union
#           of boxes, spheres and tori standing in the unit cube); the
#           reference has no human asset, so this union is this repo's.
SCENE_PRIMS = {
    "sphere": [(0, (0.0, 0.0, 0.0), (0.3, 0.0, 0.0))],
    "torus": [(2, (0.0, 0.0, 0.0), (0.25, 0.1, 0.0))],
    "human": [
        (0, (0.0, 0.335, 0.0), (0.065, 0.0, 0.0)),        # head
        (1, (0.0, 0.255, 0.0), (0.025, 0.03, 0.025)),     # neck
        (1, (0.0, 0.10, 0.0), (0.115, 0.135, 0.06)),      # torso
        (2, (0.0, -0.045, 0.0), (0.1, 0.03, 0.0)),        # belt
        (1, (0.0, -0.07, 0.0), (0.1, 0.05, 0.055)),       # pelvis
        (1, (-0.055, -0.265, 0.0), (0.04, 0.16, 0.042)),  # legs
        (1, (0.055, -0.265, 0.0), (0.04, 0.16, 0.042)),
        (1, (-0.055, -0.43, 0.025), (0.042, 0.018, 0.07)),  # feet
        (1, (0.055, -0.43, 0.025), (0.042, 0.018, 0.07)),
        (0, (-0.15, 0.215, 0.0), (0.045, 0.0, 0.0)),      # shoulders
        (0, (0.15, 0.215, 0.0), (0.045, 0.0, 0.0)),
        (1, (-0.175, 0.075, 0.0), (0.03, 0.13, 0.03)),    # arms
        (1, (0.175, 0.075, 0.0), (0.03, 0.13, 0.03)),
        (0, (-0.175, -0.07, 0.0), (0.035, 0.0, 0.0)),     # hands
        (0, (0.175, -0.07, 0.0), (0.035, 0.0, 0.0)),
    ],
}


def init_grid_analytic(cfg: GridConfig, prims, ncam=0, mlp_seed=0) -> HostGrid:
    """A grid allocated and filled from a union of primitives (the reference's
    dense-overwrite pattern, test_grid.cpp:29-43, with init_common's tile
    rule, grid.cpp:359-398): `prims` is a list for analytic_sdf or a key of
    SCENE_PRIMS."""
    if isinstance(prims, str):
        prims = SCENE_PRIMS[prims]
    return init_grid_sphere(cfg, (0, 0, 0), 0.0, ncam=ncam, mlp_seed=mlp_seed, sdf_fn=analytic_sdf(prims))


# ----------------------------------------------------------------- context
def _fptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


def _iptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


def _train_mask(m):
    """A training / evaluation mask as the ABI's 0/1 bytes.  Floats follow the
    reference's ImageGray test `mask > 0.5` (trainer.cpp:166, metrics.cpp:203);
    uint8 images are 8-bit masks as loaded from disk (value / 255 > 0.5, i.e.
    the `> 127` of MaskImage::foreground, grid.hpp:143-146) so that every entry
    point, the visual hull included, classifies a byte mask the same way; bool
    masks pass through."""
    m = np.asarray(m)
    if m.dtype == np.bool_:
        return np.ascontiguousarray(m, np.uint8)
    if m.dtype == np.uint8:
        return np.ascontiguousarray(m > 127, np.uint8)
    return np.ascontiguousarray(m > 0.5, np.uint8)


class Context:
    """One GPU's hot-path state (psdf_ctx)."""

    def __init__(self, device=0):
        self.L = _lib.load()
        h = C.c_void_p()
        check(self.L.psdf_create(device, C.byref(h)))
        self.h = h
        self.grid = None

    def close(self):
        if getattr(self, "h", None):
            self.L.psdf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        check(rc, self.h)

    # -- state
    def upload(self, grid: HostGrid, smooth=True):
        self.grid = grid
        sm = grid.smooth if (smooth and grid.smooth is not None) else None
        d = grid.desc()
        self._check(self.L.psdf_upload_grid(self.h, C.byref(d), _iptr(grid.tile_coords),
                                            _iptr(grid.probe_ids), _iptr(grid.probe_coords),
                                            _fptr(grid.raw), _fptr(sm), _fptr(grid.planes),
                                            _fptr(grid.probes)))
        self._check(self.L.psdf_upload_mlp(self.h, _fptr(grid.mlp), grid.mlp.size))

    def download(self):
        g = self.grid
        out = dict(raw=np.zeros((g.T, 4096), np.float32), smooth=np.zeros((g.T, 4096), np.float32),
                   planes=np.zeros(g.planes.shape, np.float32), probes=np.zeros(g.probes.shape, np.float32),
                   mlp=np.zeros(g.mlp.shape, np.float32))
        self._check(self.L.psdf_download_params(self.h, _fptr(out["raw"]), _fptr(out["smooth"]),
                                                _fptr(out["planes"]), _fptr(out["probes"]),
                                                _fptr(out["mlp"])))
        return out

    def info(self):
        """psdf_grid_info: the device grid's metadata at the caller's widths."""
        d = psdf_grid_desc()
        self._check(self.L.psdf_grid_info(self.h, C.byref(d)))
        return d

    # -- LOD transitions (trainer.cpp:105, 213)
    def _refresh_grid(self):
        """Re-reads the device grid's structure and parameters into self.grid."""
        d = self.info()
        old = self.grid.cfg
        cfg = GridConfig(voxel_size=d.voxel_size, origin=tuple(d.origin), resolution=tuple(d.res),
                         n_s=d.n_s, n_a=d.n_a, sh_order=d.sh_order, far_field_voxels=d.far_field_voxels,
                         band_voxels=old.band_voxels)
        tc = np.zeros((d.T, 3), np.int32)
        pid = np.zeros((d.T, 8), np.int32)
        pco = np.zeros((d.P, 3), np.int32)
        self._check(self.L.psdf_download_structure(self.h, _iptr(tc), _iptr(pid), _iptr(pco)))
        nc = d.sh_order * d.sh_order
        g = HostGrid(cfg, tc, pid, pco, np.zeros((d.T, 4096), np.float32),
                     np.zeros(d.T * 3 * 256 * d.n_s, np.float32), np.zeros(d.P * nc * d.n_a, np.float32),
                     np.zeros(self.grid.mlp.shape, np.float32), ncam=d.ncam,
                     smooth=np.zeros((d.T, 4096), np.float32))
        self._check(self.L.psdf_download_params(self.h, _fptr(g.raw), _fptr(g.smooth), _fptr(g.planes),
                                                _fptr(g.probes), _fptr(g.mlp)))
        self.grid = g
        return g

    def subdivide(self, band_voxels=None):
        """grid = grid.subdivide() (grid.cpp:271-345) on the device; returns the new HostGrid."""
        bv = self.grid.cfg.band_voxels if band_voxels is None else band_voxels
        self._check(self.L.psdf_subdivide(self.h, float(bv), None, None))
        return self._refresh_grid()

    def save_checkpoint(self, path, lod=0, lod_cursor=0, iteration=0, seed=0):
        """save_checkpoint (checkpoint.cpp:54-104) of the device grid + decoder."""
        self._check(self.L.psdf_save_checkpoint(self.h, str(path).encode(), int(lod),
                                                int(self.grid.cfg.band_voxels), int(lod_cursor),
                                                int(iteration), int(seed)))

    def load_checkpoint(self, path):
        """load_checkpoint (checkpoint.cpp:106-181) into the device; returns
        (HostGrid, dict(lod, band_voxels, lod_cursor, iteration, seed))."""
        lod, band, cur = C.c_int32(), C.c_int32(), C.c_int32()
        it, sd = C.c_int64(), C.c_uint64()
        self._check(self.L.psdf_load_checkpoint(self.h, str(path).encode(), C.byref(lod), C.byref(band),
                                                C.byref(cur), C.byref(it), C.byref(sd)))
        d = psdf_grid_desc()
        self._check(self.L.psdf_grid_info(self.h, C.byref(d)))
        cfg = GridConfig(voxel_size=d.voxel_size, origin=tuple(d.origin), resolution=tuple(d.res), n_s=d.n_s,
                         n_a=d.n_a, sh_order=d.sh_order, far_field_voxels=d.far_field_voxels,
                         band_voxels=band.value)
        self.grid = HostGrid(cfg, np.zeros((0, 3)), np.zeros((0, 8)), np.zeros((0, 3)), np.zeros((0, 4096)),
                             np.zeros(0), np.zeros(0), np.zeros(self.L.psdf_mlp_size(d.n_s, d.n_a, d.ncam)),
                             ncam=d.ncam)
        g = self._refresh_grid()
        return g, dict(lod=lod.value, band_voxels=band.value, lod_cursor=cur.value, iteration=it.value,
                       seed=sd.value)

    def init_visual_hull(self, cfg: GridConfig, cameras, masks, ncam=0):
        """init_grid_visual_hull (grid.cpp:470-504) on the device; masks are uint8
        images (> 127 = foreground).  Returns the new HostGrid (MLP zero)."""
        d = psdf_grid_desc()
        d.n_s, d.n_a, d.sh_order = cfg.n_s, cfg.n_a, cfg.sh_order
        d.res[:] = list(cfg.resolution)
        d.voxel_size = cfg.voxel_size
        d.origin[:] = list(cfg.origin)
        d.far_field_voxels = cfg.far_field_voxels
        d.ncam = ncam
        n = len(cameras)
        cam_arr = (psdf_camera * n)(*cameras)
        ms = [np.ascontiguousarray(m, np.uint8) for m in masks]
        mp = (C.POINTER(C.c_uint8) * n)(*[m.ctypes.data_as(C.POINTER(C.c_uint8)) for m in ms])
        self._check(self.L.psdf_init_visual_hull(self.h, C.byref(d), int(cfg.band_voxels), n, cam_arr, mp,
                                                 None, None))
        self.grid = HostGrid(cfg, np.zeros((0, 3)), np.zeros((0, 8)), np.zeros((0, 3)), np.zeros((0, 4096)),
                             np.zeros(0), np.zeros(0), np.zeros(self.L.psdf_mlp_size(cfg.n_s, cfg.n_a, ncam)), ncam=ncam)
        return self._refresh_grid()

    def raise_sh_order(self, order):
        """SparseGrid::raise_sh_order (grid.cpp:252-262) on the device."""
        self._check(self.L.psdf_raise_sh_order(self.h, int(order)))
        return self._refresh_grid()

    def grads(self, stage=1):
        g = self.grid
        out = dict(raw=np.zeros((g.T, 4096), np.float32), smooth=np.zeros((g.T, 4096), np.float32),
                   planes=np.zeros(g.planes.shape, np.float32), probes=np.zeros(g.probes.shape, np.float32),
                   mlp=np.zeros(g.mlp.shape, np.float32))
        self._check(self.L.psdf_download_grads(self.h, stage, _fptr(out["raw"]), _fptr(out["smooth"]),
                                               _fptr(out["planes"]), _fptr(out["probes"]),
                                               _fptr(out["mlp"])))
        return out

    def keep_raypass_grads(self, keep=True):
        self._check(self.L.psdf_set_keep_raypass_grads(self.h, int(keep)))

    def smooth_all(self):
        self._check(self.L.psdf_smooth_all(self.h))

    # -- render (render_image, renderer.cpp:321-337)
    def render_image(self, camera, opts: RenderOptions, depth=True):
        cam = camera_from(camera)
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        alpha = np.zeros((cam.height, cam.width), np.float32)
        dep = np.zeros((cam.height, cam.width), np.float32) if depth else None
        counts = psdf_counts()
        o = opts.to_c()
        self._check(self.L.psdf_render(self.h, C.byref(cam), C.byref(o), _fptr(rgb), _fptr(alpha),
                                       _fptr(dep), C.byref(counts)))
        return rgb, alpha, dep, counts.as_dict()

    def eval_psnr(self, camera, opts: RenderOptions, gt_rgb, mask):
        """psnr_masked(render_image(...).rgb, gt, mask) (metrics.cpp:196-211) with
        the render and the masked reduction on the GPU; `mask` as in train_step
        (see _train_mask)."""
        cam = camera_from(camera)
        gt = np.ascontiguousarray(gt_rgb, np.float32)
        m = _train_mask(mask)
        if gt.shape != (cam.height, cam.width, 3) or m.shape != (cam.height, cam.width):
            raise ValueError("psnr_masked: image shape mismatch")
        out = C.c_double()
        counts = psdf_counts()
        o = opts.to_c()
        self._check(self.L.psdf_eval_psnr(self.h, C.byref(cam), C.byref(o), _fptr(gt),
                                          m.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(out),
                                          C.byref(counts)))
        return out.value

    def point_mesh_distance(self, points, verts, tris):
        """MeshDistance(mesh).distance(p) for every point (metrics.cpp:131-135),
        on the GPU; returns (n,) f64."""
        p = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        v, t = _mesh(verts, tris)
        out = np.zeros(len(p))
        self._check(self.L.psdf_point_mesh_distance(self.h, _dptr(p), len(p), _dptr(v), len(v), _iptr(t),
                                                    len(t), _dptr(out)))
        return out

    def chamfer(self, pred_points, pred_verts, pred_tris, gt_points, gt_verts, gt_tris, max_dist=0.0):
        """chamfer(pred_points, pred_mesh, gt_points, gt_mesh, max_dist)
        (metrics.cpp:182-194) -> dict(accuracy, completeness, mean), x1000."""
        pp = np.ascontiguousarray(pred_points, np.float64).reshape(-1, 3)
        gp = np.ascontiguousarray(gt_points, np.float64).reshape(-1, 3)
        pv, pt = _mesh(pred_verts, pred_tris)
        gv, gt = _mesh(gt_verts, gt_tris)
        out = np.zeros(3)
        self._check(self.L.psdf_chamfer(self.h, _dptr(pp), len(pp), _dptr(pv), len(pv), _iptr(pt), len(pt),
                                        _dptr(gp), len(gp), _dptr(gv), len(gv), _iptr(gt), len(gt),
                                        float(max_dist), _dptr(out)))
        return dict(accuracy=out[0], completeness=out[1], mean=out[2])

    def marching_cubes(self):
        """marching_cubes(grid) (mesh.cpp:363-394) of the device grid's smoothed
        SDF, on the GPU -> (verts (nv, 3) f64, tris (nt, 3) i32), the reference's
        mesh exactly."""
        nv, nt = C.c_int64(), C.c_int64()
        self._check(self.L.psdf_marching_cubes(self.h, C.byref(nv), C.byref(nt)))
        v = np.zeros((nv.value, 3))
        t = np.zeros((nt.value, 3), np.int32)
        self._check(self.L.psdf_download_mesh(self.h, _dptr(v), _iptr(t)))
        return v, t

    # -- train (trainer.cpp:136-195)
    def train_reset(self):
        self._check(self.L.psdf_train_reset(self.h))

    def train_step(self, cameras, gt_rgb, masks, hp: psdf_step_params):
        n = len(cameras)
        cams = (psdf_camera * n)(*[camera_from(c) for c in cameras])
        gts = [np.ascontiguousarray(g, np.float32) for g in gt_rgb]
        mks = [_train_mask(m) for m in masks]
        gp = (C.POINTER(C.c_float) * n)(*[_fptr(g) for g in gts])
        mp = (C.POINTER(C.c_uint8) * n)(*[m.ctypes.data_as(C.POINTER(C.c_uint8)) for m in mks])
        losses, counts = psdf_losses(), psdf_counts()
        self._check(self.L.psdf_train_step(self.h, n, cams, gp, mp, C.byref(hp), C.byref(losses),
                                           C.byref(counts)))
        return losses.as_dict(), counts.as_dict()

    def upload_views(self, cameras, gt_rgb, masks):
        n = len(cameras)
        cams = (psdf_camera * n)(*[camera_from(c) for c in cameras])
        gts = [np.ascontiguousarray(g, np.float32) for g in gt_rgb]
        mks = [_train_mask(m) for m in masks]
        gp = (C.POINTER(C.c_float) * n)(*[_fptr(g) for g in gts])
        mp = (C.POINTER(C.c_uint8) * n)(*[m.ctypes.data_as(C.POINTER(C.c_uint8)) for m in mks])
        self._check(self.L.psdf_upload_views(self.h, n, cams, gp, mp))

    def train_step_views(self, view_ids, hp: psdf_step_params):
        ids = np.ascontiguousarray(view_ids, np.int32)
        losses, counts = psdf_losses(), psdf_counts()
        self._check(self.L.psdf_train_step_views(self.h, ids.size, _iptr(ids), C.byref(hp),
                                                 C.byref(losses), C.byref(counts)))
        return losses.as_dict(), counts.as_dict()

    def march_rays(self, origins, dirs, n_max=512):
        """Device march_ray t-lists (renderer.cpp:55-86) for explicit rays."""
        o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        n = o.shape[0]
        ts = np.zeros((n, max(n_max, 1)), np.float64)
        cnt = np.zeros(n, np.int32)
        dp = C.POINTER(C.c_double)
        self._check(self.L.psdf_march_rays(self.h, n, o.ctypes.data_as(dp), d.ctypes.data_as(dp), n_max,
                                           ts.ctypes.data_as(dp), _iptr(cnt)))
        return [ts[i, :cnt[i]].copy() for i in range(n)]

    def last_k2_breakdown(self):
        """Device ms of K2a/K2b/K2d/K2e of the last train step, and the number of
        ray entries / shading records it produced."""
        ms = (C.c_double * 4)()
        ne, nr = C.c_int64(), C.c_int64()
        self._check(self.L.psdf_last_k2_breakdown(self.h, ms, C.byref(ne), C.byref(nr)))
        return list(ms), ne.value, nr.value

    def last_wave_counts(self):
        """Queue sizes of the last train step's ray pass: dict(entries, records,
        handovers, continuations, alpha_samples)."""
        out = (C.c_int64 * 5)()
        self._check(self.L.psdf_last_wave_counts(self.h, out))
        return dict(zip(("entries", "records", "handovers", "continuations", "alpha_samples"), list(out)))

    def last_timing(self):
        r, s, n = C.c_double(), C.c_double(), C.c_int()
        self._check(self.L.psdf_last_timing(self.h, C.byref(r), C.byref(s), C.byref(n)))
        return r.value, s.value, n.value

    # -- multi-GPU
    GRAD_EXCHANGE = {"allreduce": 0, "bucketed": 1, "sharded": 2}

    def set_grad_exchange(self, mode):
        """How ranks combine gradients (psdf.h psdf_set_grad_exchange):
        'allreduce' (default), 'bucketed' (planes/probes/MLP bucket reduced
        under the fold) or 'sharded' (reduce-scatter, Adam on this rank's
        chunk, all-gather)."""
        self._check(self.L.psdf_set_grad_exchange(self.h, self.GRAD_EXCHANGE[mode]))

    @staticmethod
    def unique_id() -> bytes:
        L = _lib.load()
        buf = C.create_string_buffer(128)
        check(L.psdf_comm_unique_id(buf))
        return buf.raw

    def comm_init(self, uid: bytes, rank, world):
        buf = C.create_string_buffer(uid, 128)
        self._check(self.L.psdf_comm_init(self.h, buf, rank, world))

    def debug_set_shard(self, rank, world):
        """Test hook: process only `rank`'s 1/world slice, no all-reduce."""
        self._check(self.L.psdf_debug_set_shard(self.h, int(rank), int(world)))

    def last_h2d_bytes(self):
        return int(self.L.psdf_last_h2d_bytes(self.h))


def pixel_dirs(camera) -> np.ndarray:
    """Device Camera::pixel_dir at all pixel centres, [h][w][3] f64."""
    L = _lib.load()
    cam = camera_from(camera)
    out = np.zeros((cam.height, cam.width, 3), np.float64)
    check(L.psdf_pixel_dirs(C.byref(cam), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def shard(n, rank, world):
    """Contiguous 1/world slice [begin, end) of n units: the data-parallel
    partition psdf.cu applies to the batch's 8x4 work tiles (ray pass), the
    allocated tiles (sdf / eikonal / normal / feature regularizers) and the
    probe pool (probe regularizer) — SURVEY.md section 8e."""
    return (n * rank) // world, (n * (rank + 1)) // world


def work_tiles(cameras):
    """8x4-pixel work tiles of a batch (views concatenated, row-major per view)."""
    return sum(((c.width + 7) // 8) * ((c.height + 3) // 4) for c in cameras)


def render_image(ctx: Context, camera, opts: RenderOptions):
    """render_image(grid, mlp, camera, opt) (renderer.hpp:98-99) on the GPU."""
    return ctx.render_image(camera, opts)


def psnr_masked_view(ctx: Context, camera, opts: RenderOptions, gt_rgb, mask) -> float:
    """psnr_masked(render_image(grid, mlp, cam, opt).rgb, gt, mask)
    (metrics.cpp:196-211) on the GPU: the evaluation loop of main.cpp's
    `eval` per view."""
    return ctx.eval_psnr(camera, opts, gt_rgb, mask)



def _mesh(verts, tris):
    return (np.ascontiguousarray(verts, np.float64).reshape(-1, 3),
            np.ascontiguousarray(tris, np.int32).reshape(-1, 3))


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


