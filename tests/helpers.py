"""Scene builders and metrics shared by the parity tests."""
import numpy as np


# --------------------------------------------------------------------------
# Scene construction shared by the parity tests (product host code + numpy).
# --------------------------------------------------------------------------
def make_scene(res=32, n_s=2, n_a=2, sh_order=2, band=32, radius=0.3, seed=4, ncam=1, jitter=0.004,
               plane_amp=0.2, probe_amp=0.3, bias_amp=0.1, prims=None):
    """A seeded "trained-like" scene in the pattern of test_renderer.cpp:21-45 /
    gradcheck.cpp:28-53, built with the product's host API, all values
    fp32-representable.  Returns (HostGrid, GridArrays-like for the oracle)."""
    from paper_2412_10084_b200 import api
    from oracle.refcore import GridArrays
    cfg = api.GridConfig(voxel_size=1.0 / res, resolution=(res, res, res), n_s=n_s, n_a=n_a,
                         sh_order=sh_order, band_voxels=band)
    sdf_fn = api.analytic_sdf(prims) if prims else None
    g = api.init_grid_sphere(cfg, (0, 0, 0), radius, ncam=ncam, mlp_seed=seed + 1, sdf_fn=sdf_fn)
    rng = np.random.default_rng(seed)
    raw = g.raw.astype(np.float64) + jitter * rng.uniform(-1, 1, g.raw.shape)
    g.raw = raw.astype(np.float32)
    g.planes = (0.5 + plane_amp * rng.uniform(-1, 1, g.planes.shape)).astype(np.float32)
    g.probes = (probe_amp * rng.uniform(-1, 1, g.probes.shape)).astype(np.float32)
    if ncam:
        mlp = g.mlp.copy()
        mlp[-ncam * 32:] = (bias_amp * rng.uniform(-1, 1, ncam * 32)).astype(np.float32)
        g.mlp = mlp
    a = GridArrays(T=g.T, P=g.P, n_s=n_s, n_a=n_a, sh_order=sh_order, res=(res, res, res),
                   voxel_size=1.0 / res, origin=(-0.5, -0.5, -0.5), far_field_voxels=4.0,
                   tile_coords=g.tile_coords, probe_ids=g.probe_ids, probe_coords=g.probe_coords,
                   raw=g.raw.astype(np.float64), smooth=np.zeros((g.T, 4096)),
                   planes=g.planes.astype(np.float64), probes=g.probes.astype(np.float64),
                   mlp=g.mlp.astype(np.float64), ncam=ncam)
    return g, a


def oracle_with_f32_smooth(a):
    """Oracle grid whose smoothed SDF is the oracle's own f64 smoothing rounded
    to fp32, i.e. exactly what gets uploaded to the GPU (SURVEY hard part 2)."""
    from oracle.port import OracleGrid
    og0 = OracleGrid(a, smooth=False)
    sm = og0.export()["smooth"].astype(np.float32)
    b = a.copy()
    b.smooth = sm.astype(np.float64)
    return OracleGrid(b, smooth=True), sm


def check_grads(got, want, what, tol=1e-3, kink_outliers=False):
    """The gradient contract (north_star 1e-3; SURVEY hard part 6): per tensor
    ||d||_2 <= tol ||g||_2 and element-wise |d| <= tol max|g|.

    kink_outliers: the decoder runs in fp32 and the oracle in f64, so a
    ReLU mask (decoder.cpp:93-101), the n.v clamp (decoder.cpp:57) or a plane
    tap boundary can be decided differently for a sample whose pre-activation
    is within fp32 rounding of the kink; that one sample's feature gradient
    then differs by O(its own size).  Over ~10^6 shaded samples (the bench
    step) a few such samples occur (measured: 20 of 3.5 M plane entries, all
    in one tile, identical on every GPU run and in the serialised and
    overlapped schedules, profiles/r02/prod_diag.log).  With this flag up to
    max(32, 1e-5 n) entries may exceed the element-wise bound, each by at
    most 50x; the L2 bound is unchanged."""
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        g = np.asarray(got[k], np.float64)
        w = np.asarray(want[k], np.float64)
        scale = np.abs(w).max()
        if scale == 0:
            assert np.abs(g).max() == 0, (what, k)
            continue
        assert rel_l2(g, w) <= tol, (what, k, rel_l2(g, w))
        d = np.abs(g - w)
        if not kink_outliers:
            assert d.max() <= tol * scale, (what, k, d.max() / scale)
        else:
            n_out = int((d > tol * scale).sum())
            assert n_out <= max(32, 1e-5 * d.size), (what, k, n_out)
            assert d.max() <= 50 * tol * scale, (what, k, d.max() / scale)


def check_same_schedule(got, ref, what, tol=2e-5):
    """Two GPU runs of the same step (e.g. the overlapped production schedule
    against the serialised one): only the fp32 atomic order may differ, so
    every entry agrees to tol x max (measured 1e-7 .. 7e-7 at the bench
    step); a missing stream-ordering edge would clear or double-count whole
    blocks of gradient and fail this by orders of magnitude."""
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        g = np.asarray(got[k], np.float64)
        r = np.asarray(ref[k], np.float64)
        scale = max(np.abs(r).max(), 1e-30)
        assert np.abs(g - r).max() <= tol * scale, (what, k, np.abs(g - r).max() / scale)


def rel_l2(x, y):
    x = np.asarray(x, np.float64).ravel()
    y = np.asarray(y, np.float64).ravel()
    den = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / den) if den > 0 else float(np.linalg.norm(x - y))


# --------------------------------------------------------------------------
# Golden fixtures (tests/golden/, generated by tests/golden/make_golden.py
# from the unmodified reference).
# --------------------------------------------------------------------------
import os as _os

GOLDEN = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden")


def golden(name):
    return dict(np.load(_os.path.join(GOLDEN, name)))


def cam_from_array(v):
    from oracle.refcore import RefCamera
    c = RefCamera()
    c.fx, c.fy, c.cx, c.cy = (float(x) for x in v[:4])
    c.width, c.height = int(v[4]), int(v[5])
    c.rot[:] = [float(x) for x in v[6:15]]
    c.pos[:] = [float(x) for x in v[15:18]]
    c.id = int(v[18])
    return c


def scene32_arrays(z):
    """GridArrays of the golden 32^3 scene (its smoothed SDF included)."""
    from oracle.refcore import GridArrays
    n_s, n_a, order, res, ncam = (int(x) for x in z["meta"])
    g = z["geom"]
    return GridArrays(T=z["raw"].shape[0], P=z["probes"].shape[0], n_s=n_s, n_a=n_a, sh_order=order,
                      res=(res, res, res), voxel_size=float(g[0]), origin=tuple(float(x) for x in g[1:4]),
                      far_field_voxels=float(g[4]), tile_coords=z["tile_coords"],
                      probe_ids=z["probe_ids"], probe_coords=z["probe_coords"], raw=z["raw"],
                      smooth=z["smooth"], planes=z["planes"], probes=z["probes"], mlp=z["mlp"],
                      ncam=ncam)


def step_params_from(hpv):
    from oracle.port import step_params
    return step_params(tau=hpv[0], lr_vox=hpv[1], lr_mlp=hpv[2], l_sdf=hpv[3], l_eik=hpv[4],
                       l_norm=hpv[5], l_feat=hpv[6], l_probe=hpv[7], photo_scale=hpv[8],
                       use_camera_bias=bool(hpv[9]))
