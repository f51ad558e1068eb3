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


def rel_l2(x, y):
    x = np.asarray(x, np.float64).ravel()
    y = np.asarray(y, np.float64).ravel()
    den = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / den) if den > 0 else float(np.linalg.norm(x - y))
