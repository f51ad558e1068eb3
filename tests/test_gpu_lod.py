"""LOD transitions on the GPU against the unmodified
reference's own SparseGrid::subdivide / raise_sh_order (oracle/_ref, through
oracle/refcore.py), on the same fp32-representable grids.

Contract: tile and probe structure (coordinates, order, probe ids) identical;
child raw SDF values and allocation decisions computed in f64 in the
reference's operation order, stored as fp32 (|d| <= 1 fp32 ulp of the f64
value); planes / probes likewise; the re-smoothed grid within 1e-5 (fp32
smoothing vs the reference's f64, as in test_gpu_train).
"""
import numpy as np
import pytest

from helpers import make_scene

pytestmark = pytest.mark.gpu


def _ref_scene(a, case):
    from oracle.refcore import RefScene
    s = RefScene.sphere(res=case["res"], n_s=case["n_s"], n_a=case["n_a"], sh_order=case["sh_order"],
                        band_voxels=case["band"], radius=case["radius"], ncam=0)
    e = s.export()
    assert np.array_equal(e.tile_coords, a.tile_coords) and np.array_equal(e.probe_coords, a.probe_coords)
    s.import_(raw=a.raw, planes=a.planes.reshape(e.planes.shape), probes=a.probes.reshape(e.probes.shape),
              mlp=a.mlp)
    return s


def _close_f32(got, want, what):
    want = np.asarray(want, np.float64).ravel()
    got = np.asarray(got, np.float64).ravel()
    assert got.shape == want.shape, what
    ulp = np.spacing(np.abs(want).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got - want) <= ulp + 1e-30), (what, np.abs(got - want).max())


CASES = [
    dict(res=32, n_s=4, n_a=4, sh_order=3, band=4, radius=0.3, jitter=0.004),
    dict(res=64, n_s=2, n_a=2, sh_order=2, band=6, radius=0.27, jitter=0.002),
    # widths without their own kernels (zero-padded to (4, 8) on the device)
    dict(res=32, n_s=3, n_a=5, sh_order=3, band=4, radius=0.3, jitter=0.004),
]


@pytest.mark.parametrize("case", CASES)
def test_subdivide_parity(ctx, case):
    g, a = make_scene(res=case["res"], n_s=case["n_s"], n_a=case["n_a"], sh_order=case["sh_order"],
                      band=case["band"], radius=case["radius"], ncam=0, jitter=case["jitter"])
    s = _ref_scene(a, case)
    ctx.upload(g, smooth=False)
    ng = ctx.subdivide(band_voxels=case["band"])
    s.subdivide()
    b = s.export()
    assert ng.T == b.T and ng.P == b.P, (ng.T, b.T, ng.P, b.P)
    assert np.array_equal(ng.tile_coords, b.tile_coords)
    assert np.array_equal(ng.probe_ids, b.probe_ids)
    assert np.array_equal(ng.probe_coords, b.probe_coords)
    assert ng.cfg.resolution == b.res and ng.cfg.voxel_size == b.voxel_size
    _close_f32(ng.raw, b.raw, "raw")
    _close_f32(ng.planes, b.planes, "planes")
    _close_f32(ng.probes, b.probes, "probes")
    assert np.abs(ng.smooth - b.smooth).max() <= 1e-5
    np.testing.assert_array_equal(ng.mlp, g.mlp)


def test_subdivide_then_train_step(ctx):
    """The subdivided grid is a working training state (ray pass + Adam run,
    counts equal the oracle's on the same grid)."""
    from paper_2412_10084_b200 import api
    from oracle.port import step_params as ostep
    from oracle.refcore import RefCamera
    from helpers import oracle_with_f32_smooth
    from oracle.refcore import GridArrays
    g, a = make_scene(res=32, n_s=4, n_a=4, sh_order=2, band=4, ncam=0)
    ctx.upload(g, smooth=False)
    ng = ctx.subdivide(band_voxels=4)
    b = GridArrays(T=ng.T, P=ng.P, n_s=4, n_a=4, sh_order=2, res=tuple(ng.cfg.resolution),
                   voxel_size=ng.cfg.voxel_size, origin=tuple(ng.cfg.origin), far_field_voxels=4.0,
                   tile_coords=ng.tile_coords, probe_ids=ng.probe_ids, probe_coords=ng.probe_coords,
                   raw=ng.raw.astype(np.float64), smooth=np.zeros((ng.T, 4096)),
                   planes=ng.planes.astype(np.float64), probes=ng.probes.astype(np.float64),
                   mlp=ng.mlp.astype(np.float64), ncam=0)
    og, sm = oracle_with_f32_smooth(b)
    ng.smooth = sm
    ctx.upload(ng, smooth=True)
    cam = api.make_lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 38.4, 38.4, 32, 32)
    oc = RefCamera()
    for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
        setattr(oc, k, getattr(cam, k))
    oc.rot[:] = list(cam.rot)
    oc.pos[:] = list(cam.pos)
    gt = np.random.default_rng(0).uniform(0, 1, (32, 32, 3)).astype(np.float32)
    mask = np.ones((32, 32))
    kw = dict(tau=30.0 * 64, lr_vox=1e-4, lr_mlp=6e-5, photo_scale=40.0)
    ctx.train_reset()
    losses, cnt = ctx.train_step([cam], [gt], [mask], api.step_params(**kw))
    ol, oc2 = og.train_step([oc], [gt.astype(np.float64)], [mask], ostep(**kw))
    assert list(oc2) == [cnt[k] for k in ("n_rays", "n_marched", "n_extra", "n_shaded", "n_alpha",
                                          "n_bwd_rays")]
    assert abs(losses["photo"] - ol[0]) <= 1e-4 * abs(ol[0])


@pytest.mark.parametrize("ns,na", [(4, 4), (3, 5)])
def test_raise_sh_order(ctx, ns, na):
    from paper_2412_10084_b200 import _lib
    case = dict(res=32, n_s=ns, n_a=na, sh_order=2, band=4, radius=0.3)
    g, a = make_scene(res=32, n_s=ns, n_a=na, sh_order=2, band=4, ncam=0)
    s = _ref_scene(a, case)
    ctx.upload(g, smooth=False)
    ng = ctx.raise_sh_order(4)
    s.raise_sh_order(4)
    b = s.export()
    assert ng.cfg.sh_order == 4 and b.sh_order == 4
    np.testing.assert_array_equal(ng.probes.astype(np.float64), b.probes.ravel())
    with pytest.raises(_lib.PsdfInvalidArgument):
        ctx.raise_sh_order(3)
    with pytest.raises(ValueError):
        s.raise_sh_order(3)


def _sphere_masks(cams, radius):
    """uint8 silhouettes (255 / 0) of a sphere at the origin, pixel-centre rays."""
    out = []
    for c in cams:
        R = np.array(list(c.rot)).reshape(3, 3)
        o = np.array(list(c.pos))
        u, v = np.meshgrid(np.arange(c.width) + 0.5, np.arange(c.height) + 0.5)
        d = np.stack([(u - c.cx) / c.fx, (v - c.cy) / c.fy, np.ones_like(u)], -1) @ R.T
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        b = d @ o
        disc = b * b - (o @ o - radius * radius)
        out.append(np.where((disc >= 0) & (-b > 0), 255, 0).astype(np.uint8))
    return out


@pytest.mark.parametrize("res,band,ns,na", [(32, 4, 2, 2), (64, 6, 2, 2), (48, 4, 3, 5)])
def test_visual_hull_parity(ctx, res, band, ns, na):
    """init_grid_visual_hull on the device vs the reference's own (occupancy,
    EDTs, seed SDF, allocation and order bit-exact; raw stored as fp32;
    planes 0.5 / probes 0 / MLP 0 at the caller's widths, also for a pair
    the device zero-pads)."""
    from paper_2412_10084_b200 import api
    from oracle.refcore import RefCamera, RefScene
    cams = api.make_ring_cameras(8, 48)
    masks = _sphere_masks(cams, 0.3)
    rcams = []
    for c in cams:
        rc = RefCamera()
        for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
            setattr(rc, k, getattr(c, k))
        rc.rot[:] = list(c.rot)
        rc.pos[:] = list(c.pos)
        rcams.append(rc)
    cfg = api.GridConfig(voxel_size=1.0 / res, resolution=(res, res, res), n_s=ns, n_a=na, sh_order=2,
                         band_voxels=band)
    ng = ctx.init_visual_hull(cfg, cams, masks)
    b = RefScene.hull(rcams, masks, res=res, n_s=ns, n_a=na, sh_order=2, band_voxels=band).export()
    assert ng.T == b.T and ng.P == b.P and ng.T > 0, (ng.T, b.T, ng.P, b.P)
    assert np.array_equal(ng.tile_coords, b.tile_coords)
    assert np.array_equal(ng.probe_ids, b.probe_ids)
    assert np.array_equal(ng.probe_coords, b.probe_coords)
    _close_f32(ng.raw, b.raw, "raw")
    _close_f32(ng.planes, b.planes, "planes")
    _close_f32(ng.probes, b.probes, "probes")
    assert np.abs(ng.smooth - b.smooth).max() <= 1e-5
    assert not np.any(ng.mlp)


def test_visual_hull_errors(ctx):
    from paper_2412_10084_b200 import api, _lib
    cfg = api.GridConfig(voxel_size=1.0 / 24, resolution=(24, 24, 24), n_s=2, n_a=2, sh_order=2)
    cams = api.make_ring_cameras(2, 16)
    with pytest.raises(_lib.PsdfInvalidArgument):
        ctx.init_visual_hull(cfg, cams, _sphere_masks(cams, 0.3))
    with pytest.raises(_lib.PsdfInvalidArgument):
        ctx.init_visual_hull(api.GridConfig(voxel_size=1 / 32, resolution=(32, 32, 32)), [], [])
