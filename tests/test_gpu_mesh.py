"""Marching cubes on the GPU (mesh.cpp:305-394) against
the unmodified reference's own marching_cubes(grid) (oracle/_ref) on the same
grid: the reference scene is built by the reference (sphere / analytic
torus / human union, sparse bands, seeded jitter), uploaded to the device,
smoothed there, and the device's fp32 smoothed SDF is installed back into the
reference scene, so both sides polygonise identical values.

Contract: bit-exact — the same vertex count, every vertex position equal as
f64 (the same interpolation direction and operation order), the same
triangles in the same order (zero-area triangles dropped alike)."""
import numpy as np
import pytest

from conftest import have_ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")]


def _device_and_ref(ctx, scene, smooth_on_device=True):
    from paper_2412_10084_b200 import api
    a = scene.export()
    g = api.HostGrid.from_arrays(a, ncam=a.ncam)
    ctx.upload(g, smooth=not smooth_on_device)
    sm = ctx.download()["smooth"].astype(np.float64)
    scene.import_(smooth=sm)
    return a


def _check(ctx, scene):
    v, t = ctx.marching_cubes()
    rv, rt = scene.marching_cubes()
    assert v.shape == rv.shape and t.shape == rt.shape, (v.shape, rv.shape, t.shape, rt.shape)
    assert np.array_equal(v, rv)
    assert np.array_equal(t, rt)
    return v, t


@pytest.mark.parametrize("res,band,jitter", [(32, 6, 0.004), (64, 6, 0.002), (128, 6, 0.0)])
def test_marching_cubes_sphere(ctx, res, band, jitter):
    from oracle.refcore import RefScene
    s = RefScene.sphere(res=res, n_s=2, n_a=2, sh_order=2, band_voxels=band, radius=0.3, ncam=0)
    s.randomize(7, sdf_jitter=jitter)
    s.round_to_f32()
    _device_and_ref(ctx, s)
    v, t = _check(ctx, s)
    assert len(t) > 100


@pytest.mark.parametrize("shape", ["torus", "human"])
@pytest.mark.parametrize("res", [64, 128])
def test_marching_cubes_shapes(ctx, shape, res):
    """Several surface sheets, thin limbs and the torus hole: edges shared by
    cells of different tiles in every configuration."""
    from oracle.refcore import RefScene
    from paper_2412_10084_b200 import api
    s = RefScene.analytic(api.SCENE_PRIMS[shape], res=res, n_s=2, n_a=2, sh_order=2, band_voxels=4, ncam=0)
    s.randomize(3, sdf_jitter=0.001)
    s.round_to_f32()
    _device_and_ref(ctx, s)
    _check(ctx, s)


def test_marching_cubes_vetoes_and_boundary(ctx):
    """A sphere cut by the grid boundary (cells at res - 1 skipped) with a thin
    band (cells whose corners reach unallocated tiles vetoed), and values
    exactly 0 at lattice points (t = 0 / 1 clamps, coincident vertices:
    zero-area triangles dropped)."""
    from oracle.refcore import RefScene
    s = RefScene.sphere(res=48, n_s=2, n_a=2, sh_order=2, band_voxels=2, radius=0.45,
                        center=(0.2, 0.0, -0.1), ncam=0)
    s.round_to_f32()
    a = _device_and_ref(ctx, s)
    sm = ctx.download()["smooth"].astype(np.float64)
    # snap a band of values to exactly 0 (the reference's t = v0 / (v0 - v1)
    # then hits 0 and 1, vertices coincide with lattice points)
    snap = np.abs(sm) < 0.25 * (1.0 / 48)
    sm[snap] = 0.0
    from paper_2412_10084_b200 import api
    g = api.HostGrid.from_arrays(a, ncam=a.ncam)
    g.smooth = sm.astype(np.float32)
    ctx.upload(g, smooth=True)
    s.import_(smooth=sm)
    v, t = _check(ctx, s)
    assert snap.sum() > 0 and len(t) > 0


def test_marching_cubes_after_train_steps(ctx):
    """The mesh of a grid the GPU has trained (values no analytic init gives)."""
    from oracle.refcore import RefScene, ring_cameras
    from paper_2412_10084_b200 import api
    s = RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=6, radius=0.3, ncam=0)
    s.randomize(1, sdf_jitter=0.003)
    s.round_to_f32()
    a = _device_and_ref(ctx, s)
    cams = [api.camera_from(c) for c in ring_cameras(4, 32, 2.0, 0.35, 3)]
    rng = np.random.default_rng(0)
    gts = [rng.uniform(0, 1, (32, 32, 3)).astype(np.float32) for _ in cams]
    masks = [np.ones((32, 32), np.uint8) for _ in cams]
    ctx.train_reset()
    for _ in range(3):
        ctx.train_step(cams, gts, masks, api.step_params(tau=30.0 * 32, lr_vox=2e-3, lr_mlp=1e-3))
    d = ctx.download()
    s.import_(raw=d["raw"].astype(np.float64), smooth=d["smooth"].astype(np.float64))
    _check(ctx, s)


def test_marching_cubes_empty_and_no_surface(ctx):
    from oracle.refcore import RefScene
    # all values positive: no sign change anywhere -> empty mesh
    s = RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=4, radius=0.3, ncam=0)
    a = _device_and_ref(ctx, s)
    from paper_2412_10084_b200 import api
    g = api.HostGrid.from_arrays(a, ncam=a.ncam)
    g.smooth = np.full((a.T, 4096), 0.25, np.float32)
    ctx.upload(g, smooth=True)
    v, t = ctx.marching_cubes()
    assert v.shape == (0, 3) and t.shape == (0, 3)
