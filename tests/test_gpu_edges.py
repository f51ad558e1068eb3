"""Edge cases of the render and train paths against the C oracle: ragged image
sizes (not multiples of the 8x4 work tile, down to 1x1), cameras inside the
grid's box and inside the surface (rays that start in occupied / negative-SDF
space), an empty grid (T = 0: every ray misses), and batches that mix view
sizes.  Same contract as test_gpu_render / test_gpu_train: sample counts
exact, colours / alpha / depth within 1e-4, losses within 1e-4, gradients
within 1e-3.
"""
import numpy as np
import pytest

from helpers import check_grads, make_scene, oracle_with_f32_smooth

pytestmark = pytest.mark.gpu


def _ocam(cam):
    from oracle.refcore import RefCamera
    c = RefCamera()
    for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
        setattr(c, k, getattr(cam, k))
    c.rot[:] = list(cam.rot)
    c.pos[:] = list(cam.pos)
    return c


def _render_cmp(ctx, og, cam, tau, bg=(0.0, 0.0, 0.0)):
    from paper_2412_10084_b200 import api
    from oracle.refcore import render_opts
    opts = api.RenderOptions(tau=tau, camera_id=0, background=bg)
    rgb, alpha, depth, counts = ctx.render_image(cam, opts)
    orgb, oalpha, odepth, oc = og.render_image(_ocam(cam), render_opts(tau=tau, camera_id=0, bg=bg))
    assert rgb.shape == (cam.height, cam.width, 3)
    assert (counts["n_marched"], counts["n_extra"], counts["n_shaded"]) == (oc[1], oc[2], oc[3])
    tol = 1e-4
    assert np.all(np.abs(rgb - orgb) <= tol * np.maximum(np.abs(orgb), 1e-2)), np.abs(rgb - orgb).max()
    assert np.all(np.abs(alpha - oalpha) <= tol * np.maximum(np.abs(oalpha), 1e-2))
    assert np.all(np.abs(depth - odepth) <= tol * np.maximum(np.abs(odepth), 1e-2))
    return counts


def _scene(ctx, **kw):
    g, a = make_scene(**kw)
    og, sm = oracle_with_f32_smooth(a)
    g.smooth = sm
    ctx.upload(g, smooth=True)
    return g, a, og


@pytest.mark.parametrize("w,h", [(1, 1), (37, 23), (7, 45), (9, 4)])
@pytest.mark.parametrize("tau_vox", [30.0, 3000.0])
def test_render_ragged_sizes(ctx, w, h, tau_vox):
    from paper_2412_10084_b200 import api
    _, _, og = _scene(ctx, res=64, n_s=4, n_a=4, sh_order=4, band=6)
    f = 1.2 * max(w, h)
    cam = api.make_lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), f, f, w, h)
    _render_cmp(ctx, og, cam, tau_vox * 64)


@pytest.mark.parametrize("eye,target", [((0.42, 0.1, 0.05), (0, 0, 0)),     # inside the box, outside the surface
                                        ((0.0, 0.02, 0.05), (1, 0.3, 0.2)),  # inside the surface, looking out
                                        ((0.3, -0.31, 0.0), (-1, 0.2, 0.1))])  # inside the band, grazing
def test_render_camera_inside_volume(ctx, eye, target):
    from paper_2412_10084_b200 import api
    _, _, og = _scene(ctx, res=64, n_s=4, n_a=4, sh_order=3, band=6)
    cam = api.make_lookat_camera(0, eye, target, (0, 1, 0), 30.0, 30.0, 40, 32)
    for tau_vox in (30.0, 3000.0):
        _render_cmp(ctx, og, cam, tau_vox * 64)


def _empty_grid():
    """A grid with no allocated tiles (the surface lies outside the volume)."""
    from paper_2412_10084_b200 import api
    from oracle.refcore import GridArrays
    cfg = api.GridConfig(voxel_size=1.0 / 32, resolution=(32, 32, 32), n_s=2, n_a=2, sh_order=2, band_voxels=2)
    g = api.init_grid_sphere(cfg, (10.0, 10.0, 10.0), 0.1, ncam=1, mlp_seed=3)
    assert g.T == 0 and g.P == 0
    a = GridArrays(T=0, P=0, n_s=2, n_a=2, sh_order=2, res=(32, 32, 32), voxel_size=1.0 / 32,
                   origin=(-0.5, -0.5, -0.5), far_field_voxels=4.0, tile_coords=g.tile_coords,
                   probe_ids=g.probe_ids, probe_coords=g.probe_coords, raw=np.zeros((0, 4096)),
                   smooth=np.zeros((0, 4096)), planes=np.zeros(0), probes=np.zeros(0),
                   mlp=g.mlp.astype(np.float64), ncam=1)
    return g, a


def test_empty_grid_render_and_train(ctx):
    """T = 0: every ray is background with zero alpha (test_renderer.cpp:141-149)
    and a train step yields only the empty-ray (opacity) loss."""
    from paper_2412_10084_b200 import api
    from oracle.port import OracleGrid, step_params as ostep
    g, a = _empty_grid()
    ctx.upload(g, smooth=False)
    og = OracleGrid(a, smooth=False)
    cam = api.make_lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 24.0, 24.0, 20, 12)
    counts = _render_cmp(ctx, og, cam, 3000.0 * 32, bg=(0.25, 0.5, 0.75))
    assert counts["n_marched"] == 0
    rng = np.random.default_rng(1)
    gt = rng.uniform(0, 1, (12, 20, 3)).astype(np.float32)
    mask = (rng.uniform(0, 1, (12, 20)) > 0.5).astype(np.float64)
    kw = dict(tau=300.0 * 32, lr_vox=1e-4, lr_mlp=6e-5, photo_scale=20.0)
    ctx.train_reset()
    losses, cnt = ctx.train_step([cam], [gt], [mask], api.step_params(**kw))
    ol, oc = og.train_step([_ocam(cam)], [gt.astype(np.float64)], [mask], ostep(**kw))
    assert [cnt[k] for k in ("n_rays", "n_marched", "n_extra", "n_shaded", "n_alpha", "n_bwd_rays")] == list(oc)
    for i, k in enumerate(("photo", "sdf", "eik", "normal", "features", "probes")):
        assert abs(losses[k] - ol[i]) <= 1e-4 * max(abs(ol[i]), 1e-6), (k, losses[k], ol[i])


@pytest.mark.parametrize("sizes", [[(37, 23), (1, 1), (16, 9)], [(9, 4), (40, 32)]])
def test_train_step_mixed_ragged_views(ctx, sizes):
    """One batch of views with different, ragged sizes (the work-tile grid of
    each view is padded; rays past the edge must not count), plus a camera
    inside the box: counts exact, losses 1e-4, gradients 1e-3."""
    from paper_2412_10084_b200 import api
    from oracle.port import step_params as ostep
    _, _, og = _scene(ctx, res=64, n_s=4, n_a=4, sh_order=3, band=6, ncam=0)
    ctx.keep_raypass_grads(True)
    ctx.train_reset()
    og.train_reset()
    eyes = [(1.3, 0.2, 0.4), (0.42, 0.1, 0.05), (-1.1, -0.4, 0.9)]
    cams = []
    for i, (w, h) in enumerate(sizes):
        f = 1.2 * max(w, h)
        cams.append(api.make_lookat_camera(i, eyes[i % 3], (0, 0, 0), (0, 1, 0), f, f, w, h))
    rng = np.random.default_rng(9)
    gts = [rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32) for c in cams]
    masks = [(rng.uniform(0, 1, (c.height, c.width)) > 0.3).astype(np.float64) for c in cams]
    kw = dict(tau=300.0 * 64, lr_vox=1e-4, lr_mlp=6e-5, photo_scale=20.0)
    losses, cnt = ctx.train_step(cams, gts, masks, api.step_params(**kw))
    ol, oc = og.train_step([_ocam(c) for c in cams], [x.astype(np.float64) for x in gts], masks, ostep(**kw))
    assert [cnt[k] for k in ("n_rays", "n_marched", "n_extra", "n_shaded", "n_alpha", "n_bwd_rays")] == list(oc)
    assert cnt["n_rays"] == sum(w * h for w, h in sizes)
    for i, k in enumerate(("photo", "sdf", "eik", "normal", "features", "probes")):
        assert abs(losses[k] - ol[i]) <= 1e-4 * max(abs(ol[i]), 1e-6), (k, losses[k], ol[i])
    g0, g1 = og.last_grads
    got0, got1 = ctx.grads(0), ctx.grads(1)
    check_grads(got0, g0, "ray pass")
    check_grads(got1, g1, "final")
