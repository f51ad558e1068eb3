"""K1 (fused render) parity on the GPU against the C oracle (which is itself
pinned bit-exactly to the reference, tests/test_oracle_vs_reference.py).

Contract (BASELINE.json north_star): colours and depth within 1e-4 relative,
ray / sample indexing bit-exact.
"""
import numpy as np
import pytest

from helpers import make_scene, oracle_with_f32_smooth

pytestmark = pytest.mark.gpu


def _oracle_cam(cam):
    from oracle.refcore import RefCamera
    c = RefCamera()
    for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
        setattr(c, k, getattr(cam, k))
    c.rot[:] = list(cam.rot)
    c.pos[:] = list(cam.pos)
    return c


def _oracle_opts(o):
    from oracle.refcore import render_opts
    return render_opts(tau=o.tau, n_max=o.n_max, early_stop=o.early_stop_transmittance,
                       bg=o.background, camera_id=o.camera_id, no_spatial=o.no_spatial,
                       no_angular=o.no_angular, no_fresnel=o.no_fresnel,
                       sh_order_override=o.sh_order_override, need_colors=o.need_colors)


def _upload(ctx, g, sm):
    g.smooth = sm
    ctx.upload(g, smooth=True)


def test_pixel_dirs_bit_exact():
    from paper_2412_10084_b200 import api
    from oracle.port import pixel_dir
    cam = api.make_lookat_camera(3, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 38.4, 38.4, 40, 24)
    d = api.pixel_dirs(cam)
    oc = _oracle_cam(cam)
    for v in range(cam.height):
        for u in range(cam.width):
            assert np.array_equal(d[v, u], pixel_dir(oc, u + 0.5, v + 0.5))


def _march_rays(n, seed, span=1.5, tgt_span=0.45):
    rng = np.random.default_rng(seed)
    o = rng.uniform(-span, span, (n, 3))
    o[:100] = [1.2, 0.1, 0.2]
    # far cameras: t crosses several powers of two before the grid
    o[100:400] *= rng.uniform(2.0, 12.0, (300, 1))
    tgt = rng.uniform(-tgt_span, tgt_span, (n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    # axis-aligned and grazing rays exercise the parallel-slab branch
    d[:50] = [[-1, 0, 0]] * 50
    o[:50, 1:] = rng.uniform(-0.6, 0.6, (50, 2))
    return o, d


def test_pixel_dirs_bit_exact_full_view():
    """A bench-sized view (1600x1200): every ray direction bit for bit."""
    from paper_2412_10084_b200 import api
    from oracle.port import pixel_dirs
    for cam in api.make_ring_cameras(3, 1600, height=1200):
        assert np.array_equal(api.pixel_dirs(cam), pixel_dirs(_oracle_cam(cam)))


@pytest.mark.parametrize("res,band,radius,n", [(32, 32, 0.3, 3000), (64, 3, 0.3, 3000),
                                               (256, 3, 0.25, 20000), (512, 2, 0.3, 20000)])
def test_march_bit_exact(ctx, res, band, radius, n):
    """march_ray t-lists bit for bit, including the empty-space jumps of the
    tile distance field (tile_dist, psdf_device.cuh Marcher)."""
    g, a = make_scene(res=res, band=band, radius=radius)
    og, sm = oracle_with_f32_smooth(a)
    _upload(ctx, g, sm)
    o, d = _march_rays(n, 11)
    got = ctx.march_rays(o, d, 512)
    for i in range(len(o)):
        want = og.march_ray(o[i], d[i], 512)
        assert got[i].shape == want.shape and np.array_equal(got[i], want), i
    # n_max cap
    got = ctx.march_rays(o[:200], d[:200], 7)
    for i in range(200):
        assert np.array_equal(got[i], og.march_ray(o[i], d[i], 7))


@pytest.mark.parametrize("margin", ["0.02", "0.45"])
def test_march_exact_paths(ctx, monkeypatch, margin):
    """A widened decision margin sends most tile / skip decisions (and every
    decision after an empty-space jump near a face) down the exact and rewind
    paths; the t-lists must not change by a bit."""
    g, a = make_scene(res=256, band=3, radius=0.25)
    og, sm = oracle_with_f32_smooth(a)
    _upload(ctx, g, sm)
    o, d = _march_rays(6000, 12)
    # rays along tile faces / through tile edges (lattice-aligned decisions)
    h = 1.0 / 256
    o[400:600] = [[-1.3, -0.5 + 16 * h * k, -0.5 + 16 * h * (k % 7)] for k in range(200)]
    d[400:600] = [[1.0, 0.0, 0.0]] * 200
    monkeypatch.setenv("PSDF_TEST_MARGIN", margin)
    got = ctx.march_rays(o, d, 512)
    for i in range(len(o)):
        want = og.march_ray(o[i], d[i], 512)
        assert got[i].shape == want.shape and np.array_equal(got[i], want), i


SCENES = [
    dict(res=32, n_s=2, n_a=2, sh_order=2, band=32),
    dict(res=64, n_s=4, n_a=4, sh_order=4, band=6),
    dict(res=32, n_s=8, n_a=8, sh_order=3, band=32),
    dict(res=256, n_s=4, n_a=4, sh_order=4, band=3),  # empty-space jumps
    dict(res=32, n_s=3, n_a=5, sh_order=3, band=32),  # no own kernels: zero-padded to (4, 8)
]


@pytest.mark.parametrize("scene", SCENES)
@pytest.mark.parametrize("tau_vox", [0.75, 30.0, 3000.0])
def test_render_parity(ctx, scene, tau_vox):
    _render_parity(ctx, scene, tau_vox)


@pytest.mark.parametrize("tau_vox", [300.0, 3000.0])
def test_render_parity_production_grid(ctx, tau_vox):
    """configs[1] / [3] grid (512^3, (4, 4, 4), T = 2848) on a 48x48 view."""
    _render_parity(ctx, dict(res=512, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32), tau_vox)


def test_render_parity_wave_overflow(monkeypatch):
    """Undersized ray-pass buffers: the render overflows, grows and redoes."""
    from paper_2412_10084_b200 import api
    monkeypatch.setenv("PSDF_WAVE_INIT", "32")
    c = api.Context(0)
    try:
        _render_parity(c, SCENES[1], 0.75)
    finally:
        c.close()


def _render_parity(ctx, scene, tau_vox):
    from paper_2412_10084_b200 import api
    g, a = make_scene(**scene)
    og, sm = oracle_with_f32_smooth(a)
    _upload(ctx, g, sm)
    res = scene["res"]
    cam = api.make_lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 1.2 * 48, 1.2 * 48, 48, 48)
    opts = api.RenderOptions(tau=tau_vox * res, camera_id=0)
    rgb, alpha, depth, counts = ctx.render_image(cam, opts)
    orgb, oalpha, odepth, ocounts = og.render_image(_oracle_cam(cam), _oracle_opts(opts))
    # indexing: identical sample counts (march + early termination + shaded set)
    assert counts["n_marched"] == ocounts[1]
    assert counts["n_extra"] == ocounts[2]
    assert counts["n_shaded"] == ocounts[3]
    tol = 1e-4
    assert np.all(np.abs(rgb - orgb) <= tol * np.maximum(np.abs(orgb), 1e-2)), np.abs(rgb - orgb).max()
    assert np.all(np.abs(alpha - oalpha) <= tol * np.maximum(np.abs(oalpha), 1e-2))
    assert np.all(np.abs(depth - odepth) <= tol * np.maximum(np.abs(odepth), 1e-2))


@pytest.mark.parametrize("flag", ["no_spatial", "no_angular", "no_fresnel", "sh_order_override",
                                  "background", "no_early_stop", "early_stop_above_one", "alpha_only"])
def test_render_options(ctx, flag):
    from paper_2412_10084_b200 import api
    g, a = make_scene(res=32, n_s=4, n_a=4, sh_order=4, band=32)
    og, sm = oracle_with_f32_smooth(a)
    _upload(ctx, g, sm)
    cam = api.make_lookat_camera(0, (1.0, 0.15, 0.2), (0, 0.2, 0.05), (0, 1, 0), 38.4, 38.4, 32, 32)
    kw = dict(tau=2000.0, camera_id=0)
    if flag == "sh_order_override":
        kw[flag] = 1
    elif flag == "background":
        kw[flag] = (0.25, 0.5, 0.75)
    elif flag == "no_early_stop":
        kw["early_stop_transmittance"] = 0.0
    elif flag == "early_stop_above_one":  # stops after the first settled sample
        kw["early_stop_transmittance"] = 1.5
    elif flag == "alpha_only":
        kw["need_colors"] = False
    else:
        kw[flag] = True
    opts = api.RenderOptions(**kw)
    rgb, alpha, depth, counts = ctx.render_image(cam, opts)
    orgb, oalpha, odepth, ocounts = og.render_image(_oracle_cam(cam), _oracle_opts(opts))
    assert counts["n_marched"] == ocounts[1] and counts["n_shaded"] == ocounts[3]
    assert np.abs(rgb - orgb).max() <= 1e-4 * max(1.0, np.abs(orgb).max())
    assert np.abs(alpha - oalpha).max() <= 1e-6


def test_render_errors(ctx):
    from paper_2412_10084_b200 import api
    from paper_2412_10084_b200._lib import PsdfOutOfRange
    g, a = make_scene(res=32, ncam=1)
    ctx.upload(g)
    cam = api.make_lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 38.4, 38.4, 8, 8)
    with pytest.raises(PsdfOutOfRange):  # decoder.cpp:73-74
        ctx.render_image(cam, api.RenderOptions(tau=100.0, camera_id=5))
    # a ray missing the volume: background, zero alpha (test_renderer.cpp:141-149)
    far = api.make_lookat_camera(0, (5, 5, 5), (10, 10, 10), (0, 1, 0), 8, 8, 4, 4)
    rgb, alpha, _, counts = ctx.render_image(far, api.RenderOptions(tau=100.0, background=(0.25, 0.5, 0.75)))
    assert counts["n_marched"] == 0 and np.all(alpha == 0)
    assert np.allclose(rgb, [0.25, 0.5, 0.75])


@pytest.mark.parametrize("scene", [SCENES[1], dict(res=512, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32)])
def test_eval_psnr(ctx, scene):
    """psdf_eval_psnr (metrics.cpp:196-211 on the device): the masked-error
    reduction of the GPU's own render matches the restated psnr_masked on
    that render to 1e-9 dB (only the f64 summation order differs), and the
    oracle's f64 render to 1e-3 dB; an empty mask and an exact match give 99."""
    from oracle.port import psnr_masked
    from paper_2412_10084_b200 import api
    g, a = make_scene(**scene)
    og, sm = oracle_with_f32_smooth(a)
    _upload(ctx, g, sm)
    cam = api.make_lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 1.2 * 48, 1.2 * 48, 48, 40)
    opts = api.RenderOptions(tau=300.0 * scene["res"], camera_id=0)
    rng = np.random.default_rng(7)
    gt = rng.uniform(0, 1, (40, 48, 3)).astype(np.float32)
    mask = rng.uniform(0, 1, (40, 48))
    got = ctx.eval_psnr(cam, opts, gt, mask)
    rgb, _, _, _ = ctx.render_image(cam, opts)
    assert abs(got - psnr_masked(rgb, gt, mask)) <= 1e-9
    orgb = og.render_image(_oracle_cam(cam), _oracle_opts(opts))[0]
    assert abs(got - psnr_masked(orgb, gt.astype(np.float64), mask)) <= 1e-3
    assert ctx.eval_psnr(cam, opts, gt, np.zeros((40, 48))) == 99.0
    assert ctx.eval_psnr(cam, opts, rgb, mask) == 99.0
    with pytest.raises(ValueError, match="shape mismatch"):
        ctx.eval_psnr(cam, opts, gt[:-1], mask)


@pytest.mark.parametrize("tau_vox", [300.0, 3000.0])
def test_render_parity_bench_view(ctx, tau_vox):
    """Maximum size: a full configs[1] view (1600x1200 = 1.92 M rays) of the
    512^3 production grid — sample counts (march, early termination, shaded
    set) identical to the oracle over every ray, colours / alpha / depth
    within the 1e-4 contract."""
    from paper_2412_10084_b200 import api
    g, a = make_scene(res=512, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32)
    og, sm = oracle_with_f32_smooth(a)
    _upload(ctx, g, sm)
    cam = api.make_ring_cameras(2, 1600, height=1200)[1]
    opts = api.RenderOptions(tau=tau_vox * 512, camera_id=0)
    rgb, alpha, depth, counts = ctx.render_image(cam, opts)
    orgb, oalpha, odepth, ocounts = og.render_image(_oracle_cam(cam), _oracle_opts(opts))
    assert counts["n_rays"] == 1600 * 1200
    assert (counts["n_marched"], counts["n_extra"], counts["n_shaded"]) == tuple(ocounts[1:4])
    assert counts["n_marched"] > 10 * counts["n_shaded"] > 0
    tol = 1e-4
    assert np.all(np.abs(rgb - orgb) <= tol * np.maximum(np.abs(orgb), 1e-2)), np.abs(rgb - orgb).max()
    assert np.all(np.abs(alpha - oalpha) <= tol * np.maximum(np.abs(oalpha), 1e-2))
    assert np.all(np.abs(depth - odepth) <= tol * np.maximum(np.abs(odepth), 1e-2))


def test_render_parity_bench_view_after_overflow(monkeypatch):
    """Regression: a context whose ray-pass buffers were sized for tiny passes
    (PSDF_WAVE_INIT) renders a full 1600x1200 view — the first pass overflows
    by orders of magnitude (records allocated past an overflowed entry stay
    unwritten), the kernels after the march must ignore its queues, and the
    redo matches the oracle."""
    from paper_2412_10084_b200 import api
    monkeypatch.setenv("PSDF_WAVE_INIT", "64")
    c = api.Context(0)
    try:
        test_render_parity_bench_view(c, 300.0)
    finally:
        c.close()
