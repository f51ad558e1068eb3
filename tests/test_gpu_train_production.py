"""Parity of the train-step schedule the bench and the drop-in actually run.

Every other train test keeps the ray pass's own gradients
(psdf_set_keep_raypass_grads(1)), which serialises the step.  Here that switch
is OFF, so the production schedule is live (psdf.cu do_train_step):

* the gradient clear on the low-priority side stream (ev_zeroed),
* the regularizers and the empty rays' photo terms on the side stream, forked
  at the step start (small grids: T * 1000 > rays, or PSDF_REGS_EARLY) or
  after the first composite round (ev_fork), joined before the fold (ev_join),
* with host images (psdf_train_step): masks / colours copied on the copy
  stream under the scan (ev_masks / ev_rgb),
* a render on the same context right before each step (the view table and
  the scan's hand-over bits are shared between the two).

The comparison is with the oracle's full step (trainer.cpp:136-195): exact
counts, losses within 1e-4 relative, final (stage-1) gradients within 1e-3
(per tensor L2 and element-wise against the max), post-Adam parameters.
Each case is repeated from the same state to shake out ordering races, and
every repeat is also compared with the serialised schedule on the GPU itself
(check_same_schedule: atomic-order noise only), which is the sharp race test.
(compute-sanitizer is closed on the GPU pool, so races and bad accesses are
caught by these comparisons and the redo / overflow tests.)
"""
import numpy as np
import pytest

from helpers import check_grads, check_same_schedule, make_scene, oracle_with_f32_smooth

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-3


def _ocam(c):
    from oracle.refcore import RefCamera
    oc = RefCamera()
    for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
        setattr(oc, k, getattr(c, k))
    oc.rot[:] = list(c.rot)
    oc.pos[:] = list(c.pos)
    return oc


def _views(og, ocams, seed, res):
    from oracle.refcore import render_opts
    rng = np.random.default_rng(seed)
    gts, masks = [], []
    for c in ocams:
        _, alpha, _, _ = og.render_image(c, render_opts(tau=3000.0 * res))
        masks.append((alpha > 0.5).astype(np.float64))
        gts.append(rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32).astype(np.float64))
    return gts, masks


def _production_parity(ctx, scene, tau, size, height=None, n_views=4, batch=(0, 1, 2, 3), repeats=3,
                       resident=False, render_first=True, lr=(5e-3 / 50, 3e-3 / 50), kink_outliers=False):
    from paper_2412_10084_b200 import api
    from oracle.port import step_params as ostep
    g, a = make_scene(ncam=0, **scene)
    og, sm = oracle_with_f32_smooth(a)
    g.smooth = sm
    res = scene["res"]
    cams = api.make_ring_cameras(n_views, size, height=height)
    ocams = [_ocam(c) for c in cams]
    gts, masks = _views(og, ocams, 7, res)
    batch = list(batch)
    kw = dict(tau=tau * res, lr_vox=lr[0], lr_mlp=lr[1], photo_scale=40.0 / len(batch))
    og.train_reset()
    ol, oc = og.train_step([ocams[i] for i in batch], [gts[i] for i in batch], [masks[i] for i in batch],
                           ostep(**kw))
    want_g = og.last_grads[1]
    want_p = og.export()
    ro = api.RenderOptions(tau=3000.0 * res)
    # the serialised schedule on the same inputs: the GPU's own reference for
    # the race check (check_same_schedule)
    ctx.upload(g, smooth=True)
    ctx.keep_raypass_grads(True)
    ctx.train_reset()
    ctx.train_step([cams[i] for i in batch], [gts[i] for i in batch], [masks[i] for i in batch],
                   api.step_params(**kw))
    serial = ctx.grads(1)
    for rep in range(repeats):
        ctx.upload(g, smooth=True)
        ctx.keep_raypass_grads(False)
        ctx.train_reset()
        if resident:
            ctx.upload_views(cams, [gts[i].astype(np.float32) for i in range(n_views)], masks)
        if render_first:  # a render right before: shared view table / hand-over bits
            ctx.render_image(cams[(rep + 1) % n_views], ro)
        hp = api.step_params(**kw)
        if resident:
            losses, counts = ctx.train_step_views(batch, hp)
        else:
            losses, counts = ctx.train_step([cams[i] for i in batch], [gts[i] for i in batch],
                                            [masks[i] for i in batch], hp)
        what = f"rep{rep} {'views' if resident else 'host'}"
        assert [counts[k] for k in ("n_rays", "n_marched", "n_extra", "n_shaded", "n_alpha",
                                    "n_bwd_rays")] == list(oc), (what, counts, oc)
        for i, k in enumerate(("photo", "sdf", "eik", "normal", "features", "probes")):
            assert abs(losses[k] - ol[i]) <= 1e-4 * max(abs(ol[i]), 1e-6), (what, k, losses[k], ol[i])
        assert abs(losses["psnr"] - ol[7]) <= 1e-3, (what, losses["psnr"], ol[7])
        got = ctx.grads(1)
        check_same_schedule(got, serial, what)
        check_grads(got, want_g, what, GRAD_TOL, kink_outliers)
        p = ctx.download()
        for k in ("raw", "planes", "probes", "mlp"):
            gk = want_g[k]
            sig = np.abs(gk) > 1e-4 * max(np.abs(gk).max(), 1e-30)
            d = np.abs(p[k].astype(np.float64) - want_p[k])
            assert d[sig].max(initial=0) <= 2e-3 * kw["lr_vox"] + 1e-6, (what, k, d[sig].max(initial=0))
        tol_sm = 1e-5 + 0.3 * kw["lr_vox"]
        assert np.abs(p["smooth"] - want_p["smooth"]).max() <= tol_sm, (what, np.abs(p["smooth"] - want_p["smooth"]).max())


@pytest.mark.parametrize("resident", [False, True])
def test_production_small_early_fork(ctx, resident):
    """64^3, 32x32 views: T * 1000 > rays, so the regularizers fork at the step
    start and the empty-ray loss must wait for the scan (ev_scanned)."""
    _production_parity(ctx, dict(res=64, n_s=4, n_a=4, sh_order=4, band=6), tau=30.0, size=32,
                       resident=resident)


@pytest.mark.parametrize("resident", [False, True])
def test_production_late_fork(ctx, resident):
    """Rays >> 1000 per tile: the regularizers fork after the first composite
    round (the bench's schedule)."""
    _production_parity(ctx, dict(res=64, n_s=4, n_a=4, sh_order=4, band=6), tau=300.0, size=256,
                       resident=resident)


def test_production_forced_early(ctx, monkeypatch):
    from paper_2412_10084_b200 import api
    monkeypatch.setenv("PSDF_REGS_EARLY", "1")
    c = api.Context(0)
    try:
        _production_parity(c, dict(res=128, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32), tau=300.0,
                           size=128)
    finally:
        c.close()


@pytest.mark.parametrize("resident", [False, True])
def test_production_bench_config(ctx, resident):
    """The bench's configs[1] step exactly: 512^3 grid, (4,4,4), a batch of
    4 views at 1600x1200 (7.68 M rays), tau = 300 / voxel, production
    schedule, three repeats."""
    _production_parity(ctx, dict(res=512, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32), tau=300.0,
                       size=1600, height=1200, n_views=4, repeats=3, resident=resident, kink_outliers=True)
