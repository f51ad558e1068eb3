"""The product's own multi-rank decomposition, on one GPU (psdf.cu
do_train_step with psdf_debug_set_shard: rank r of N processes its
contiguous 1/N of the batch's 8x4 work tiles, tiles [r T/N, (r+1) T/N) of
the tile regularizers and probes [r P/N, (r+1) P/N) of the probe term, and
psdf_train_step copies only the pixel rows of its slice).  Without the
all-reduce, the N ranks' stage-1 gradients (after the per-rank G^T fold,
which is linear), loss statistics and counts must sum to the one-rank step —
the NCCL all-reduce then makes every rank hold that sum (GradBuffers::add
across GPUs, trainer.cpp:184-185)."""
import numpy as np
import pytest

from helpers import make_scene

pytestmark = pytest.mark.gpu


def _setup(seed=3, n_views=3, size=48):
    from paper_2412_10084_b200 import api
    g, _ = make_scene(res=64, n_s=4, n_a=4, sh_order=4, band=6, ncam=0)
    cams = api.make_ring_cameras(n_views, size, height=size - 8)
    rng = np.random.default_rng(seed)
    gts = [rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32) for c in cams]
    return g, cams, gts


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("resident", [False, True])
def test_shards_sum_to_one_rank(world, resident):
    from paper_2412_10084_b200 import api
    g, cams, gts = _setup()
    c1 = api.Context(0)
    try:
        c1.upload(g)
        masks = [c1.render_image(c, api.RenderOptions(tau=3000.0 * 64))[1] > 0.5 for c in cams]
        hp = api.step_params(tau=30.0 * 64, lr_vox=1e-4, lr_mlp=6e-5, photo_scale=40.0 / len(cams))

        def step(ctx):
            ctx.upload(g)
            ctx.train_reset()
            if resident:
                ctx.upload_views(cams, gts, masks)
                return ctx.train_step_views(list(range(len(cams))), hp)
            return ctx.train_step(cams, gts, masks, hp)

        l1, n1 = step(c1)
        full_h2d = c1.last_h2d_bytes()
        g1 = c1.grads(1)
        parts = []
        for r in range(world):
            c = api.Context(0)
            try:
                c.debug_set_shard(r, world)
                l, n = step(c)
                parts.append((l, n, c.grads(1), c.last_h2d_bytes()))
            finally:
                c.close()
    finally:
        c1.close()
    for k in ("n_marched", "n_extra", "n_shaded", "n_alpha", "n_bwd_rays"):
        assert sum(p[1][k] for p in parts) == n1[k], k
    for k in ("photo", "sdf", "eik", "normal", "features", "probes", "sq_err", "mask_px"):
        s = sum(p[0][k] for p in parts)
        assert abs(s - l1[k]) <= 1e-6 * max(abs(l1[k]), 1e-9), (k, s, l1[k])
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        s = sum(p[2][k].astype(np.float64) for p in parts)
        scale = max(np.abs(g1[k]).max(), 1e-30)
        assert np.abs(s - g1[k]).max() <= 2e-5 * scale, (k, np.abs(s - g1[k]).max() / scale)
    if not resident:
        # each rank copies only its slice's rows (plus at most one partial
        # 4-row band per view boundary)
        h2d = [p[3] for p in parts]
        assert sum(h2d) <= full_h2d * 1.2 and max(h2d) < full_h2d * (1.0 / world + 0.25), (h2d, full_h2d)
