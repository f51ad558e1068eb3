"""Pins the C restatement (oracle/psdf_oracle.c) to the UNMODIFIED reference
(oracle/_ref/libsdfrecon_ref.so) on randomized scenes: the forward pass, the
march t-lists, the per-ray backward, every regularizer and full train steps
must agree bit for bit (f64 arithmetic in the same operation order).
Skipped where the reference build is absent."""
import numpy as np
import pytest

from conftest import have_ref

pytestmark = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built (needs /root/reference)")


@pytest.fixture(scope="module")
def scene():
    from oracle import refcore as R
    from oracle.port import OracleGrid
    s = R.RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=32, radius=0.3, ncam=1)
    s.randomize(4, sdf_jitter=0.004)
    return s, OracleGrid(s.export())


def test_render_bit_exact(scene):
    from oracle import refcore as R
    s, og = scene
    cam = R.lookat_camera(0, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 38.4, 38.4, 32, 32)
    for tau in (0.75 * 32, 24.0, 2000.0):
        for kw in ({}, dict(no_spatial=True), dict(no_angular=True), dict(no_fresnel=True),
                   dict(sh_order_override=1), dict(bg=(0.2, 0.4, 0.6)), dict(early_stop=0.0)):
            o = R.render_opts(tau=tau, camera_id=0, **kw)
            r1 = s.render_image(cam, o, threads=1)
            r2 = og.render_image(cam, o)
            for x, y in zip(r1, r2):
                assert np.array_equal(np.asarray(x), np.asarray(y)), (tau, kw)


def test_march_bit_exact(scene):
    s, og = scene
    rng = np.random.default_rng(0)
    for _ in range(3000):
        o = rng.uniform(-1.5, 1.5, 3)
        d = rng.uniform(-0.4, 0.4, 3) - o
        d /= np.linalg.norm(d)
        assert np.array_equal(s.march_ray(o, d), og.march_ray(o, d))
    for d in ([1, 0, 0], [0, -1, 0], [0, 0, 1]):  # axis-parallel rays
        o = np.array([0.1, 0.2, -0.3]) - 2 * np.array(d)
        assert np.array_equal(s.march_ray(o, d), og.march_ray(o, d))


def test_ray_backward_bit_exact(scene):
    from oracle import refcore as R
    s, og = scene
    rng = np.random.default_rng(1)
    for i in range(20):
        o = rng.uniform(-1.2, 1.2, 3)
        d = rng.uniform(-0.3, 0.3, 3) - o
        d /= np.linalg.norm(d)
        opts = R.render_opts(tau=24.0, early_stop=0.0 if i % 2 else 1e-4, camera_id=0)
        up = rng.uniform(-1, 1, 3)
        g1 = s.ray_backward(o, d, opts, up, 0.7)
        g2 = og.ray_backward(o, d, opts, up, 0.7)
        for k in g1:
            assert np.array_equal(g1[k], g2[k]), (i, k)


def test_regularizers_bit_exact(scene):
    s, og = scene
    for which in range(5):
        (o1, g1), (o2, g2) = s.regularizer(which, 0.3), og.regularizer(which, 0.3)
        assert np.array_equal(o1, o2)
        for k in g1:
            if k == "mlp":
                continue
            assert np.array_equal(g1[k], g2[k]), (which, k)


def test_train_steps_bit_exact():
    from oracle import refcore as R
    from oracle.port import OracleGrid, step_params
    s = R.RefScene.sphere(res=32, n_s=4, n_a=4, sh_order=3, band_voxels=6, radius=0.32, ncam=0)
    s.randomize(1)
    og = OracleGrid(s.export())
    cams = R.ring_cameras(4, 24)
    gts, masks = zip(*[R.raytrace(R.GLOSSY_SPHERE, c) for c in cams])
    hp = step_params(tau=30 * 32, lr_vox=5e-3 / 50, lr_mlp=3e-3 / 50, photo_scale=20.0)
    for it in range(3):
        b = slice(2 * (it % 2), 2 * (it % 2) + 2)
        l1, c1 = s.train_step(cams[b], gts[b], masks[b], hp, threads=1)
        l2, c2 = og.train_step(cams[b], gts[b], masks[b], hp)
        assert np.array_equal(c1, c2)
        assert np.allclose(l1, l2, rtol=1e-13, atol=0)
        for st in (0, 1):
            ga, gb = s.grads(st), og.last_grads[st]
            for k in ga:
                assert np.array_equal(ga[k], gb[k]), (it, st, k)
        b_ = s.export()
        e = og.export()
        for k in e:
            assert np.array_equal(getattr(b_, k), e[k]), (it, k)


def test_step_mirror_matches_reference_train():
    """The harness's step mirror (ref_harness.cpp) equals the reference's own
    train() for a one-LOD schedule (same batch order from mt19937_64)."""
    from oracle import refcore as R
    from oracle.port import step_params
    mk = lambda: R.RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=6, radius=0.32, ncam=0)
    cams = R.ring_cameras(3, 16)
    gts, masks = zip(*[R.raytrace(R.GLOSSY_SPHERE, c) for c in cams])
    a, b = mk(), mk()
    br = [5e-3, 5e-3, 3e-3, 3e-3, 0.3, 0.3, 0.7, 0.7, 0.15, 0.15, 0.2, 0.2, 0.25, 0.25, 30.0, 30.0]
    a.train_full(list(cams), list(gts), list(masks), iterations=1, images_per_batch=3, brackets=br,
                 seed=0, threads=1)
    hp = step_params(tau=30 * 32, lr_vox=5e-3 / 50, lr_mlp=3e-3 / 50, l_sdf=0.7, l_eik=0.3, l_norm=0.2,
                     l_feat=0.15, l_probe=0.25, photo_scale=40.0 / 3)
    # train() shuffles the view order with mt19937_64(seed); with 3 views in one
    # batch every permutation gives the same gradient sum up to float order, so
    # compare at a tolerance
    b.train_step(list(cams), list(gts), list(masks), hp, threads=1)
    pa, pb = a.export(), b.export()
    for k in ("raw", "planes", "probes", "mlp"):
        assert np.allclose(getattr(pa, k), getattr(pb, k), rtol=0, atol=1e-12), k


def test_psnr_masked_bit_exact():
    """oracle.port.psnr_masked against the reference's psnr_masked
    (metrics.cpp:196-211) through the harness: random images, a random mask,
    an empty mask and an exact match."""
    import ctypes as C
    from oracle import refcore as R
    from oracle.port import psnr_masked
    L = R.reflib()
    rng = np.random.default_rng(3)
    h, w = 23, 37
    img, gt = rng.uniform(0, 1, (h, w, 3)), rng.uniform(0, 1, (h, w, 3))
    for mask in (rng.uniform(0, 1, (h, w)), np.zeros((h, w)), np.ones((h, w))):
        for a in (img, gt):
            out = np.zeros(1)
            R._check(L.ref_psnr_masked(R.ptr(np.ascontiguousarray(a)), R.ptr(gt), R.ptr(mask), w, h,
                                       R.ptr(out)), L)
            assert psnr_masked(a, gt, mask) == out[0]


@pytest.fixture(scope="module")
def mc_mesh():
    """The reference's own marching_cubes (mesh.cpp:363) of a jittered sphere scene."""
    from oracle import refcore as R
    s = R.RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=6, radius=0.3, ncam=0)
    s.randomize(5, sdf_jitter=0.004)
    return s.marching_cubes()


def test_point_mesh_distance_bit_exact(mc_mesh):
    """oracle.port.point_mesh_distance (brute-force restatement of
    metrics.cpp:11-47) against MeshDistance (BVH, metrics.cpp:48-135)."""
    from oracle import refcore as R
    from oracle.port import point_mesh_distance
    v, t = mc_mesh
    assert len(t) > 500
    rng = np.random.default_rng(11)
    pts = np.concatenate([rng.uniform(-0.7, 0.7, (150, 3)), v[:50] + rng.normal(0, 1e-3, (50, 3)), v[50:60]])
    assert np.array_equal(point_mesh_distance(pts, v, t), R.ref_point_mesh_distance(pts, v, t))


def test_chamfer_bit_exact(mc_mesh):
    """oracle.port.chamfer against chamfer (metrics.cpp:182-194) on the
    reference's sampled surface points, with and without max_dist clipping."""
    from oracle import refcore as R
    from oracle.port import chamfer
    v, t = mc_mesh
    # a second mesh: the same surface shifted by a fraction of a voxel
    v2 = v + np.array([0.004, -0.002, 0.001])
    p1 = R.ref_sample_mesh_points(v, t, 300, 1)
    p2 = R.ref_sample_mesh_points(v2, t, 300, 2)
    for md in (0.0, 0.0045):
        assert np.array_equal(chamfer(p1, v, t, p2, v2, t, md), R.ref_chamfer(p1, v, t, p2, v2, t, md))
    with pytest.raises(RuntimeError, match="empty mesh"):
        R.ref_point_mesh_distance(p1, v, t[:0])


def test_point_mesh_distance_degenerate_soup():
    """Unstructured triangles with a repeated corner and a collinear sliver
    (NaN closest-point parameters): the restatement keeps std::min's NaN
    behaviour."""
    from oracle import refcore as R
    from oracle.port import point_mesh_distance
    rng = np.random.default_rng(0)
    nt = 300
    v = rng.uniform(-0.5, 0.5, (3 * nt, 3))
    v[3 * 5 + 1] = v[3 * 5]
    v[3 * 9 + 2] = 0.5 * (v[3 * 9] + v[3 * 9 + 1])
    t = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
    pts = np.concatenate([rng.uniform(-0.8, 0.8, (100, 3)), v[:40]])
    assert np.array_equal(point_mesh_distance(pts, v, t), R.ref_point_mesh_distance(pts, v, t))
