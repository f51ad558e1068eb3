"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libsdfrecon_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run in the dev container:  python tests/golden/make_golden.py

Fixtures (small; committed):
  kat.npz        known-answer values of the reference's unit tests, computed
                 by the reference itself (alpha, SH basis, Fresnel powers,
                 Gaussian taps, Adam, photo pixel, brackets).
  scene32.npz    a seeded 32^3 scene (test_renderer.cpp:21-45 pattern, all
                 parameters fp32-representable), two 16x16 training views and
                 a 24x24 render camera, with the reference's render outputs
                 (colour, alpha, depth, sample counts) at two tau, march
                 t-lists of 64 rays, and one train step (losses, counts,
                 ray-pass and final gradients, post-step parameters).
  init64.npz     init_grid_sphere at 64^3 (tile / probe ordering, raw SDF)
                 and reference cameras (make_lookat_camera, make_ring_cameras).
  mesh32.npz     the reference's marching_cubes of a jittered 32^3 sphere
                 scene and of a shifted copy, sample_mesh_points on both,
                 MeshDistance distances of probe points, and chamfer with and
                 without max_dist clipping (metrics.cpp).

    python tests/golden/make_golden.py [kat scene32 init64 mesh32]
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refcore as R  # noqa: E402


def cam_array(c):
    return np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height, *c.rot, *c.pos, c.id], np.float64)


def kat():
    L = R.reflib()
    out = {}
    out["alpha_1_m1_1"] = L.ref_alpha_from_sdf(1.0, -1.0, 1.0)
    out["alpha_m1_1_1"] = L.ref_alpha_from_sdf(-1.0, 1.0, 1.0)
    out["alpha_flat"] = L.ref_alpha_from_sdf(0.4, 0.4, 10.0)
    rng = np.random.default_rng(0)
    dirs = rng.normal(size=(16, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dirs[0] = [0, 0, 1]
    sh = np.zeros((16, 4, 16))
    for i, d in enumerate(dirs):
        for o in range(1, 5):
            buf = np.zeros(16)
            L.ref_eval_sh_basis(R.ptr(np.ascontiguousarray(d)), o, R.ptr(buf))
            sh[i, o - 1] = buf
    out["sh_dirs"], out["sh_values"] = dirs, sh
    ndv = np.array([-0.5, 0.0, 0.25, 0.75, 1.0, 1.5])
    fr = np.zeros((len(ndv), 6))
    for i, v in enumerate(ndv):
        L.ref_fresnel_powers(v, R.ptr(fr[i]))
    out["fresnel_ndv"], out["fresnel"] = ndv, fr
    taps = np.zeros(5)
    L.ref_gaussian_kernel(R.ptr(taps))
    out["gaussian"] = taps
    # Adam: the scalar-reference test of test_losses.cpp:277-310, 100 steps
    p0 = rng.uniform(-1, 1, 5)
    gs = rng.uniform(-1, 1, (100, 5))
    lrs = np.full(100, 0.01)
    p = p0.copy()
    L.ref_adam_steps(5, R.ptr(p), R.ptr(np.ascontiguousarray(gs)), 100, R.ptr(lrs))
    out["adam_p0"], out["adam_grads"], out["adam_lrs"], out["adam_p"] = p0, gs, lrs, p
    pp = np.zeros((2, 6))
    L.ref_photo_pixel(R.ptr(np.array([0.25] * 3)), R.ptr(np.array([0.5] * 3)), 1, 1.0, 1.0, R.ptr(pp[0]))
    L.ref_photo_pixel(R.ptr(np.array([0.25] * 3)), R.ptr(np.array([0.5] * 3)), 0, 0.5, 2.0, R.ptr(pp[1]))
    out["photo"] = pp
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)


def scene32():
    s = R.RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=32, radius=0.3, ncam=2,
                          mlp_seed=5)
    s.randomize(4, sdf_jitter=0.004)
    s.round_to_f32()
    a = s.export()
    out = dict(tile_coords=a.tile_coords, probe_ids=a.probe_ids, probe_coords=a.probe_coords,
               raw=a.raw, smooth=a.smooth, planes=a.planes, probes=a.probes, mlp=a.mlp,
               meta=np.array([a.n_s, a.n_a, a.sh_order, a.res[0], a.ncam], np.int64),
               geom=np.array([a.voxel_size, *a.origin, a.far_field_voxels]))
    rcam = R.lookat_camera(1, (1.3, 0.2, 0.4), (0, 0, 0), (0, 1, 0), 28.8, 28.8, 24, 24)
    out["render_cam"] = cam_array(rcam)
    for tag, tau in (("soft", 24.0), ("sharp", 2000.0)):
        rgb, alpha, depth, counts = s.render_image(rcam, R.render_opts(tau=tau, camera_id=1), threads=1)
        out[f"render_{tag}_rgb"], out[f"render_{tag}_alpha"] = rgb, alpha
        out[f"render_{tag}_depth"], out[f"render_{tag}_counts"] = depth, counts
    rng = np.random.default_rng(3)
    o = rng.uniform(-1.2, 1.2, (64, 3))
    t = rng.uniform(-0.4, 0.4, (64, 3))
    d = t - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ts = np.full((64, 512), np.nan)
    n = np.zeros(64, np.int64)
    for i in range(64):
        x = s.march_ray(o[i], d[i], 512)
        n[i] = len(x)
        ts[i, : len(x)] = x
    out["march_o"], out["march_d"], out["march_n"], out["march_ts"] = o, d, n, ts
    # one train step: 2 views of 16x16, GT = random colours, mask = silhouette
    cams = [R.lookat_camera(i, e, (0, 0, 0), (0, 1, 0), 19.2, 19.2, 16, 16)
            for i, e in enumerate([(1.6, 0.4, 0.9), (-1.2, -0.5, 1.3)])]
    gts, masks = [], []
    for c in cams:
        _, alpha, _, _ = s.render_image(c, R.render_opts(tau=2000.0), threads=1)
        masks.append((alpha > 0.5).astype(np.float64))
        gts.append(rng.uniform(0, 1, (16, 16, 3)).astype(np.float32).astype(np.float64))
    out["train_cams"] = np.stack([cam_array(c) for c in cams])
    out["train_gt"], out["train_mask"] = np.stack(gts), np.stack(masks)
    hp = R.RefStepParams()
    hp.tau, hp.lr_vox, hp.lr_mlp = 30.0 * 32, 1e-4, 6e-5
    hp.l_sdf, hp.l_eik, hp.l_norm, hp.l_feat, hp.l_probe, hp.photo_scale = 0.7, 0.3, 0.2, 0.15, 0.25, 20.0
    hp.use_camera_bias = 1
    out["train_hp"] = np.array([hp.tau, hp.lr_vox, hp.lr_mlp, hp.l_sdf, hp.l_eik, hp.l_norm, hp.l_feat,
                                hp.l_probe, hp.photo_scale, hp.use_camera_bias])
    s.train_reset()
    losses, counts = s.train_step(cams, gts, masks, hp, threads=1)
    out["train_losses"], out["train_counts"] = losses, counts
    for st in (0, 1):
        g = s.grads(st)
        for k, v in g.items():
            out[f"grad{st}_{k}"] = v.astype(np.float32)
    p = s.export()
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        out[f"post_{k}"] = getattr(p, k).astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "scene32.npz"), **out)


def init64():
    s = R.RefScene.sphere(res=64, n_s=4, n_a=4, sh_order=4, band_voxels=6, radius=0.32, ncam=0)
    a = s.export()
    out = dict(tile_coords=a.tile_coords, probe_ids=a.probe_ids, probe_coords=a.probe_coords,
               raw=a.raw.astype(np.float32))
    out["lookat"] = cam_array(R.lookat_camera(2, (1.3, 0.2, 0.4), (0.1, 0, -0.2), (0, 1, 0), 50.0, 40.0,
                                              40, 30))
    out["ring"] = np.stack([cam_array(c) for c in R.ring_cameras(6, 48, 2.0, 0.35, 17)])
    np.savez_compressed(os.path.join(HERE, "init64.npz"), **out)


def mesh32():
    s = R.RefScene.sphere(res=32, n_s=2, n_a=2, sh_order=2, band_voxels=6, radius=0.3, ncam=0)
    s.randomize(5, sdf_jitter=0.004)
    v, t = s.marching_cubes()
    v2 = v + np.array([0.004, -0.002, 0.001])
    rng = np.random.default_rng(11)
    probes = np.concatenate([rng.uniform(-0.7, 0.7, (300, 3)), v[:100] + rng.normal(0, 1e-3, (100, 3)),
                             v[100:120]])
    p1 = R.ref_sample_mesh_points(v, t, 2000, 1)
    p2 = R.ref_sample_mesh_points(v2, t, 2000, 2)
    out = dict(verts=v, tris=t, verts2=v2, probes=probes, probe_dist=R.ref_point_mesh_distance(probes, v, t),
               pred_pts=p1, gt_pts=p2, chamfer0=R.ref_chamfer(p1, v, t, p2, v2, t, 0.0),
               chamfer_clip=R.ref_chamfer(p1, v, t, p2, v2, t, 0.0045))
    np.savez_compressed(os.path.join(HERE, "mesh32.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kat", "scene32", "init64", "mesh32"]
    for name in which:
        globals()[name]()
        f = name + ".npz"
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
