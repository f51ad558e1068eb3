"""The C oracle (oracle/psdf_oracle.c) against golden fixtures produced by the
unmodified reference (tests/golden/make_golden.py) and against the published
known-answer constants of the reference's own unit tests."""
import math
import os

import numpy as np
import pytest

from conftest import have_ref
from helpers import cam_from_array, golden, scene32_arrays, step_params_from


@pytest.fixture(scope="module")
def kat():
    return golden("kat.npz")


def test_alpha_known_answer(kat):
    from oracle.port import kat_alpha
    # test_renderer.cpp:49-61 / acceptance.cpp:238-240
    assert abs(kat_alpha(1.0, -1.0, 1.0) - 0.6321206) < 1e-6
    assert kat_alpha(1.0, -1.0, 1.0) == kat["alpha_1_m1_1"]
    assert kat_alpha(-1.0, 1.0, 1.0) == kat["alpha_m1_1_1"] == 0.0
    assert kat_alpha(0.4, 0.4, 10.0) == kat["alpha_flat"] == 0.0
    assert kat_alpha(0.5, -0.5, 2.0) > kat_alpha(0.5, -0.1, 2.0)


def test_sh_basis_known_answer(kat):
    from oracle.port import kat_sh
    # test_sh.cpp:84-93: Y_0 = 1/(2 sqrt(pi)); at +z only Y_0, Y_2, Y_6, Y_12 are non-zero
    y = kat_sh((0, 0, 1), 4)
    assert abs(y[0] - 0.2820948) < 1e-7
    for i, d in enumerate(kat["sh_dirs"]):
        for o in range(1, 5):
            assert np.array_equal(kat_sh(d, o), kat["sh_values"][i, o - 1, : o * o])


def test_fresnel_known_answer(kat):
    from oracle.port import kat_fresnel
    # test_decoder.cpp:62-74: u = 1 - 0.75 = 0.25 -> powers 0.25^k
    assert np.allclose(kat_fresnel(0.75), [0.25 ** k for k in range(6)], atol=0, rtol=1e-15)
    for v, want in zip(kat["fresnel_ndv"], kat["fresnel"]):
        assert np.array_equal(kat_fresnel(v), want)


def test_gaussian_taps_known_answer(kat):
    from oracle.port import kat_gaussian
    w = kat_gaussian()
    assert np.array_equal(w, kat["gaussian"])
    # test_grid.cpp:47-57: ratios exp(-1/2), exp(-2); normalised
    assert abs(w[1] / w[2] - math.exp(-0.5)) < 1e-12 and abs(w[0] / w[2] - math.exp(-2.0)) < 1e-12
    assert abs(w.sum() - 1.0) < 1e-12


def test_adam_known_answer(kat):
    from oracle.port import kat_adam
    # test_losses.cpp:277-310 scalar reference, 100 steps
    p = kat_adam(kat["adam_p0"], kat["adam_grads"], kat["adam_lrs"])
    assert np.array_equal(p, kat["adam_p"])
    # a single unit-gradient step moves by just under lr; zero gradient is a no-op
    assert abs(kat_adam([0.0], [[1.0]], [0.5])[0] + 0.5) < 1e-6
    assert kat_adam([0.4], [[0.0]], [0.5])[0] == 0.4


def test_photo_pixel_known_answer(kat):
    from oracle.port import lib
    from oracle.refcore import ptr
    out = np.zeros(6)
    lib().og_photo_pixel(ptr(np.array([0.25] * 3)), ptr(np.array([0.5] * 3)), 1, 1.0, 1.0, ptr(out))
    assert abs(out[2] - (-0.998004)) < 1e-6  # test_losses.cpp:59-76
    assert np.array_equal(out, kat["photo"][0])
    lib().og_photo_pixel(ptr(np.array([0.25] * 3)), ptr(np.array([0.5] * 3)), 0, 0.5, 2.0, ptr(out))
    assert np.array_equal(out, kat["photo"][1])


@pytest.fixture(scope="module")
def scene():
    from oracle.port import OracleGrid
    z = golden("scene32.npz")
    return z, OracleGrid(scene32_arrays(z), smooth=True)


def test_scene_smoothing_matches(scene):
    """The oracle's own smoothing of the golden raw SDF reproduces the golden
    smoothed field (fp32-rounded by the generator) to fp32 rounding."""
    from oracle.port import OracleGrid
    z, _ = scene
    og = OracleGrid(scene32_arrays(z), smooth=False)
    # the generator smoothed the raw field before rounding it to fp32, so the
    # difference is the smoothing of <= 1 ulp raw rounding: a few fp32 ulps of
    # the field's magnitude
    scale = float(np.spacing(np.float32(np.abs(z["raw"]).max())))
    assert np.abs(og.export()["smooth"] - z["smooth"]).max() <= 4 * scale


def test_scene_march_bit_exact(scene):
    z, og = scene
    for i in range(len(z["march_n"])):
        ts = og.march_ray(z["march_o"][i], z["march_d"][i], 512)
        n = int(z["march_n"][i])
        assert len(ts) == n and np.array_equal(ts, z["march_ts"][i, :n])


@pytest.mark.parametrize("tag,tau", [("soft", 24.0), ("sharp", 2000.0)])
def test_scene_render_bit_exact(scene, tag, tau):
    from oracle.refcore import render_opts
    z, og = scene
    cam = cam_from_array(z["render_cam"])
    rgb, alpha, depth, counts = og.render_image(cam, render_opts(tau=tau, camera_id=1))
    assert np.array_equal(counts, z[f"render_{tag}_counts"])
    assert np.array_equal(rgb, z[f"render_{tag}_rgb"])
    assert np.array_equal(alpha, z[f"render_{tag}_alpha"])
    assert np.array_equal(depth, z[f"render_{tag}_depth"])


def test_scene_train_step(scene):
    from oracle.port import OracleGrid
    z, _ = scene
    og = OracleGrid(scene32_arrays(z), smooth=True)
    cams = [cam_from_array(v) for v in z["train_cams"]]
    og.train_reset()
    losses, counts = og.train_step(cams, list(z["train_gt"]), list(z["train_mask"]),
                                   step_params_from(z["train_hp"]))
    assert np.array_equal(counts, z["train_counts"])
    assert np.allclose(losses, z["train_losses"], rtol=1e-12, atol=1e-12)
    for st in (0, 1):
        for k, v in og.last_grads[st].items():
            want = z[f"grad{st}_{k}"]
            assert np.array_equal(v.astype(np.float32), want), (st, k)
    p = og.export()
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        assert np.array_equal(p[k].astype(np.float32), z[f"post_{k}"]), k


def test_host_init_matches_reference():
    """The product's host-side init_grid_sphere (numpy) allocates tiles and
    corner probes in the reference's order (grid.cpp:58-76, 359-398)."""
    from paper_2412_10084_b200 import api
    z = golden("init64.npz")
    cfg = api.GridConfig(voxel_size=1 / 64, resolution=(64, 64, 64), n_s=4, n_a=4, sh_order=4,
                         band_voxels=6)
    g = api.init_grid_sphere(cfg, (0, 0, 0), 0.32)
    assert np.array_equal(g.tile_coords, z["tile_coords"])
    assert np.array_equal(g.probe_ids, z["probe_ids"])
    assert np.array_equal(g.probe_coords, z["probe_coords"])
    assert np.abs(g.raw - z["raw"]).max() < 1e-6


def test_host_cameras_match_reference():
    from paper_2412_10084_b200 import api
    z = golden("init64.npz")

    def arr(c):
        return np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height, *c.rot, *c.pos, c.id])

    c = api.make_lookat_camera(2, (1.3, 0.2, 0.4), (0.1, 0, -0.2), (0, 1, 0), 50.0, 40.0, 40, 30)
    assert np.allclose(arr(c), z["lookat"], rtol=0, atol=1e-15)
    for c, want in zip(api.make_ring_cameras(6, 48, 2.0, 0.35, 17), z["ring"]):
        assert np.allclose(arr(c), want, rtol=0, atol=1e-15)


def test_mesh_distance_golden():
    """oracle.port.point_mesh_distance / chamfer against the reference's
    MeshDistance and chamfer on its own marching-cubes mesh (mesh32.npz)."""
    from oracle.port import chamfer, point_mesh_distance
    g = golden("mesh32.npz")
    v, t, v2 = g["verts"], g["tris"], g["verts2"]
    assert np.array_equal(point_mesh_distance(g["probes"], v, t), g["probe_dist"])
    p1, p2 = g["pred_pts"][:400], g["gt_pts"][:400]
    full = chamfer(g["pred_pts"], v, t, g["gt_pts"], v2, t, 0.0)
    assert np.array_equal(full, g["chamfer0"])
    assert np.array_equal(chamfer(g["pred_pts"], v, t, g["gt_pts"], v2, t, 0.0045), g["chamfer_clip"])
    with pytest.raises(ValueError, match="empty input"):
        chamfer(p1[:0], v, t, p2, v2, t, 0.0)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_mc_case_table_matches_reference():
    """The device's packed 256-case triangle table (psdf_mesh.cuh kMcTri)
    emits, for every case of a single cell, the reference's triangles in the
    reference's order (marching_cubes_field over a 2x2x2 field of +-1)."""
    import re
    from oracle.refcore import ref_marching_cubes_field
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2412_10084_b200", "csrc",
                            "psdf_mesh.cuh")).read()
    body = src[src.index("kMcTri[256] = {"):]
    words = [int(w, 16) for w in re.findall(r"0x([0-9a-f]{16})ull", body[:body.index("};")])]
    assert len(words) == 256
    corner = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    edges = [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4), (0, 4), (1, 5), (2, 6), (3, 7)]
    mid = {tuple((np.array(corner[a]) + np.array(corner[b])) / 2): e for e, (a, b) in enumerate(edges)}
    for ci in range(256):
        f = np.zeros((2, 2, 2))
        for c, (x, y, z) in enumerate(corner):
            f[x, y, z] = -1.0 if (ci >> c) & 1 else 1.0
        v, t = ref_marching_cubes_field(f)
        want = [mid[tuple(v[i])] for tri in t for i in tri]
        w = words[ci]
        got = [(w >> (4 * k)) & 15 for k in range(3 * (w >> 60))]
        assert got == want, (ci, got, want)
