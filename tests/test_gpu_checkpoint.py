"""SDFC v1 checkpoints against the unmodified reference's
own save_checkpoint / load_checkpoint (oracle/_ref): a file the reference
writes loads onto the device with identical values, and the device's save of
it is byte-identical to the reference's file (the reference's own
save(load(save(x))) contract, checkpoint.hpp:11-12); a device save loads in
the reference with identical values; errors map to std::runtime_error."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref_scene(n_s=4, n_a=4):
    from oracle.refcore import RefScene
    s = RefScene.sphere(res=32, n_s=n_s, n_a=n_a, sh_order=3, band_voxels=4, radius=0.3, ncam=3, mlp_seed=7)
    s.randomize(11, sdf_jitter=0.003, plane_amp=0.2, probe_amp=0.3, bias_amp=0.1)
    return s


@pytest.mark.parametrize("ns,na", [(4, 4), (3, 5)])
def test_checkpoint_roundtrip_bytes(ctx, tmp_path, ns, na):
    """(3, 5) has no kernel instantiation: the device holds it zero-padded to
    (4, 8) and the file keeps the reference's widths byte for byte."""
    s = _ref_scene(ns, na)
    f_ref, f_gpu = tmp_path / "ref.sdfc", tmp_path / "gpu.sdfc"
    s.save_checkpoint(f_ref, lod_cursor=2, iteration=17, seed=12345678901)
    g, meta = ctx.load_checkpoint(f_ref)
    assert meta == dict(lod=0, band_voxels=4, lod_cursor=2, iteration=17, seed=12345678901)
    a = s.export()
    assert np.array_equal(g.tile_coords, a.tile_coords) and np.array_equal(g.probe_coords, a.probe_coords)
    assert np.array_equal(g.probe_ids, a.probe_ids)
    np.testing.assert_array_equal(g.raw, a.raw.astype(np.float32))
    np.testing.assert_array_equal(g.planes, a.planes.astype(np.float32).ravel())
    np.testing.assert_array_equal(g.probes, a.probes.astype(np.float32).ravel())
    np.testing.assert_array_equal(g.mlp, a.mlp.astype(np.float32))
    ctx.save_checkpoint(f_gpu, lod=meta["lod"], lod_cursor=2, iteration=17, seed=12345678901)
    assert f_gpu.read_bytes() == f_ref.read_bytes()


def test_checkpoint_device_save_loads_in_reference(ctx, tmp_path):
    from oracle.refcore import RefScene
    from paper_2412_10084_b200 import api
    from helpers import make_scene
    g, _ = make_scene(res=32, n_s=2, n_a=2, sh_order=2, band=4, ncam=2)
    ctx.upload(g, smooth=False)
    f = tmp_path / "gpu.sdfc"
    ctx.save_checkpoint(f, lod=1, lod_cursor=1, iteration=5, seed=9)
    r, meta = RefScene.load_checkpoint(f)
    assert meta == (1, 5, 9)
    b = r.export()
    assert np.array_equal(b.tile_coords, g.tile_coords) and np.array_equal(b.probe_coords, g.probe_coords)
    np.testing.assert_array_equal(b.raw, g.raw.astype(np.float64))
    np.testing.assert_array_equal(b.planes.ravel(), g.planes.astype(np.float64).ravel())
    np.testing.assert_array_equal(b.probes.ravel(), g.probes.astype(np.float64).ravel())
    np.testing.assert_array_equal(b.mlp, g.mlp.astype(np.float64))


def test_checkpoint_errors(ctx, tmp_path):
    from paper_2412_10084_b200 import _lib
    s = _ref_scene()
    f = tmp_path / "ref.sdfc"
    s.save_checkpoint(f)
    data = f.read_bytes()
    bad = tmp_path / "bad.sdfc"
    bad.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(_lib.PsdfError, match="bad magic"):
        ctx.load_checkpoint(bad)
    bad.write_bytes(data[: len(data) // 2])
    with pytest.raises(_lib.PsdfError, match="truncated"):
        ctx.load_checkpoint(bad)
    with pytest.raises(_lib.PsdfError, match="cannot open"):
        ctx.load_checkpoint(tmp_path / "missing.sdfc")
