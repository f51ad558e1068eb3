"""Multi-GPU decomposition on CPU (gloo, world_size 2): each rank runs the
oracle's ray pass over its contiguous slice of the batch's work tiles and the
regularizers over its slice of tiles / probes, folds its own smooth-staged
gradient (G^T is linear), and the flat gradients are all-reduced.  The result
must equal the single-process step gradient — the exchange psdf.cu performs
with ncclAllReduce before Adam."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import cam_from_array, golden, scene32_arrays, step_params_from


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_grads(rank, world, z):
    from oracle.port import OracleGrid
    from paper_2412_10084_b200.api import shard
    og = OracleGrid(scene32_arrays(z), smooth=True)
    cams = [cam_from_array(v) for v in z["train_cams"]]
    hp = step_params_from(z["train_hp"])
    gb = og.new_grads()
    n_tiles = sum(((c.width + 7) // 8) * ((c.height + 3) // 4) for c in cams)
    t0, t1 = shard(n_tiles, rank, world)
    stats = og.raypass_tiles(cams, list(z["train_gt"]), list(z["train_mask"]), hp, t0, t1, gb)
    a = og.a
    lam = [hp.l_sdf, hp.l_eik, hp.l_norm, hp.l_feat, hp.l_probe]
    losses = [stats[0]]
    for which in range(5):
        n = a.P if which == 4 else a.T
        b, e = shard(n, rank, world)
        losses.append(og.regularizer_range(which, lam[which], b, e, gb)[0])
    og.gt_fold_into(gb)
    g = og.grads_of(gb)
    og.free_grads(gb)
    flat = np.concatenate([g[k].ravel() for k in ("raw", "planes", "probes", "mlp")])
    return flat, np.array(losses + [stats[1], stats[2]])


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = golden("scene32.npz")
    flat, losses = _rank_grads(rank, world, z)
    t = torch.from_numpy(flat)
    l = torch.from_numpy(losses)
    dist.all_reduce(t)
    dist.all_reduce(l)
    if rank == 0:
        np.savez(out_path, flat=t.numpy(), losses=l.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dp_shards_allreduce_equal_single_step(tmp_path, world):
    from oracle.port import OracleGrid
    z = golden("scene32.npz")
    out = str(tmp_path / "dp.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    # single-process reference step (the oracle's train step, stage-1 grads)
    og = OracleGrid(scene32_arrays(z), smooth=True)
    og.train_reset()
    losses, _ = og.train_step([cam_from_array(v) for v in z["train_cams"]], list(z["train_gt"]),
                              list(z["train_mask"]), step_params_from(z["train_hp"]))
    g = og.last_grads[1]
    want = np.concatenate([g[k].ravel() for k in ("raw", "planes", "probes", "mlp")])
    scale = np.abs(want).max()
    assert np.abs(got["flat"] - want).max() <= 1e-12 * scale
    # photo + the five regularizer values, and the PSNR partials
    assert np.allclose(got["losses"][:6], losses[:6], rtol=1e-12)
    assert np.allclose(got["losses"][6:], losses[8:10], rtol=1e-12)


def test_shard_partition_covers_exactly_once():
    from paper_2412_10084_b200.api import shard
    for n in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                b, e = shard(n, r, world)
                seen.extend(range(b, e))
            assert seen == list(range(n))
