"""Times the evaluation kernels (metrics.cpp on the GPU) against the
reference's CPU implementation (oracle/_ref) on acceptance-style inputs:
the reference's marching cubes of a sphere scene, sample_mesh_points on it
and on a scaled copy, two-way chamfer.  Prints one JSON line per size.

    python profiles/eval_timing.py [RES ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import refcore as R  # noqa: E402
from paper_2412_10084_b200 import api  # noqa: E402


def run(res, n_pts=20000, reps=5):
    s = R.RefScene.sphere(res=res, n_s=2, n_a=2, sh_order=2, band_voxels=6, radius=0.3, ncam=0)
    s.randomize(2, sdf_jitter=0.004)
    v, t = s.marching_cubes()
    v2 = v * 1.01
    p1 = R.ref_sample_mesh_points(v, t, n_pts, 1)
    p2 = R.ref_sample_mesh_points(v2, t, n_pts, 2)
    ctx = api.Context(0)
    ctx.chamfer(p1, v, t, p2, v2, t)  # warm-up
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = ctx.chamfer(p1, v, t, p2, v2, t)
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    ref = R.ref_chamfer(p1, v, t, p2, v2, t, 0.0)
    t_ref = time.perf_counter() - t0
    ctx.close()
    return dict(workload=f"chamfer: reference marching cubes of a {res}^3 sphere scene ({len(t)} triangles), "
                         f"{n_pts} sampled points per side", gpu_ms_median=1e3 * float(np.median(ts)),
                gpu_note="host wall clock of psdf_chamfer incl. H2D of meshes/points and D2H of distances",
                ref_ms=1e3 * t_ref, ref_note="reference chamfer (BVH MeshDistance, single thread)",
                bit_exact=[r["accuracy"], r["completeness"], r["mean"]] == list(ref))


if __name__ == "__main__":
    for res in [int(a) for a in sys.argv[1:]] or [128, 512]:
        print(json.dumps(run(res)), flush=True)
