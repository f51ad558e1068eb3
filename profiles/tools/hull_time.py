# Visual-hull init wall time at 256^3 / 512^3 with 49 views of 1600x1200 (profiles/r02/v36_hull_time.log).
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from paper_2412_10084_b200 import api
ctx = api.Context(0)
cams = api.make_ring_cameras(49, 1600, height=1200)
masks = []
for c in cams:
    yy, xx = np.mgrid[0:1200, 0:1600]
    masks.append((((xx - 800) ** 2 + (yy - 600) ** 2) < 330 ** 2).astype(np.uint8) * 255)
for res in (256, 512):
    cfg = api.GridConfig(voxel_size=1.0 / res, resolution=(res,) * 3, n_s=4, n_a=4, sh_order=4, band_voxels=6)
    for rep in range(3):
        t = time.perf_counter()
        g = ctx.init_visual_hull(cfg, cams, masks)
        print(res, rep, f"{time.perf_counter() - t:.3f} s", g.T, flush=True)
ctx.close()
