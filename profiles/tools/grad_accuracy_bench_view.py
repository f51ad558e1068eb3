# Gradient accuracy of one full 1600x1200 bench-view train step against the f64 oracle (per-tensor rel-L2, max/scale, count over 1e-3); v43/v44/v45 logs.
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np
import test_gpu_train as T
from paper_2412_10084_b200 import api

def chk(got, want, what):
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        g = np.asarray(got[k], np.float64); w = np.asarray(want[k], np.float64)
        sc = np.abs(w).max()
        if sc == 0:
            print(what, k, "zero"); continue
        d = np.abs(g - w)
        print(what, k, "rel_l2 %.2e" % T.rel_l2(g, w), "max/scale %.2e" % (d.max() / sc),
              "n>1e-3 %d" % int((d > 1e-3 * sc).sum()), "of", d.size, flush=True)
T._check_grads = chk
ctx = api.Context(0)
T._train_parity(ctx, dict(scene=dict(res=512, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32), tau=300.0,
                          size=1600, height=1200, n_views=1, batches=[[0]], ncam=0, bias=False))
ctx.close()
