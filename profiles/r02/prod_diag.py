import sys, os, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from helpers import make_scene, oracle_with_f32_smooth, rel_l2
from test_gpu_train_production import _ocam, _views
from paper_2412_10084_b200 import api
from oracle.port import step_params as ostep
res = 512
g, a = make_scene(ncam=0, res=512, n_s=4, n_a=4, sh_order=4, band=6, radius=0.32)
og, sm = oracle_with_f32_smooth(a)
g.smooth = sm
cams = api.make_ring_cameras(4, 1600, height=1200)
ocams = [_ocam(c) for c in cams]
gts, masks = _views(og, ocams, 7, res)
kw = dict(tau=300.0 * res, lr_vox=1e-4, lr_mlp=6e-5, photo_scale=10.0)
og.train_reset()
ol, oc = og.train_step(ocams, gts, masks, ostep(**kw))
g0w, g1w = og.last_grads
ctx = api.Context(0)
outs = {}
for mode in ["serial", "prod", "prod2", "serial2"]:
    ctx.upload(g, smooth=True)
    ctx.keep_raypass_grads(mode.startswith("serial"))
    ctx.train_reset()
    losses, counts = ctx.train_step(cams, gts, masks, api.step_params(**kw))
    G1 = ctx.grads(1)
    outs[mode] = G1
    if mode.startswith("serial"):
        G0 = ctx.grads(0)
    for k in ("raw", "smooth", "planes", "probes", "mlp"):
        for stage, (G, W) in enumerate([(G1, g1w)] + ([(G0, g0w)] if mode.startswith("serial") else [])):
            d = np.abs(G[k].astype(np.float64) - W[k]).ravel()
            sc = np.abs(W[k]).max()
            idx = np.argsort(d)[-5:][::-1]
            print(mode, "stage", 1 - stage if stage == 0 else 0, k, "rel_l2 %.2e" % rel_l2(G[k], W[k]), "max/scale %.2e" % (d.max() / sc),
                  "n>1e-3:", int((d > 1e-3 * sc).sum()), "top", [(int(i), float(d[i]), float(W[k].ravel()[i])) for i in idx[:3]])
for k in ("raw", "planes", "probes", "mlp", "smooth"):
    d = np.abs(outs["prod"][k] - outs["prod2"][k]).max(); d2 = np.abs(outs["serial"][k] - outs["prod"][k]).max()
    print("gpu-vs-gpu", k, "prod/prod2 %.3e" % d, "serial/prod %.3e" % d2, "scale %.3e" % np.abs(outs["prod"][k]).max())
