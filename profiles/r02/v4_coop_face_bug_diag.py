import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from helpers import make_scene, oracle_with_f32_smooth
from paper_2412_10084_b200 import api
from oracle.refcore import RefCamera, render_opts

res = 64
g, a = make_scene(ncam=0, res=64, n_s=4, n_a=4, sh_order=4, band=6)
og, sm = oracle_with_f32_smooth(a)
g.smooth = sm
cams = api.make_ring_cameras(4, 32)
ocams = []
for c in cams:
    oc = RefCamera()
    for k in ("fx", "fy", "cx", "cy", "width", "height", "id"):
        setattr(oc, k, getattr(c, k))
    oc.rot[:] = list(c.rot); oc.pos[:] = list(c.pos)
    ocams.append(oc)
rng = np.random.default_rng(5)
gts, masks = [], []
for c in ocams:
    _, alpha, _, _ = og.render_image(c, render_opts(tau=3000.0 * 32))
    masks.append((alpha > 0.5).astype(np.float64))
    gts.append(rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32).astype(np.float64))
kw = dict(tau=30.0 * res, lr_vox=5e-3 / 50, lr_mlp=3e-3 / 50, photo_scale=40.0 / 2)
Q = {0: ("e_slot", np.int32, 1), 1: ("e_acc", np.float64, 1), 2: ("e_craw", np.float64, 3), 3: ("e_nlive", np.int32, 1),
     4: ("e_cfirst", np.int32, 1), 5: ("e_tfirst", np.float64, 1), 6: ("r_pos", np.float64, 3), 7: ("r_w", np.float64, 1),
     8: ("r_tile", np.int32, 1), 9: ("r_entry", np.int32, 1), 10: ("a_t", np.float64, 2), 11: ("a_s", np.float64, 3),
     12: ("a_i", np.int32, 4), 13: ("e_head", np.int32, 1), 14: ("e_ahead", np.int32, 1), 15: ("r_next", np.int32, 1)}
def dump(ctx):
    w = ctx.last_wave_counts()
    out = {}
    for k, (name, dt, m) in Q.items():
        n = w["entries"] if name.startswith("e_") else (w["records"] if name.startswith("r_") else w["alpha_samples"])
        arr = np.zeros((n, m), dt)
        ctx._check(ctx.L.psdf_debug_wave(ctx.h, k, arr.ctypes.data_as(C.c_void_p), n))
        out[name] = arr
    return out
def run(coop):
    os.environ["PSDF_COOP"] = coop
    os.environ["PSDF_COMPOSITE_STEPS"] = "1"
    ctx = api.Context(0)
    ctx.upload(g, smooth=True)
    ctx.keep_raypass_grads(True)
    ctx.train_reset()
    for step, batch in enumerate([[0, 1], [2, 3]]):
        losses, counts = ctx.train_step([cams[i] for i in batch], [gts[i] for i in batch], [masks[i] for i in batch], api.step_params(**kw))
    d = dump(ctx)
    ctx.close()
    return losses["photo"], d
p0, d0 = run("0")
p1, d1 = run("1")
print("photo", p0, p1)
def per_entry(d):
    m = {}
    for e in range(len(d["e_slot"])):
        s = int(d["e_slot"][e, 0])
        recs = np.where(d["r_entry"][:, 0] == e)[0]
        rr = sorted([(tuple(d["r_pos"][r]), float(d["r_w"][r, 0]), int(d["r_tile"][r, 0])) for r in recs])
        al = []
        a = int(d["e_ahead"][e, 0])
        while a >= 0:
            al.append((tuple(d["a_t"][a]), tuple(d["a_s"][a]), int(d["a_i"][a, 0]), int(d["a_i"][a, 1]), int(d["a_i"][a, 2]) >= 0))
            a = int(d["a_i"][a, 3])
        m[s] = dict(acc=float(d["e_acc"][e, 0]), craw=tuple(d["e_craw"][e]), nlive=int(d["e_nlive"][e, 0]),
                    cfirst=int(d["e_cfirst"][e, 0]), tfirst=float(d["e_tfirst"][e, 0]), recs=rr, alphas=al)
    return m
m0, m1 = per_entry(d0), per_entry(d1)
print("entries", len(m0), len(m1), "same slots", set(m0) == set(m1))
nd = 0
for s in sorted(m0):
    if s not in m1: print("missing", s); continue
    x, y = m0[s], m1[s]
    for k in x:
        if k == "craw" and np.allclose(x[k], y[k], rtol=1e-12, atol=0):
            continue
        if x[k] != y[k]:
            nd += 1
            if nd < 12:
                print("slot", s, "field", k)
                if k in ("recs", "alphas"):
                    for i, (u, v) in enumerate(zip(x[k], y[k])):
                        if u != v: print("   ", i, u, "\n    ", v)
                    if len(x[k]) != len(y[k]): print("   len", len(x[k]), len(y[k]))
                else:
                    print("   ", x[k], y[k])
print("n diffs", nd)

# host photo of the entries (photo_term, losses.cpp:8-38) from the dumps
def entry_photo(d, scale=40.0 / 2):
    tot = 0.0
    H = W = 32
    for e in range(len(d["e_slot"])):
        slot = int(d["e_slot"][e, 0]); wi, ln = slot >> 5, slot & 31
        tpv = ((W + 7) // 8) * ((H + 3) // 4)
        v = 2 + wi // tpv  # batch [2, 3]
        lt = wi % tpv
        u = (lt % ((W + 7) // 8)) * 8 + (ln & 7); vv = (lt // ((W + 7) // 8)) * 4 + (ln >> 3)
        acc = d["e_acc"][e, 0]; col = d["e_craw"][e] + 0.0 * (1 - acc)
        if masks[v][vv, u] > 0.5:
            gt = gts[v][vv, u]
            tot += scale * ((col - gt) ** 2).sum()
        else:
            tot += scale * acc * acc
    return tot
print("entry photo", entry_photo(d0), entry_photo(d1))
for k, name in ((13, "e_head"), (15, "r_next")):
    pass
def chains(d):
    out = {}
    for e in range(len(d["e_slot"])):
        r = int(d["e_head"][e, 0]); c = []
        while r >= 0 and len(c) < 10000:
            c.append(tuple(d["r_pos"][r])); r = int(d["r_next"][r, 0])
        out[int(d["e_slot"][e, 0])] = c
    return out
c0, c1 = chains(d0), chains(d1)
bad = [s for s in c0 if c0[s] != c1.get(s)]
print("record chains differing:", len(bad), bad[:10])
for s in bad[:3]:
    print(s, len(c0[s]), len(c1[s]))
