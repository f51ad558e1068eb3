#!/usr/bin/env python
"""Benchmark of the B200-native ProbeSDF hot path (BASELINE.json configs[1]).

A "step" is one iteration of train()'s loop body (trainer.cpp:136-195) on a
batch of views (the DTU LOD-0 batch of 4 views per GPU, PAPER.md supp.
Table 5): fused ray pass (K2) + regularizers + G^T fold + [all-reduce] + Adam
+ re-smoothing.

Workload (config.workload, default = configs[1]): a synthetic DTU-scale
object — a 512^3 sparse grid, sphere-initialised (r = 0.32, band 6 voxels,
T = 2848 tiles, P = 4830 probes at tile corners, (n_s, n_a, l) = (4, 4, 4))
with seeded trained-like features — and 49 ring views at 1600x1200 whose
ground truth is rendered from a differently-seeded target model.  tau = 300 /
voxel (the geometric middle of the default [30, 3000] bracket).
`--config 2`: configs[2], the MVMannequins-scale synthetic human (a union of
boxes, spheres and tori, api.SCENE_PRIMS["human"]) with 68 cameras at
2048x1536 and a fixed global batch of 8 views (strong scaling).

Metric: marched samples per second (N_m, counted after early termination —
identical to the reference's RayWorkspace counts, tests/test_gpu_train*.py),
whole job over all ranks.  `value` is device-timed with inputs resident in
HBM; `e2e` goes through the C ABI call psdf_train_step with pinned host image
buffers, host->device copies (each rank copies only its slice's rows) and the
loss read-back inside the timed region.

Multi-GPU: `--gpus N` re-launches itself under torch.distributed.run (one
process per GPU, NCCL); ray-batch data parallelism, each rank renders its
contiguous 1/N of the batch's work tiles, grid gradients all-reduced before
Adam.  Weak scaling by default (4 views per GPU); `--scaling strong` keeps the
global batch fixed.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libsdfrecon_ref.so, the unmodified /root/reference sources
through its public API, trainer.cpp:136-195 step body) on all host cores: the
same global batch of views per step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NS = NA = 4
SH_ORDER = 4
RADIUS = 0.32
TAU_VOX = 300.0
LAMBDA_PHOTO = 40.0
BATCH_PER_GPU = 4

CONFIGS = {
    1: dict(scene="sphere", res=512, views=49, width=1600, height=1200, batch=BATCH_PER_GPU, scaling="weak",
            name="configs[1]: DTU-scale synthetic object"),
    2: dict(scene="human", res=512, views=68, width=2048, height=1536, batch=8, scaling="strong",
            name="configs[2]: MVMannequins-scale synthetic human (union of boxes, spheres, tori)"),
}
W = dict(CONFIGS[1])
# DTU LOD-0 loss weights (PAPER.md supp. Table 5); learning rates are the
# acceptance schedule's final-LOD values (acceptance.cpp:98-100) scaled by the
# 64^3 -> R^3 voxel-size ratio, so the timed steps keep a surface-like SDF
# (the paper's 0.01 is 5 voxels per Adam step at 512^3 and destroys the scene).
HP = dict(lr_vox=8e-4 * 64 / 512, lr_mlp=8e-4, l_sdf=0.2, l_eik=0.1, l_norm=0.05, l_feat=0.05, l_probe=0.2)


def algorithmic_bytes(c, mode="train"):
    """fp32 gather model, no cross-sample reuse."""
    f_sh = 6 * 8 + 3 * 4 * NS + 8 * SH_ORDER * SH_ORDER * NA  # 608 floats at (4,4,4)
    b_fwd = 32 * (c["n_marched"] + c["n_extra"]) + 4 * f_sh * c["n_shaded"] + 16 * c["n_rays"]
    if mode == "render":
        return b_fwd
    return b_fwd + 64 * c["n_alpha"] + 4 * f_sh * c["n_shaded"]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for t, r in self.rows if t0 - 0.15 <= t <= t1 + 0.15] or [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def grid_config(api):
    return api.GridConfig(voxel_size=1.0 / W["res"], resolution=(W["res"],) * 3, n_s=NS, n_a=NA,
                          sh_order=SH_ORDER, band_voxels=6)


def build_scene(api, seed):
    """The trained-like model and the differently-seeded target model (same
    geometry), as fp32 host grids."""
    cfg = grid_config(api)
    if W["scene"] == "sphere":
        g = api.init_grid_sphere(cfg, (0, 0, 0), RADIUS, ncam=0, mlp_seed=seed)
    else:
        g = api.init_grid_analytic(cfg, W["scene"], ncam=0, mlp_seed=seed)
    rng = np.random.default_rng(seed)
    g.planes = (0.5 + 0.2 * rng.uniform(-1, 1, g.planes.shape)).astype(np.float32)
    g.probes = (0.3 * rng.uniform(-1, 1, g.probes.shape)).astype(np.float32)
    tgt = api.HostGrid(cfg, g.tile_coords, g.probe_ids, g.probe_coords, g.raw,
                       (0.5 + 0.2 * rng.uniform(-1, 1, g.planes.shape)).astype(np.float32),
                       (0.3 * rng.uniform(-1, 1, g.probes.shape)).astype(np.float32),
                       api.glorot_mlp(NS, NA, 0, seed + 100))
    return g, tgt


def cameras(api):
    return api.make_ring_cameras(W["views"], W["width"], height=W["height"])


def make_views(api, ctx, tgt, cams):
    ctx.upload(tgt)
    gts, masks = [], []
    for c in cams:
        rgb, alpha, _, _ = ctx.render_image(c, api.RenderOptions(tau=3000.0 * W["res"]), depth=False)
        gts.append(rgb)
        masks.append(alpha > 0.5)
    return gts, masks


def pinned_copy(L, arr):
    """Copies a numpy array into page-locked host memory (psdf_host_alloc)."""
    p = L.psdf_host_alloc(arr.nbytes)
    if not p:
        raise MemoryError("psdf_host_alloc failed")
    buf = (C.c_uint8 * arr.nbytes).from_address(p)
    out = np.frombuffer(buf, dtype=arr.dtype).reshape(arr.shape)
    out[...] = arr
    return p, out


def global_batch(world):
    return W["batch"] * world if W["scaling"] == "weak" else W["batch"]


def batch_ids(it, world):
    """The global batch of step `it`: every rank holds all views and renders its
    contiguous 1/N of the batch's work tiles."""
    n = global_batch(world)
    base = (it * n) % W["views"]
    return [(base + k) % W["views"] for k in range(n)]


def hp_kwargs(world):
    return dict(tau=TAU_VOX * W["res"], photo_scale=LAMBDA_PHOTO / global_batch(world), **HP)


# --------------------------------------------------------------------------
# the reference's own CPU implementation (oracle/_ref, unmodified sources)
# --------------------------------------------------------------------------
def ref_scene(g):
    """The reference's grid with the same structure and values as `g`."""
    from oracle import refcore as R
    if W["scene"] == "sphere":
        s = R.RefScene.sphere(res=W["res"], n_s=NS, n_a=NA, sh_order=SH_ORDER, band_voxels=6, radius=RADIUS,
                              ncam=0)
    else:
        from paper_2412_10084_b200 import api
        s = R.RefScene.analytic(api.SCENE_PRIMS[W["scene"]], res=W["res"], n_s=NS, n_a=NA, sh_order=SH_ORDER,
                                band_voxels=6, ncam=0)
    a = s.export()
    assert a.T == g.T and np.array_equal(a.tile_coords, g.tile_coords)
    s.import_(raw=g.raw.astype(np.float64), planes=g.planes.astype(np.float64),
              probes=g.probes.astype(np.float64), mlp=g.mlp.astype(np.float64))
    return s


def ref_cam(c, i):
    from oracle import refcore as R
    return R.camera_from_dict(dict(fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy, width=c.width, height=c.height,
                                   rot=list(c.rot), pos=list(c.pos), id=i))


def ref_steps(s, cams, gts, masks, ids_per_step, hp_kw, threads):
    """Times reference train steps (trainer.cpp:136-195 through the public API,
    oracle/ref_harness.cpp): per-thread gradient replicas kept across steps
    and cleared per step, as train() does; the parity copies of the
    gradients are off.  Returns per-step (ms, marched samples, phase ms)."""
    from oracle.port import step_params
    s.keep_grads(False)
    s.train_reset()
    hp = step_params(**hp_kw)
    out = []
    for ids in ids_per_step:
        rc = [ref_cam(cams[v], v) for v in ids]
        gt = [gts[v].astype(np.float64) for v in ids]
        mk = [masks[v].astype(np.float64) for v in ids]
        _, counts = s.train_step(rc, gt, mk, hp, threads=threads)
        ph = s.last_phase_ms()
        out.append((float(ph.sum()), int(counts[1]), [float(x) for x in ph]))
    return out


def ref_sample(g, cams, gts, masks, world, threads, steps, warmup):
    """Full reference steps on the global batch.  Beyond one GPU's batch (weak
    scaling at N > 1) the ray pass scales with the views and the grid work
    does not: the timed step is the BATCH_PER_GPU-view step, extrapolated as
    ray-pass ms x (global views / 4) + grid-tail ms (reported as such)."""
    s = ref_scene(g)
    n_glob = global_batch(world)
    n_run = min(n_glob, BATCH_PER_GPU) if world > 1 else n_glob
    ids = [batch_ids(it, world)[:n_run] for it in range(warmup + steps)]
    res = ref_steps(s, cams, gts, masks, ids, hp_kwargs(world), threads)[warmup:]
    scale = n_glob / n_run
    ms = [r[2][0] * scale + r[2][1] + r[2][2] for r in res]
    samples = [r[1] * scale for r in res]
    return sum(samples) / (sum(ms) / 1000.0), ms, samples, res, n_run


def run_reference(args, rank, world):
    """--impl reference: the reference CPU path on this box's host cores."""
    if rank != 0:
        return
    from paper_2412_10084_b200 import api
    from oracle import refcore as R
    cores = os.cpu_count() or 1
    g, tgt = build_scene(api, seed=1)
    cams = cameras(api)
    steps, warmup = max(1, min(args.steps, 2)), 1
    need = sorted({v for it in range(warmup + steps) for v in batch_ids(it, world)})
    # ground truth from the reference itself (this arm does not touch the GPU)
    st = ref_scene(tgt)
    gts, masks = {}, {}
    for v in need:
        rgb, alpha = st.render_image_api(ref_cam(cams[v], v), R.render_opts(tau=3000.0 * W["res"]),
                                         threads=cores)
        gts[v] = rgb.astype(np.float32)
        masks[v] = alpha > 0.5
    del st
    sps, ms, samples, res, n_run = ref_sample(g, cams, gts, masks, world, cores, steps, warmup)
    line = {
        "impl": "reference", "metric": "train samples/sec (fwd+bwd)", "value": sps, "unit": "samples/s",
        "n_gpus": world, "steps": steps, "warmup": warmup, "steps_requested": args.steps,
        "ms_per_step": statistics.mean(ms), "higher_is_better": True, "scaling": W["scaling"],
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(world),
        "cpu_baseline": {"value": sps, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": sample_text(world, n_run, steps, warmup)},
        "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "samples_per_step": statistics.mean(samples),
        "phase_ms": {"ray_pass": statistics.mean(r[2][0] for r in res),
                     "regularizers_fold": statistics.mean(r[2][1] for r in res),
                     "adam_smoothing": statistics.mean(r[2][2] for r in res)},
    }
    print(json.dumps(line), flush=True)


def sample_text(world, n_run, steps, warmup):
    n_glob = global_batch(world)
    t = (f"{steps} timed full train steps (after {warmup} warm-up) of the unmodified reference "
         f"(oracle/_ref, trainer.cpp:136-195 body: clear, ray pass over {n_run} views of "
         f"{W['width']}x{W['height']}, replica reduction, 5 regularizers, G^T fold, Adam, smoothing)")
    if n_run != n_glob:
        t += (f"; the global batch is {n_glob} views, so the step time is extrapolated as "
              f"ray-pass ms x {n_glob}/{n_run} + grid-tail ms")
    return t


def workload_name():
    for k, c in CONFIGS.items():
        if all(W[x] == c[x] for x in ("scene", "res", "views", "width", "height")):
            return c["name"]
    return f"configs[4] sweep point: synthetic {W['scene']} at {W['res']}^3"


EXCHANGE = ["allreduce"]  # --grad-exchange (set in main)


def config_dict(world):
    shape = "sphere r=0.32" if W["scene"] == "sphere" else f"{W['scene']} union (api.SCENE_PRIMS)"
    return {"workload": f"{workload_name()}, {W['res']}^3 sparse SDF grid ({shape}, band 6), probes at tile "
                        f"corners ({W['res'] // 16 + 1}^3 lattice; the reference fixes the probe lattice, "
                        f"SURVEY 8d), (n_s,n_a,l)=({NS},{NA},{SH_ORDER}), {W['views']} views at "
                        f"{W['width']}x{W['height']}, global batch {global_batch(world)} views/step "
                        f"({W['scaling']} scaling), tau={TAU_VOX:g}/voxel",
            "global_batch_views": global_batch(world),
            "rays_per_step": global_batch(world) * W["width"] * W["height"],
            "parallelism": f"dp{world} (ray-batch data parallel, NCCL {EXCHANGE[0]} of grid gradients)",
            "l2": "no flush; per-step working set (params+grads+Adam moments 4x83 MB, smoothed SDF "
                  "47 MB + apron 66 MB, the batch's images >= 100 MB) exceeds the 126 MB L2"}


# --------------------------------------------------------------------------
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None)
    ap.add_argument("--batch", type=int, default=None, help="views per step (per GPU if weak, global if strong)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--res", type=int, default=None, help="grid resolution (configs[4] sweep)")
    ap.add_argument("--views", type=int, default=None)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--height", type=int, default=None)
    ap.add_argument("--grad-exchange", choices=["allreduce", "bucketed", "sharded"], default="allreduce",
                    help="how ranks combine gradients (psdf_set_grad_exchange; N > 1 only)")
    ap.add_argument("--profile", action="store_true",
                    help="setup + warm-up + 2 train steps + 1 render, no JSON (for ncu)")
    ap.add_argument("--profile-render", action="store_true",
                    help="setup + warm-up, then one configs[3] render inside cudaProfilerStart/Stop (for ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    W.update(CONFIGS[args.config])
    for k in ("res", "views", "width", "height", "batch", "scaling"):
        if getattr(args, k) is not None:
            W[k] = getattr(args, k)
    HP["lr_vox"] = 8e-4 * 64 / W["res"]  # acceptance final-LOD rate scaled to the voxel size

    # one process per GPU: re-launch under torch.distributed.run
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2412_10084_b200 import api, _lib
    import torch

    L = _lib.load()
    ctx = api.Context(local_rank)
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(api.Context.unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ctx.comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world)
        ctx.set_grad_exchange(args.grad_exchange)
    EXCHANGE[0] = {"allreduce": "all-reduce", "bucketed": "bucketed all-reduce (planes/probes/MLP under the fold)",
                   "sharded": "reduce-scatter + sharded Adam + all-gather"}[args.grad_exchange]

    g, tgt = build_scene(api, seed=1)
    cams = cameras(api)
    gts, masks = make_views(api, ctx, tgt, cams)
    ctx.upload(g)
    ctx.upload_views(cams, gts, masks)
    ctx.train_reset()
    hp_kw = hp_kwargs(world)
    hp = api.step_params(**hp_kw)

    stream = torch.cuda.ExternalStream(L.psdf_stream(ctx.h))
    for it in range(args.warmup):
        ctx.train_step_views(batch_ids(it, world), hp)
    if args.profile_render:
        render_fps(api, torch, ctx, 6455.3, frames=1, profile=True)
        ctx.close()
        return
    if args.profile:
        # the second step runs inside cudaProfilerStart/Stop, so
        # `ncu --profile-from-start off` captures exactly one train step
        for it in range(2):
            if it == 1:
                torch.cuda.synchronize()
                torch.cuda.cudart().cudaProfilerStart()
            print(ctx.train_step_views(batch_ids(args.warmup + it, world), hp))
            if it == 1:
                torch.cuda.synchronize()
                torch.cuda.cudart().cudaProfilerStop()
            print(ctx.last_timing(), ctx.last_k2_breakdown())
        print(render_fps(api, torch, ctx, 6455.3, frames=1))
        ctx.close()
        return

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    counts_tot = dict(n_rays=0, n_marched=0, n_extra=0, n_shaded=0, n_alpha=0, n_bwd_rays=0)
    ray_ms, step_ms, launches, k2_parts = [], [], 0, []
    bytes_tot = 0
    t_wall0 = time.time()
    ev0.record(stream)
    for it in range(args.steps):
        losses, counts = ctx.train_step_views(batch_ids(args.warmup + it, world), hp)
        r_ms, s_ms, n_l = ctx.last_timing()
        k2_parts.append(ctx.last_k2_breakdown()[0])
        ray_ms.append(r_ms)
        step_ms.append(s_ms)
        launches += n_l
        for k in counts_tot:
            counts_tot[k] += counts[k]
        if not all(math.isfinite(v) for v in losses.values()):
            raise FloatingPointError(f"non-finite loss at timed step {it}: {losses}")
        bytes_tot += algorithmic_bytes(counts)
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if dist:
        dist.barrier()
    time.sleep(0.2)
    sampler.stop()
    total_ms = ev0.elapsed_time(ev1)
    if dist:
        # counts from psdf are already all-reduced over ranks; take the max time
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = counts_tot["n_marched"] / (total_ms / 1000.0)

    # roofline of the dominant kernel (K2, the fused ray pass), from CUDA events
    # on the context stream around its launches
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback"
    # per-rank bytes: counts are global, each rank ran 1/world of them
    k2_bytes = bytes_tot / args.steps / world
    k2_ms = statistics.mean(ray_ms)
    achieved = k2_bytes / (k2_ms / 1000.0) / 1e9
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_k2_traffic.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            if tj.get("workload") in (None, workload_name()):
                traffic = tj.get("dram_bytes_per_launch")
                traffic_src = tj.get("source")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "K2 ray pass: tile_raster + march_scan + march_fwd (round 0) + march_coop (round 1) + "
                          "record sort + shade_fwd<4,4> + alpha_bwd + shade_bwd<4,4> + shade_geo<4,4>",
                "algorithmic_bytes_per_launch": k2_bytes, "kernel_ms": k2_ms, "peak_source": peak_src,
                "k2_share_of_step": k2_ms / statistics.mean(step_ms),
                "k2_kernels_ms": dict(zip(["scan+march+sort", "shade_fwd", "alpha_bwd", "shade_bwd+geo"],
                                          [statistics.mean(p[k] for p in k2_parts) for k in range(4)])),
                "note": "K2 = the ray-pass kernels (psdf_train.cuh) timed together as one unit with CUDA "
                        "events on the context stream; bytes per SURVEY 8(d); the regularizer kernels "
                        "run concurrently on a side stream"}

    # e2e: the reference-facing C-ABI call with pinned host buffers; H2D of the
    # step's images (this rank's rows) and the D2H loss read inside the timed
    # region (host wall clock)
    pinned = {}
    for v in range(W["views"]):
        pinned[v] = (pinned_copy(L, np.ascontiguousarray(gts[v], np.float32)),
                     pinned_copy(L, np.ascontiguousarray(masks[v], np.uint8)))
    from paper_2412_10084_b200._lib import psdf_camera, psdf_losses, psdf_counts

    def e2e_args(it):  # the C-ABI arguments of step `it` (camera array, host image pointers)
        ids = batch_ids(it, world)
        n = len(ids)
        cam_arr = (psdf_camera * n)(*[cams[i] for i in ids])
        rp = (C.POINTER(C.c_float) * n)(*[C.cast(pinned[i][0][0], C.POINTER(C.c_float)) for i in ids])
        mp = (C.POINTER(C.c_uint8) * n)(*[C.cast(pinned[i][1][0], C.POINTER(C.c_uint8)) for i in ids])
        return n, cam_arr, rp, mp

    step_args = {}

    def e2e_step(it):
        n, cam_arr, rp, mp = step_args[it] if it in step_args else e2e_args(it)
        lo, co = psdf_losses(), psdf_counts()
        _lib.check(L.psdf_train_step(ctx.h, n, cam_arr, rp, mp, C.byref(hp), C.byref(lo), C.byref(co)),
                   ctx.h)
        return co.n_marched

    for it in range(2):
        e2e_step(it)
    # argument arrays built ahead (a caller holds its dataset's cameras and
    # image pointers; the timed region is the API call: copies + step)
    step_args = {it: e2e_args(it) for it in range(args.steps)}
    e2e_dev_ms, e2e_k2 = [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_e2e = 0
    h2d_tot = 0
    for it in range(args.steps):
        n_e2e += e2e_step(it)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    # the same steps again, untimed, for the per-step H2D bytes and device
    # times (kept out of the timed loop: instrumentation only)
    for it in range(args.steps):
        e2e_step(it)
        h2d_tot += L.psdf_last_h2d_bytes(ctx.h)
        e2e_dev_ms.append(ctx.last_timing()[1])
        e2e_k2.append(ctx.last_k2_breakdown()[0])
    h2d = torch.tensor([float(h2d_tot) / args.steps], dtype=torch.float64, device="cuda")
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        dist.all_reduce(h2d)  # each rank copies its own slice's rows
    e2e = {"value": n_e2e / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": float(h2d.item()),
           "d2h_bytes_per_step": (16 * 8 + 8 * 8) * world, "ms_per_step": 1000 * e2e_s / args.steps,
           "device_ms_per_step": statistics.mean(e2e_dev_ms),
           "device_k2_parts_ms": [statistics.mean(x[k] for x in e2e_k2) for k in range(4)],
           "timing": "host wall clock around K psdf_train_step calls (pinned host images, each rank "
                     "copies the pixel rows of its slice), max over ranks"}
    for v in pinned.values():
        L.psdf_host_free(C.c_void_p(v[0][0]))
        L.psdf_host_free(C.c_void_p(v[1][0]))

    line = {
        "metric": "train samples/sec (fwd+bwd)", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": W["scaling"], "vs_baseline": None, "dtype": "f32 (f64 ray geometry)", "data": "synthetic",
        "config": config_dict(world), "roofline": roofline,
        "clocks": sampler.summary(t_wall0, t_wall1), "e2e": e2e,
        "gpu_launches": launches,
        "counts_per_step": {k: v / args.steps for k, v in counts_tot.items()},
        "losses_last_step": losses,
    }

    if rank == 0 and not args.no_render:
        line["render"] = render_fps(api, torch, ctx, peak)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            sps, ms, samples, res, n_run = ref_sample(g, cams, gts, masks, world, cores, steps=1, warmup=1)
            sps1, ms1, _, res1, _ = ref_sample(g, cams, gts, masks, world, 1, steps=1, warmup=0)
            line["cpu_baseline"] = {
                "value": sps, "unit": "samples/s", "cores": cores, "kind": "reference",
                "sample": sample_text(world, n_run, 1, 1) + f": {ms[0] / 1000:.1f} s per step "
                          f"(ray pass {res[0][2][0]:.0f} ms, regularizers + fold {res[0][2][1]:.0f} ms, "
                          f"Adam + smoothing {res[0][2][2]:.0f} ms)",
                "one_thread": {"value": sps1, "unit": "samples/s", "cores": 1,
                               "sample": f"the same step on 1 thread (no warm-up): {ms1[0] / 1000:.1f} s"}}
        except Exception as e:  # the reference build is a checker; report, don't fail the bench
            line["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def render_fps(api, torch, ctx, peak, frames=20, profile=False):
    """configs[3]: 1080p inference render of the R^3 scene (K1) — device
    outputs (kernel / FPS) and through psdf_render with host outputs (e2e,
    the D2H of the RGB and alpha images — render_image's RenderedImage,
    renderer.hpp:93-96 — inside the timed region)."""
    from paper_2412_10084_b200 import _lib
    L = _lib.load()
    cam = api.make_ring_cameras(8, 1920, height=1080)[1]
    opts = api.RenderOptions(tau=3000.0 * W["res"]).to_c()
    px = 1920 * 1080
    buf = torch.empty(5 * px, dtype=torch.float32, device="cuda")
    rgb, alpha, depth = buf.data_ptr(), buf.data_ptr() + 12 * px, buf.data_ptr() + 16 * px
    cnt = _lib.psdf_counts()
    for _ in range(3):
        _lib.check(L.psdf_render_device(ctx.h, C.byref(cam), C.byref(opts), C.c_void_p(rgb),
                                        C.c_void_p(alpha), C.c_void_p(depth), C.byref(cnt)), ctx.h)
    if profile:  # one frame for `ncu --profile-from-start off`
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        _lib.check(L.psdf_render_device(ctx.h, C.byref(cam), C.byref(opts), C.c_void_p(rgb),
                                        C.c_void_p(alpha), C.c_void_p(depth), C.byref(cnt)), ctx.h)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        print(cnt.as_dict())
        return None
    kms = []
    stream = torch.cuda.ExternalStream(L.psdf_stream(ctx.h))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(frames):
        _lib.check(L.psdf_render_device(ctx.h, C.byref(cam), C.byref(opts), C.c_void_p(rgb),
                                        C.c_void_p(alpha), C.c_void_p(depth), C.byref(cnt)), ctx.h)
        kms.append(ctx.last_timing()[0])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / frames
    # e2e: host output buffers (pinned), D2H inside the call
    hp = L.psdf_host_alloc(5 * 4 * px)
    fp = C.POINTER(C.c_float)
    hrgb, halpha, hdepth = C.cast(hp, fp), C.cast(hp + 12 * px, fp), None  # no depth in RenderedImage
    _lib.check(L.psdf_render(ctx.h, C.byref(cam), C.byref(opts), hrgb, halpha, hdepth, C.byref(cnt)), ctx.h)
    t0 = time.perf_counter()
    for _ in range(frames):
        _lib.check(L.psdf_render(ctx.h, C.byref(cam), C.byref(opts), hrgb, halpha, hdepth, C.byref(cnt)), ctx.h)
    e2e_ms = 1000 * (time.perf_counter() - t0) / frames
    L.psdf_host_free(C.c_void_p(hp))
    c = cnt.as_dict()
    b = algorithmic_bytes(c, "render")
    # measured DRAM bytes per marched sample of the render kernels (one ncu
    # capture of `bench.py --profile-render`, profiles/render_traffic.json)
    meas = None
    rp = os.path.join(ROOT, "profiles", "render_traffic.json")
    if os.path.exists(rp):
        try:
            rj = json.load(open(rp))
            if rj.get("res") == W["res"]:
                meas = {"dram_bytes_per_marched_sample": rj["dram_bytes"] / max(rj["n_marched"], 1),
                        "dram_bytes_per_frame": rj["dram_bytes"], "source": rj.get("source")}
        except Exception:
            meas = None
    return {"config": f"configs[3]: 1920x1080 view of the {W['res']}^3 scene, tau=3000/voxel",
            "measured_traffic": meas,
            "fps": 1000.0 / ms, "ms_per_frame": ms, "kernel_ms": statistics.mean(kms),
            "e2e_fps": 1000.0 / e2e_ms, "e2e_ms_per_frame": e2e_ms, "e2e_d2h_bytes_per_frame": 16 * px,
            "marched_samples": c["n_marched"], "shaded_samples": c["n_shaded"],
            "samples_per_s": c["n_marched"] / (ms / 1000.0),
            "algorithmic_bytes_per_marched_sample": b / max(c["n_marched"], 1),
            "roofline_frac": b / (statistics.mean(kms) / 1000.0) / 1e9 / peak}


if __name__ == "__main__":
    main()
