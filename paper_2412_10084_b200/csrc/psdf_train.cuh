// psdf_train.cuh — K2, the ray pass of one train step (trainer.cpp:157-182:
// render_ray + photo_pixel + render_ray_backward + scatter_smooth_grad) as a
// wavefront pipeline (render, K1, reuses its forward half):
//
//  K2a-scan  march_scan   one lane per ray (8x4 pixel tile per warp): the
//                         saturated prefix of the exact f64 march (empty-space
//                         jumps, cell-saturated runs; no image read); rays that
//                         reach a cell that can hold sigmoid < 1 are handed
//                         over, the others only counted.
//  K2a       march_fwd    two rounds (16 steps, then the still-alive rays
//                         compacted): the exact alpha / T / weight chain of the
//                         handed-over rays; shading records (samples the
//                         reference decodes), ray entries and alpha-sample
//                         lists appended with warp-aggregated atomics.
//            rec_tile_*   shading records grouped by tile (counting sort).
//  K2b       shade_fwd    one lane per record: decode_fused, colour stored in
//                         the record, c_raw[ray] += w C (f64 atomics).
//            empty_ray_loss  (side stream) photo terms of the finished rays.
//  K2d       alpha_bwd    one lane per ray entry: photo_pixel, then the alpha /
//                         transmittance chain of renderer.cpp:247-276 over the
//                         ray's alpha > 0 samples (no second march), SDF-sample
//                         gradient scatters; each record's upstream w g.
//  K2e       shade_bwd    32 records per warp: decoder MLP backward as
//                         3xTF32 mma.sync GEMMs, weight gradients in
//                         registers, feature gradients per record.
//  K2e-geo   shade_geo    tri-plane / probe / normal-chain gradients (probe
//                         gradients aggregated over the records of one tile).
//
// Item counts are read on device (no host round trip inside the pass).
//
// Suffix sums: the reverse traversal of renderer.cpp:254-261 is replaced by
// suffix_i = Total - prefix_i, Total = g.(c_raw - bg acc) + dA acc (known
// after K2b); the subtraction's rounding error enters ds only multiplied by
// (1 - alpha_i).
#pragma once

#include "psdf_mma.cuh"
#include "psdf_raypass.cuh"

#ifndef PSDF_MARCH_MINB
#define PSDF_MARCH_MINB 3  // r02: round 0 218 vs 229 us at 4
#endif

namespace psdf {

// Full state of a K2a ray at a sample boundary (the marcher is synchronised
// with the reference there), for the compacted second round.
struct ContRec {
    double t, t_cur, a_cur, acc, trans, depth, t_first, t1, dir[3];
    int slot, count, tile, n_live, entry, prev, head, cnt_first, flags;  // flags: have_cur | in_mask << 1
    int ahead, aprev;
    unsigned n_exact;
};

struct WaveBufs {
    // ray entries: rays with at least one alpha > 0 sample
    int* e_slot;       // local work tile * 32 + lane
    double* e_dir;     // [cap][3] unit ray direction
    double* e_tfirst;  // t of the first alpha > 0 sample
    int* e_cfirst;     // its sample index
    int* e_nlive;      // samples kept after early termination
    double* e_acc;     // accumulated opacity
    int* e_head;       // first record of the ray, -1 if none
    double* e_craw;    // [cap][3] sum_i w_i C_i (K2b)
    double* e_t1;      // box exit of the ray
    // shading records: samples with w > 0 on in-mask rays, append order
    double* r_pos;     // [cap][3]
    double* r_w;
    int* r_tile;
    int* r_entry;
    int* r_next;       // next record of the same ray, -1 at the end
    float* r_c;        // [cap][4] decoded colour (K2b)
    float* r_up;       // [cap][4] upstream w g (K2d)
    float* r_geo;      // [cap][GeoRec::STRIDE] geometry + features (K2b -> K2e)
    // handovers K2a-scan -> K2a: rays that reach a sample which can have
    // sigmoid < 1 (or whose final settle can), with the scan's state there
    int* h_slot;       // local work tile * 32 + lane
    int* h_count;      // samples before it (all saturated)
    int* h_tileprev;   // tile of the last of them
    double* h_t;       // t of that sample (marcher t at exhaustion for a final settle)
    double* h_tprev;   // t of the last saturated sample
    double* h_dir;     // [cap][3]
    double* h_t1;      // box exit
    int* r_perm;       // shading records grouped by tile (K2b / K2e order; rec_tile_*_kernel)
    float* r_fg;       // [cap][FgDims::STRIDE] feature gradients (K2e-mlp -> K2e-geo)
    ContRec* k_rec;    // continuations: rays still alive after K2a's first round
    // alpha samples (K2a -> K2d): every settle with alpha > 0, linked per ray
    // entry in march order — all the backward's alpha / transmittance chain
    // needs, so K2d does not march again
    double* a_t;       // [cap][2] t of the sample, t of the point it settled against
    double* a_s;       // [cap][3] sigmoid at both, transmittance before the sample
    int4* a_i;         // [cap] (tile of the sample, tile of the next point or -1 for the
                       //        one-past-the-end point, record or -1, next alpha sample or -1)
    int* e_ahead;      // first alpha sample of the entry
    unsigned* hand_bits;  // [work tiles] lanes of each 8x4 pixel tile handed over by the scan (train)
    unsigned* counters;  // [0] entries, [1] records, [2] handovers, [3] continuations, [4] alpha samples
    int e_cap, r_cap, h_cap, k_cap, a_cap;
};

// True when any wave buffer overflowed this pass (the host redoes it).
__device__ __forceinline__ bool wave_over(const WaveBufs& W) {
    const volatile unsigned* c = W.counters;
    return c[0] > (unsigned)W.e_cap || c[1] > (unsigned)W.r_cap || c[2] > (unsigned)W.h_cap ||
           c[3] > (unsigned)W.k_cap || c[4] > (unsigned)W.a_cap;
}

// Items in the entry / record queues, read on device by the kernels after the
// march.  An overflowed pass is redone, and its queues can hold allocated but
// unwritten slots (a record whose entry overflowed), so after an overflow the
// downstream kernels see empty queues.
__device__ __forceinline__ int n_entries(const WaveBufs& W) {
    return wave_over(W) ? 0 : (int)min(*(volatile unsigned*)W.counters, (unsigned)W.e_cap);
}
__device__ __forceinline__ int n_records(const WaveBufs& W) {
    return wave_over(W) ? 0 : (int)min(*(volatile unsigned*)(W.counters + 1), (unsigned)W.r_cap);
}
// The records in the tile-sorted permutation r_perm (the queue minus the
// holes of abandoned allocation chunks), counted by rec_tile_count_kernel.
__device__ __forceinline__ int n_sorted(const WaveBufs& W) {
    return wave_over(W) ? 0 : (int)min(*(volatile unsigned*)(W.counters + 5), (unsigned)W.r_cap);
}

// Warp-aggregated slot allocation inside divergent code.
__device__ __forceinline__ int warp_alloc(unsigned* counter, bool want, int lane) {
    const unsigned am = __activemask();
    const unsigned m = __ballot_sync(am, want);
    if (!want) return -1;
    const int leader = __ffs(m) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    return (int)(base + __popc(m & ((1u << lane) - 1u)));
}

// Per-warp chunked allocation from a queue counter: the warp takes slots
// for its (warp-uniform) k requests from a private chunk and fetches a fresh
// chunk of max(CH, k) slots with one atomic when the chunk runs short, instead
// of one same-address atomic per step (those were 19 % of round 0's stalls).
// The rest of an abandoned chunk becomes holes, marked by `hole(slot)` so the
// queue's readers skip them (records: tile -1; entries: slot -1, head -1).
struct WarpChunk {
    unsigned base, left;
};
constexpr unsigned kChunk = 64;
template <class F>
__device__ __forceinline__ unsigned chunk_take(unsigned* counter, WarpChunk& c, unsigned k, int lane, F hole) {
    if (k > c.left) {
        for (unsigned i = lane; i < c.left; i += 32) hole(c.base + i);
        const unsigned n = k > kChunk ? k : kChunk;
        unsigned b = 0;
        if (lane == 0) b = atomicAdd(counter, n);
        c.base = __shfl_sync(FULL, b, 0);
        c.left = n;
    }
    const unsigned r = c.base;
    c.base += k;
    c.left -= k;
    return r;
}
template <class F>
__device__ __forceinline__ void chunk_close(WarpChunk& c, int lane, F hole) {
    for (unsigned i = lane; i < c.left; i += 32) hole(c.base + i);
    c.left = 0;
}

constexpr float kTminNone = 3.0e38f;  // at or above: "no tile" (the byte memset 0x7F7F7F7F is 3.396e38; tile_raster_kernel)

struct LaneRay {
    const ViewDev* V;
    int u, v;
    bool valid;
    int64_t px;
};

__device__ __forceinline__ LaneRay lane_ray(const RayPassParams& P, int wi, int lane) {
    const int64_t tile_id = P.tile_begin + wi;
    const int vi = locate_view(P, tile_id);
    LaneRay r;
    r.V = &P.views[vi];
    // the tile inside its view (< 2^31: 32-bit division)
    const int lt = (int)(tile_id - r.V->tile_begin);
    const int ty = lt / r.V->tiles_x;
    r.u = (lt - ty * r.V->tiles_x) * 8 + (lane & 7);
    r.v = ty * 4 + (lane >> 3);
    r.valid = r.u < r.V->cam.width && r.v < r.V->cam.height;
    r.px = r.valid ? (int64_t)r.v * r.V->cam.width + r.u : 0;
    return r;
}

// photo_pixel (losses.cpp:8-38) in f64; returns whether the ray has a
// non-zero gradient (trainer.cpp:179).
__device__ __forceinline__ bool photo_term(const RayPassParams& P, bool in_mask, const float* gtp,
                                           const double col[3], double acc, double& g0, double& g1,
                                           double& g2, double& dA, double& st_photo,
                                           double& st_sq, unsigned long long& st_mask) {
    const double scale = P.photo_scale;
    g0 = g1 = g2 = dA = 0.0;
    if (in_mask) {
        double gg[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double gtk = (double)__ldg(gtp + k);
            const double d = dsub(col[k], gtk);
            const double wk = __drcp_rn(dadd(col[k] > gtk ? col[k] : gtk, kPhotoEps));  // = 1.0 / x
            st_photo = dadd(st_photo, dmul(dmul(scale, d), d));
            st_sq = dadd(st_sq, dmul(d, d));
            gg[k] = dmul(dmul(dmul(scale, 2.0), wk), d);
        }
        g0 = gg[0];
        g1 = gg[1];
        g2 = gg[2];
        st_mask += 3;
    } else {
        const double am = acc > 0.0 ? acc : 0.0;
        const double wa = __drcp_rn(dadd(am, kPhotoEps));  // = 1.0 / x
        st_photo = dadd(st_photo, dmul(dmul(scale, acc), acc));
        dA = dmul(dmul(dmul(scale, 2.0), wa), acc);
    }
    return dadd(dadd(dmul(g0, g0), dmul(g1, g1)), dmul(g2, g2)) > 0.0 || dA != 0.0;
}

// ------------------------------------------------------------------ K2a-scan
// The saturated prefix of every ray: march (jumps, skips, saturated runs)
// until the first sample whose block can hold sigmoid < 1, with no SDF
// evaluation.  Saturated samples settle with alpha exactly 0 and change
// nothing but the counts, so a ray that never leaves them (or misses the
// grid) is finished here — its loss is the empty-ray term — and the others
// are handed over, compacted, to K2a with the state at that sample.
#ifndef PSDF_SCAN_MINB
#define PSDF_SCAN_MINB 6
#endif
__global__ void __launch_bounds__(BLOCK, PSDF_SCAN_MINB) march_scan_kernel(RayPassParams P, WaveBufs W) {
    extern __shared__ __align__(16) uint32_t sm_bits[];
    const int lane = threadIdx.x & 31;
    const GridView& g = P.g;
    const uint32_t* bits = stage_tile_bits(g, sm_bits, P.bits_sm_words);
    __syncthreads();
    const double tau = P.tau;
    const double tau_run = P.early_stop > 1.0 ? 0.0 : tau;  // see render_kernel
    double st_photo = 0.0, st_sq = 0.0;
    unsigned long long st_mask = 0;
    unsigned c_m = 0, c_x = 0, c_bwd = 0, c_ex = 0;
    for (;;) {
        // the next active work tile (overlapping some view's projected box of
        // the allocated tiles) inside this rank's slice
        long long ak = 0;
        if (lane == 0) ak = (long long)(P.scan_lo + atomicAdd(P.work_counter, 1ull));
        ak = __shfl_sync(FULL, ak, 0);
        if (ak >= P.scan_hi) break;
        const int64_t gt = active_tile(P, ak);
        if (gt < P.tile_begin || gt >= P.tile_end) continue;
        const float tl = __ldg(P.tile_tmin + gt);
        if (tl >= kTminNone) continue;  // no allocated tile in this work tile's frustum: no sample
        const int wi = (int)(gt - P.tile_begin);
        const LaneRay R = lane_ray(P, wi, lane);
        Marcher mr;
        int k = 0, tile_prev = -1;
        double t_prev = 0.0, h_t = 0.0;
        bool hand = false;
        const ViewDev& V = *R.V;
        if (R.valid && R.u >= V.occ_u0 && R.u <= V.occ_u1 && R.v >= V.occ_v0 && R.v <= V.occ_v1) {
            const D3 dir = pixel_dir(R.V->cam, (double)R.u + 0.5, (double)R.v + 0.5);
            const double dd[3] = {dir.x, dir.y, dir.z};
            if (mr.init(g, R.V->cam.pos, dd, P.n_max) && mr.enter_occupied(g)) {
                mr.jump_to(g, (double)tl);
                // no sample lies beyond the work tile's farthest allocated
                // tile: the march ends there instead of at the grid exit
                // (t1 only bounds the loop; every sample before it is kept)
                const double tf = (double)__ldg(P.tile_tmax + gt);
                if (tf < mr.t1) mr.t1 = tf;
                for (;;) {
                    double ts;
                    int tile;
                    int4 tc;
                    SampleRun run;
                    if (!mr.next_run(g, ts, tile, bits, &tc, tau_run, run)) {
                        if (k > 0) {  // the final settle against the one-past-the-end point
                            double pn[3];
                            mr.pos(dadd(t_prev, g.h), pn);
                            if (sigmoid_sat(dmul(tau, sample_sdf(g, pn[0], pn[1], pn[2]))) != 1.0) {
                                hand = true;
                                h_t = mr.t;
                            }
                        }
                        break;
                    }
                    if (!run.sat) {
                        hand = true;
                        h_t = ts;
                        break;
                    }
                    k += run.n;
                    t_prev = run.t_last;
                    tile_prev = tile;
                }
            }
            c_ex += mr.n_exact;
            if (k > 0) ++c_x;  // the ray's first sample (n_extra)
        }
        const int h = warp_alloc(W.counters + 2, hand, lane);
        if (hand) {
            if (h < W.h_cap) {
                W.h_slot[h] = wi * 32 + lane;
                W.h_count[h] = k;
                W.h_tileprev[h] = tile_prev;
                W.h_t[h] = h_t;
                W.h_tprev[h] = t_prev;
                W.h_dir[3 * (int64_t)h] = mr.d[0];
                W.h_dir[3 * (int64_t)h + 1] = mr.d[1];
                W.h_dir[3 * (int64_t)h + 2] = mr.d[2];
                W.h_t1[h] = mr.t1;
            }
        } else if (R.valid && P.mode == 1) {  // render: background, zero opacity and depth
            c_m += k;
            P.out_rgb[3 * R.px] = (float)P.bg[0];
            P.out_rgb[3 * R.px + 1] = (float)P.bg[1];
            P.out_rgb[3 * R.px + 2] = (float)P.bg[2];
            P.out_alpha[R.px] = 0.f;
            if (P.out_depth) P.out_depth[R.px] = 0.f;
        } else if (R.valid) {
            // every settle had alpha 0: acc = 0, nothing shaded, nothing to
            // back-propagate; its photo term (stats only) is taken by
            // empty_ray_loss_kernel once the images are in HBM, so the scan
            // itself reads no image and can run under the image copies
            c_m += k;
        }
        if (P.mode != 1) {
            const unsigned hb = __ballot_sync(FULL, hand);
            if (lane == 0) W.hand_bits[wi] = hb;
        }
    }
    st_photo = warp_sum_d(st_photo);
    st_sq = warp_sum_d(st_sq);
    st_mask = warp_sum_u(st_mask);
    const unsigned long long m = warp_sum_u(c_m), x = warp_sum_u(c_x), bw = warp_sum_u(c_bwd),
                             ex = warp_sum_u(c_ex);
    if (lane == 0) {
        atomicAdd(P.counts + 6, ex);
        atomicAdd(P.stats + 0, st_photo);
        atomicAdd(P.stats + 1, st_sq);
        atomicAdd(P.stats + 2, (double)st_mask);
        atomicAdd(P.counts + 1, m);
        atomicAdd(P.counts + 2, x);
        atomicAdd(P.counts + 5, bw);
    }
}

// Per 8x4 work tile of every view, a lower bound on the distance along its
// rays to the first allocated tile (the scan jumps there at once; a work tile
// with no bound has no sample at all).  One warp per (allocated tile, view):
// the tile's AABB projected through its 8 corners (padded by a pixel) marks
// the work tiles whose pixel rays can meet it, each receiving the camera's
// distance to the AABB minus 2 voxels (a point of the ray at parameter t is
// at distance t from the camera: directions are unit).  Tiles with a corner
// beside or behind the camera mark the whole view.  atomicMin on the float
// bits (non-negative floats order as integers).
__global__ void __launch_bounds__(128) tile_raster_kernel(GridView g, const ViewDev* views, int n_views,
                                                          float* __restrict__ tmin, float* __restrict__ tmax) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw >= (int64_t)g.T * n_views) return;
    const int tile = (int)(gw / n_views), vi = (int)(gw - (int64_t)tile * n_views);
    const ViewDev& V = views[vi];
    const Cam& k = V.cam;
    const int4 tc = __ldg(g.tile_coords + tile);
    const double s16 = 16.0 * g.h;
    const double lo[3] = {g.org[0] + s16 * tc.x, g.org[1] + s16 * tc.y, g.org[2] + s16 * tc.z};
    float u = 0.f, v = 0.f;
    bool bad = false;
    if (lane < 8) {
        const double p[3] = {lo[0] + ((lane & 1) ? s16 : 0.0), lo[1] + ((lane & 2) ? s16 : 0.0),
                             lo[2] + ((lane & 4) ? s16 : 0.0)};
        const double d[3] = {p[0] - k.pos[0], p[1] - k.pos[1], p[2] - k.pos[2]};
        const double cx = k.rot[0] * d[0] + k.rot[3] * d[1] + k.rot[6] * d[2];
        const double cy = k.rot[1] * d[0] + k.rot[4] * d[1] + k.rot[7] * d[2];
        const double cz = k.rot[2] * d[0] + k.rot[5] * d[1] + k.rot[8] * d[2];
        bad = !(cz > 1e-6);
        u = bad ? 0.f : (float)(k.fx * cx / cz + k.cx);
        v = bad ? 0.f : (float)(k.fy * cy / cz + k.cy);
    }
    float umin = lane < 8 ? u : 3e38f, umax = lane < 8 ? u : -3e38f;
    float vmin = lane < 8 ? v : 3e38f, vmax = lane < 8 ? v : -3e38f;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        umin = fminf(umin, __shfl_xor_sync(FULL, umin, o));
        umax = fmaxf(umax, __shfl_xor_sync(FULL, umax, o));
        vmin = fminf(vmin, __shfl_xor_sync(FULL, vmin, o));
        vmax = fmaxf(vmax, __shfl_xor_sync(FULL, vmax, o));
    }
    umin = __shfl_sync(FULL, umin, 0);
    umax = __shfl_sync(FULL, umax, 0);
    vmin = __shfl_sync(FULL, vmin, 0);
    vmax = __shfl_sync(FULL, vmax, 0);
    bad = __any_sync(FULL, bad);
    // distance from the camera to the AABB, minus 2 voxels, rounded down
    double q = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double e = fmax(fmax(lo[a] - k.pos[a], k.pos[a] - (lo[a] + s16)), 0.0);
        q += e * e;
    }
    const float tv = __double2float_rd(fmax(sqrt(q) - 2.0 * g.h, 0.0));
    // and to its farthest corner, plus 2 voxels, rounded up: no sample in the
    // tile lies farther along a unit-direction ray from the camera
    double qf = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double e = fmax(fabs(lo[a] - k.pos[a]), fabs(lo[a] + s16 - k.pos[a]));
        qf += e * e;
    }
    const float tf = __double2float_ru(sqrt(qf) + 2.0 * g.h);
    int tx0 = 0, tx1 = V.tiles_x - 1, ty0 = 0, ty1 = V.tiles_y - 1;
    if (!bad) {  // work tile tx spans image points [8 tx + 0.5, 8 tx + 7.5]
        tx0 = max(tx0, (int)ceilf((umin - 1.f - 7.5f) * 0.125f));
        tx1 = min(tx1, (int)floorf((umax + 1.f - 0.5f) * 0.125f));
        ty0 = max(ty0, (int)ceilf((vmin - 1.f - 3.5f) * 0.25f));
        ty1 = min(ty1, (int)floorf((vmax + 1.f - 0.5f) * 0.25f));
    }
    const int w = tx1 - tx0 + 1, n = w > 0 && ty1 >= ty0 ? w * (ty1 - ty0 + 1) : 0;
    for (int i = lane; i < n; i += 32) {
        const int ty = ty0 + i / w, tx = tx0 + (i - (i / w) * w);
        atomicMin(reinterpret_cast<int*>(tmin) + V.tile_begin + (int64_t)ty * V.tiles_x + tx, __float_as_int(tv));
        atomicMax(reinterpret_cast<int*>(tmax) + V.tile_begin + (int64_t)ty * V.tiles_x + tx, __float_as_int(tf));
    }
}

// K1: every pixel of this pass's work tiles starts as background with zero
// opacity and depth (renderer.cpp:330-335 for a ray without samples); the
// scan / composite pass overwrite the pixels of the active tiles.
__global__ void __launch_bounds__(256) render_fill_kernel(RayPassParams P, int64_t n_work) {
    const int64_t n = n_work * 32;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const LaneRay R = lane_ray(P, (int)(q >> 5), (int)(q & 31));
        if (!R.valid) continue;
        P.out_rgb[3 * R.px] = (float)P.bg[0];
        P.out_rgb[3 * R.px + 1] = (float)P.bg[1];
        P.out_rgb[3 * R.px + 2] = (float)P.bg[2];
        P.out_alpha[R.px] = 0.f;
        if (P.out_depth) P.out_depth[R.px] = 0.f;
    }
}

// photo_pixel (losses.cpp:8-38) of the rays the scan finished and of the
// handed-over rays the composite pass ended without an alpha > 0 settle (it
// clears their hand-over bit) (no alpha > 0
// settle: colour = background, acc = 0, so only the loss statistics and the
// backward-ray count change — nothing is back-propagated).  One warp per
// 8x4 pixel work tile.
__global__ void __launch_bounds__(BLOCK) empty_ray_loss_kernel(RayPassParams P, WaveBufs W, int64_t n_work) {
    const int lane = threadIdx.x & 31;
    double st_photo = 0.0, st_sq = 0.0;
    unsigned long long st_mask = 0, c_bwd = 0;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    // four work tiles per warp and iteration, their hand-over words and mask
    // bytes loaded before any is used (the one-tile loop was latency bound on
    // these two dependent loads)
    constexpr int U = 4;
    for (int64_t w0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * U; w0 < n_work;
         w0 += warps * U) {
        unsigned hb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) hb[u] = w0 + u < n_work ? __ldg(W.hand_bits + w0 + u) : FULL;
        LaneRay R[U];
        bool act[U];
        uint8_t m[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            act[u] = hb[u] != FULL;
            if (act[u]) {
                R[u] = lane_ray(P, (int)(w0 + u), lane);
                act[u] = R[u].valid && !((hb[u] >> lane) & 1u);
            }
            m[u] = act[u] ? __ldg(R[u].V->mask + R[u].px) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!act[u]) continue;
            const double col[3] = {P.bg[0], P.bg[1], P.bg[2]};
            double g0, g1, g2, dA;
            if (photo_term(P, m[u] != 0, R[u].V->gt + 3 * R[u].px, col, 0.0, g0, g1, g2, dA, st_photo, st_sq,
                           st_mask))
                ++c_bwd;
        }
    }
    // block-wide sums, one atomic per value per block
    st_photo = warp_sum_d(st_photo);
    st_sq = warp_sum_d(st_sq);
    st_mask = warp_sum_u(st_mask);
    c_bwd = warp_sum_u(c_bwd);
    __shared__ double red[WARPS_PER_BLOCK][4];
    if (lane == 0) {
        red[threadIdx.x >> 5][0] = st_photo;
        red[threadIdx.x >> 5][1] = st_sq;
        red[threadIdx.x >> 5][2] = (double)st_mask;
        red[threadIdx.x >> 5][3] = (double)c_bwd;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double v = 0.0;
        for (int w = 0; w < WARPS_PER_BLOCK; ++w) v += red[w][threadIdx.x];
        if (v != 0.0) {
            if (threadIdx.x < 3) atomicAdd(P.stats + threadIdx.x, v);
            else atomicAdd(P.counts + 5, (unsigned long long)v);
        }
    }
}

// ------------------------------------------------------------------ K2a
// The rest of each handed-over ray, one lane per handover (full warps):
// sigmoid, alpha compositing, early termination, ray entries and shading
// records.
//
// Round 0 takes the handovers and stops after `cap` steps: rays still alive
// then (grazing rays with long tails, a few per warp) are written out as
// continuations and finished, compacted into full warps, by round 1.
__global__ void __launch_bounds__(BLOCK, PSDF_MARCH_MINB) march_fwd_kernel(RayPassParams P, WaveBufs W, int round,
                                                                          int cap) {
    extern __shared__ __align__(16) uint32_t sm_bits[];
    const int n_hand = round == 0 ? (int)min(*(volatile unsigned*)(W.counters + 2), (unsigned)W.h_cap)
                                  : (int)min(*(volatile unsigned*)(W.counters + 3), (unsigned)W.k_cap);
    const int lane = threadIdx.x & 31;
    const GridView& g = P.g;
    const uint32_t* bits = stage_tile_bits(g, sm_bits, P.bits_sm_words);
    __syncthreads();
    const double tau = P.tau;
    const double tau_run = P.early_stop > 1.0 ? 0.0 : tau;  // see render_kernel
    double st_photo = 0.0, st_sq = 0.0;
    unsigned long long st_mask = 0, c_m = 0, c_x = 0, c_sh = 0, c_bwd = 0, c_ex = 0;
    WarpChunk ch_e{0, 0}, ch_r{0, 0}, ch_a{0, 0};
    auto hole_e = [&](unsigned e) {
        if (e < (unsigned)W.e_cap) {
            W.e_slot[e] = -1;
            W.e_head[e] = -1;
        }
    };
    auto hole_r = [&](unsigned r) {
        if (r < (unsigned)W.r_cap) W.r_tile[r] = -1;
    };
    auto hole_a = [](unsigned) {};  // alpha samples are reached only through their entry's list
    for (;;) {
        int base = 0;
        if (lane == 0) base = (int)atomicAdd(P.work_counter, 32ull);
        base = __shfl_sync(FULL, base, 0);
        if (base >= n_hand) break;
        const bool valid = base + lane < n_hand;
        const int hi = valid ? base + lane : 0;
        const ContRec* kr = W.k_rec + hi;
        const int slot = valid ? (round == 0 ? W.h_slot[hi] : kr->slot) : 0;
        const LaneRay R = lane_ray(P, slot >> 5, slot & 31);
        Marcher mr;
        double t_cur = 0.0, a_cur = 1.0, acc = 0.0, trans = 1.0, depth = 0.0;
        int tile_cur = -1, n_live = 0, entry = -1, prev = -1, head = -1, ahead = -1, aprev = -1;
        double t_first = 0.0;
        int cnt_first = -1;
        bool have_cur = false, in_mask = false, cont = false;
        bool alive = valid;
        if (valid && round == 0) {
            // train: only in-mask rays are shaded (trainer.cpp:163); render: all, if colours are wanted
            in_mask = P.mode == 1 ? P.need_colors != 0 : __ldg(R.V->mask + R.px) != 0;
            const double dd[3] = {W.h_dir[3 * (int64_t)hi], W.h_dir[3 * (int64_t)hi + 1], W.h_dir[3 * (int64_t)hi + 2]};
            mr.init_from(g, R.V->cam.pos, dd, P.n_max, W.h_t1[hi]);
            mr.t = W.h_t[hi];
            mr.count = W.h_count[hi];
            have_cur = mr.count > 0;
            n_live = have_cur ? mr.count - 1 : 0;  // settles among the saturated prefix
            t_cur = W.h_tprev[hi];
            tile_cur = W.h_tileprev[hi];
        } else if (valid) {
            mr.init_from(g, R.V->cam.pos, kr->dir, P.n_max, kr->t1);
            mr.t = kr->t;
            mr.count = kr->count;
            mr.n_exact = kr->n_exact;
            t_cur = kr->t_cur;
            a_cur = kr->a_cur;
            acc = kr->acc;
            trans = kr->trans;
            depth = kr->depth;
            t_first = kr->t_first;
            tile_cur = kr->tile;
            n_live = kr->n_live;
            entry = kr->entry;
            prev = kr->prev;
            head = kr->head;
            cnt_first = kr->cnt_first;
            ahead = kr->ahead;
            aprev = kr->aprev;
            have_cur = kr->flags & 1;
            in_mask = (kr->flags >> 1) & 1;
        }
        // One sample per iteration, warp-synchronous so that the record
        // allocation below uses full-warp ballots (single call sites also
        // keep the loop small): fetch the next march sample (or the
        // one-past-the-end position), evaluate its sigmoid, then settle the
        // alpha of the previous sample.
#ifdef PSDF_MARCH_STATS
        int nsteps = 0;
#endif
        for (int step = 0; __any_sync(FULL, alive); ++step) {
#ifdef PSDF_MARCH_STATS
            nsteps += alive ? 1 : 0;
#endif
            if (step == cap) {  // warp-uniform: hand the remaining rays to round 1
                const unsigned km = __ballot_sync(FULL, alive);
                unsigned kb = 0;
                if (lane == 0) kb = atomicAdd(W.counters + 3, (unsigned)__popc(km));
                kb = __shfl_sync(FULL, kb, 0);
                if (alive) {
                    cont = true;
                    const int k = (int)(kb + __popc(km & ((1u << lane) - 1u)));
                    if (k < W.k_cap) {
                        ContRec& o = W.k_rec[k];
                        o.t = mr.t;
                        o.t_cur = t_cur;
                        o.a_cur = a_cur;
                        o.acc = acc;
                        o.trans = trans;
                        o.depth = depth;
                        o.t_first = t_first;
                        o.t1 = mr.t1;
                        o.dir[0] = mr.d[0];
                        o.dir[1] = mr.d[1];
                        o.dir[2] = mr.d[2];
                        o.slot = slot;
                        o.count = mr.count;
                        o.tile = tile_cur;
                        o.n_live = n_live;
                        o.entry = entry;
                        o.prev = prev;
                        o.head = head;
                        o.cnt_first = cnt_first;
                        o.ahead = ahead;
                        o.aprev = aprev;
                        o.flags = (have_cur ? 1 : 0) | (in_mask ? 2 : 0);
                        o.n_exact = mr.n_exact;
                    }
                }
                break;
            }
            double t_nxt = 0.0, w = 0.0;
            int tile_nxt = -1;
            bool has_next = false, settle = false, want_entry = false, shade = false, want_alpha = false;
            double a_nxt = 0.0, alpha = 0.0;
            int n_settle = 0;
            if (alive) {
                int4 tc_nxt;
                SampleRun run;
                has_next = mr.next_run(g, t_nxt, tile_nxt, bits, &tc_nxt, tau_run, run);
                if (!has_next && !have_cur) {
                    alive = false;  // no sample at all
                } else if (has_next && run.sat) {
                    // a run of saturated samples: sigmoid 1, every alpha
                    // settled against them is exactly 0 (no weight, no entry,
                    // no record, transmittance unchanged); the run's last
                    // sample becomes the pending one
                    a_nxt = 1.0;
                    n_settle = run.n - (have_cur ? 0 : 1);
                    if (!have_cur) {
                        have_cur = true;
                        ++c_x;
                    }
                    settle = n_settle > 0;
                    t_nxt = run.t_last;
                } else {
                    double pn[3];
                    mr.pos(has_next ? t_nxt : dadd(t_cur, g.h), pn);
                    const double s_nxt = has_next ? sample_sdf_in(g, pn[0], pn[1], pn[2], tile_nxt, tc_nxt)
                                                  : sample_sdf(g, pn[0], pn[1], pn[2]);
                    a_nxt = sigmoid_sat(dmul(tau, s_nxt));
                    if (!have_cur) {
                        have_cur = true;
                        ++c_x;
                    } else {
                        settle = true;
                        n_settle = 1;
                        alpha = a_nxt == 1.0 ? 0.0 : alpha_from(a_cur, a_nxt);
                        w = dmul(trans, alpha);
                        if (alpha > 0.0 && cnt_first < 0) {
                            cnt_first = mr.count - 1 - (has_next ? 1 : 0);
                            t_first = t_cur;
                        }
                        want_entry = alpha > 0.0 && entry < 0;
                        want_alpha = alpha > 0.0 && P.mode != 1;
                        shade = in_mask && w > 0.0 && tile_cur >= 0;
                    }
                }
            }
            // warp-chunked allocation of ray entries / shading records / alpha samples
            {
                const unsigned me = __ballot_sync(FULL, want_entry);
                const unsigned mr_ = __ballot_sync(FULL, shade);
                const unsigned ma = __ballot_sync(FULL, want_alpha);
                const unsigned below = (1u << lane) - 1u;
                unsigned be = 0, br = 0, ba = 0;
                if (me) be = chunk_take(W.counters + 0, ch_e, (unsigned)__popc(me), lane, hole_e);
                if (mr_) br = chunk_take(W.counters + 1, ch_r, (unsigned)__popc(mr_), lane, hole_r);
                if (ma) ba = chunk_take(W.counters + 4, ch_a, (unsigned)__popc(ma), lane, hole_a);
                if (want_entry) {
                    const int e = (int)(be + __popc(me & below));
                    entry = e < W.e_cap ? e : -2;  // -2: overflow, host retries
                }
                int rec_now = -1;
                if (shade) {
                    ++c_sh;
                    const int r = (int)(br + __popc(mr_ & below));
                    if (r < W.r_cap && entry >= 0) {
                        rec_now = r;
                        double pc[3];
                        mr.pos(t_cur, pc);
                        W.r_pos[3 * (int64_t)r] = pc[0];
                        W.r_pos[3 * (int64_t)r + 1] = pc[1];
                        W.r_pos[3 * (int64_t)r + 2] = pc[2];
                        W.r_w[r] = w;
                        W.r_tile[r] = tile_cur;
                        W.r_entry[r] = entry;
                        W.r_next[r] = -1;
                        if (prev >= 0) W.r_next[prev] = r;
                        else head = r;
                        prev = r;
                    }
                }
                if (want_alpha) {
                    const int a = (int)(ba + __popc(ma & below));
                    if (a < W.a_cap && entry >= 0) {
                        W.a_t[2 * (int64_t)a] = t_cur;
                        W.a_t[2 * (int64_t)a + 1] = has_next ? t_nxt : dadd(t_cur, g.h);
                        W.a_s[3 * (int64_t)a] = a_cur;
                        W.a_s[3 * (int64_t)a + 1] = a_nxt;
                        W.a_s[3 * (int64_t)a + 2] = trans;
                        W.a_i[a] = make_int4(tile_cur, has_next ? tile_nxt : -1, rec_now, -1);
                        if (aprev >= 0) W.a_i[aprev].w = a;
                        else ahead = a;
                        aprev = a;
                    }
                }
            }
            if (alive) {
                if (settle) {
                    acc = dadd(acc, w);
                    if (P.mode == 1) depth = dadd(depth, dmul(w, t_cur));  // render_ray (renderer.cpp:149-210)
                    trans = dmul(trans, dsub(1.0, alpha));
                    n_live += n_settle;
                    if ((P.early_stop > 0.0 && trans < P.early_stop) || !has_next) alive = false;
                }
                t_cur = t_nxt;
                tile_cur = tile_nxt;
                a_cur = a_nxt;
            }
        }
#ifdef PSDF_MARCH_STATS
        if (valid && !cont) atomicAdd(&g_cont_hist[round][min(15, 32 - __clz(nsteps))], 1ull);
#endif
        if (cont) continue;
        c_m += n_live;
        if (valid) c_ex += mr.n_exact;
        if (entry >= 0) {
            W.e_slot[entry] = slot;
            W.e_dir[3 * (int64_t)entry] = mr.d[0];
            W.e_dir[3 * (int64_t)entry + 1] = mr.d[1];
            W.e_dir[3 * (int64_t)entry + 2] = mr.d[2];
            W.e_tfirst[entry] = t_first;
            W.e_cfirst[entry] = cnt_first;
            W.e_nlive[entry] = n_live;
            W.e_acc[entry] = acc;
            W.e_t1[entry] = mr.t1;
            W.e_head[entry] = head;
            W.e_ahead[entry] = ahead;
            W.e_craw[3 * (int64_t)entry] = 0.0;
            W.e_craw[3 * (int64_t)entry + 1] = 0.0;
            W.e_craw[3 * (int64_t)entry + 2] = 0.0;
        }
        if (valid && P.mode == 1) {
            // render outputs; with shaded samples the colour is completed by
            // render_finish after K2b (c_raw + bg (1 - acc))
            P.out_alpha[R.px] = (float)acc;
            if (P.out_depth) P.out_depth[R.px] = (float)depth;
            if (head < 0) {
                const double om = dsub(1.0, acc);
                P.out_rgb[3 * R.px] = (float)dmul(P.bg[0], om);
                P.out_rgb[3 * R.px + 1] = (float)dmul(P.bg[1], om);
                P.out_rgb[3 * R.px + 2] = (float)dmul(P.bg[2], om);
            }
        } else if (valid && entry < 0 && cnt_first < 0) {
            // no alpha > 0 sample: acc = 0, colour = background, nothing to
            // back-propagate — exactly the empty-ray term, taken by
            // empty_ray_loss_kernel once the colours are in HBM (this kernel
            // only waits for the masks)
            atomicAnd(W.hand_bits + (slot >> 5), ~(1u << (slot & 31)));
        }
    }
    chunk_close(ch_e, lane, hole_e);
    chunk_close(ch_r, lane, hole_r);
    st_photo = warp_sum_d(st_photo);
    st_sq = warp_sum_d(st_sq);
    st_mask = warp_sum_u(st_mask);
    c_m = warp_sum_u(c_m);
    c_x = warp_sum_u(c_x);
    c_sh = warp_sum_u(c_sh);
    c_bwd = warp_sum_u(c_bwd);
    c_ex = warp_sum_u(c_ex);
    if (lane == 0) {
        atomicAdd(P.counts + 6, c_ex);
        atomicAdd(P.stats + 0, st_photo);
        atomicAdd(P.stats + 1, st_sq);
        atomicAdd(P.stats + 2, (double)st_mask);
        atomicAdd(P.counts + 1, c_m);
        atomicAdd(P.counts + 2, c_x);
        atomicAdd(P.counts + 3, c_sh);
        atomicAdd(P.counts + 5, c_bwd);
    }
}

// ------------------------------------------------------------------ K2a round 1
#ifndef PSDF_COOP_MINB
#define PSDF_COOP_MINB 4  // <= 128 registers: 16 warps (rays) per SM
#endif
// The continuations (rays still alive after round 0's `cap` steps: grazing
// rays with long tails, ~12 K at the bench step with 16-64 more samples
// each) as ONE WARP PER RAY.  With one lane per ray they leave a few warps per
// SM in a latency-bound tail (round 1 of march_fwd: 6.5 % warps active, 9
// threads per instruction): such a ray alternates short saturated runs (~4
// samples) with short unsaturated stretches, ~20 sequential marcher steps.
// Here the marcher's control (tile decisions, jumps) runs warp-uniformly, and
// the first lattice point of an allocated tile opens a batch of up to 32
// consecutive lattice points of that tile (Marcher::run_length), one per
// lane, whose SDF and sigmoid are evaluated in parallel — exactly the samples
// the reference visits (a point of a saturated cell evaluates to sigmoid 1
// exactly, so no saturated-run shortcut is needed).  The settles stay in the reference's order: lane j's
// transmittance is trans * (1 - alpha_0) * ... * (1 - alpha_{j-1}) multiplied
// left to right through shuffles, acc / depth are summed in lane order, and
// early termination cuts the batch at the first lane below the threshold, so
// every value, count and queue entry equals the one-lane march's.
__global__ void __launch_bounds__(BLOCK, PSDF_COOP_MINB) march_coop_kernel(RayPassParams P, WaveBufs W) {
    extern __shared__ __align__(16) uint32_t sm_bits[];
    const int n_cont = (int)min(*(volatile unsigned*)(W.counters + 3), (unsigned)W.k_cap);
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const GridView& g = P.g;
    const uint32_t* bits = stage_tile_bits(g, sm_bits, P.bits_sm_words);
    __syncthreads();
    const double tau = P.tau, h = g.h;
    double st_photo = 0.0, st_sq = 0.0;
    unsigned long long st_mask = 0, c_m = 0, c_x = 0, c_sh = 0, c_bwd = 0, c_ex = 0;
    WarpChunk ch_e{0, 0}, ch_r{0, 0}, ch_a{0, 0};  // chunked queue allocation (chunk_take)
    auto hole_e = [&](unsigned e) {
        if (e < (unsigned)W.e_cap) {
            W.e_slot[e] = -1;
            W.e_head[e] = -1;
        }
    };
    auto hole_r = [&](unsigned r) {
        if (r < (unsigned)W.r_cap) W.r_tile[r] = -1;
    };
    for (;;) {
        int ki = 0;
        if (lane == 0) ki = (int)atomicAdd(P.work_counter, 1ull);
        ki = __shfl_sync(FULL, ki, 0);
        if (ki >= n_cont) break;
        const ContRec* kr = W.k_rec + ki;
        const int slot = kr->slot;
        const LaneRay R = lane_ray(P, slot >> 5, slot & 31);
        Marcher mr;
        mr.init_from(g, R.V->cam.pos, kr->dir, P.n_max, kr->t1);
        mr.t = kr->t;
        mr.count = kr->count;
        mr.n_exact = kr->n_exact;
        double t_cur = kr->t_cur, a_cur = kr->a_cur, acc = kr->acc, trans = kr->trans, depth = kr->depth,
               t_first = kr->t_first;
        int tile_cur = kr->tile, n_live = kr->n_live, entry = kr->entry, prev = kr->prev, head = kr->head,
            cnt_first = kr->cnt_first, ahead = kr->ahead, aprev = kr->aprev;
        bool have_cur = kr->flags & 1;
        const bool in_mask = (kr->flags >> 1) & 1;
#ifdef PSDF_MARCH_STATS
        if (lane == 0) atomicAdd(&g_coop_stats[0], 1ull);
#endif
        for (;;) {
#ifdef PSDF_MARCH_STATS
            if (lane == 0) atomicAdd(&g_coop_stats[1], 1ull);
#endif
            double t_nxt = 0.0;
            int tile_nxt = -1;
            int4 tc_nxt;
            SampleRun run;
            // no saturated-run shortcut here: a batch evaluates a whole tile's
            // lattice points at once (saturated ones to sigmoid 1 exactly)
            const bool has_next = mr.next_run(g, t_nxt, tile_nxt, bits, &tc_nxt, 0.0, run);
            if (!has_next && !have_cur) break;  // no sample at all
            if (has_next && run.sat) {
#ifdef PSDF_MARCH_STATS
                if (lane == 0) atomicAdd(&g_coop_stats[2], 1ull);
#endif
                // saturated run: every settle has alpha 0 (acc, trans, depth
                // unchanged; never terminates); its last sample is pending
                n_live += run.n - (have_cur ? 0 : 1);
                if (!have_cur) {
                    have_cur = true;
                    c_x += lane == 0;
                }
                t_cur = run.t_last;
                tile_cur = tile_nxt;
                a_cur = 1.0;
                continue;
            }
            // the batch: sample 0 at t_nxt (or the one-past-the-end point
            // t_cur + h), then the tile's next lattice points
            const int cnt0 = mr.count;  // samples fetched including sample 0
            int n = 1;
            if (has_next) {
                double v[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) v[a] = fma(mr.vd[a], t_nxt, mr.vo[a]);
                n = (int)fmin(fmin(mr.run_length(g, v, t_nxt, h), 32.0), (double)(mr.n_max - cnt0 + 1));
                if (n > 1) {  // the marcher continues after the batch's last point
                    mr.t = lattice_advance(t_nxt, (double)n, h);
                    mr.count = cnt0 + n - 1;
                }
            }
#ifdef PSDF_MARCH_STATS
            if (lane == 0) {
                atomicAdd(&g_coop_stats[3], 1ull);
                atomicAdd(&g_coop_stats[4], (unsigned long long)n);
                if (n == 1) atomicAdd(&g_coop_stats[5], 1ull);
            }
#endif
            const bool act = lane < n;
            double tj = t_nxt, aj = 1.0;
            if (act) {
                if (lane > 0) tj = lattice_advance(t_nxt, (double)lane, h);
                double pn[3];
                mr.pos(has_next ? tj : dadd(t_cur, h), pn);
                const double sv = has_next ? sample_sdf_in(g, pn[0], pn[1], pn[2], tile_nxt, tc_nxt)
                                           : sample_sdf(g, pn[0], pn[1], pn[2]);
                aj = sigmoid_sat(dmul(tau, sv));
            }
            // lane j settles the sample before it (the pending one for lane 0)
            const double a_up = __shfl_up_sync(FULL, aj, 1), t_up = __shfl_up_sync(FULL, tj, 1);
            const double a_prev = lane == 0 ? a_cur : a_up;
            const double t_prev = lane == 0 ? t_cur : t_up;
            const int tile_prev = lane == 0 ? tile_cur : tile_nxt;
            const bool settles = act && (lane > 0 || have_cur);
            const double alpha = (settles && aj != 1.0) ? alpha_from(a_prev, aj) : 0.0;
            const double om = dsub(1.0, alpha);
            double tj_before = trans;  // trans * om_0 * ... * om_{lane-1}, in order
            for (int i = 0; i + 1 < n; ++i) {
                const double omi = __shfl_sync(FULL, om, i);
                if (i < lane) tj_before = dmul(tj_before, omi);
            }
            const double t_after = dmul(tj_before, om);
            const bool term = settles && P.early_stop > 0.0 && t_after < P.early_stop;
            const unsigned tm = __ballot_sync(FULL, term);
            const int n_eff = tm ? __ffs(tm) : n;  // lanes [0, n_eff) take part
            const bool live = settles && lane < n_eff;
            const double w = live ? dmul(tj_before, alpha) : 0.0;
            // first alpha > 0 settle (trainer statistics)
            const unsigned mpos = __ballot_sync(FULL, live && alpha > 0.0);
            if (mpos && cnt_first < 0) {
                const int j = __ffs(mpos) - 1;
                cnt_first = cnt0 + j - 1 - (has_next ? 1 : 0);
                t_first = __shfl_sync(FULL, t_prev, j);
            }
            // ray entry (once), shading records, alpha samples
            if (mpos && entry < 0) {
                const unsigned e0 = chunk_take(W.counters + 0, ch_e, 1u, lane, hole_e);
                entry = (int)e0 < W.e_cap ? (int)e0 : -2;  // -2: overflow, host retries
            }
            const bool shade = live && in_mask && w > 0.0 && tile_prev >= 0;
            const unsigned msh = __ballot_sync(FULL, shade);
            const unsigned mal = P.mode != 1 ? mpos : 0u;
            unsigned br = 0, ba = 0;
            if (msh) br = chunk_take(W.counters + 1, ch_r, (unsigned)__popc(msh), lane, hole_r);
            if (mal) ba = chunk_take(W.counters + 4, ch_a, (unsigned)__popc(mal), lane, [](unsigned) {});
            int rec_now = -1;
            if (msh) {
                c_sh += lane == 0 ? (unsigned long long)__popc(msh) : 0ull;
                const int r_first = (int)br, r_last = (int)br + __popc(msh) - 1;
                if (shade) {
                    const int r = (int)br + __popc(msh & below);
                    if (r < W.r_cap && entry >= 0) {
                        rec_now = r;
                        double pc[3];
                        mr.pos(t_prev, pc);
                        W.r_pos[3 * (int64_t)r] = pc[0];
                        W.r_pos[3 * (int64_t)r + 1] = pc[1];
                        W.r_pos[3 * (int64_t)r + 2] = pc[2];
                        W.r_w[r] = w;
                        W.r_tile[r] = tile_prev;
                        W.r_entry[r] = entry;
                        W.r_next[r] = (r < r_last && r + 1 < W.r_cap) ? r + 1 : -1;
                    }
                }
                if (entry >= 0 && r_first < W.r_cap) {
                    if (prev >= 0) {
                        if (lane == 0) W.r_next[prev] = r_first;
                    } else {
                        head = r_first;
                    }
                    prev = min(r_last, W.r_cap - 1);
                }
            }
            if (mal) {
                const int a_first = (int)ba, a_last = (int)ba + __popc(mal) - 1;
                if ((mal >> lane) & 1u) {
                    const int a = (int)ba + __popc(mal & below);
                    if (a < W.a_cap && entry >= 0) {
                        W.a_t[2 * (int64_t)a] = t_prev;
                        W.a_t[2 * (int64_t)a + 1] = has_next ? tj : dadd(t_cur, h);
                        W.a_s[3 * (int64_t)a] = a_prev;
                        W.a_s[3 * (int64_t)a + 1] = aj;
                        W.a_s[3 * (int64_t)a + 2] = tj_before;
                        W.a_i[a] = make_int4(tile_prev, has_next ? tile_nxt : -1, rec_now,
                                             (a < a_last && a + 1 < W.a_cap) ? a + 1 : -1);
                    }
                }
                if (entry >= 0 && a_first < W.a_cap) {
                    if (aprev >= 0) {
                        if (lane == 0) W.a_i[aprev].w = a_first;
                    } else {
                        ahead = a_first;
                    }
                    aprev = min(a_last, W.a_cap - 1);
                }
            }
            // acc / depth in march order; the batch's settles
            for (int i = 0; i < n_eff; ++i) {
                const double wi = __shfl_sync(FULL, w, i);
                if (P.mode == 1) depth = dadd(depth, dmul(wi, __shfl_sync(FULL, t_prev, i)));
                acc = dadd(acc, wi);
            }
            n_live += __popc(__ballot_sync(FULL, live));
            trans = __shfl_sync(FULL, t_after, n_eff - 1);
            if (!have_cur) {
                have_cur = true;
                c_x += lane == 0;
            }
            if (tm || !has_next) break;  // early termination / end of the ray
            t_cur = __shfl_sync(FULL, tj, n - 1);
            a_cur = __shfl_sync(FULL, aj, n - 1);
            tile_cur = tile_nxt;
        }
        if (lane != 0) continue;
        c_m += n_live;
        c_ex += mr.n_exact;
        if (entry >= 0) {
            W.e_slot[entry] = slot;
            W.e_dir[3 * (int64_t)entry] = mr.d[0];
            W.e_dir[3 * (int64_t)entry + 1] = mr.d[1];
            W.e_dir[3 * (int64_t)entry + 2] = mr.d[2];
            W.e_tfirst[entry] = t_first;
            W.e_cfirst[entry] = cnt_first;
            W.e_nlive[entry] = n_live;
            W.e_acc[entry] = acc;
            W.e_t1[entry] = mr.t1;
            W.e_head[entry] = head;
            W.e_ahead[entry] = ahead;
            W.e_craw[3 * (int64_t)entry] = 0.0;
            W.e_craw[3 * (int64_t)entry + 1] = 0.0;
            W.e_craw[3 * (int64_t)entry + 2] = 0.0;
        }
        if (P.mode == 1) {
            P.out_alpha[R.px] = (float)acc;
            if (P.out_depth) P.out_depth[R.px] = (float)depth;
            if (head < 0) {
                const double om = dsub(1.0, acc);
                P.out_rgb[3 * R.px] = (float)dmul(P.bg[0], om);
                P.out_rgb[3 * R.px + 1] = (float)dmul(P.bg[1], om);
                P.out_rgb[3 * R.px + 2] = (float)dmul(P.bg[2], om);
            }
        } else if (entry < 0 && cnt_first < 0) {  // the empty-ray term (see march_fwd_kernel)
            atomicAnd(W.hand_bits + (slot >> 5), ~(1u << (slot & 31)));
        }
    }
    chunk_close(ch_e, lane, hole_e);
    chunk_close(ch_r, lane, hole_r);
    st_photo = warp_sum_d(st_photo);
    st_sq = warp_sum_d(st_sq);
    st_mask = warp_sum_u(st_mask);
    c_m = warp_sum_u(c_m);
    c_x = warp_sum_u(c_x);
    c_sh = warp_sum_u(c_sh);
    c_bwd = warp_sum_u(c_bwd);
    c_ex = warp_sum_u(c_ex);
    if (lane == 0) {
        atomicAdd(P.counts + 6, c_ex);
        atomicAdd(P.stats + 0, st_photo);
        atomicAdd(P.stats + 1, st_sq);
        atomicAdd(P.stats + 2, (double)st_mask);
        atomicAdd(P.counts + 1, c_m);
        atomicAdd(P.counts + 2, c_x);
        atomicAdd(P.counts + 3, c_sh);
        atomicAdd(P.counts + 5, c_bwd);
    }
}

// K1 tail: colour of every rendered ray with shaded samples, c_raw + bg (1 - acc)
// (renderer.cpp:330-335).
__global__ void __launch_bounds__(BLOCK) render_finish_kernel(RayPassParams P, WaveBufs W) {
    const int n_ent = n_entries(W);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_ent; e += gridDim.x * blockDim.x) {
        if (W.e_head[e] < 0) continue;
        const int slot = W.e_slot[e];
        const LaneRay R = lane_ray(P, slot >> 5, slot & 31);
        const double om = dsub(1.0, W.e_acc[e]);
#pragma unroll
        for (int k = 0; k < 3; ++k)
            P.out_rgb[3 * R.px + k] = (float)dadd(W.e_craw[3 * (int64_t)e + k], dmul(P.bg[k], om));
    }
}

// Camera-bias row of a ray entry's view.
__device__ __forceinline__ const ViewDev& entry_view(const RayPassParams& P, const WaveBufs& W,
                                                     int e) {
    const int slot = __ldg(W.e_slot + e);
    return P.views[locate_view(P, P.tile_begin + (slot >> 5))];
}

// ------------------------------------------------------------------ counts
// The ray pass runs without host round trips: every kernel after K2a reads
// its item count from the wave counters (clamped to the buffer capacity; an
// overflow is detected by the host after the step and the step is redone with
// larger buffers, Adam being skipped on device meanwhile).

// 1 in *flag when any wave buffer overflowed this pass (the step is redone).
__global__ void wave_overflow_kernel(WaveBufs W, unsigned long long* flag) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *flag = wave_over(W) ? 1ull : 0ull;
}

// Shading records grouped by tile (K2b / K2e order: decode gathers and the
// per-tile probe / plane gradient aggregation see runs of one tile): a
// counting sort, warp-aggregated per tile with __match_any_sync.
__global__ void __launch_bounds__(256) rec_tile_count_kernel(WaveBufs W, int* __restrict__ cnt) {
    const int n = n_records(W);
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    __shared__ unsigned s_valid;  // records of this block (holes excluded), one atomic per block
    if (threadIdx.x == 0) s_valid = 0;
    __syncthreads();
    unsigned valid = 0;
    for (int b = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; b < n; b += warps * 32) {
        const int i = b + lane;
        const int t = i < n ? W.r_tile[i] : -1;
        const unsigned m = __match_any_sync(FULL, t);
        if (t >= 0 && lane == __ffs(m) - 1) atomicAdd(cnt + t, __popc(m));
        valid += (unsigned)__popc(__ballot_sync(FULL, t >= 0));
    }
    if (lane == 0 && valid) atomicAdd(&s_valid, valid);
    __syncthreads();
    if (threadIdx.x == 0 && s_valid) atomicAdd(W.counters + 5, s_valid);
}
__global__ void __launch_bounds__(256) rec_tile_scatter_kernel(WaveBufs W, int* __restrict__ off) {
    const int n = n_records(W);
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int b = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; b < n; b += warps * 32) {
        const int i = b + lane;
        const int t = i < n ? W.r_tile[i] : -1;
        const unsigned m = __match_any_sync(FULL, t);
        const int leader = __ffs(m) - 1;
        int base = 0;
        if (t >= 0 && lane == leader) base = atomicAdd(off + t, __popc(m));
        base = __shfl_sync(FULL, base, leader);
        if (t >= 0) W.r_perm[base + __popc(m & ((1u << lane) - 1u))] = i;
    }
}

// ------------------------------------------------------------------ K2b
template <int NS, int NA, bool GEO>
#ifndef PSDF_FWD_MINB
#define PSDF_FWD_MINB 4  // 4 blocks per SM (r02: 299 vs 332 us at 5; with FFMA2 the register cap cost more)
#endif
__global__ void __launch_bounds__(BLOCK, PSDF_FWD_MINB) shade_fwd_kernel(RayPassParams P, WaveBufs W) {
    const int n_rec = n_sorted(W);
    constexpr int IN = NS + NA + NPOW;
    extern __shared__ __align__(16) float smem[];
    __shared__ uint64_t s_bar[WARPS_PER_BLOCK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const SmemMlp L = SmemMlp::make(IN);
    const MlpLayout G = MlpLayout::make(IN);
    ProbeStage ps;
    ps.init(smem + up4i(L.total) + warp * probe_stage_floats<NA>(), &s_bar[warp], P.g.order * P.g.order * NA);
    load_mlp_smem(P.mlp, smem, G, L);
    __syncthreads();
    const bool stage = P.stage_fwd && !P.no_angular;
    // one record per lane; a warp's 32 records are consecutive in tile order,
    // and the probe blocks of their first / last tile are bulk-copied into
    // this warp's staging slots
    for (int base = (blockIdx.x * WARPS_PER_BLOCK + warp) * 32; base < n_rec; base += gridDim.x * BLOCK) {
        const bool in_range = base + lane < n_rec;
        const int i = in_range ? W.r_perm[base + lane] : 0;
        const int tile = in_range ? W.r_tile[i] : -1;
        const float* psm = nullptr;
        if (stage) {
            const int tA = __shfl_sync(FULL, tile, 0), tB = __shfl_sync(FULL, tile, min(31, n_rec - 1 - base));
            psm = ps.fetch(tA, tB, tile, P.g.probes, P.g.probe_ids);
        }
        if (!in_range) continue;
        const int e = W.r_entry[i];
        const ViewDev& V = entry_view(P, W, e);
        const float* cam_row =
            (P.ncam > 0 && V.cam_bias_row >= 0) ? P.mlp + G.cam + V.cam_bias_row * HID : nullptr;
        const double pc[3] = {W.r_pos[3 * (int64_t)i], W.r_pos[3 * (int64_t)i + 1],
                              W.r_pos[3 * (int64_t)i + 2]};
        const double dneg[3] = {-W.e_dir[3 * (int64_t)e], -W.e_dir[3 * (int64_t)e + 1],
                                -W.e_dir[3 * (int64_t)e + 2]};
        float rgb[3];
        ShadeGeo geo;
        decode_forward<NS, NA>(P, smem, L, tile, pc, dneg, cam_row, rgb, geo,
                               GEO ? W.r_geo + (int64_t)i * GeoRec<NS, NA>::STRIDE : nullptr, psm);
        reinterpret_cast<float4*>(W.r_c)[i] = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
        const double w = W.r_w[i];
        atomicAdd(W.e_craw + 3 * (int64_t)e, dmul((double)rgb[0], w));
        atomicAdd(W.e_craw + 3 * (int64_t)e + 1, dmul((double)rgb[1], w));
        atomicAdd(W.e_craw + 3 * (int64_t)e + 2, dmul((double)rgb[2], w));
    }
}

// K2b on the tensor cores: decode_features per lane (one shading record per
// lane, records in tile order), then the decoder MLP for the warp's 32
// records as three warp GEMMs (3xTF32 mma.sync, weights pre-split in shared
// memory once per block): A1 = relu(X W1^T + b1 (+ camera bias)), A2 =
// relu(A1 W2^T + b2), Z = A2 W3^T + b3, colour = sigmoid(Z).  The FFMA
// form (shade_fwd_kernel) spends ~42 % of its instructions on the MLP
// (profiles/r02/v3); here it is ~170 MMAs per 32 records.
template <int IN>
struct FwdDims {
    static constexpr int K1 = (IN + 7) & ~7;  // input width padded to the MMA k step
    static_assert(K1 > IN, "the bias-gradient ones column needs a padding slot");
    static constexpr int XS = K1 + 4;         // row stride of W1 (conflict-free B fragments)
    static constexpr int HS = 36;             // row stride of 32-wide rows
    // pre-split weights (uint32 TF32 words): hi, then lo
    static constexpr int W1 = 0;              // [32][XS]
    static constexpr int W2 = W1 + 32 * XS;   // [32][HS]
    static constexpr int W3 = W2 + 32 * HS;   // [8][HS], rows 3..7 zero
    static constexpr int WN = W3 + 8 * HS;    // words per split half
    static constexpr int B1 = 2 * WN, B2 = B1 + 32, B3 = B2 + 32;  // biases (float)
    static constexpr int MLP = B3 + 4;
    // per-warp scratch: S0 = X (row stride HS), later A2; S1 = A1, later Z
    static constexpr int S0 = 0, S1 = 32 * HS, SCR = 64 * HS;
};

template <int NS, int NA>
size_t shade_fwd_mma_smem_bytes() {
    using D = FwdDims<NS + NA + NPOW>;
    return sizeof(float) * (D::MLP + WARPS_PER_BLOCK * (D::SCR + probe_stage_floats<NA>()));
}

#ifndef PSDF_FWDM_MINB
#define PSDF_FWDM_MINB 4
#endif
template <int NS, int NA, bool GEO>
__global__ void __launch_bounds__(BLOCK, PSDF_FWDM_MINB) shade_fwd_mma_kernel(RayPassParams P, WaveBufs W) {
    const int n_rec = n_sorted(W);
    constexpr int IN = NS + NA + NPOW;
    using D = FwdDims<IN>;
    extern __shared__ __align__(16) float smem[];
    uint32_t* wsp = reinterpret_cast<uint32_t*>(smem);
    const MlpLayout G = MlpLayout::make(IN);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // weights, split once: W1 [32][IN] (zero padded to K1), W2 [32][32], W3 [3][32]
    for (int i = threadIdx.x; i < D::WN; i += blockDim.x) {
        float v = 0.f;
        if (i < D::W2) {
            const int j = i / D::XS, k = i % D::XS;
            if (k < IN) v = __ldg(P.mlp + G.w1 + j * IN + k);
        } else if (i < D::W3) {
            const int j = (i - D::W2) / D::HS, k = (i - D::W2) % D::HS;
            if (k < 32) v = __ldg(P.mlp + G.w2 + j * 32 + k);
        } else {
            const int j = (i - D::W3) / D::HS, k = (i - D::W3) % D::HS;
            if (j < 3 && k < 32) v = __ldg(P.mlp + G.w3 + j * 32 + k);
        }
        const uint32_t hi = tf32(v);
        wsp[i] = hi;
        wsp[D::WN + i] = tf32(v - __uint_as_float(hi));
    }
    for (int i = threadIdx.x; i < 32; i += blockDim.x) {
        smem[D::B1 + i] = __ldg(P.mlp + G.b1 + i);
        smem[D::B2 + i] = __ldg(P.mlp + G.b2 + i);
        if (i < 3) smem[D::B3 + i] = __ldg(P.mlp + G.b3 + i);
    }
    __syncthreads();
    float* S0 = smem + D::MLP + warp * D::SCR + D::S0;
    float* S1 = smem + D::MLP + warp * D::SCR + D::S1;
    __shared__ uint64_t s_bar[WARPS_PER_BLOCK];
    ProbeStage ps;
    ps.init(smem + D::MLP + WARPS_PER_BLOCK * D::SCR + warp * probe_stage_floats<NA>(), &s_bar[warp],
            P.g.order * P.g.order * NA);
    __shared__ int s_cam[WARPS_PER_BLOCK][32];
    int* cam = s_cam[warp];
    const float* cam_base = P.mlp + G.cam;
    const int warps_total = gridDim.x * WARPS_PER_BLOCK;
    for (int base = (blockIdx.x * WARPS_PER_BLOCK + warp) * 32; base < n_rec; base += warps_total * 32) {
        const bool in_range = base + lane < n_rec;
        int i = 0, e = 0, cam_row = -1;
        float x[IN];
#pragma unroll
        for (int k = 0; k < IN; ++k) x[k] = 0.f;
        if (in_range) i = W.r_perm[base + lane];
        const int tile = in_range ? W.r_tile[i] : -1;
        const float* psm = nullptr;
        if (P.stage_fwd && !P.no_angular) {
            const int tA = __shfl_sync(FULL, tile, 0), tB = __shfl_sync(FULL, tile, min(31, n_rec - 1 - base));
            psm = ps.fetch(tA, tB, tile, P.g.probes, P.g.probe_ids);
        }
        if (in_range) {
            e = W.r_entry[i];
            const ViewDev& V = entry_view(P, W, e);
            if (P.ncam > 0 && V.cam_bias_row >= 0) cam_row = V.cam_bias_row;
            const double pc[3] = {W.r_pos[3 * (int64_t)i], W.r_pos[3 * (int64_t)i + 1],
                                  W.r_pos[3 * (int64_t)i + 2]};
            const double dneg[3] = {-W.e_dir[3 * (int64_t)e], -W.e_dir[3 * (int64_t)e + 1],
                                    -W.e_dir[3 * (int64_t)e + 2]};
            ShadeGeo geo;
            float pv[3][NS];
            decode_features<NS, NA>(P, tile, pc, dneg, geo, x, pv, psm);
            if (GEO) store_geo<NS, NA>(geo, pv, x, W.r_geo + (int64_t)i * GeoRec<NS, NA>::STRIDE);
        }
#pragma unroll
        for (int k = 0; k < D::K1; ++k) S0[lane * D::HS + k] = k < IN ? x[k] : 0.f;
        cam[lane] = cam_row;
        __syncwarp();
        {  // A1 = relu(X W1^T + b1 + camera bias)
            float c[2][4][4];
            zero_c(c);
            warp_gemm3w<2, 4, D::K1 / 8>(
                c, [&](int m, int k) { return S0[m * D::HS + k]; },
                [&](int n, int k) { return wsp[D::W1 + n * D::XS + k]; },
                [&](int n, int k) { return wsp[D::WN + D::W1 + n * D::XS + k]; });
            for_c(c, [&](int m, int n, float& v) {
                float z = v + smem[D::B1 + n];
                if (cam[m] >= 0) z += __ldg(cam_base + cam[m] * HID + n);
                S1[m * D::HS + n] = z > 0.f ? z : 0.f;
            });
        }
        __syncwarp();
        {  // A2 = relu(A1 W2^T + b2)  (into S0: X is dead)
            float c[2][4][4];
            zero_c(c);
            warp_gemm3w<2, 4, 4>(
                c, [&](int m, int k) { return S1[m * D::HS + k]; },
                [&](int n, int k) { return wsp[D::W2 + n * D::HS + k]; },
                [&](int n, int k) { return wsp[D::WN + D::W2 + n * D::HS + k]; });
            __syncwarp();
            for_c(c, [&](int m, int n, float& v) {
                const float z = v + smem[D::B2 + n];
                S0[m * D::HS + n] = z > 0.f ? z : 0.f;
            });
        }
        __syncwarp();
        {  // Z = A2 W3^T (columns 0..2 of one 8-wide tile), into S1
            float c[2][1][4];
            zero_c(c);
            warp_gemm3w<2, 1, 4>(
                c, [&](int m, int k) { return S0[m * D::HS + k]; },
                [&](int n, int k) { return wsp[D::W3 + n * D::HS + k]; },
                [&](int n, int k) { return wsp[D::WN + D::W3 + n * D::HS + k]; });
            __syncwarp();
            for_c(c, [&](int m, int n, float& v) {
                if (n < 3) S1[m * 4 + n] = v;
            });
        }
        __syncwarp();
        if (in_range) {
            float rgb[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) rgb[j] = sigmoidf_(S1[lane * 4 + j] + smem[D::B3 + j]);
            reinterpret_cast<float4*>(W.r_c)[i] = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
            const double w = W.r_w[i];
            atomicAdd(W.e_craw + 3 * (int64_t)e, dmul((double)rgb[0], w));
            atomicAdd(W.e_craw + 3 * (int64_t)e + 1, dmul((double)rgb[1], w));
            atomicAdd(W.e_craw + 3 * (int64_t)e + 2, dmul((double)rgb[2], w));
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ K2d
__global__ void __launch_bounds__(BLOCK) alpha_bwd_kernel(RayPassParams P, WaveBufs W) {
    const int n_ent = n_entries(W);
    const int lane = threadIdx.x & 31;
    const GridView& g = P.g;
    const double tau = P.tau;
    double st_photo = 0.0, st_sq = 0.0;
    unsigned long long st_mask = 0, c_al = 0, c_bwd = 0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_ent; e += gridDim.x * blockDim.x) {
        const int slot = W.e_slot[e];
        if (slot < 0) continue;  // a hole of an abandoned allocation chunk
        const LaneRay R = lane_ray(P, slot >> 5, slot & 31);
        const bool in_mask = __ldg(R.V->mask + R.px) != 0;
        const double acc = W.e_acc[e];
        const double om = dsub(1.0, acc);
        const double c0 = W.e_craw[3 * (int64_t)e], c1 = W.e_craw[3 * (int64_t)e + 1],
                     c2 = W.e_craw[3 * (int64_t)e + 2];
        const double col[3] = {dadd(c0, dmul(P.bg[0], om)), dadd(c1, dmul(P.bg[1], om)),
                               dadd(c2, dmul(P.bg[2], om))};
        double gx, gy, gz, dA;
        const bool need_bwd = photo_term(P, in_mask, R.V->gt + 3 * R.px, col, acc, gx, gy, gz, dA,
                                         st_photo, st_sq, st_mask);
        int rec = W.e_head[e];
        if (!need_bwd) {  // no gradient: records carry a zero upstream
            for (; rec >= 0; rec = W.r_next[rec])
                reinterpret_cast<float4*>(W.r_up)[rec] = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        ++c_bwd;
        const double total = dadd(dadd(dadd(dmul(gx, dsub(c0, dmul(P.bg[0], acc))),
                                            dmul(gy, dsub(c1, dmul(P.bg[1], acc)))),
                                       dmul(gz, dsub(c2, dmul(P.bg[2], acc)))),
                                  dmul(dA, acc));
        const double gbg = dadd(dadd(dmul(gx, P.bg[0]), dmul(gy, P.bg[1])), dmul(gz, P.bg[2]));
        const double* o = R.V->cam.pos;
        const double dd[3] = {W.e_dir[3 * (int64_t)e], W.e_dir[3 * (int64_t)e + 1],
                              W.e_dir[3 * (int64_t)e + 2]};
        auto pos = [&](double t, double p[3]) {
#pragma unroll
            for (int k = 0; k < 3; ++k) p[k] = dadd(o[k], dmul(dd[k], t));
        };
        // the alpha > 0 samples in march order; the samples between them have
        // alpha == 0 and w == 0 and only pass the previous sample's
        // d/ds_{i+1} term on to their own position (renderer.cpp:254-276)
        double pre = 0.0, carry = 0.0, t_carry = -1.0;
        int tile_carry = -1;
        for (int a = W.e_ahead[e]; a >= 0;) {
            const int4 ai = W.a_i[a];
            const double t_i = W.a_t[2 * (int64_t)a], t_n = W.a_t[2 * (int64_t)a + 1];
            const double a_cur = W.a_s[3 * (int64_t)a], a_nxt = W.a_s[3 * (int64_t)a + 1],
                         T = W.a_s[3 * (int64_t)a + 2];
            const double alpha = alpha_from(a_cur, a_nxt);
            const double w = dmul(T, alpha);
            ++c_al;
            // dL/dw_i = g.(C_i - bg) + dA (renderer.cpp:249-253)
            double dw = dadd(-gbg, dA);
            if (ai.z >= 0) {
                const float4 cr = reinterpret_cast<const float4*>(W.r_c)[ai.z];
                dw = dadd(dsub(dadd(dadd(dmul(gx, (double)cr.x), dmul(gy, (double)cr.y)),
                                    dmul(gz, (double)cr.z)),
                               gbg),
                          dA);
                reinterpret_cast<float4*>(W.r_up)[ai.z] =
                    make_float4((float)(w * gx), (float)(w * gy), (float)(w * gz), 0.f);
            }
            pre = dadd(pre, dmul(dw, w));
            double own = 0.0, nxt = 0.0;
            const double om_a = dsub(1.0, alpha);
            const double dalpha = dsub(dmul(dw, T), om_a > 1e-12 ? ddiv_fast(dsub(total, pre), om_a) : 0.0);
            if (dalpha != 0.0) {  // renderer.cpp:266-276
                const double da = dmul(dmul(tau, a_cur), dsub(1.0, a_cur));
                const double db = dmul(dmul(tau, a_nxt), dsub(1.0, a_nxt));
                own = ddiv_fast(dmul(dmul(dalpha, a_nxt), da), dmul(a_cur, a_cur));
                nxt = dmul(dalpha, ddiv_fast(-db, a_cur));
            }
            double p[3];
            // the previous alpha sample's term lands here, or at a sample of its own
            double ds_i = own;
            if (carry != 0.0) {
                if (t_carry == t_i) {
                    ds_i = dadd(carry, own);
                } else {
                    pos(t_carry, p);
                    scatter_smooth_in(g, P.g_smooth, tile_carry, __ldg(g.tile_coords + tile_carry), p, carry);
                }
            }
            if (ds_i != 0.0) {
                pos(t_i, p);
                scatter_smooth_in(g, P.g_smooth, ai.x, __ldg(g.tile_coords + ai.x), p, ds_i);
            }
            carry = nxt;
            t_carry = t_n;
            tile_carry = ai.y;
            a = ai.w;
            if (a < 0 && carry != 0.0) {
                pos(t_n, p);
                if (tile_carry >= 0)
                    scatter_smooth_in(g, P.g_smooth, tile_carry, __ldg(g.tile_coords + tile_carry), p, carry);
                else  // the one-past-the-end point
                    scatter_smooth(g, P.g_smooth, p[0], p[1], p[2], carry);
            }
        }
    }
    st_photo = warp_sum_d(st_photo);
    st_sq = warp_sum_d(st_sq);
    st_mask = warp_sum_u(st_mask);
    c_al = warp_sum_u(c_al);
    c_bwd = warp_sum_u(c_bwd);
    if (lane == 0) {
        atomicAdd(P.stats + 0, st_photo);
        atomicAdd(P.stats + 1, st_sq);
        atomicAdd(P.stats + 2, (double)st_mask);
        atomicAdd(P.counts + 4, c_al);
        atomicAdd(P.counts + 5, c_bwd);
    }
}

// Per-record feature gradients handed from the MLP backward to the geometry
// backward: gfs[NS] | gfa[NA] | d(n.v), padded to a float4 multiple.
template <int NS, int NA>
struct FgDims {
    static constexpr int STRIDE = ((NS + NA + 1) + 3) & ~3;
};

// ------------------------------------------------------------------ K2e
// decode_backward's MLP half (decoder.cpp:111-176) for batches of 32 shading
// records per warp (tile order), every product on the tensor cores
// (psdf_mma.cuh, 3xTF32): the forward is recomputed (A1 = relu(X W1^T + b1),
// A2 = relu(A1 W2^T + b2)), then DZ2 = (DZ3 W3) [A2 > 0], DZ1 = (DZ2 W2) [A1 > 0],
// DIN = DZ1 W1 and the weight gradients dW3 += DZ3^T A2, dW2 += DZ2^T A1,
// dW1 += DZ1^T X into per-warp accumulators (C fragments kept in shared
// memory), flushed once per block.  Rows of non-shading lanes are zero.
template <int IN>
struct MmaDims {
    static constexpr int K1 = (IN + 7) & ~7;  // input width padded to the MMA k step
    static constexpr int XS = K1 + 4;         // row stride of X / W1 (conflict-free fragments)
    static constexpr int HS = 36;             // row stride of 32-wide rows
    static constexpr int DS = 12;             // row stride of DZ3 (8 used)
    // shared MLP copy
    static constexpr int W1 = 0;              // [32][XS]   W1, zero padded
    static constexpr int W1T = W1 + 32 * XS;  // [K1][HS]   W1^T
    static constexpr int W2 = W1T + K1 * HS;  // [32][HS]
    static constexpr int W2T = W2 + 32 * HS;  // [32][HS]   W2^T
    static constexpr int W3 = W2T + 32 * HS;  // [8][HS]    rows 3..7 zero
    static constexpr int B1 = W3 + 8 * HS, B2 = B1 + 32, B3 = B2 + 32;
    static constexpr int MLP = B3 + 4;
    // the weights [0, B1) are kept pre-split for the 3xTF32 products: TF32
    // high halves in place, low halves at WLO + the same offset
    static constexpr int WLO = MLP;
    static constexpr int MLPX = WLO + B1;     // shared MLP incl. the low halves
    // per-warp scratch
    static constexpr int SX = 0;                // [32][XS]  X, later DIN
    static constexpr int SA1 = SX + 32 * XS;    // [32][HS]  A1, later DZ1
    static constexpr int SA2 = SA1 + 32 * HS;   // [32][HS]  A2, later DZ2
    static constexpr int SD3 = SA2 + 32 * HS;   // [32][DS]  DZ3
    static constexpr int SCR = SD3 + 32 * DS;
    // per-warp gradient accumulators
    static constexpr int GW1 = 0;               // [32][XS]
    static constexpr int GW2 = GW1 + 32 * XS;   // [32][HS]
    static constexpr int GW3 = GW2 + 32 * HS;   // [3][HS]
    static constexpr int GB1 = GW3 + 3 * HS, GB2 = GB1 + 32, GB3 = GB2 + 32;
    static constexpr int GACC = (GB3 + 4 + 3) & ~3;
};

template <int NS, int NA>
#ifndef PSDF_BWD_MINB
#define PSDF_BWD_MINB 1  // measured: 224 registers / 2 blocks per SM beat a 170-register cap (297 vs 318 us); after the conversion-free split all caps are within noise (profiles/r02/v50_bwd_regcap_ab.txt)
#endif
__global__ void __launch_bounds__(BLOCK, PSDF_BWD_MINB) shade_bwd_kernel(RayPassParams P, WaveBufs W) {
    const int n_rec = n_sorted(W);
    constexpr int IN = NS + NA + NPOW;
    using D = MmaDims<IN>;
    using GR = GeoRec<NS, NA>;
    extern __shared__ __align__(16) float smem[];
    const MlpLayout G = MlpLayout::make(IN);
    float* sm = smem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* scr = smem + D::MLPX + warp * D::SCR;
    __shared__ int s_cam[WARPS_PER_BLOCK][32];
    int* cam = s_cam[warp];
    // MLP into shared memory: padded W1 / W1^T / W2 / W2^T / W3, biases
    for (int i = threadIdx.x; i < D::MLP; i += blockDim.x) sm[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * IN; i += blockDim.x) {
        const int j = i / IN, k = i % IN;
        const float v = __ldg(P.mlp + G.w1 + i);
        sm[D::W1 + j * D::XS + k] = v;
        sm[D::W1T + k * D::HS + j] = v;
    }
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        const float v = __ldg(P.mlp + G.w2 + i);
        sm[D::W2 + (i >> 5) * D::HS + (i & 31)] = v;
        sm[D::W2T + (i & 31) * D::HS + (i >> 5)] = v;
    }
    for (int i = threadIdx.x; i < 96; i += blockDim.x) sm[D::W3 + (i >> 5) * D::HS + (i & 31)] = __ldg(P.mlp + G.w3 + i);
    for (int i = threadIdx.x; i < 32; i += blockDim.x) {
        sm[D::B1 + i] = __ldg(P.mlp + G.b1 + i);
        sm[D::B2 + i] = __ldg(P.mlp + G.b2 + i);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < D::B1; i += blockDim.x) {  // pre-split weights (once per block)
        uint32_t hi, lo;
        split1(sm[i], hi, lo);
        sm[i] = __uint_as_float(hi);
        sm[D::WLO + i] = __uint_as_float(lo);
    }
    __syncthreads();
    auto wh = [&](int a) { return __float_as_uint(sm[a]); };
    auto wl = [&](int a) { return __float_as_uint(sm[D::WLO + a]); };
    // weight-gradient accumulators: this warp's C fragments, kept in registers
    // across its batches (dW2 32x32, dW1 32xK1, dW3 rows 0..2) + bias sums
    float gw2[2][4][4], gw1[2][D::K1 / 8][4], gw3[1][4][4];
    zero_c(gw2);
    zero_c(gw1);
    zero_c(gw3);
    float gb2 = 0.f, gb3 = 0.f;  // db1 comes out of the dW1 GEMM (ones column)
    const float* cam_base = P.mlp + G.cam;
    const bool has_cam = P.ncam > 0;
    float* X = scr + D::SX;
    float* A1 = scr + D::SA1;
    float* A2 = scr + D::SA2;
    float* D3 = scr + D::SD3;
    const int warps_total = gridDim.x * WARPS_PER_BLOCK;
    for (int base = (blockIdx.x * WARPS_PER_BLOCK + warp) * 32; base < n_rec; base += warps_total * 32) {
        const bool in_range = base + lane < n_rec;
        const int i = in_range ? W.r_perm[base + lane] : 0;
        float4 up = make_float4(0.f, 0.f, 0.f, 0.f);
        int cam_row = -1;
        if (in_range) {
            up = reinterpret_cast<const float4*>(W.r_up)[i];
            if (P.ncam > 0) cam_row = entry_view(P, W, W.r_entry[i]).cam_bias_row;
        }
        const bool shade = in_range && (up.x != 0.f || up.y != 0.f || up.z != 0.f);
        const unsigned smask = __ballot_sync(FULL, shade);
        if (!smask) continue;
        // row `lane` of X and DZ3 (zero for non-shading lanes)
        float ndv = 0.f;
        {
            float x[D::K1];
#pragma unroll
            for (int q = 0; q < D::K1; ++q) x[q] = 0.f;
            float d3[3] = {0.f, 0.f, 0.f};
            if (shade) {
                const float* rg = W.r_geo + (int64_t)i * GR::STRIDE;
#pragma unroll
                for (int q = 0; q < IN; ++q) x[q] = rg[GR::X + q];
                // a ones column in the first padding slot: the dW1 GEMM's
                // column IN is then db1 = sum_m DZ1[m] (W1's padding is zero,
                // so the forward recompute and DIN are unchanged)
                x[IN] = 1.f;
                ndv = rg[7];
                const float4 cr = reinterpret_cast<const float4*>(W.r_c)[i];
                d3[0] = up.x * cr.x * (1.f - cr.x);  // sigmoid'
                d3[1] = up.y * cr.y * (1.f - cr.y);
                d3[2] = up.z * cr.z * (1.f - cr.z);
            }
#pragma unroll
            for (int q = 0; q < D::K1; ++q) X[lane * D::XS + q] = x[q];
#pragma unroll
            for (int q = 0; q < 8; ++q) D3[lane * D::DS + q] = q < 3 ? d3[q] : 0.f;
            cam[lane] = shade ? cam_row : -1;
        }
        __syncwarp();
        // A1 = relu(X W1^T + b1 (+ camera bias))
        {
            float c[2][4][4];
            zero_c(c);
            warp_gemm3w<2, 4, D::K1 / 8>(
                c, [&](int m, int k) { return X[m * D::XS + k]; },
                [&](int n, int k) { return wh(D::W1 + n * D::XS + k); },
                [&](int n, int k) { return wl(D::W1 + n * D::XS + k); });
            if (has_cam) {
                for_c(c, [&](int m, int n, float& v) {
                    float z = v + sm[D::B1 + n];
                    if (cam[m] >= 0) z += __ldg(cam_base + cam[m] * HID + n);
                    A1[m * D::HS + n] = z > 0.f ? z : 0.f;
                });
            } else {
                for_c(c, [&](int m, int n, float& v) {
                    const float z = v + sm[D::B1 + n];
                    A1[m * D::HS + n] = z > 0.f ? z : 0.f;
                });
            }
        }
        __syncwarp();
        // A2 = relu(A1 W2^T + b2)
        {
            float c[2][4][4];
            zero_c(c);
            warp_gemm3w<2, 4, 4>(
                c, [&](int m, int k) { return A1[m * D::HS + k]; },
                [&](int n, int k) { return wh(D::W2 + n * D::HS + k); },
                [&](int n, int k) { return wl(D::W2 + n * D::HS + k); });
            for_c(c, [&](int m, int n, float& v) {
                const float z = v + sm[D::B2 + n];
                A2[m * D::HS + n] = z > 0.f ? z : 0.f;
            });
        }
        __syncwarp();
        // dW3 += DZ3^T A2 (rows 0..2 of one 16-row tile), db3
        {
            warp_gemm3<1, 4, 4>(
                gw3, [&](int m, int k) { return m < 3 ? D3[k * D::DS + m] : 0.f; },
                [&](int n, int k) { return A2[k * D::HS + n]; });
            if (lane < 3)
                for (int r = 0; r < 32; ++r) gb3 += D3[r * D::DS + lane];
        }
        __syncwarp();
        // DZ2 = (DZ3 W3) [A2 > 0]  (in place of A2)
        {
            float c[2][4][4];
            zero_c(c);
            warp_gemm3w<2, 4, 1>(
                c, [&](int m, int k) { return D3[m * D::DS + k]; },
                [&](int n, int k) { return wh(D::W3 + k * D::HS + n); },
                [&](int n, int k) { return wl(D::W3 + k * D::HS + n); });
            __syncwarp();
            for_c(c, [&](int m, int n, float& v) {
                float& a = A2[m * D::HS + n];
                a = a > 0.f ? v : 0.f;
            });
        }
        __syncwarp();
        // dW2 += DZ2^T A1, db2
        {
            warp_gemm3<2, 4, 4>(
                gw2, [&](int m, int k) { return A2[k * D::HS + m]; },
                [&](int n, int k) { return A1[k * D::HS + n]; });
            for (int r = 0; r < 32; ++r) gb2 += A2[r * D::HS + lane];
        }
        __syncwarp();
        // DZ1 = (DZ2 W2) [A1 > 0]  (in place of A1)
        {
            float c[2][4][4];
            zero_c(c);
            warp_gemm3w<2, 4, 4>(
                c, [&](int m, int k) { return A2[m * D::HS + k]; },
                [&](int n, int k) { return wh(D::W2T + n * D::HS + k); },
                [&](int n, int k) { return wl(D::W2T + n * D::HS + k); });
            __syncwarp();
            for_c(c, [&](int m, int n, float& v) {
                float& a = A1[m * D::HS + n];
                a = a > 0.f ? v : 0.f;
            });
        }
        __syncwarp();
        // dW1 += DZ1^T X, db1, camera-bias rows (grouped by camera row)
        {
            warp_gemm3<2, D::K1 / 8, 4>(
                gw1, [&](int m, int k) { return A1[k * D::HS + m]; },
                [&](int n, int k) { return X[k * D::XS + n]; });
            if (P.ncam > 0) {
                const int my = cam[lane];
                unsigned rem = __ballot_sync(FULL, my >= 0);
                while (rem) {
                    const int row = __shfl_sync(FULL, my, __ffs(rem) - 1);
                    const unsigned grp = __ballot_sync(FULL, ((rem >> lane) & 1u) && my == row);
                    rem &= ~grp;
                    float cs = 0.f;
                    for (unsigned m = grp; m; m &= m - 1) cs += A1[(__ffs(m) - 1) * D::HS + lane];
                    if (cs != 0.f) atomicAdd(P.g_mlp + G.cam + row * HID + lane, cs);
                }
            }
        }
        __syncwarp();
        // DIN = DZ1 W1  (into X)
        {
            float c[2][D::K1 / 8][4];
            zero_c(c);
            warp_gemm3w<2, D::K1 / 8, 4>(
                c, [&](int m, int k) { return A1[m * D::HS + k]; },
                [&](int n, int k) { return wh(D::W1T + n * D::HS + k); },
                [&](int n, int k) { return wl(D::W1T + n * D::HS + k); });
            __syncwarp();
            for_c(c, [&](int m, int n, float& v) { X[m * D::XS + n] = v; });
        }
        __syncwarp();
        if (shade) {  // feature gradients for K2e-geo: gfs | gfa | d(n.v)
            const float* din = X + lane * D::XS;
            float* fg = W.r_fg + (int64_t)i * FgDims<NS, NA>::STRIDE;
#pragma unroll
            for (int k = 0; k < NS + NA; ++k) fg[k] = din[k];
            float d_ndotv = 0.f;
            if (!P.no_fresnel && ndv >= 0.f && ndv <= 1.f) {  // decoder.cpp:162-175
                const float uu = 1.f - ndv;
                float du = 0.f, upw = 1.f;
#pragma unroll
                for (int k = 1; k < NPOW; ++k) {
                    du += din[NS + NA + k] * (float)k * upw;
                    upw *= uu;
                }
                d_ndotv = -du;
            }
            fg[NS + NA] = d_ndotv;
        }
        __syncwarp();
    }
    // flush: each warp's accumulators into its scratch (GACC layout), then the
    // block sums the warps, one atomic per weight
    __syncwarp();
    float* gacc = scr;
    for_c(gw2, [&](int m, int n, float& v) { gacc[D::GW2 + m * D::HS + n] = v; });
    for_c(gw1, [&](int m, int n, float& v) { gacc[D::GW1 + m * D::XS + n] = v; });
    for_c(gw3, [&](int m, int n, float& v) {
        if (m < 3) gacc[D::GW3 + m * D::HS + n] = v;
    });
    gacc[D::GB2 + lane] = gb2;
    if (lane < 3) gacc[D::GB3 + lane] = gb3;
    __syncthreads();
    for (int q = threadIdx.x; q < G.total_nocam; q += blockDim.x) {
        int a;
        if (q < G.b1) a = D::GW1 + (q / IN) * D::XS + (q % IN);
        else if (q < G.w2) a = D::GW1 + (q - G.b1) * D::XS + IN;  // db1: the ones column
        else if (q < G.b2) a = D::GW2 + ((q - G.w2) >> 5) * D::HS + ((q - G.w2) & 31);
        else if (q < G.w3) a = D::GB2 + (q - G.b2);
        else if (q < G.b3) a = D::GW3 + ((q - G.w3) >> 5) * D::HS + ((q - G.w3) & 31);
        else a = D::GB3 + (q - G.b3);
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < WARPS_PER_BLOCK; ++w) v += smem[D::MLPX + w * D::SCR + a];
        if (v != 0.f) atomicAdd(P.g_mlp + q, v);
    }
}

// ------------------------------------------------------------------ K2e-geo
// The geometry half of decode_backward and the normal chain, one lane per
// shading record in tile order (no MLP state: high occupancy): tri-plane
// atomics (grid.cpp:189-202), the probe direction gradient (sh.cpp:151-169),
// probe coefficient gradients aggregated over the warp's lanes sharing a
// tile, and the SDF-gradient chain of the normal (renderer.cpp:216-235).
constexpr int PWS = 36;  // row stride of the per-warp probe staging (w8 | Y[16] | gfa), float4 aligned
template <int NS, int NA>
__global__ void __launch_bounds__(BLOCK) shade_geo_kernel(RayPassParams P, WaveBufs W) {
    const int n_rec = n_sorted(W);
    __shared__ __align__(16) float s_pw[WARPS_PER_BLOCK][32 * PWS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* PW = s_pw[warp];
    const GridView& g = P.g;
    const int warps_total = gridDim.x * WARPS_PER_BLOCK;
    using GR = GeoRec<NS, NA>;
    for (int base = (blockIdx.x * WARPS_PER_BLOCK + warp) * 32; base < n_rec; base += warps_total * 32) {
        const bool in_range = base + lane < n_rec;
        const int i = in_range ? W.r_perm[base + lane] : 0;
        float4 up = make_float4(0.f, 0.f, 0.f, 0.f);
        int e = -1, tile = -1;
        if (in_range) {
            up = reinterpret_cast<const float4*>(W.r_up)[i];
            e = W.r_entry[i];
            tile = W.r_tile[i];
        }
        const bool shade = in_range && (up.x != 0.f || up.y != 0.f || up.z != 0.f);
        const unsigned smask = __ballot_sync(FULL, shade);
        if (!smask) continue;
        float gfs[NS], gfa[NA], d_ndotv = 0.f, drx = 0.f, dry = 0.f, drz = 0.f;
        ShadeGeo geo;
        float pv[3][NS];
        if (shade) {
            constexpr int NQ = (GR::X + 3) / 4;
            float r[4 * NQ];
            const float4* src = reinterpret_cast<const float4*>(W.r_geo + (int64_t)i * GR::STRIDE);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float4 v4 = src[q];
                r[4 * q] = v4.x;
                r[4 * q + 1] = v4.y;
                r[4 * q + 2] = v4.z;
                r[4 * q + 3] = v4.w;
            }
            geo.n[0] = r[0];
            geo.n[1] = r[1];
            geo.n[2] = r[2];
            geo.glen = r[3];
            geo.refl[0] = r[4];
            geo.refl[1] = r[5];
            geo.refl[2] = r[6];
            geo.ndv = r[7];
            const int packed = __float_as_int(r[11]);
            geo.tx = Tap{packed & 15, r[8]};
            geo.ty = Tap{(packed >> 4) & 15, r[9]};
            geo.tz = Tap{(packed >> 8) & 15, r[10]};
            geo.degenerate = (packed >> 12) & 1;
#pragma unroll
            for (int c = 0; c < 8; ++c) geo.w8[c] = r[12 + c];
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int k = 0; k < NS; ++k) pv[q][k] = r[GR::PV + q * NS + k];
            const float* fg = W.r_fg + (int64_t)i * FgDims<NS, NA>::STRIDE;
#pragma unroll
            for (int k = 0; k < NS; ++k) gfs[k] = fg[k];
#pragma unroll
            for (int k = 0; k < NA; ++k) gfa[k] = fg[NS + k];
            d_ndotv = fg[NS + NA];
            // tri-plane backward (grid.cpp:189-202), plane samples from the record
            if (!P.no_spatial) {
                float* gpl = P.g_planes + (int64_t)tile * 3 * 256 * NS;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const Tap ta = q == 0 ? geo.ty : geo.tx;
                    const Tap tb = q == 2 ? geo.ty : geo.tz;
                    float gq[NS];
#pragma unroll
                    for (int k = 0; k < NS; ++k)
                        gq[k] = gfs[k] * (q == 0 ? pv[1][k] * pv[2][k]
                                                 : (q == 1 ? pv[0][k] * pv[2][k] : pv[0][k] * pv[1][k]));
                    float* bp = gpl + q * 256 * NS;
                    const float wq[4] = {(1.f - ta.f) * (1.f - tb.f), (1.f - ta.f) * tb.f,
                                         ta.f * (1.f - tb.f), ta.f * tb.f};
                    const int off[4] = {(ta.a0 * TE + tb.a0) * NS, (ta.a0 * TE + tb.a0 + 1) * NS,
                                        ((ta.a0 + 1) * TE + tb.a0) * NS,
                                        ((ta.a0 + 1) * TE + tb.a0 + 1) * NS};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float vv4[NS];
#pragma unroll
                        for (int k = 0; k < NS; ++k) vv4[k] = wq[c] * gq[k];
                        red_vec<NS>(bp + off[c], vv4);
                    }
                }
            }
            // probe direction gradient (sh.cpp:151-169)
            if (!P.no_angular) {
                const int nc = P.order * P.order;
                const int stride = g.order * g.order * NA;
                const int32_t* pid = g.probe_ids + (int64_t)tile * 8;
                float sj[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) sj[j] = 0.f;
#pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    const float wc = geo.w8[c];
                    if (wc == 0.f) continue;
                    const float* cp = g.probes + (int64_t)__ldg(pid + c) * stride;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (j < nc) {
                            const VecF<NA> cv = ldg_vec<NA>(cp + j * NA);
                            float sacc = 0.f;
#pragma unroll
                            for (int k = 0; k < NA; ++k) sacc += cv.v[k] * gfa[k];
                            sj[j] += wc * sacc;
                        }
                    }
                }
                sh_basis_grad_dot(geo.refl[0], geo.refl[1], geo.refl[2], P.order, sj, drx, dry, drz);
            }
        }
        // ---- probe coefficient gradients, aggregated over lanes sharing a tile
        if (!P.no_angular) {
            if (shade) {
                float Y[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) Y[j] = 0.f;
                sh_basis(geo.refl[0], geo.refl[1], geo.refl[2], P.order, Y);
#pragma unroll
                for (int c = 0; c < 8; ++c) PW[lane * PWS + c] = geo.w8[c];
#pragma unroll
                for (int j = 0; j < 16; ++j) PW[lane * PWS + 8 + j] = Y[j];
#pragma unroll
                for (int k = 0; k < NA; ++k) PW[lane * PWS + 24 + k] = gfa[k];
            }
            __syncwarp();
            const int nc = P.order * P.order;
            const int stride = g.order * g.order * NA;
            unsigned rem = smask;
            while (rem) {
                const int t0 = __shfl_sync(FULL, tile, __ffs(rem) - 1);
                const unsigned grp = __ballot_sync(FULL, ((rem >> lane) & 1u) && tile == t0);
                rem &= ~grp;
                const int32_t* pid = g.probe_ids + (int64_t)t0 * 8;
                // A[c][j][k] = sum_s w_c(s) Y_j(s) gfa_k(s): lane = (corner half, j),
                // all k; the group's rows are shared-memory broadcasts
                const int half = lane >> 4, j = lane & 15;
                if (j < nc) {
                    float a[4][NA];
                    bool anyc[4] = {false, false, false, false};
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                        for (int k = 0; k < NA; ++k) a[cc][k] = 0.f;
                    for (unsigned m = grp; m; m &= m - 1) {
                        const float* row = PW + (__ffs(m) - 1) * PWS;
                        const float4 w4 = *reinterpret_cast<const float4*>(row + 4 * half);
                        const float wc[4] = {w4.x, w4.y, w4.z, w4.w};
                        const float y = row[8 + j];
                        VecF<NA> u;
#pragma unroll
                        for (int k = 0; k < NA; ++k) u.v[k] = y * row[24 + k];
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) {
                            anyc[cc] |= wc[cc] != 0.f;
                            axpy_pairs<NA>(a[cc], u, wc[cc]);  // FFMA2
                        }
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc)
                        if (anyc[cc])
                            red_vec<NA>(P.g_probes + (int64_t)__ldg(pid + 4 * half + cc) * stride + j * NA, a[cc]);
                }
            }
            __syncwarp();
        }
        // ---- normal chain (renderer.cpp:216-235)
        if (shade && !geo.degenerate) {
            const double n[3] = {geo.n[0], geo.n[1], geo.n[2]};
            const double dneg[3] = {-W.e_dir[3 * (int64_t)e], -W.e_dir[3 * (int64_t)e + 1],
                                    -W.e_dir[3 * (int64_t)e + 2]};
            const double pc[3] = {W.r_pos[3 * (int64_t)i], W.r_pos[3 * (int64_t)i + 1],
                                  W.r_pos[3 * (int64_t)i + 2]};
            const double dr[3] = {(double)drx, (double)dry, (double)drz};
            const double drn = dr[0] * n[0] + dr[1] * n[1] + dr[2] * n[2];
            const double nv = n[0] * dneg[0] + n[1] * dneg[1] + n[2] * dneg[2];
            double dn[3], dgv[3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                dn[a] = 2.0 * drn * dneg[a] + 2.0 * nv * dr[a] + (double)d_ndotv * dneg[a];
            const double dnn = dn[0] * n[0] + dn[1] * n[1] + dn[2] * n[2];
#pragma unroll
            for (int a = 0; a < 3; ++a) dgv[a] = (dn[a] - n[a] * dnn) / geo.glen;
            const double inv2h = 1.0 / (2.0 * g.h);
            scatter_gradient_stencil(g, P.g_smooth, tile, pc, dgv[0] * inv2h, dgv[1] * inv2h,
                                     dgv[2] * inv2h);
        }
    }
}

template <int NS, int NA>
size_t shade_bwd_smem_bytes() {
    using D = MmaDims<NS + NA + NPOW>;
    static_assert(D::GACC <= D::SCR, "accumulator flush reuses the warp scratch");
    return sizeof(float) * (D::MLPX + WARPS_PER_BLOCK * D::SCR);
}

}  // namespace psdf
