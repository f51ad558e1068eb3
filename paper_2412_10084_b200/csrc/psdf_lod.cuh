// psdf_lod.cuh — LOD transition kernels: the GPU side
// of SparseGrid::subdivide (grid.cpp:271-338).  The allocation decision and
// every resampled value are computed in f64 in the reference's operation
// order from the (fp32) parent parameters; only the host-side bookkeeping of
// the new tile / probe lists (allocate_tile / ensure_probe order,
// grid.cpp:44-72) runs on the CPU.
#pragma once

#include "psdf_device.cuh"

namespace psdf {

// raw_value (grid.cpp:74-81) of the parent grid.
__device__ __forceinline__ double raw_value(const GridView& g, const float* __restrict__ raw, int vx, int vy,
                                            int vz) {
    if (vx < 0 || vy < 0 || vz < 0 || vx >= g.res[0] || vy >= g.res[1] || vz >= g.res[2]) return g.far;
    const int t = tile_lookup(g, vx >> 4, vy >> 4, vz >> 4);
    if (t < 0) return g.far;
    return (double)__ldg(raw + (int64_t)t * TV + vox_index(vx & 15, vy & 15, vz & 15));
}

// One block per (parent tile, child): the child's 16^3 raw values, sampled
// from the parent's raw grid at the child voxel centres (sample_raw,
// grid.cpp:120-125 / 96-117), and whether the child is allocated: it is
// dropped only when min |s| > band and the values do not change sign
// (grid.cpp:294-305).
__global__ void __launch_bounds__(256) subdiv_raw_kernel(GridView g, const float* __restrict__ raw,
                                                         double h_new, double band,
                                                         float* __restrict__ child_raw,
                                                         uint8_t* __restrict__ keep) {
    const int tile = blockIdx.x >> 3, child = blockIdx.x & 7;
    const int4 tc = __ldg(g.tile_coords + tile);
    const int cx = 2 * tc.x + (child & 1), cy = 2 * tc.y + ((child >> 1) & 1), cz = 2 * tc.z + ((child >> 2) & 1);
    double mn = 1.79769313486231570e308;
    bool pos = false, neg = false;
    float* out = child_raw + (int64_t)blockIdx.x * TV;
    for (int i = threadIdx.x; i < TV; i += blockDim.x) {
        const int x = i >> 8, y = (i >> 4) & 15, z = i & 15;
        // voxel_center (grid.hpp:75-77) of the child grid
        const double p[3] = {dadd(g.org[0], dmul((double)(cx * TE + x) + 0.5, h_new)),
                             dadd(g.org[1], dmul((double)(cy * TE + y) + 0.5, h_new)),
                             dadd(g.org[2], dmul((double)(cz * TE + z) + 0.5, h_new))};
        double c[3];
        int b[3];
        double f[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            c[a] = dsub(w2v(g, p[a], a), 0.5);
            b[a] = (int)floor(c[a]);
            f[a] = dsub(c[a], (double)b[a]);
        }
        double v8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v8[k] = raw_value(g, raw, b[0] + (k & 1), b[1] + ((k >> 1) & 1), b[2] + ((k >> 2) & 1));
        const double s = trilerp8(f[0], f[1], f[2], v8);
        out[vox_index(x, y, z)] = (float)s;
        mn = fmin(mn, fabs(s));
        (s >= 0.0 ? pos : neg) = true;
    }
    __shared__ double s_mn[8];
    __shared__ int s_flags[8];
    int fl = (pos ? 1 : 0) | (neg ? 2 : 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_mn[threadIdx.x >> 5] = mn;
        s_flags[threadIdx.x >> 5] = fl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mn = fmin(mn, s_mn[w]);
            fl |= s_flags[w];
        }
        keep[blockIdx.x] = (mn > band && fl != 3) ? 0 : 1;
    }
}

// Child raw values of the kept children, in the new tile order.
__global__ void __launch_bounds__(256) subdiv_gather_raw_kernel(const float* __restrict__ child_raw,
                                                                const int* __restrict__ src, int n_new,
                                                                float* __restrict__ raw_new) {
    const int t = blockIdx.x;
    if (t >= n_new) return;
    const float4* s4 = reinterpret_cast<const float4*>(child_raw + (int64_t)__ldg(src + t) * TV);
    float4* d4 = reinterpret_cast<float4*>(raw_new + (int64_t)t * TV);
    for (int i = threadIdx.x; i < TV / 4; i += blockDim.x) d4[i] = __ldg(s4 + i);
}

// Planes of a child: each 16x16 plane covers half of the parent's
// (grid.cpp:309-322): bilinear plane_sample at offs*8 + (a + 1/2)/2.
__global__ void __launch_bounds__(256) subdiv_planes_kernel(const float* __restrict__ planes, int n_s,
                                                            const int* __restrict__ src, int n_new,
                                                            float* __restrict__ planes_new) {
    const int t = blockIdx.x;
    if (t >= n_new) return;
    const int s = __ldg(src + t);
    const int parent = s >> 3, child = s & 7;
    const int offs[3] = {child & 1, (child >> 1) & 1, (child >> 2) & 1};
    const int per_plane = 256 * n_s;
    for (int i = threadIdx.x; i < 3 * per_plane; i += blockDim.x) {
        const int q = i / per_plane, r = i - q * per_plane;
        const int a = r / (TE * n_s), bb = (r / n_s) % TE, k = r % n_s;
        // plane_x: axes (y, z); plane_y: (x, z); plane_z: (x, y)
        const int axis_a = q == 0 ? 1 : 0, axis_b = q == 2 ? 1 : 2;
        const Tap ta = plane_tap(offs[axis_a] * 8.0 + ((double)a + 0.5) * 0.5);
        const Tap tb = plane_tap(offs[axis_b] * 8.0 + ((double)bb + 0.5) * 0.5);
        const float* P = planes + ((int64_t)parent * 3 + q) * per_plane;
        const double v00 = P[(ta.a0 * TE + tb.a0) * n_s + k], v01 = P[(ta.a0 * TE + tb.a0 + 1) * n_s + k];
        const double v10 = P[((ta.a0 + 1) * TE + tb.a0) * n_s + k], v11 = P[((ta.a0 + 1) * TE + tb.a0 + 1) * n_s + k];
        const double fa = ta.f, fb = tb.f;
        const double v = dadd(dmul(dsub(1.0, fa), dadd(dmul(dsub(1.0, fb), v00), dmul(fb, v01))),
                              dmul(fa, dadd(dmul(dsub(1.0, fb), v10), dmul(fb, v11))));
        planes_new[((int64_t)t * 3 + q) * per_plane + r] = (float)v;
    }
}

// Probe coefficients on the twice-as-dense lattice (grid.cpp:325-345):
// weighted over the existing parent-lattice neighbours, renormalised.
__global__ void __launch_bounds__(128) subdiv_probes_kernel(const int32_t* __restrict__ probe_table,
                                                            int3 pdim, const float* __restrict__ probes,
                                                            int stride, const int4* __restrict__ coords_new,
                                                            int n_new, float* __restrict__ probes_new) {
    const int p = blockIdx.x;
    if (p >= n_new) return;
    const int4 gc = __ldg(coords_new + p);
    int ids[8];
    double ws[8];
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int gx = gc.x / 2 + ((gc.x & 1) ? (i & 1) : 0);
        const int gy = gc.y / 2 + ((gc.y & 1) ? ((i >> 1) & 1) : 0);
        const int gz = gc.z / 2 + ((gc.z & 1) ? ((i >> 2) & 1) : 0);
        const double w = dmul(dmul((gc.x & 1) ? 0.5 : ((i & 1) ? 0.0 : 1.0),
                                   (gc.y & 1) ? 0.5 : ((i & 2) ? 0.0 : 1.0)),
                              (gc.z & 1) ? 0.5 : ((i & 4) ? 0.0 : 1.0));
        ids[i] = -1;
        ws[i] = 0.0;
        if (w == 0.0) continue;
        if (gx < 0 || gy < 0 || gz < 0 || gx >= pdim.x || gy >= pdim.y || gz >= pdim.z) continue;
        const int opi = __ldg(probe_table + ((int64_t)gx * pdim.y + gy) * pdim.z + gz);
        if (opi < 0) continue;
        total = dadd(total, w);
        ids[i] = opi;
        ws[i] = w;
    }
    for (int q = threadIdx.x; q < stride; q += blockDim.x) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (ids[i] >= 0) acc = dadd(acc, dmul(ws[i], (double)__ldg(probes + (int64_t)ids[i] * stride + q)));
        probes_new[(int64_t)p * stride + q] = (float)(total > 0.0 ? ddiv(acc, total) : acc);
    }
}

}  // namespace psdf

namespace psdf {

// ------------------------------------------------------------ visual hull
// init_grid_visual_hull (grid.cpp:470-504) on the device:
// occupancy by projection into every mask, two exact squared EDTs
// (Felzenszwalb, grid.cpp:400-468), the seed SDF, and init_common's
// allocation decision (grid.cpp:358-397) per tile.  f64 in the reference's
// operation order throughout, so occupancy, distances and decisions are the
// reference's bit for bit.

// voxel (x, y, z) -> index (x * ry + y) * rz + z, as the reference's idx
__global__ void __launch_bounds__(256) hull_occ_kernel(const Cam* __restrict__ cams,
                                                       const uint8_t* const* __restrict__ masks, int n_cams,
                                                       int3 res, double3 org, double h,
                                                       uint8_t* __restrict__ occ) {
    const int64_t n = (int64_t)res.x * res.y * res.z;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(i % res.z), y = (int)((i / res.z) % res.y), x = (int)(i / ((int64_t)res.y * res.z));
        const double p[3] = {dadd(org.x, dmul((double)x + 0.5, h)), dadd(org.y, dmul((double)y + 0.5, h)),
                             dadd(org.z, dmul((double)z + 0.5, h))};
        uint8_t o = 1;
        for (int c = 0; c < n_cams; ++c) {
            const Cam& k = cams[c];
            // Camera::project (camera.hpp:38-44): rotate_inv(p - pos)
            const double d[3] = {dsub(p[0], k.pos[0]), dsub(p[1], k.pos[1]), dsub(p[2], k.pos[2])};
            const double cx = dadd(dadd(dmul(k.rot[0], d[0]), dmul(k.rot[3], d[1])), dmul(k.rot[6], d[2]));
            const double cy = dadd(dadd(dmul(k.rot[1], d[0]), dmul(k.rot[4], d[1])), dmul(k.rot[7], d[2]));
            const double cz = dadd(dadd(dmul(k.rot[2], d[0]), dmul(k.rot[5], d[1])), dmul(k.rot[8], d[2]));
            bool fg = false;
            if (cz > 1e-9) {
                const double u = dadd(ddiv(dmul(k.fx, cx), cz), k.cx);
                const double v = dadd(ddiv(dmul(k.fy, cy), cz), k.cy);
                const long lu = lround(u), lv = lround(v);  // MaskImage::foreground (grid.hpp:143-146)
                fg = lu >= 0 && lv >= 0 && lu < k.width && lv < k.height &&
                     __ldg(masks[c] + (size_t)lv * k.width + lu) > 127;
            }
            if (!fg) {
                o = 0;
                break;
            }
        }
        occ[i] = o;
    }
}

// One pass of edt3d (grid.cpp:430-468): dt1d along every line of `n` elements
// at `stride` (line l starts at base(l)); one thread per line, the lower
// envelope in global scratch interleaved across the batch's lines.
struct EdtLines {
    int n_lines, n, stride;
    int64_t step_a, step_b;  // line l = (la, lb): base = la * step_a + lb * step_b
    int n_b;
};
__global__ void __launch_bounds__(128) edt_pass_kernel(double* __restrict__ d, EdtLines L, int line0, int n_batch,
                                                       double* __restrict__ fbuf, int* __restrict__ vbuf,
                                                       double* __restrict__ zbuf) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_batch || line0 + t >= L.n_lines) return;
    const int l = line0 + t;
    double* line = d + (int64_t)(l / L.n_b) * L.step_a + (int64_t)(l % L.n_b) * L.step_b;
    const int n = L.n;
    // scratch interleaved across the batch (element q of every line's copy
    // adjacent): the lock-step f[q] loads / stores of a warp coalesce
    const int64_t nb = n_batch;
    double* f = fbuf + t;
    int* v = vbuf + t;
    double* z = zbuf + t;
    for (int q = 0; q < n; ++q) f[q * nb] = line[(int64_t)q * L.stride];
    // Felzenszwalb 1D squared distance transform (grid.cpp:400-427)
    int k = 0;
    v[0] = 0;
    z[0] = -INFINITY;
    z[nb] = INFINITY;
    for (int q = 1; q < n; ++q) {
        double s;
        const double fq = dadd(f[q * nb], (double)(q * q));
        for (;;) {
            const int vk = v[k * nb];
            s = ddiv(dsub(fq, dadd(f[vk * nb], (double)(vk * vk))), dsub(dmul(2.0, (double)q), dmul(2.0, (double)vk)));
            if (s <= z[k * nb]) --k;
            else break;
        }
        ++k;
        v[k * nb] = q;
        z[k * nb] = s;
        z[(k + 1) * nb] = INFINITY;
    }
    k = 0;
    for (int q = 0; q < n; ++q) {
        while (z[(k + 1) * nb] < (double)q) ++k;
        const int vk = v[k * nb];
        const int dq = q - vk;
        line[(int64_t)q * L.stride] = dadd(dmul((double)dq, (double)dq), f[vk * nb]);
    }
}

// planes of freshly allocated tiles (allocate_tile, grid.cpp:66-69): `value`
// in the first `hs` of every `ks` channels, zero in padded ones
__global__ void __launch_bounds__(256) plane_fill_kernel(float* __restrict__ p, int64_t n, int ks, int hs,
                                                         float value) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int)(i % ks) < hs ? value : 0.f;
}

__global__ void __launch_bounds__(256) edt_init_kernel(const uint8_t* __restrict__ occ, int64_t n, int want,
                                                       double* __restrict__ d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (occ[i] != 0) == (want != 0) ? 0.0 : 1e18;  // edt3d: the `inside` set is at distance 0
}

// The seed SDF of every voxel of tile (tx, ty, tz) and init_common's
// allocation decision (grid.cpp:376-393): raw in tile layout, keep flag.
__global__ void __launch_bounds__(256) hull_tiles_kernel(const double* __restrict__ d_occ,
                                                         const double* __restrict__ d_free, int3 res, double h,
                                                         double max_s, double band, float* __restrict__ raw,
                                                         uint8_t* __restrict__ keep) {
    const int nty = res.y / TE, ntz = res.z / TE;
    const int t = blockIdx.x;
    const int tx = t / (nty * ntz), ty = (t / ntz) % nty, tz = t % ntz;
    double mn = 1.79769313486231570e308;
    int fl = 0;
    for (int i = threadIdx.x; i < TV; i += blockDim.x) {
        const int x = tx * TE + (i >> 8), y = ty * TE + ((i >> 4) & 15), z = tz * TE + (i & 15);
        const int64_t j = ((int64_t)x * res.y + y) * res.z + z;
        const double a = d_occ[j] < 1e12 ? d_occ[j] : 1e12, b = d_free[j] < 1e12 ? d_free[j] : 1e12;
        double s = dmul(dsub(dsqrt(a), dsqrt(b)), h);
        s = fmin(fmax(s, -max_s), max_s);  // clampd (vec.hpp:63)
        raw[(int64_t)t * TV + i] = (float)s;
        mn = fmin(mn, fabs(s));
        fl |= s >= 0.0 ? 1 : 2;
    }
    __shared__ double s_mn[8];
    __shared__ int s_fl[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_mn[threadIdx.x >> 5] = mn;
        s_fl[threadIdx.x >> 5] = fl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mn = fmin(mn, s_mn[w]);
            fl |= s_fl[w];
        }
        keep[t] = (mn > band && fl != 3) ? 0 : 1;
    }
}

}  // namespace psdf
