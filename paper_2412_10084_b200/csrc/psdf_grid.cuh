// psdf_grid.cuh — per-tile grid kernels of the train step.
//
//  K9 smooth / K7 fold : SparseGrid::smooth_all (grid.cpp:204-250) and
//                        finalize_smooth_grads (grads.cpp:67-96) share one
//                        separable 5-tap kernel over a 20^3 shared-memory
//                        halo.  Smoothing fills missing voxels with the far
//                        field; the G^T fold fills them with 0 (the reference
//                        skips unallocated / out-of-range taps, and the
//                        Gaussian is symmetric, so G^T is the same stencil).
//  K3 loss_sdf         : losses.cpp:121-142, element-wise.
//  K4 eikonal + normal : losses.cpp:144-220 on a 20^3 halo (TileHalo,
//                        losses.cpp:61-117) in an atomic-free gather form;
//                        halo cells belong to neighbour tiles and are
//                        flushed with global atomics.
//  K5 loss_features    : losses.cpp:222-257, one block per tile plane set.
//  K6 loss_probes      : losses.cpp:259-283 over the probe lattice table.
//  K8 adam             : Optimizer::step / AdamState::step
//                        (trainer.cpp:53-70, adam.hpp:28-37), one fused pass
//                        over the flat [raw | planes | probes | mlp] buffer.
// Loss values accumulate in f64 (stats[]); per-voxel arithmetic is fp32.
#pragma once

#include "psdf_device.cuh"

namespace psdf {

constexpr int HE = 20;           // 16 + 2 * kSmoothRadius
constexpr int HV = HE * HE * HE;  // 8000

struct GridMut {
    GridView g;
    const float* raw;
    const int32_t* probe_table;  // [(nt0+1)][(nt1+1)][(nt2+1)] -> probe or -1
    const int4* probe_coords;    // [P]
};

__device__ __forceinline__ int hidx(int x, int y, int z) { return (x * HE + y) * HE + z; }

// Gaussian taps of grid.cpp:10-22 (sigma = 1, radius 2, normalised), computed
// on the host in f64 and passed as fp32.
struct Taps {
    float w[5];
};

// The 27 neighbour tile ids of tile t (g.tile_nbr, -1 = unallocated or
// outside the grid) into shared memory; call before a __syncthreads.
__device__ __forceinline__ void stage_nbr(const GridView& g, int t, int* nb) {
    if (threadIdx.x < 27) nb[threadIdx.x] = __ldg(g.tile_nbr + (int64_t)t * 27 + threadIdx.x);
}

// Cube of E^3 voxels around a tile, local voxel coordinates [LO, LO + E) per
// axis (tile voxels are [0, 16)), from the per-tile array `src`; voxels of
// unallocated tiles or outside the grid get `fill`.  With `alloc` (one bit
// per cell, E^3 / 32 words) the allocation mask is recorded too.  Loads are
// issued four at a time (no dependent table lookups: the neighbour ids are
// in shared memory).
template <int E, int LO>
__device__ __forceinline__ void load_region(const float* __restrict__ src, const int* nb, float fill,
                                            float* __restrict__ buf, uint32_t* __restrict__ alloc) {
    constexpr int N = E * E * E;
    const int step = blockDim.x;
    for (int i0 = threadIdx.x; i0 < N; i0 += 4 * step) {
        float v[4];
        bool in[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * step;
            v[k] = fill;
            in[k] = false;
            if (i < N) {
                const int lx = i / (E * E) + LO, ly = (i / E) % E + LO, lz = i % E + LO;
                const int n = nb[((lx >> 4) + 1) * 9 + ((ly >> 4) + 1) * 3 + (lz >> 4) + 1];
                if (n >= 0) {
                    v[k] = __ldg(src + (int64_t)n * TV + vox_index(lx & 15, ly & 15, lz & 15));
                    in[k] = true;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * step;
            if (alloc) {
                const unsigned m = __ballot_sync(0xffffffffu, in[k]);
                if ((threadIdx.x & 31) == 0 && i < N) alloc[i >> 5] = m;
            }
            if (i < N) buf[i] = v[k];
        }
    }
}

__device__ __forceinline__ bool bit_at(const uint32_t* bits, int i) { return (bits[i >> 5] >> (i & 31)) & 1u; }

// One separable 5-tap pass along a column: out[o * os] = sum_d w[d] in[(o + d) * is],
// o in [0, NO), with the NO + 4 inputs held in registers (one load per input
// instead of five per output).  Summation order d = 0..4 (same fp32 value
// whichever block computes the voxel).
template <int NO>
__device__ __forceinline__ void column_5tap(const float* __restrict__ in, int is, float* __restrict__ out,
                                            int os, const Taps& taps) {
    float v[NO + 4];
#pragma unroll
    for (int k = 0; k < NO + 4; ++k) v[k] = in[k * is];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < 5; ++d) s += taps.w[d] * v[o + d];
        out[o * os] = s;
    }
}

// K7: the G^T fold (grads.cpp:67-96): dst[t] += G * src over a 20^3 halo of
// src filled with 0 (the reference skips unallocated / out-of-range taps, and
// the Gaussian is symmetric, so G^T is the same stencil).  Separable 5-tap
// column passes in shared memory.
constexpr int FZ = HE + 1;  // padded z stride of the y-pass output (conflict-free z columns)
#ifndef PSDF_FOLD_THREADS
#define PSDF_FOLD_THREADS 512
#endif
__global__ void __launch_bounds__(PSDF_FOLD_THREADS) smooth_fold_kernel(GridView g, const float* __restrict__ src,
                                                          float fill, float* __restrict__ dst,
                                                          int accumulate, Taps taps) {
    extern __shared__ __align__(16) float sh[];
    __shared__ int nb[27];
    float* A = sh;           // [20][20][20] halo; later [16][16][21] after the y pass
    float* B = sh + HV;      // [16][20][20] after the x pass
    const int t = blockIdx.x;
    stage_nbr(g, t, nb);
    __syncthreads();
    load_region<HE, -2>(src, nb, fill, A, nullptr);
    __syncthreads();
    for (int c = threadIdx.x; c < HE * HE; c += blockDim.x)  // x pass, column (y, z)
        column_5tap<16>(A + c, HE * HE, B + c, HE * HE, taps);
    __syncthreads();
    for (int c = threadIdx.x; c < 16 * HE; c += blockDim.x) {  // y pass, column (x, z)
        const int x = c / HE, z = c % HE;
        column_5tap<16>(B + x * HE * HE + z, HE, A + x * 16 * FZ + z, FZ, taps);
    }
    __syncthreads();
    float* out = dst + (int64_t)t * TV;
    if (threadIdx.x < 256) {  // z pass, column (x, y): 16 consecutive voxels of the tile
        const int c = threadIdx.x;  // 256 columns
        float r[16];
        column_5tap<16>(A + c * FZ, 1, r, 1, taps);
        float4* o4 = reinterpret_cast<float4*>(out + c * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float4 v = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
            if (accumulate) {
                const float4 o = o4[q];
                v.x += o.x;
                v.y += o.y;
                v.z += o.z;
                v.w += o.w;
            }
            o4[q] = v;
        }
    }
}
constexpr size_t kFoldSmem = sizeof(float) * (HV + 16 * HE * HE);

// K9: SparseGrid::smooth_all (grid.cpp:204-250) fused with the samplers'
// apron copy.  The tile's smoothed values AND its 1-voxel apron (18^3, the
// neighbours' smoothed values or the far field where the neighbour tile is
// unallocated / outside the grid) come from one 22^3 raw halo, so no second
// pass over the smoothed grid is needed; every smoothed value is the same
// fp32 expression (same taps, same summation order) whichever tile's block
// computes it.
constexpr int SE = 22;  // raw halo edge: local voxels [-3, 19)
constexpr int SZ = SE + 1;  // padded z stride of the y-pass output
constexpr size_t kSmoothApronSmem = sizeof(float) * (SE * SE * SE + AE * SE * SE);
#ifndef PSDF_SMOOTH_THREADS
#define PSDF_SMOOTH_THREADS 1024
#endif
__global__ void __launch_bounds__(PSDF_SMOOTH_THREADS) smooth_apron_kernel(GridView g, const float* __restrict__ raw,
                                                           float fill, float* __restrict__ smooth,
                                                           float* __restrict__ ap, Taps taps) {
    extern __shared__ __align__(16) float sh[];
    __shared__ int nb[27];
    float* A = sh;                  // [22][22][22] raw halo; later [18][18][23]
    float* B = sh + SE * SE * SE;   // [18][22][22] after the x pass; later the 18^3 apron
    const int t = blockIdx.x;
    stage_nbr(g, t, nb);
    __syncthreads();
    load_region<SE, -3>(raw, nb, fill, A, nullptr);
    __syncthreads();
    for (int c = threadIdx.x; c < SE * SE; c += blockDim.x)  // x pass, column (y, z)
        column_5tap<AE>(A + c, SE * SE, B + c, SE * SE, taps);
    __syncthreads();
    for (int c = threadIdx.x; c < AE * SE; c += blockDim.x) {  // y pass, column (x, z)
        const int x = c / SE, z = c % SE;
        column_5tap<AE>(B + x * SE * SE + z, SE, A + x * AE * SZ + z, SZ, taps);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < AE * AE; c += blockDim.x)  // z pass, column (x, y)
        column_5tap<AE>(A + c * SZ, 1, B + c * AE, 1, taps);
    __syncthreads();
    float* apt = ap + (int64_t)t * AV;
    float* sm = smooth + (int64_t)t * TV;
    for (int i = threadIdx.x; i < AV; i += blockDim.x) {
        const int x = i / (AE * AE), y = (i / AE) % AE, z = i % AE;  // local voxel = (x,y,z) - 1
        float s = B[i];
        const int lx = x - 1, ly = y - 1, lz = z - 1;
        const bool own = (unsigned)lx < 16u && (unsigned)ly < 16u && (unsigned)lz < 16u;
        if (own) {
            sm[vox_index(lx, ly, lz)] = s;
        } else if (nb[((lx >> 4) + 1) * 9 + ((ly >> 4) + 1) * 3 + (lz >> 4) + 1] < 0) {
            s = (float)g.far;  // smooth_value (grid.cpp:87-94)
        }
        apt[i] = s;
    }
}

// The apron copy from an already smoothed grid: used when the host uploads
// its own smoothed values (psdf_upload_grid with `smooth`).
__global__ void __launch_bounds__(256) apron_fill_kernel(GridView g, const float* __restrict__ smooth,
                                                         float* __restrict__ ap) {
    __shared__ float B[AV];
    __shared__ int nb[27];
    const int t = blockIdx.x;
    stage_nbr(g, t, nb);
    __syncthreads();
    load_region<AE, -1>(smooth, nb, (float)g.far, B, nullptr);
    __syncthreads();
    float* apt = ap + (int64_t)t * AV;
    for (int i = threadIdx.x; i < AV; i += blockDim.x) apt[i] = B[i];
}

// Saturation distances for one ray pass (its tau), per trilinear cell: cell b
// of tile t (b in [-1, 15]^3, index b + 1 over 17^3) holds the samples whose
// eight corners are voxels b .. b + 1 (apron brick entries b + 1 .. b + 2).  A
// cell is unsaturated when tau * (minimum of its corners) < kSatX (a sample in
// it can have sigmoid < 1); the value is the exact L-inf distance, in cells,
// to the nearest unsaturated cell of the same tile (0 = the cell itself), or
// kCellNone when the tile has none.  Separable chessboard transform: 1-D
// distances along x, then min over y' of max(|y - y'|, d), then over z'.
// The marcher's saturated runs (psdf_device.cuh, Marcher::next_run) read it.
constexpr int kSatThreads = 320;  // >= 17 * 17 rows of cells
__global__ void __launch_bounds__(kSatThreads) sat_dist_kernel(GridView g, double tau, uint8_t* __restrict__ sd) {
    constexpr int E = kCellE, NR = kCellE * kCellE;  // rows (x, y) of 17 cells along z: one bit each
    constexpr uint32_t FULLROW = (1u << kCellE) - 1u;
    __shared__ __align__(16) float ap[AV];
    __shared__ uint32_t M[2][NR];
    __shared__ uint8_t out[kCellN];
    const int t = blockIdx.x, r = threadIdx.x;
    const float* src = g.smooth_ap + (int64_t)t * AV;
    static_assert(AV % 4 == 0, "apron bricks are float4 aligned");
    for (int i = threadIdx.x; i < AV / 4; i += blockDim.x)
        reinterpret_cast<float4*>(ap)[i] = __ldg(reinterpret_cast<const float4*>(src) + i);
    __syncthreads();
    // unsaturated cells of row r as a bit mask
    uint32_t m = 0;
    const int x = r / E, y = r % E;
    if (r < NR) {
        const float* p = ap + (x * AE + y) * AE;
        float c0 = fminf(fminf(p[0], p[AE]), fminf(p[AE * AE], p[AE * AE + AE]));
        for (int z = 0; z < E; ++z) {
            const float c1 = fminf(fminf(p[z + 1], p[AE + z + 1]), fminf(p[AE * AE + z + 1], p[AE * AE + AE + z + 1]));
            const float mn = fminf(c0, c1);
            const bool sat = tau > 0.0 && mn > 0.0f && dmul(tau, (double)mn) >= kSatX;
            if (!sat) m |= 1u << z;
            c0 = c1;
        }
        M[0][r] = m;
#pragma unroll
        for (int z = 0; z < E; ++z) out[r * E + z] = ((m >> z) & 1u) ? 0 : kCellNone;
    }
    uint8_t* dst = sd + (int64_t)t * kCellN;
    const int any = __syncthreads_or(m != 0);
    if (any && !__syncthreads_and(r >= NR || m == FULLROW)) {
        // L-inf (chessboard) distance = number of 3x3x3 dilations that reach the cell
        int cur = 0;
        for (int k = 1; k < E; ++k) {
            bool full = true;
            if (r < NR) {
                uint32_t n = 0;
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
                    for (int dy = -1; dy <= 1; ++dy) {
                        const int xx = x + dx, yy = y + dy;
                        if ((unsigned)xx < (unsigned)E && (unsigned)yy < (unsigned)E) n |= M[cur][xx * E + yy];
                    }
                n = (n | (n << 1) | (n >> 1)) & FULLROW;
                for (uint32_t nw = n & ~M[cur][r]; nw; nw &= nw - 1) out[r * E + __ffs(nw) - 1] = (uint8_t)k;
                M[cur ^ 1][r] = n;
                full = n == FULLROW;
            }
            cur ^= 1;
            if (__syncthreads_and(full)) break;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kCellN; i += blockDim.x) dst[i] = out[i];
}

// Block-wide sums of NV doubles, one atomic per value per block.
template <int NV>
__device__ __forceinline__ void block_add_f64v(double* const* dst, double* v, double* red) {
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) red[k * nw + w] = v[k];
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += red[threadIdx.x * nw + i];
        if (s != 0.0) atomicAdd(dst[threadIdx.x], s);
    }
}

__device__ __forceinline__ void block_add_f64(double* dst, double v, double* red) {
    double* d[1] = {dst};
    double vv[1] = {v};
    block_add_f64v<1>(d, vv, red);
}

// (x, y, z) of a flat index over an E^3 cube, advanced by a constant stride
// without divisions.
template <int E, int S>
struct Walk3 {
    static constexpr int SX = S / (E * E), SY = (S / E) % E, SZ = S % E;
    int x, y, z;
    __device__ __forceinline__ explicit Walk3(int i) : x(i / (E * E)), y((i / E) % E), z(i % E) {}
    __device__ __forceinline__ void step() {
        z += SZ;
        if (z >= E) {
            z -= E;
            ++y;
        }
        y += SY;
        if (y >= E) {
            y -= E;
            ++x;
        }
        x += SX;
    }
};

// K3 + K4: loss_sdf, loss_eikonal and loss_normal (losses.cpp:121-220) of tile
// t0 + blockIdx.x in one pass over its 20^3 smoothed halo (TileHalo,
// losses.cpp:61-117).
//
// Atomic-free gather form of the TileHalo stencil scatter: every term
// deposits a vector dg at a centre w and the stencil adds +-dg_b * inv2h at
// w -+ e_b.  Phase A stores the central-difference gradient and its inverse
// length at every centre of the tile plus its +1 shell ([2,18]^3 in halo
// coordinates); phase B sums, per centre, the vectors of all terms centred
// there (the eikonal term of w, dg1 of the normal pairs (w, w+e_a), dg2 of the
// pairs (w-e_a, w)) into registers, which then overwrite the gradients; the
// sdf term of the tile's own voxels replaces their smoothed values; phase C
// gathers the stencil at every allocated cell it reaches and flushes with
// global atomics (neighbour tiles' blocks reach the same cells).
constexpr int DE = 17;                 // centres [2, 18] in halo coordinates
constexpr int DN = DE * DE * DE;       // 4913
constexpr int LG_THREADS = 512;
constexpr int LG_PER = (DN + LG_THREADS - 1) / LG_THREADS;  // centres per thread
constexpr size_t kLossGridSmem = sizeof(float) * (HV + 4 * DN) + sizeof(uint32_t) * (HV / 32);
__global__ void __launch_bounds__(LG_THREADS, 2) loss_grid_kernel(GridView g, const float* __restrict__ raw,
                                                                 int t0, float l_sdf, float l_eik,
                                                                 float l_norm, float inv2h,
                                                                 float* __restrict__ g_smooth,
                                                                 float* __restrict__ g_raw, double* stats) {
    extern __shared__ __align__(16) float sh[];
    float* val = sh;                                    // [20^3] smoothed values (far field outside)
    float4* P = reinterpret_cast<float4*>(sh + HV);     // [17^3] (gradient, proximity weight), then D
    uint32_t* alloc = reinterpret_cast<uint32_t*>(sh + HV + 4 * DN);  // [20^3] bits
    __shared__ int nb[27];
    __shared__ double red[6 * (LG_THREADS / 32)];
    const int t = t0 + blockIdx.x;
    stage_nbr(g, t, nb);
    __syncthreads();
    load_region<HE, -2>(g.smooth, nb, (float)g.far, val, alloc);
    __syncthreads();
    auto in_tile = [](int x, int y, int z) {
        return x >= 2 && x < 18 && y >= 2 && y < 18 && z >= 2 && z < 18;
    };
    auto weight = [&](int x, int y, int z) {  // proximity_weight (losses.hpp:20)
        return __frcp_rn(1.f + fabsf(val[hidx(x, y, z)]) * 5.f);
    };
    // phase A
    {
        Walk3<DE, LG_THREADS> c(threadIdx.x);
        for (int i = threadIdx.x; i < DN; i += LG_THREADS, c.step()) {
            const int x = c.x + 2, y = c.y + 2, z = c.z + 2;
            const float gx = (val[hidx(x + 1, y, z)] - val[hidx(x - 1, y, z)]) * inv2h;
            const float gy = (val[hidx(x, y + 1, z)] - val[hidx(x, y - 1, z)]) * inv2h;
            const float gz = (val[hidx(x, y, z + 1)] - val[hidx(x, y, z - 1)]) * inv2h;
            // (gradient, proximity weight): the weight once per centre; 1/|g|
            // is recomputed where needed (one rsqrt)
            P[i] = make_float4(gx, gy, gz, weight(x, y, z));
        }
    }
    __syncthreads();
    // phase B
    // sdf pl/wt, eik pl/wt, normal pl/wt: fp32 partial sums over this
    // thread's <= 30 terms, then f64 across the block (block_add_f64v)
    float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float D[LG_PER][3];
    constexpr int SX = DE * DE, SY = DE;
    {
        Walk3<DE, LG_THREADS> c(threadIdx.x);
#pragma unroll
        for (int k = 0; k < LG_PER; ++k, c.step()) {
            const int i = threadIdx.x + k * LG_THREADS;
            float dx = 0.f, dy = 0.f, dz = 0.f;
            if (i < DN) {
                const int x = c.x + 2, y = c.y + 2, z = c.z + 2;
                const float4 pc = P[i];
                const float q = pc.x * pc.x + pc.y * pc.y + pc.z * pc.z;
                const float inv = q > 0.f ? rsqrtf(q) : 0.f;
                const float len = q * inv;  // |g|
                if (in_tile(x, y, z)) {
                    const float w = pc.w;
                    const float e = len - 1.f;
                    acc[2] += l_eik * e * e;
                    acc[3] += l_eik * w * e * e;
                    if (q > 1e-24f) {  // len > 1e-12
                        const float cc = 2.f * l_eik * w * e * inv;
                        dx += cc * pc.x;
                        dy += cc * pc.y;
                        dz += cc * pc.z;
                    }
                    if (q >= 1e-16f) {  // len >= 1e-8: pairs (w, w + e_a), the dg1 side and the loss
                        const float n1x = pc.x * inv, n1y = pc.y * inv, n1z = pc.z * inv;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const int nx = x + (a == 0), ny = y + (a == 1), nz = z + (a == 2);
                            if (!bit_at(alloc, hidx(nx, ny, nz))) continue;
                            const float4 ph = P[i + (a == 0 ? SX : a == 1 ? SY : 1)];
                            const float qh = ph.x * ph.x + ph.y * ph.y + ph.z * ph.z;
                            if (qh < 1e-16f) continue;
                            const float ih = rsqrtf(qh);
                            const float ddx = ph.x * ih - n1x, ddy = ph.y * ih - n1y, ddz = ph.z * ih - n1z;
                            const float vv = ddx * ddx + ddy * ddy + ddz * ddz;
                            acc[4] += l_norm * vv;
                            acc[5] += l_norm * w * vv;
                            const float cn = 2.f * l_norm * w;
                            // dn1 = -c d ; dg1 = (dn1 - n1 (dn1 . n1)) / l1
                            const float m1x = -cn * ddx, m1y = -cn * ddy, m1z = -cn * ddz;
                            const float p1 = m1x * n1x + m1y * n1y + m1z * n1z;
                            dx += (m1x - n1x * p1) * inv;
                            dy += (m1y - n1y * p1) * inv;
                            dz += (m1z - n1z * p1) * inv;
                        }
                    }
                }
                // pairs (w - e_a, w) with w - e_a in the tile: the dg2 side
                if (q >= 1e-16f && bit_at(alloc, hidx(x, y, z))) {
                    const float n2x = pc.x * inv, n2y = pc.y * inv, n2z = pc.z * inv;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const int px = x - (a == 0), py = y - (a == 1), pz = z - (a == 2);
                        if (!in_tile(px, py, pz)) continue;
                        const float4 ph = P[i - (a == 0 ? SX : a == 1 ? SY : 1)];
                        const float qh = ph.x * ph.x + ph.y * ph.y + ph.z * ph.z;
                        if (qh < 1e-16f) continue;
                        const float ih = rsqrtf(qh);
                        const float cn = 2.f * l_norm * ph.w;
                        const float m2x = cn * (n2x - ph.x * ih), m2y = cn * (n2y - ph.y * ih),
                                    m2z = cn * (n2z - ph.z * ih);
                        const float p2 = m2x * n2x + m2y * n2y + m2z * n2z;
                        dx += (m2x - n2x * p2) * inv;
                        dy += (m2y - n2y * p2) * inv;
                        dz += (m2z - n2z * p2) * inv;
                    }
                }
            }
            D[k][0] = dx;
            D[k][1] = dy;
            D[k][2] = dz;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < LG_PER; ++k) {
        const int i = threadIdx.x + k * LG_THREADS;
        if (i < DN) P[i] = make_float4(D[k][0], D[k][1], D[k][2], 0.f);
    }
    // loss_sdf (losses.cpp:121-142) on the tile's own voxels, vectorised; the
    // smooth-side gradient replaces the voxel's smoothed value in val
    {
        const float4* r4 = reinterpret_cast<const float4*>(raw + (int64_t)t * TV);
        float4* g4 = reinterpret_cast<float4*>(g_raw + (int64_t)t * TV);
        for (int j = threadIdx.x; j < TV / 4; j += LG_THREADS) {
            const float4 r = __ldg(r4 + j);
            float4 gr = g4[j];
            const int x = (j >> 6) + 2, y = ((j >> 2) & 15) + 2, z0 = ((j & 3) << 2) + 2;
            const float* ra = &r.x;
            float* ga = &gr.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float& cell = val[hidx(x, y, z0 + k)];
                const float sv = cell;
                const float d = sv - ra[k];
                const float as = fabsf(sv), ar = fabsf(ra[k]);
                const float w = __frcp_rn((as > ar ? as : ar) + (float)kPhotoEps) * __frcp_rn(1.f + as * 5.f);
                acc[0] += l_sdf * d * d;
                acc[1] += l_sdf * w * d * d;
                const float gg = 2.f * l_sdf * w * d;
                ga[k] -= gg;
                cell = gg;
            }
            g4[j] = gr;
        }
    }
    __syncthreads();
    // phase C: cells [1, 19]^3 (everything the stencils reach)
    auto dv = [&](int x, int y, int z) -> const float4* {
        if (x < 2 || x > 18 || y < 2 || y > 18 || z < 2 || z > 18) return nullptr;
        return P + (((x - 2) * DE + (y - 2)) * DE + (z - 2));
    };
    constexpr int CE = 19;
    {
        Walk3<CE, LG_THREADS> c(threadIdx.x);
        for (int i = threadIdx.x; i < CE * CE * CE; i += LG_THREADS, c.step()) {
            const int x = c.x + 1, y = c.y + 1, z = c.z + 1;
            if (!bit_at(alloc, hidx(x, y, z))) continue;
            float s = 0.f;
            const float4* p;
            if ((p = dv(x - 1, y, z))) s += p->x;
            if ((p = dv(x + 1, y, z))) s -= p->x;
            if ((p = dv(x, y - 1, z))) s += p->y;
            if ((p = dv(x, y + 1, z))) s -= p->y;
            if ((p = dv(x, y, z - 1))) s += p->z;
            if ((p = dv(x, y, z + 1))) s -= p->z;
            float gv = s * inv2h;
            if (in_tile(x, y, z)) gv += val[hidx(x, y, z)];
            if (gv == 0.f) continue;
            const int lx = x - 2, ly = y - 2, lz = z - 2;
            const int n = nb[((lx >> 4) + 1) * 9 + ((ly >> 4) + 1) * 3 + (lz >> 4) + 1];
            atomicAdd(g_smooth + (int64_t)n * TV + vox_index(lx & 15, ly & 15, lz & 15), gv);
        }
    }
    double* dst[6] = {stats + 3, stats + 8, stats + 4, stats + 9, stats + 5, stats + 10};
    double accd[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) accd[k] = (double)acc[k];
    block_add_f64v<6>(dst, accd, red);
}

// K5: loss_features (losses.cpp:222-257); block = one (tile, plane), thread =
// one texel with its NS channels, gathering the pair terms it belongs to (one
// atomic per texel channel: the ray pass may scatter into the same planes
// concurrently).
template <int NS>
__global__ void __launch_bounds__(256) loss_features_kernel(GridView g, int t0, float lambda,
                                                            float* __restrict__ g_planes,
                                                            double* stats) {
    __shared__ __align__(16) float pl[256 * NS];
    __shared__ double red[16];  // block_add_f64v<2>: 2 values x 8 warps
    const int t = t0 + blockIdx.x / 3, q = blockIdx.x % 3;
    const float* p = g.planes + ((int64_t)t * 3 + q) * 256 * NS;
    float* gp = g_planes + ((int64_t)t * 3 + q) * 256 * NS;
    for (int i = threadIdx.x; i < 64 * NS; i += blockDim.x)
        reinterpret_cast<float4*>(pl)[i] = __ldg(reinterpret_cast<const float4*>(p) + i);
    __syncthreads();
    const int ab = threadIdx.x, a = ab >> 4, b = ab & 15;
    float pw = 0.f, ww = 0.f;  // this texel's share of the loss (pairs it starts)
    float gsum[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) gsum[k] = 0.f;
    auto pair = [&](int i0, int i1, bool starts, float sign) {
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const float v0 = pl[i0 * NS + k], v1 = pl[i1 * NS + k];
            const float d = v1 - v0;
            const float a0 = fabsf(v0), a1 = fabsf(v1);
            const float w = __frcp_rn((a0 > a1 ? a0 : a1) + (float)kPhotoEps);
            if (starts) {
                pw += lambda * d * d;
                ww += lambda * w * d * d;
            }
            gsum[k] += sign * 2.f * lambda * w * d;
        }
    };
    if (a + 1 < 16) pair(ab, ab + 16, true, -1.f);   // pair (i0, (a+1, b)): loss counted here, -g to i0
    if (b + 1 < 16) pair(ab, ab + 1, true, -1.f);    // pair (i0, (a, b+1))
    if (a >= 1) pair(ab - 16, ab, false, 1.f);       // pair ((a-1, b), i0): +g to i0
    if (b >= 1) pair(ab - 1, ab, false, 1.f);        // pair ((a, b-1), i0)
    // atomic (the kernel may run beside the ray pass's plane-gradient
    // scatters), one vector reduction per texel
    bool any = false;
#pragma unroll
    for (int k = 0; k < NS; ++k) any |= gsum[k] != 0.f;
    if (any) red_vec<NS>(gp + ab * NS, gsum);
    double* dst[2] = {stats + 6, stats + 11};
    double v2[2] = {(double)pw, (double)ww};
    block_add_f64v<2>(dst, v2, red);
}

// K6: loss_probes (losses.cpp:259-283) over probes [p0, p1); one thread per
// (probe, coefficient).
__global__ void __launch_bounds__(256) loss_probes_kernel(GridMut m, int p0, int p1, int stride,
                                                          float lambda,
                                                          float* __restrict__ g_probes,
                                                          double* stats) {
    __shared__ double red[8];
    const GridView& g = m.g;
    const int64_t n = (int64_t)(p1 - p0) * stride;
    double pl = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int pi = p0 + (int)(i / stride), c = (int)(i % stride);
        const int4 pc = __ldg(m.probe_coords + pi);
        const float b1 = g.probes[(int64_t)pi * stride + c];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int qx = pc.x + (a == 0), qy = pc.y + (a == 1), qz = pc.z + (a == 2);
            if (qx > g.nt[0] || qy > g.nt[1] || qz > g.nt[2]) continue;
            const int qi =
                __ldg(m.probe_table + ((int64_t)qx * (g.nt[1] + 1) + qy) * (g.nt[2] + 1) + qz);
            if (qi < 0) continue;
            const float d = b1 - g.probes[(int64_t)qi * stride + c];
            pl += (double)(lambda * d * d);
            const float gg = 2.f * lambda * d;
            atomicAdd(g_probes + (int64_t)pi * stride + c, gg);
            atomicAdd(g_probes + (int64_t)qi * stride + c, -gg);
        }
    }
    block_add_f64(stats + 7, pl, red);
}

// K8: Adam over the flat parameter buffer; [0, n_vox) uses lr_vox, the rest
// lr_mlp.  c1 = 1 - beta1^t, c2 = 1 - beta2^t precomputed on the host in f64.
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p,
                                                   const float* __restrict__ gr,
                                                   float* __restrict__ m, float* __restrict__ v,
                                                   int64_t n, int64_t n_vox, float lr_vox,
                                                   float lr_mlp, float inv_c1, float inv_c2,
                                                   const unsigned long long* __restrict__ skip) {
    if (*skip) return;  // the ray pass overflowed a buffer: the step is redone
    const float b1 = 0.9f, b2 = 0.995f, eps = 1e-8f;
    const int64_t n4 = n >> 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        float4 pp = reinterpret_cast<float4*>(p)[i];
        const float4 gg = reinterpret_cast<const float4*>(gr)[i];
        float4 mm = reinterpret_cast<float4*>(m)[i];
        float4 vv = reinterpret_cast<float4*>(v)[i];
        float* pa = &pp.x;
        const float* ga = &gg.x;
        float* ma = &mm.x;
        float* va = &vv.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t e = 4 * i + k;
            const float lr = e < n_vox ? lr_vox : lr_mlp;
            ma[k] = b1 * ma[k] + (1.f - b1) * ga[k];
            va[k] = b2 * va[k] + (1.f - b2) * ga[k] * ga[k];
            pa[k] -= lr * (ma[k] * inv_c1) / (sqrtf(va[k] * inv_c2) + eps);
        }
        reinterpret_cast<float4*>(p)[i] = pp;
        reinterpret_cast<float4*>(m)[i] = mm;
        reinterpret_cast<float4*>(v)[i] = vv;
    }
    // tail
    for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const float lr = e < n_vox ? lr_vox : lr_mlp;
        m[e] = b1 * m[e] + (1.f - b1) * gr[e];
        v[e] = b2 * v[e] + (1.f - b2) * gr[e] * gr[e];
        p[e] -= lr * (m[e] * inv_c1) / (sqrtf(v[e] * inv_c2) + eps);
    }
}

}  // namespace psdf
