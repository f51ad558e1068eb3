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

// Loads a 20^3 halo of `src` around tile t; missing voxels get `fill`.
// Optionally records the allocation mask.
__device__ __forceinline__ void load_halo(const GridView& g, const float* __restrict__ src, int t,
                                          float fill, float* __restrict__ buf,
                                          unsigned char* __restrict__ alloc) {
    const int4 tc = __ldg(g.tile_coords + t);
    const int ox = tc.x * TE - 2, oy = tc.y * TE - 2, oz = tc.z * TE - 2;
    for (int i = threadIdx.x; i < HV; i += blockDim.x) {
        const int x = i / (HE * HE), y = (i / HE) % HE, z = i % HE;
        const int vx = ox + x, vy = oy + y, vz = oz + z;
        float v = fill;
        bool in = false;
        if (vx >= 0 && vy >= 0 && vz >= 0 && vx < g.res[0] && vy < g.res[1] && vz < g.res[2]) {
            const int nt = tile_lookup(g, vx >> 4, vy >> 4, vz >> 4);
            if (nt >= 0) {
                v = __ldg(src + (int64_t)nt * TV + vox_index(vx & 15, vy & 15, vz & 15));
                in = true;
            }
        }
        buf[i] = v;
        if (alloc) alloc[i] = in;
    }
}

// Separable 5-tap pass over the halo: out(tile voxels) = G * halo.
// mode 0: dst[t] = result (smoothing); mode 1: dst[t] += result (fold).
__global__ void __launch_bounds__(256) smooth_fold_kernel(GridView g, const float* __restrict__ src,
                                                          float fill, float* __restrict__ dst,
                                                          int accumulate, Taps taps) {
    extern __shared__ __align__(16) float sh[];
    float* A = sh;           // [20][20][20]
    float* B = sh + HV;      // [16][20][20] after the x pass
    const int t = blockIdx.x;
    load_halo(g, src, t, fill, A, nullptr);
    __syncthreads();
    // x pass: B[x][y][z] = sum_d w[d] A[x+d+2][y][z], x in [0,16)
    for (int i = threadIdx.x; i < 16 * HE * HE; i += blockDim.x) {
        const int x = i / (HE * HE), yz = i % (HE * HE);
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < 5; ++d) s += taps.w[d] * A[(x + d) * HE * HE + yz];
        B[i] = s;
    }
    __syncthreads();
    // y pass: A'[x][y][z] = sum_d w[d] B[x][y+d][z], y in [0,16)  (reuse A as [16][16][20])
    for (int i = threadIdx.x; i < 16 * 16 * HE; i += blockDim.x) {
        const int x = i / (16 * HE), y = (i / HE) % 16, z = i % HE;
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < 5; ++d) s += taps.w[d] * B[(x * HE + y + d) * HE + z];
        A[i] = s;
    }
    __syncthreads();
    // z pass into the tile
    float* out = dst + (int64_t)t * TV;
    for (int i = threadIdx.x; i < TV; i += blockDim.x) {
        const int x = i >> 8, y = (i >> 4) & 15, z = i & 15;
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < 5; ++d) s += taps.w[d] * A[(x * 16 + y) * HE + z + d];
        if (accumulate)
            out[i] += s;
        else
            out[i] = s;
    }
}

// Apron copy of the smoothed SDF (psdf_device.cuh, sample_sdf_in): cell
// (x, y, z) in [-1, 16]^3 of tile t holds smooth_value at that global voxel,
// i.e. the owning tile's value or the far field.
__global__ void __launch_bounds__(256) apron_fill_kernel(GridView g, const float* __restrict__ smooth,
                                                         float* __restrict__ ap) {
    const int t = blockIdx.x;
    const int4 tc = __ldg(g.tile_coords + t);
    for (int i = threadIdx.x; i < AV; i += blockDim.x) {
        const int x = i / (AE * AE) - 1, y = (i / AE) % AE - 1, z = i % AE - 1;
        const int vx = tc.x * TE + x, vy = tc.y * TE + y, vz = tc.z * TE + z;
        float v = (float)g.far;
        if ((unsigned)x < 16u && (unsigned)y < 16u && (unsigned)z < 16u) {
            v = smooth[(int64_t)t * TV + vox_index(x, y, z)];
        } else if (vx >= 0 && vy >= 0 && vz >= 0 && vx < g.res[0] && vy < g.res[1] && vz < g.res[2]) {
            const int nt = tile_lookup(g, vx >> 4, vy >> 4, vz >> 4);
            if (nt >= 0) v = smooth[(int64_t)nt * TV + vox_index(vx & 15, vy & 15, vz & 15)];
        }
        ap[(int64_t)t * AV + i] = v;
    }
}

__device__ __forceinline__ void block_add_f64(double* dst, double v, double* red) {
    // block-wide sum of one double per thread, one atomic per block
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
        if (s != 0.0) atomicAdd(dst, s);
    }
}

// K3: loss_sdf (losses.cpp:121-142) over tiles [t0, t1)
__global__ void __launch_bounds__(256) loss_sdf_kernel(GridView g, const float* __restrict__ raw,
                                                       int t0, int t1, float lambda,
                                                       float* __restrict__ g_smooth,
                                                       float* __restrict__ g_raw, double* stats) {
    __shared__ double red[8];
    const int64_t n = (int64_t)(t1 - t0) * TV;
    const int64_t base = (int64_t)t0 * TV;
    double pl = 0.0, wt = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float s = g.smooth[base + i], r = raw[base + i];
        const float d = s - r;
        const float as = fabsf(s), ar = fabsf(r);
        const float w = (1.f / ((as > ar ? as : ar) + (float)kPhotoEps)) * (1.f / (1.f + as * 5.f));
        pl += (double)(lambda * d * d);
        wt += (double)(lambda * w * d * d);
        const float gg = 2.f * lambda * w * d;
        if (gg != 0.f) {
            g_smooth[base + i] += gg;
            g_raw[base + i] -= gg;
        }
    }
    block_add_f64(stats + 3, pl, red);
    block_add_f64(stats + 8, wt, red);
}

// K4: loss_eikonal + loss_normal (losses.cpp:144-220) for tile blockIdx.x + t0.
//
// Atomic-free gather form of the TileHalo stencil scatter (losses.cpp:61-117):
// every term deposits a vector dg at a centre w and the stencil adds
// +-dg_b * inv2h at w -+ e_b.  Phase 1 sums, per centre w in the tile plus its
// +1 shell ([2,18]^3 in halo coordinates), the vectors of all terms centred
// there: the eikonal term of w, dg1 of the normal pairs (w, w+e_a) and dg2 of
// the pairs (w-e_a, w).  Phase 2 gathers the stencil at every halo cell.
constexpr int DE = 17;  // centres [2, 18] in halo coordinates
__global__ void __launch_bounds__(256) loss_eik_normal_kernel(GridView g, int t0, float l_eik,
                                                              float l_norm, float inv2h,
                                                              float* __restrict__ g_smooth,
                                                              double* stats) {
    extern __shared__ __align__(16) float sh[];
    float* val = sh;                          // [20^3] smoothed values (far field outside)
    float* D = sh + HV;                       // [17^3][3] stencil vectors per centre
    unsigned char* alloc = reinterpret_cast<unsigned char*>(sh + HV + 3 * DE * DE * DE);
    __shared__ double red[8];
    const int t = t0 + blockIdx.x;
    load_halo(g, g.smooth, t, (float)g.far, val, alloc);
    __syncthreads();
    auto grad_at = [&](int x, int y, int z, float& gx, float& gy, float& gz) {
        gx = (val[hidx(x + 1, y, z)] - val[hidx(x - 1, y, z)]) * inv2h;
        gy = (val[hidx(x, y + 1, z)] - val[hidx(x, y - 1, z)]) * inv2h;
        gz = (val[hidx(x, y, z + 1)] - val[hidx(x, y, z - 1)]) * inv2h;
    };
    auto in_tile = [](int x, int y, int z) {
        return x >= 2 && x < 18 && y >= 2 && y < 18 && z >= 2 && z < 18;
    };
    double e_pl = 0.0, e_wt = 0.0, n_pl = 0.0, n_wt = 0.0;
    for (int i = threadIdx.x; i < DE * DE * DE; i += blockDim.x) {
        const int x = i / (DE * DE) + 2, y = (i / DE) % DE + 2, z = i % DE + 2;
        float dx = 0.f, dy = 0.f, dz = 0.f;
        float gx, gy, gz;
        grad_at(x, y, z, gx, gy, gz);
        const float len = sqrtf(gx * gx + gy * gy + gz * gz);
        const bool own = in_tile(x, y, z);
        if (own) {
            const float w = 1.f / (1.f + fabsf(val[hidx(x, y, z)]) * 5.f);  // losses.hpp:20
            const float e = len - 1.f;
            e_pl += (double)(l_eik * e * e);
            e_wt += (double)(l_eik * w * e * e);
            if (len > 1e-12f) {
                const float c = 2.f * l_eik * w * e / len;
                dx += c * gx;
                dy += c * gy;
                dz += c * gz;
            }
            if (len >= 1e-8f) {  // pairs (w, w + e_a): the dg1 side, and the loss
                const float n1x = gx / len, n1y = gy / len, n1z = gz / len;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int nx = x + (a == 0), ny = y + (a == 1), nz = z + (a == 2);
                    if (!alloc[hidx(nx, ny, nz)]) continue;
                    float hx, hy, hz;
                    grad_at(nx, ny, nz, hx, hy, hz);
                    const float l2 = sqrtf(hx * hx + hy * hy + hz * hz);
                    if (l2 < 1e-8f) continue;
                    const float ddx = hx / l2 - n1x, ddy = hy / l2 - n1y, ddz = hz / l2 - n1z;
                    const float vv = ddx * ddx + ddy * ddy + ddz * ddz;
                    n_pl += (double)(l_norm * vv);
                    n_wt += (double)(l_norm * w * vv);
                    const float c = 2.f * l_norm * w;
                    // dn1 = -c d ; dg1 = (dn1 - n1 (dn1 . n1)) / l1
                    const float m1x = -c * ddx, m1y = -c * ddy, m1z = -c * ddz;
                    const float p1 = m1x * n1x + m1y * n1y + m1z * n1z;
                    dx += (m1x - n1x * p1) / len;
                    dy += (m1y - n1y * p1) / len;
                    dz += (m1z - n1z * p1) / len;
                }
            }
        }
        // pairs (w - e_a, w) with w - e_a in the tile: the dg2 side
        if (len >= 1e-8f && alloc[hidx(x, y, z)]) {
            const float n2x = gx / len, n2y = gy / len, n2z = gz / len;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int px = x - (a == 0), py = y - (a == 1), pz = z - (a == 2);
                if (!in_tile(px, py, pz)) continue;
                float hx, hy, hz;
                grad_at(px, py, pz, hx, hy, hz);
                const float l1 = sqrtf(hx * hx + hy * hy + hz * hz);
                if (l1 < 1e-8f) continue;
                const float w = 1.f / (1.f + fabsf(val[hidx(px, py, pz)]) * 5.f);
                const float c = 2.f * l_norm * w;
                const float m2x = c * (n2x - hx / l1), m2y = c * (n2y - hy / l1),
                            m2z = c * (n2z - hz / l1);
                const float p2 = m2x * n2x + m2y * n2y + m2z * n2z;
                dx += (m2x - n2x * p2) / len;
                dy += (m2y - n2y * p2) / len;
                dz += (m2z - n2z * p2) / len;
            }
        }
        D[3 * i] = dx;
        D[3 * i + 1] = dy;
        D[3 * i + 2] = dz;
    }
    __syncthreads();
    // phase 2: gather the stencils and flush (TileHalo::flush, losses.cpp:87-97)
    const int4 tc = __ldg(g.tile_coords + t);
    const int ox = tc.x * TE - 2, oy = tc.y * TE - 2, oz = tc.z * TE - 2;
    auto dval = [&](int x, int y, int z, int b) -> float {
        if (x < 2 || x > 18 || y < 2 || y > 18 || z < 2 || z > 18) return 0.f;
        return D[3 * (((x - 2) * DE + (y - 2)) * DE + (z - 2)) + b];
    };
    for (int i = threadIdx.x; i < HV; i += blockDim.x) {
        if (!alloc[i]) continue;
        const int x = i / (HE * HE), y = (i / HE) % HE, z = i % HE;
        const float gv = (dval(x - 1, y, z, 0) - dval(x + 1, y, z, 0) + dval(x, y - 1, z, 1) -
                          dval(x, y + 1, z, 1) + dval(x, y, z - 1, 2) - dval(x, y, z + 1, 2)) *
                         inv2h;
        if (gv == 0.f) continue;
        const int vx = ox + x, vy = oy + y, vz = oz + z;
        const int nt = tile_lookup(g, vx >> 4, vy >> 4, vz >> 4);
        atomicAdd(g_smooth + (int64_t)nt * TV + vox_index(vx & 15, vy & 15, vz & 15), gv);
    }
    block_add_f64(stats + 4, e_pl, red);
    block_add_f64(stats + 9, e_wt, red);
    block_add_f64(stats + 5, n_pl, red);
    block_add_f64(stats + 10, n_wt, red);
}
constexpr size_t kEikNormalSmem = sizeof(float) * (HV + 3 * DE * DE * DE) + HV;

// K5: loss_features (losses.cpp:222-257); block = one (tile, plane), one
// thread per texel channel, gathering the pair terms it belongs to (no
// atomics: the plane's gradient is owned by this block).
__global__ void __launch_bounds__(256) loss_features_kernel(GridView g, int t0, int n_s,
                                                            float lambda,
                                                            float* __restrict__ g_planes,
                                                            double* stats) {
    __shared__ double red[8];
    const int t = t0 + blockIdx.x / 3, q = blockIdx.x % 3;
    const int n = 256 * n_s;
    const float* p = g.planes + ((int64_t)t * 3 + q) * n;
    float* gp = g_planes + ((int64_t)t * 3 + q) * n;
    double pl = 0.0, wt = 0.0;
    auto term = [&](int i0, int i1, float& d, float& w) {
        d = p[i1] - p[i0];
        const float a0 = fabsf(p[i0]), a1 = fabsf(p[i1]);
        w = 1.f / ((a0 > a1 ? a0 : a1) + (float)kPhotoEps);
    };
    for (int i0 = threadIdx.x; i0 < n; i0 += blockDim.x) {
        const int ab = i0 / n_s, k = i0 % n_s, a = ab >> 4, b = ab & 15;
        float gsum = 0.f, d, w;
        if (a + 1 < 16) {  // pair (i0, (a+1, b)): loss counted here, -g to i0
            term(i0, ((a + 1) * 16 + b) * n_s + k, d, w);
            pl += (double)(lambda * d * d);
            wt += (double)(lambda * w * d * d);
            gsum -= 2.f * lambda * w * d;
        }
        if (b + 1 < 16) {  // pair (i0, (a, b+1))
            term(i0, (a * 16 + b + 1) * n_s + k, d, w);
            pl += (double)(lambda * d * d);
            wt += (double)(lambda * w * d * d);
            gsum -= 2.f * lambda * w * d;
        }
        if (a >= 1) {  // pair ((a-1, b), i0): +g to i0
            term(((a - 1) * 16 + b) * n_s + k, i0, d, w);
            gsum += 2.f * lambda * w * d;
        }
        if (b >= 1) {  // pair ((a, b-1), i0)
            term((a * 16 + b - 1) * n_s + k, i0, d, w);
            gsum += 2.f * lambda * w * d;
        }
        if (gsum != 0.f) gp[i0] += gsum;
    }
    block_add_f64(stats + 6, pl, red);
    block_add_f64(stats + 11, wt, red);
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
                                                   float lr_mlp, float inv_c1, float inv_c2) {
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
