// psdf_raypass.cuh — shared pieces of the ray pass (psdf_train.cuh):
// parameters, MLP layouts, decode_fused (renderer.cpp:88-147) as
// decode_features + mlp_forward, and the geometry record the shading
// backward reads.  K1 (render_image, renderer.cpp:321-337) runs through the
// same pipeline as the train ray pass with RayPassParams::mode = 1.
//
// Work decomposition of the march kernels: one ray per lane; a warp owns an
// 8x4 pixel tile (so its rays are coherent) and pulls tiles from a global
// work counter.  The march / alpha / compositing chain is exact f64
// (psdf_device.cuh).  Shaded samples are decoded in fp32.
//
// The backward is a second forward sweep instead of the reference's reverse
// traversal over a cached RayWorkspace: the suffix sum of renderer.cpp:254-261
// is rewritten as  suffix_i = Total - prefix_i  with
//   Total = sum_k dw_k w_k = g.(c_raw - bg*acc) + dA*acc
// known after the forward sweep, so no per-sample state is stored.  The sweep
// restarts at the first sample with alpha > 0 (samples before it have w = 0
// and contribute nothing), with T = 1 exactly.  The rounding error of the
// subtraction enters ds only multiplied by (1 - alpha_i), see DESIGN.md.
#pragma once

#include "psdf_bulk.cuh"
#include "psdf_device.cuh"

namespace psdf {

constexpr unsigned FULL = 0xffffffffu;
#ifndef PSDF_WARPS_PER_BLOCK
#define PSDF_WARPS_PER_BLOCK 4
#endif
constexpr int WARPS_PER_BLOCK = PSDF_WARPS_PER_BLOCK;
constexpr int BLOCK = 32 * WARPS_PER_BLOCK;

struct ViewDev {
    Cam cam;
    const float* gt;      // [h][w][3] (train)
    const uint8_t* mask;  // [h][w]   (train)
    int tiles_x, tiles_y;
    int64_t tile_begin;   // first global work tile of this view
    int cam_bias_row;     // camera-bias row for this view, -1 = none
    int pad_;
    // pixels whose ray can meet the allocated tiles' bounding box: the box's
    // projection, padded by 2 pixels (the whole image when the camera is not
    // in front of every box corner); rays outside yield no sample
    int occ_u0, occ_u1, occ_v0, occ_v1;
    // the work tiles (8x4 pixels) that overlap that rectangle: the scan's
    // work list is these tiles only (the others have no sample: their rays
    // are the empty-ray term, hand-over bits 0)
    int act_tx0, act_ty0, act_w, act_n;
    int64_t act_begin;    // first active tile of this view in the batch's active list
};

struct RayPassParams {
    GridView g;
    const float* mlp;     // device MLP (flat layout)
    int in_dim, ncam;
    int order;            // effective SH order (sh_order_override applied)
    int no_spatial, no_angular, no_fresnel, need_colors;
    int n_max;
    int mode;             // 0: train ray pass, 1: render (K1 through the same pipeline)
    int bits_sm_words;    // words of the tile bitmap staged in shared memory (0 = use global)
    int stage_fwd;        // K2b: bulk-copy the tiles' probe blocks into shared memory
    double tau, early_stop, bg[3];
    double photo_scale;
    const ViewDev* views;
    int n_views;
    int64_t tile_begin, tile_end;  // this rank's slice of the global work tiles
    int64_t scan_lo, scan_hi;      // K2a-scan: active-tile list range [lo, hi) (ViewDev::act_*)
    const float* tile_tmin;        // [global work tiles] lower bound on the first allocated-tile hit (kTminNone: none)
    const float* tile_tmax;        // [global work tiles] upper bound on the distance of any sample (last allocated tile)
    unsigned long long* work_counter;
    // render outputs (K1)
    float* out_rgb;
    float* out_alpha;
    float* out_depth;
    // gradients (K2)
    float* g_smooth;  // [T][4096] smooth-staged
    float* g_planes;  // [T][3][256][n_s]
    float* g_probes;  // [P][order^2][n_a]
    float* g_mlp;     // flat MLP layout
    // statistics
    double* stats;                // [0] photo plain, [1] sq_err, [2] mask_px
    unsigned long long* counts;   // psdf_counts layout
};

// MLP offsets in the flat layout (decoder.hpp:17-31).
struct MlpLayout {
    int w1, b1, w2, b2, w3, b3, cam, total_nocam;
    __host__ __device__ static MlpLayout make(int in) {
        MlpLayout m;
        m.w1 = 0;
        m.b1 = 32 * in;
        m.w2 = m.b1 + 32;
        m.b2 = m.w2 + 1024;
        m.w3 = m.b2 + 32;
        m.b3 = m.w3 + 96;
        m.cam = m.b3 + 3;
        m.total_nocam = m.cam;
        return m;
    }
};

// Shared-memory MLP copy, input-major for the paired-FMA forward (mlp_forward):
// w1t[i][j] = W1[j][i] (IN x 32), w2t[i][j] = W2[j][i] (32 x 32), rows of 32
// outputs 16-byte aligned; w3 row-major [3][32]; biases.
struct SmemMlp {
    int w1t, b1, w2t, b2, w3, b3, total;
    __host__ __device__ static SmemMlp make(int in) {
        SmemMlp s;
        s.w1t = 0;
        s.b1 = 32 * in;
        s.w2t = s.b1 + 32;
        s.b2 = s.w2t + 1024;
        s.w3 = s.b2 + 32;
        s.b3 = s.w3 + 96;
        s.total = s.b3 + 4;
        return s;
    }
};

// Per-warp scratch rows (train only).  Row strides are 4*(odd) floats so
// 128-bit row writes by 8 lanes hit distinct bank groups.
//   A1[32][RS] : a1 rows, later overwritten by dz1
//   A2[32][RS] : a2 rows, later dz2, later the probe-gradient factors
//   X [32][XS] : MLP inputs
//   D3[32][4]  : dz3
constexpr int RS = 36;
template <int IN>
struct ScratchDims {
    static constexpr int XS = ((((IN + 3) / 4) % 2) ? ((IN + 3) / 4) : ((IN + 3) / 4 + 1)) * 4;
    static constexpr int A1 = 0;
    static constexpr int A2 = A1 + 32 * RS;
    static constexpr int X = A2 + 32 * RS;
    static constexpr int D3 = X + 32 * XS;
    static constexpr int TOTAL = D3 + 32 * 4;
};

// Per-block MLP-gradient accumulator (rows padded to odd strides so lane j
// updating row j hits distinct banks).
template <int IN>
struct GAccDims {
    static constexpr int W1S = IN | 1;
    static constexpr int W1 = 0;
    static constexpr int B1 = W1 + 32 * W1S;
    static constexpr int W2 = B1 + 32;
    static constexpr int B2 = W2 + 32 * 33;
    static constexpr int W3 = B2 + 32;
    static constexpr int B3 = W3 + 96;
    static constexpr int TOTAL = ((B3 + 3) + 3) & ~3;
};

__device__ __forceinline__ float sigmoidf_(float z) { return 1.f / (1.f + __expf(-z)); }

// State of a shaded sample kept for its backward.
struct ShadeGeo {
    double n[3], glen;
    float refl[3];
    float ndv;        // n.v (raw)
    bool degenerate;
    Tap tx, ty, tz;
    float w8[8];
};

// Per-record geometry + features written by K2b for K2e (floats):
//   [0,3) normal  [3] |grad|  [4,7) refl  [7] n.v  [8,11) tap fractions
//   [11] tap a0 | degenerate flag (int bits)  [12,20) probe corner weights
//   [20, 20+3 NS) plane samples  [20+3 NS, +IN) MLP input
template <int NS, int NA>
struct GeoRec {
    static constexpr int IN = NS + NA + NPOW;
    static constexpr int PV = 20;
    static constexpr int X = PV + 3 * NS;
    static constexpr int STRIDE = (X + IN + 3) & ~3;
};

// c += a * (b, b) on a pair of fp32 lanes (FFMA2, sm_100): two outputs per
// instruction, each rounded exactly as a scalar FFMA.
__device__ __forceinline__ void ffma2(float2& c, float2 a, float b) {
    unsigned long long& cc = *reinterpret_cast<unsigned long long*>(&c);
    const float2 bb = make_float2(b, b);
    asm("fma.rn.f32x2 %0, %1, %2, %0;"
        : "+l"(cc)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&bb)));
}

// acc[k] += y * v[k] over an even channel count, two channels per FFMA2.
template <int N>
__device__ __forceinline__ void axpy_pairs(float (&acc)[N], const VecF<N>& v, float y) {
    static_assert(N % 2 == 0, "channel counts are even");
#pragma unroll
    for (int k = 0; k < N; k += 2) {
        float2 a = make_float2(acc[k], acc[k + 1]);
        ffma2(a, make_float2(v.v[k], v.v[k + 1]), y);
        acc[k] = a.x;
        acc[k + 1] = a.y;
    }
}

// decode_fused (renderer.cpp:88-147), geometry + feature part, for one sample
// at p (f64 world point); dneg = -dir = view vector toward the camera.
// Produces the MLP input x and the tri-plane samples pv.
template <int NS, int NA>
__device__ __forceinline__ void decode_features(const RayPassParams& P, int tile, const double p[3],
                                                const double dneg[3], ShadeGeo& geo,
                                                float x[NS + NA + NPOW], float pv[3][NS],
                                                const float* psm = nullptr) {
    const GridView& g = P.g;
    const double h = g.h;
    // central-difference normal of the smoothed SDF, exact f64
    const double sxp = sample_sdf(g, dadd(p[0], h), p[1], p[2]);
    const double sxm = sample_sdf(g, dsub(p[0], h), p[1], p[2]);
    const double syp = sample_sdf(g, p[0], dadd(p[1], h), p[2]);
    const double sym = sample_sdf(g, p[0], dsub(p[1], h), p[2]);
    const double szp = sample_sdf(g, p[0], p[1], dadd(p[2], h));
    const double szm = sample_sdf(g, p[0], p[1], dsub(p[2], h));
    const double h2 = dmul(2.0, h);
    // x / (2h): exact multiply for a power-of-two h (see div_h)
    const double inv2h = g.h_pow2 ? dmul(0.5, g.inv_h) : 0.0;
    auto div2h = [&](double x_) { return g.h_pow2 ? dmul(x_, inv2h) : ddiv(x_, h2); };
    const D3 gv = d3(div2h(dsub(sxp, sxm)), div2h(dsub(syp, sym)), div2h(dsub(szp, szm)));
    const double glen = dsqrt(ddot(gv, gv));
    geo.degenerate = glen < 1e-8;
    geo.glen = glen;
    const D3 v = d3(dneg[0], dneg[1], dneg[2]);
    double ndv;
    if (geo.degenerate) {
        geo.n[0] = geo.n[1] = geo.n[2] = 0.0;
        geo.refl[0] = (float)v.x;
        geo.refl[1] = (float)v.y;
        geo.refl[2] = (float)v.z;
        ndv = 1.0;
    } else {
        const D3 n = d3(ddiv(gv.x, glen), ddiv(gv.y, glen), ddiv(gv.z, glen));
        geo.n[0] = n.x;
        geo.n[1] = n.y;
        geo.n[2] = n.z;
        ndv = ddot(n, v);
        const double s2 = dmul(2.0, ndv);  // reflect_about (vec.hpp:59-61)
        geo.refl[0] = (float)dsub(dmul(n.x, s2), v.x);
        geo.refl[1] = (float)dsub(dmul(n.y, s2), v.y);
        geo.refl[2] = (float)dsub(dmul(n.z, s2), v.z);
    }
    geo.ndv = (float)ndv;
    // tile-local position (renderer.cpp:117-118)
    const int4 tc = __ldg(g.tile_coords + tile);
    const double lx = dsub(w2v(g, p[0], 0), (double)(tc.x * 16));
    const double ly = dsub(w2v(g, p[1], 1), (double)(tc.y * 16));
    const double lz = dsub(w2v(g, p[2], 2), (double)(tc.z * 16));
    geo.tx = plane_tap(lx);
    geo.ty = plane_tap(ly);
    geo.tz = plane_tap(lz);
    {  // trilinear_weights(local/16) (sh.cpp:172-181); /16 is an exact multiply
        const double fx = dmul(lx, 0.0625), fy = dmul(ly, 0.0625), fz = dmul(lz, 0.0625);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            geo.w8[i] = (float)dmul(dmul((i & 1) ? fx : dsub(1.0, fx), (i & 2) ? fy : dsub(1.0, fy)),
                                    (i & 4) ? fz : dsub(1.0, fz));
    }
#pragma unroll
    for (int k = 0; k < NS + NA; ++k) x[k] = 0.f;
    // F_s: channel-wise tri-plane product (grid.cpp:179-187)
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int k = 0; k < NS; ++k) pv[q][k] = 0.f;
    if (!P.no_spatial) {
        const float* pl = g.planes + (int64_t)tile * 3 * 256 * NS;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const Tap ta = q == 0 ? geo.ty : geo.tx;
            const Tap tb = q == 2 ? geo.ty : geo.tz;
            const float* base = pl + q * 256 * NS;
            const VecF<NS> v00 = ldg_vec<NS>(base + (ta.a0 * TE + tb.a0) * NS);
            const VecF<NS> v01 = ldg_vec<NS>(base + (ta.a0 * TE + tb.a0 + 1) * NS);
            const VecF<NS> v10 = ldg_vec<NS>(base + ((ta.a0 + 1) * TE + tb.a0) * NS);
            const VecF<NS> v11 = ldg_vec<NS>(base + ((ta.a0 + 1) * TE + tb.a0 + 1) * NS);
#pragma unroll
            for (int k = 0; k < NS; ++k)
                pv[q][k] = (1.f - ta.f) * ((1.f - tb.f) * v00.v[k] + tb.f * v01.v[k]) +
                           ta.f * ((1.f - tb.f) * v10.v[k] + tb.f * v11.v[k]);
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) x[k] = pv[0][k] * pv[1][k] * pv[2][k];
    }
    // F_a: coefficient-blended probes evaluated along refl (sh.cpp:104-123)
    if (!P.no_angular) {
        float Y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) Y[j] = 0.f;
        sh_basis(geo.refl[0], geo.refl[1], geo.refl[2], P.order, Y);
        const int nc = P.order * P.order;
        const int stride = g.order * g.order * NA;
        const int32_t* pid = g.probe_ids + (int64_t)tile * 8;
        // psm: the tile's 8 probe blocks staged in shared memory (ProbeStage)
#pragma unroll 1
        for (int i = 0; i < 8; ++i) {
            const float w = geo.w8[i];
            if (w == 0.f) continue;
            float acc[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) acc[k] = 0.f;
            if (psm) {
                const float* c = psm + i * stride;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j < nc) {
                        axpy_pairs<NA>(acc, lds_vec<NA>(c + j * NA), Y[j]);
                    }
                }
            } else {
                const float* c = g.probes + (int64_t)__ldg(pid + i) * stride;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j < nc) {
                        axpy_pairs<NA>(acc, ldg_vec<NA>(c + j * NA), Y[j]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < NA; ++k) x[NS + k] += w * acc[k];
        }
    }
    {  // Fresnel powers (decoder.cpp:55-59)
        const float nv = P.no_fresnel ? 1.f : geo.ndv;
        const float u = 1.f - fminf(fmaxf(nv, 0.f), 1.f);
        x[NS + NA] = 1.f;
#pragma unroll
        for (int k = 1; k < NPOW; ++k) x[NS + NA + k] = x[NS + NA + k - 1] * u;
    }
}

// decode_color (decoder.cpp:61-109) from the MLP input.  Layers 1 and 2 run
// input-major: for each input i one broadcast float4 of the transposed weight
// row feeds two paired FMAs (FFMA2), half the issue of per-output FFMA dot
// products (those were ~35 % of shade_fwd's instructions, profiles/r02/v15).
template <int IN>
__device__ __forceinline__ void mlp_forward(const float* __restrict__ sm, const SmemMlp& L,
                                            const float x[IN], const float* cam_row, float rgb[3],
                                            float* a1_row, float* a2_row) {
    float2 z[HID / 2];
#pragma unroll
    for (int j = 0; j < HID / 2; ++j) {
        z[j] = reinterpret_cast<const float2*>(sm + L.b1)[j];
        if (cam_row) {
            z[j].x += __ldg(cam_row + 2 * j);
            z[j].y += __ldg(cam_row + 2 * j + 1);
        }
    }
#pragma unroll
    for (int i = 0; i < IN; ++i) {
        const float4* row = reinterpret_cast<const float4*>(sm + L.w1t + i * HID);
#pragma unroll
        for (int q = 0; q < HID / 4; ++q) {
            const float4 w = row[q];
            ffma2(z[2 * q], make_float2(w.x, w.y), x[i]);
            ffma2(z[2 * q + 1], make_float2(w.z, w.w), x[i]);
        }
    }
    float a1[HID];
#pragma unroll
    for (int j = 0; j < HID / 2; ++j) {
        a1[2 * j] = z[j].x > 0.f ? z[j].x : 0.f;
        a1[2 * j + 1] = z[j].y > 0.f ? z[j].y : 0.f;
    }
#pragma unroll
    for (int j = 0; j < HID / 2; ++j) z[j] = reinterpret_cast<const float2*>(sm + L.b2)[j];
#pragma unroll
    for (int i = 0; i < HID; ++i) {
        const float4* row = reinterpret_cast<const float4*>(sm + L.w2t + i * HID);
#pragma unroll
        for (int q = 0; q < HID / 4; ++q) {
            const float4 w = row[q];
            ffma2(z[2 * q], make_float2(w.x, w.y), a1[i]);
            ffma2(z[2 * q + 1], make_float2(w.z, w.w), a1[i]);
        }
    }
    float a2[HID];
#pragma unroll
    for (int j = 0; j < HID / 2; ++j) {
        a2[2 * j] = z[j].x > 0.f ? z[j].x : 0.f;
        a2[2 * j + 1] = z[j].y > 0.f ? z[j].y : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        float zz = sm[L.b3 + j];
        const float4* row = reinterpret_cast<const float4*>(sm + L.w3 + j * HID);
#pragma unroll
        for (int i = 0; i < HID / 4; ++i) {
            const float4 w = row[i];
            zz += w.x * a2[4 * i] + w.y * a2[4 * i + 1] + w.z * a2[4 * i + 2] + w.w * a2[4 * i + 3];
        }
        rgb[j] = sigmoidf_(zz);
    }
    if (a1_row) {
#pragma unroll
        for (int i = 0; i < HID / 4; ++i) {
            reinterpret_cast<float4*>(a1_row)[i] =
                make_float4(a1[4 * i], a1[4 * i + 1], a1[4 * i + 2], a1[4 * i + 3]);
            reinterpret_cast<float4*>(a2_row)[i] =
                make_float4(a2[4 * i], a2[4 * i + 1], a2[4 * i + 2], a2[4 * i + 3]);
        }
    }
}

template <int NS, int NA>
__device__ __forceinline__ void store_geo(const ShadeGeo& geo, const float (&pv)[3][NS],
                                          const float (&x)[NS + NA + NPOW], float* geo_out);

// decode_fused (renderer.cpp:88-147): features + MLP.  geo_out (optional)
// receives the GeoRec block for the backward.
template <int NS, int NA>
__device__ __forceinline__ void decode_forward(const RayPassParams& P, const float* __restrict__ sm,
                                               const SmemMlp& L, int tile, const double p[3],
                                               const double dneg[3], const float* cam_row,
                                               float rgb[3], ShadeGeo& geo, float* geo_out,
                                               const float* psm = nullptr) {
    constexpr int IN = NS + NA + NPOW;
    float x[IN], pv[3][NS];
    decode_features<NS, NA>(P, tile, p, dneg, geo, x, pv, psm);
    mlp_forward<IN>(sm, L, x, cam_row, rgb, nullptr, nullptr);
    if (geo_out) store_geo<NS, NA>(geo, pv, x, geo_out);
}

// The GeoRec block of a shaded sample (K2b -> K2e): geometry, plane taps,
// probe weights, plane samples and the MLP input.
template <int NS, int NA>
__device__ __forceinline__ void store_geo(const ShadeGeo& geo, const float (&pv)[3][NS],
                                          const float (&x)[NS + NA + NPOW], float* geo_out) {
    constexpr int IN = NS + NA + NPOW;
    {
        using GR = GeoRec<NS, NA>;
        float r[GR::STRIDE];
        r[0] = (float)geo.n[0];
        r[1] = (float)geo.n[1];
        r[2] = (float)geo.n[2];
        r[3] = (float)geo.glen;
        r[4] = geo.refl[0];
        r[5] = geo.refl[1];
        r[6] = geo.refl[2];
        r[7] = geo.ndv;
        r[8] = geo.tx.f;
        r[9] = geo.ty.f;
        r[10] = geo.tz.f;
        r[11] = __int_as_float(geo.tx.a0 | (geo.ty.a0 << 4) | (geo.tz.a0 << 8) |
                               (geo.degenerate ? (1 << 12) : 0));
#pragma unroll
        for (int i = 0; i < 8; ++i) r[12 + i] = geo.w8[i];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
            for (int k = 0; k < NS; ++k) r[GR::PV + q * NS + k] = pv[q][k];
#pragma unroll
        for (int i = 0; i < IN; ++i) r[GR::X + i] = x[i];
#pragma unroll
        for (int i = GR::X + IN; i < GR::STRIDE; ++i) r[i] = 0.f;
#pragma unroll
        for (int i = 0; i < GR::STRIDE / 4; ++i)
            reinterpret_cast<float4*>(geo_out)[i] = make_float4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
    }
}

// Block-wide f64 / u64 accumulation helpers.
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// The scan's k-th active work tile (ViewDev::act_*) as a global work tile.
__device__ __forceinline__ int64_t active_tile(const RayPassParams& P, int64_t k) {
    int v = 0;
    while (v + 1 < P.n_views && P.views[v + 1].act_begin <= k) ++v;
    const ViewDev& V = P.views[v];
    const int a = (int)(k - V.act_begin);  // < the view's tile count: 32-bit division
    const int ay = a / V.act_w, ax = a - ay * V.act_w;
    return V.tile_begin + (int64_t)(V.act_ty0 + ay) * V.tiles_x + V.act_tx0 + ax;
}

// Maps a global work tile to (view, pixel) for this lane.
__device__ __forceinline__ int locate_view(const RayPassParams& P, int64_t tile) {
    int v = 0;
    while (v + 1 < P.n_views && P.views[v + 1].tile_begin <= tile) ++v;
    return v;
}

// Copies the flat MLP (without camera bias) into the shared-memory layout
// (W1 and W2 transposed to input-major).
__device__ __forceinline__ void load_mlp_smem(const float* __restrict__ mlp, float* sm,
                                              const MlpLayout& G, const SmemMlp& L) {
    const int in = G.b1 / HID;
    for (int i = threadIdx.x; i < G.total_nocam; i += blockDim.x) {
        int dst;
        if (i < G.b1) dst = L.w1t + (i % in) * HID + i / in;                   // W1[j][k] -> w1t[k][j]
        else if (i < G.w2) dst = L.b1 + (i - G.b1);
        else if (i < G.b2) dst = L.w2t + ((i - G.w2) & 31) * HID + ((i - G.w2) >> 5);  // W2[j][k] -> w2t[k][j]
        else if (i < G.w3) dst = L.b2 + (i - G.b2);
        else if (i < G.b3) dst = L.w3 + (i - G.w3);
        else dst = L.b3 + (i - G.b3);
        sm[dst] = __ldg(mlp + i);
    }
}

// Per-warp probe staging (ProbeStage): two slots of 8 probe blocks of at most
// 16 coefficients x n_a floats.
template <int NA>
constexpr int probe_stage_floats() {
    return 2 * 8 * 16 * NA;
}
__host__ __device__ constexpr int up4i(int x) { return (x + 3) & ~3; }

template <int NS, int NA>
size_t render_smem_bytes() {
    return sizeof(float) * (up4i(SmemMlp::make(NS + NA + NPOW).total) + WARPS_PER_BLOCK * probe_stage_floats<NA>());
}

}  // namespace psdf
