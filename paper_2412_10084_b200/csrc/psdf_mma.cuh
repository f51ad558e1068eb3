// psdf_mma.cuh — warp-level tensor-core GEMM helpers for the decoder MLP
// (2 x 32 hidden, decoder.hpp:17-31) on shading-record batches of 32.
//
// mma.sync m16n8k8 TF32 with the 3xTF32 split (x = hi + lo, both TF32;
// a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi, fp32 accumulate): fp32-level
// accuracy (~1e-6 relative) from the tensor pipe, which the decoder's
// 1e-4 colour / 1e-3 gradient tolerances need (plain TF32 is ~5e-4).
//
// Fragment layouts (PTX ISA, mma.m16n8k8 .tf32): g = lane / 4, t = lane % 4;
//   A (16x8, row): a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
//   B (8x8,  col): b0 (k=t, n=g), b1 (k=t+4, n=g)
//   C (16x8):      c0 (g, 2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1)
#pragma once

#include <cstdint>

namespace psdf {

__device__ __forceinline__ uint32_t tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mma_tf32(float c[4], const uint32_t a[4], const uint32_t b[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

struct Split4 {
    uint32_t hi[4], lo[4];
};
struct Split2 {
    uint32_t hi[2], lo[2];
};
// hi = v with the 13 mantissa bits of a TF32 operand cleared (an exact
// prefix of v, one LOP), lo = v - hi (exact in fp32) rounded to TF32 by an
// integer add + mask (round half away from zero on the magnitude, as
// cvt.rna): |v - hi - lo| <= 2^-22 |v|.  Measured on the bench step
// (profiles/r02/v42-v45): cvt.rna for both halves 0.705 ms for shade_bwd +
// shade_geo, this split 0.636 ms, same accuracy (ray-pass plane gradients
// 6e-7 relative to the f64 oracle); passing lo unrounded is NOT equivalent —
// the tensor core does not simply ignore the low 13 bits (plane gradients
// drifted to 2e-4).
__device__ __forceinline__ void split1(float v, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(v) & 0xffffe000u;
    lo = (__float_as_uint(v - __uint_as_float(hi)) + 0x1000u) & 0xffffe000u;
}
template <int N, class S>
__device__ __forceinline__ void split(const float* v, S& s) {
#pragma unroll
    for (int i = 0; i < N; ++i) split1(v[i], s.hi[i], s.lo[i]);
}

// C[MT*16 x NT*8] += A(m, k) B(n, k) over k in [0, KT*8); A and B are element
// accessors (m, k) -> float and (n, k) -> float.
template <int MT, int NT, int KT, class FA, class FB>
__device__ __forceinline__ void warp_gemm3(float (&c)[MT][NT][4], FA A, FB B) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
        const int k0 = kt * 8;
        Split4 a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m0 = mt * 16;
            const float v[4] = {A(m0 + g, k0 + t), A(m0 + g + 8, k0 + t), A(m0 + g, k0 + t + 4),
                                A(m0 + g + 8, k0 + t + 4)};
            split<4>(v, a[mt]);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int n0 = nt * 8;
            const float v[2] = {B(n0 + g, k0 + t), B(n0 + g, k0 + t + 4)};
            Split2 b;
            split<2>(v, b);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                mma_tf32(c[mt][nt], a[mt].lo, b.hi);
                mma_tf32(c[mt][nt], a[mt].hi, b.lo);
                mma_tf32(c[mt][nt], a[mt].hi, b.hi);
            }
        }
    }
}

// As warp_gemm3, with B already split (constant weights staged once per block
// as TF32 hi / lo words): Bh(n, k) / Bl(n, k) -> uint32.  Halves the split
// work of the weight GEMMs.
template <int MT, int NT, int KT, class FA, class FBH, class FBL>
__device__ __forceinline__ void warp_gemm3w(float (&c)[MT][NT][4], FA A, FBH Bh, FBL Bl) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
        const int k0 = kt * 8;
        Split4 a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m0 = mt * 16;
            const float v[4] = {A(m0 + g, k0 + t), A(m0 + g + 8, k0 + t), A(m0 + g, k0 + t + 4),
                                A(m0 + g + 8, k0 + t + 4)};
            split<4>(v, a[mt]);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int n0 = nt * 8;
            const uint32_t bh[2] = {Bh(n0 + g, k0 + t), Bh(n0 + g, k0 + t + 4)};
            const uint32_t bl[2] = {Bl(n0 + g, k0 + t), Bl(n0 + g, k0 + t + 4)};
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                mma_tf32(c[mt][nt], a[mt].lo, bh);
                mma_tf32(c[mt][nt], a[mt].hi, bl);
                mma_tf32(c[mt][nt], a[mt].hi, bh);
            }
        }
    }
}

// Visits every C element held by this lane: f(m, n, value&).
template <int MT, int NT, class F>
__device__ __forceinline__ void for_c(float (&c)[MT][NT][4], F f) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) f(mt * 16 + g + ((i >> 1) << 3), nt * 8 + 2 * t + (i & 1), c[mt][nt][i]);
}

template <int MT, int NT>
__device__ __forceinline__ void zero_c(float (&c)[MT][NT][4]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) c[mt][nt][i] = 0.f;
}

}  // namespace psdf
