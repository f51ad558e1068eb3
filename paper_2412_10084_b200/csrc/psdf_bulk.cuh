// psdf_bulk.cuh — bulk global->shared copies on the TMA engine
// (cp.async.bulk, SASS UBLKCP) completed on an mbarrier, for staging the small
// per-tile parameter blocks the shading kernels gather (the 8 corner probes of
// a tile: every shading record of the tile reads all of them).
//
// Protocol per warp (one mbarrier, one elected lane issues):
//   __syncwarp();                                  // readers of the slot done
//   lane 0: bulk_fence(); bulk_expect(bar, bytes); bulk_copy(...) x n;
//   all:    bulk_wait(bar, phase); phase ^= 1;
// bulk_fence orders the generic-proxy reads of the previous contents before
// the async-proxy writes of the new ones.
#pragma once

#include <cstdint>

namespace psdf {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_bar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bulk_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void bulk_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// bytes: a multiple of 16; src and dst 16-byte aligned.
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Per-warp staging of the 8 corner-probe blocks of up to two tiles (the first
// and the last tile of a warp's 32 tile-sorted shading records), cached across
// the warp's batches.  A probe block is contiguous ([order^2][n_a] floats,
// `stride`), so each corner is one bulk copy.  Records of a third tile in the
// same batch (rare: a run of tiles with very few records) read global memory.
struct ProbeStage {
    float* slot0;     // [8][stride]
    float* slot1;
    uint64_t* bar;
    int tag0, tag1;   // tile held by each slot, -1 none
    uint32_t phase;
    int stride;
    bool on;          // stride * 4 is a multiple of 16 (bulk copy granule)

    __device__ __forceinline__ void init(float* base, uint64_t* bar_, int stride_) {
        slot0 = base;
        slot1 = base + 8 * stride_;
        bar = bar_;
        tag0 = tag1 = -1;
        phase = 0;
        stride = stride_;
        on = (stride_ & 3) == 0;
        if ((threadIdx.x & 31) == 0) bulk_bar_init(bar);
        __syncwarp();
    }

    // Warp-uniform: tiles tA (lane 0's record) and tB (the last valid lane's);
    // returns this lane's staged block for `my_tile`, or nullptr.
    __device__ __forceinline__ const float* fetch(int tA, int tB, int my_tile, const float* probes,
                                                  const int32_t* probe_ids) {
        if (!on || tA < 0) return nullptr;
        const int lane = threadIdx.x & 31;
        int sA = tag0 == tA ? 0 : (tag1 == tA ? 1 : -1);
        int sB = tB == tA ? sA : (tag0 == tB ? 0 : (tag1 == tB ? 1 : -1));
        bool ldA = false, ldB = false;
        if (sA < 0) {
            sA = sB == 0 ? 1 : 0;
            ldA = true;
        }
        if (tB == tA) {
            sB = sA;
        } else if (sB < 0) {
            sB = sA == 0 ? 1 : 0;
            ldB = true;
        }
        if (ldA || ldB) {
            const uint32_t bytes = 4u * (uint32_t)stride;
            __syncwarp();  // every lane is done with the slots' previous contents
            if (lane == 0) bulk_expect(bar, (ldA ? 8u : 0u) * bytes + (ldB ? 8u : 0u) * bytes);
            __syncwarp();
            const int c = lane & 7;
            const bool mine = (lane < 8 && ldA) || (lane >= 8 && lane < 16 && ldB);
            if (mine) {
                const int t = lane < 8 ? tA : tB;
                const int s = lane < 8 ? sA : sB;
                bulk_fence();
                bulk_copy((s ? slot1 : slot0) + c * stride, probes + (int64_t)__ldg(probe_ids + (int64_t)t * 8 + c) * stride,
                          bytes, bar);
            }
            bulk_wait(bar, phase);
            phase ^= 1u;
            if (sA) tag1 = tA; else tag0 = tA;
            if (sB) tag1 = tB; else tag0 = tB;
        }
        return my_tile == tA ? (sA ? slot1 : slot0) : (my_tile == tB ? (sB ? slot1 : slot0) : nullptr);
    }
};

}  // namespace psdf
