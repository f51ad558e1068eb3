// psdf_mesh.cuh — marching cubes of the smoothed SDF on the device
// (= marching_cubes(grid), mesh.cpp:305-394), reproducing the reference's
// mesh exactly: the same vertices (bit-identical f64 positions, same ids) and
// the same triangles in the same order.
//
// The reference walks the allocated tiles in allocation order, the cells of a
// tile x-major, polygonises each cell with the 256-case table and numbers a
// vertex when an edge is first met (a hash map keyed by lattice point + axis).
// Here every cell is a thread, and the sequential numbering becomes two
// prefix sums over the cells in that same order (cell key = tile * 4096 +
// local x-major index):
//   mc_case    cell case index + validity (all 8 corners in allocated tiles,
//              inside the resolution) — the reference's veto rule;
//   mc_own     per active edge, whether this cell is the FIRST cell (smallest
//              key) among the valid cells sharing the lattice edge: that cell
//              creates the vertex, with its own corner orientation (the
//              interpolation direction decides the rounding);
//   scan       vertex base per cell;
//   mc_vert    owned vertices: p0 + (p1 - p0) t, t = clamp(v0 / (v0 - v1));
//   mc_tri     triangles of the table per cell, vertex ids looked up through
//              the owner cell of each edge, zero-area triangles dropped
//              (|e1 x e2| / 2 <= 1e-12, exact f64); count, scan, write.
//
// Cells are 2x2x2 voxel centres (origin = voxel_center(0,0,0)); the values
// are the device's fp32 smoothed SDF, read as f64 like smooth_value
// (grid.cpp:87-94).  All f64 arithmetic is explicitly rounded in the
// reference's operation order (no FMA contraction).
#pragma once

#include "psdf_device.cuh"

namespace psdf {

// Triangle table of the 256 marching-cubes cases (Lorensen & Cline 1987; the
// public-domain table of P. Bourke / C. Bloyd, "Polygonising a scalar field",
// 1994, which is also the reference's).  One word per case: edge indices of
// the triangles in nibbles 0..14 (emission order), triangle count in bits
// 60..63.  Edge e joins corners mc_edge_c0/c1(e); corner c sits at offset
// (c&1 ^ c>>1&1, c>>1&1, c>>2&1): (0,0,0),(1,0,0),(1,1,0),(0,1,0), then z+1.
__constant__ unsigned long long kMcTri[256] = {
    0x0000000000000000ull, 0x1000000000000380ull, 0x1000000000000910ull, 0x2000000000189381ull,
    0x1000000000000a21ull, 0x2000000000a21380ull, 0x2000000000920a29ull, 0x300000089a8a2382ull,
    0x10000000000002b3ull, 0x20000000000b82b0ull, 0x2000000000b32091ull, 0x3000000b89b912b1ull,
    0x20000000003ab1a3ull, 0x3000000ab8a801a0ull, 0x30000009ab9b3093ull, 0x2000000000b8aa89ull,
    0x1000000000000874ull, 0x2000000000437034ull, 0x2000000000748910ull, 0x3000000137174914ull,
    0x2000000000748a21ull, 0x3000000a21403743ull, 0x3000000748209a29ull, 0x40004973727929a2ull,
    0x20000000002b3748ull, 0x300000040242b74bull, 0x3000000b32748109ull, 0x40001292b9b49b74ull,
    0x3000000487ab31a3ull, 0x40004b7401b41ab1ull, 0x400030bab9b09874ull, 0x3000000ab99b4b74ull,
    0x1000000000000459ull, 0x2000000000380459ull, 0x2000000000051450ull, 0x3000000513538458ull,
    0x2000000000459a21ull, 0x3000000594a21803ull, 0x3000000204245a25ull, 0x40008434535235a2ull,
    0x2000000000b32459ull, 0x3000000594b802b0ull, 0x3000000b32510450ull, 0x4000584b82852512ull,
    0x300000045931ab3aull, 0x4000ab81a8180594ull, 0x400030bab5b05045ull, 0x3000000b8aa85845ull,
    0x2000000000975879ull, 0x3000000375359039ull, 0x3000000751710870ull, 0x2000000000753351ull,
    0x300000021a759879ull, 0x400037503505921aull, 0x400025a758528208ull, 0x30000007533525a2ull,
    0x30000002b3987597ull, 0x4000b72029279759ull, 0x4000751871810b32ull, 0x300000051771b12bull,
    0x4000b3a31a758859ull, 0x50aba010b7905075ull, 0x507570805a30b0abull, 0x20000000005b75abull,
    0x100000000000056aull, 0x20000000006a5380ull, 0x20000000006a5109ull, 0x30000006a5891381ull,
    0x2000000000162561ull, 0x3000000803621561ull, 0x3000000620609569ull, 0x4000823625285895ull,
    0x200000000056ab32ull, 0x300000056a02b80bull, 0x30000006a5b32910ull, 0x4000b892b92916a5ull,
    0x3000000315356b36ull, 0x40006b51505b0b80ull, 0x40009505606306b3ull, 0x300000089bb96956ull,
    0x20000000008746a5ull, 0x3000000a56374034ull, 0x30000007486a5091ull, 0x400049737179156aull,
    0x3000000874156216ull, 0x4000743403625521ull, 0x4000620560509748ull, 0x5962695923497937ull,
    0x300000056a4872b3ull, 0x4000b720242746a5ull, 0x40006a5b32874910ull, 0x56a54b7b492b9129ull,
    0x40006b51535b3748ull, 0x5b404b7b016b5b15ull, 0x574836b630560950ull, 0x40009b7974b96956ull,
    0x2000000000a4694aull, 0x3000000380a946a4ull, 0x300000004606a10aull, 0x4000a16468618138ull,
    0x3000000462421941ull, 0x4000462942921803ull, 0x2000000000624420ull, 0x3000000624428238ull,
    0x300000032b46a94aull, 0x40006a4a94b82280ull, 0x4000a164606102b3ull, 0x51b8b12184a16146ull,
    0x400036b319639469ull, 0x514641916b0181b8ull, 0x30000004600636b3ull, 0x200000000086b846ull,
    0x3000000a98a876a7ull, 0x4000a76a907a0370ull, 0x40000818717a176aull, 0x300000037117a76aull,
    0x4000768981861621ull, 0x5937390976192962ull, 0x3000000206607087ull, 0x2000000000276237ull,
    0x400076898a86ab32ull, 0x57a9a76790b72702ull, 0x5b32a767a1871081ull, 0x400017616a71b12bull,
    0x563136b619768698ull, 0x200000000076b190ull, 0x400006b0b3607087ull, 0x10000000000006b7ull,
    0x1000000000000b67ull, 0x200000000067b803ull, 0x200000000067b910ull, 0x300000067b138918ull,
    0x20000000007b621aull, 0x30000007b6803a21ull, 0x30000007b69a2092ull, 0x400089a38a3a27b6ull,
    0x2000000000726327ull, 0x3000000026067807ull, 0x3000000910732672ull, 0x4000678891681261ull,
    0x300000073171a67aull, 0x4000801781a7167aull, 0x40007a69a0a70730ull, 0x30000009a88a7a67ull,
    0x200000000068b486ull, 0x3000000640603b63ull, 0x3000000109648b68ull, 0x400063b139369649ull,
    0x30000001a28b6486ull, 0x4000640b60b03a21ull, 0x40009a2920b648b4ull, 0x536463b34923a39aull,
    0x3000000264248328ull, 0x2000000000264240ull, 0x4000834642432091ull, 0x3000000642241491ull,
    0x40001a6648168318ull, 0x300000040660a01aull, 0x539a9303a6834364ull, 0x20000000004a649aull,
    0x2000000000b67594ull, 0x300000067b594380ull, 0x3000000b67045105ull, 0x400051345343867bull,
    0x3000000b6721a459ull, 0x4000594380a217b6ull, 0x4000204a24a45b67ull, 0x567b25a523453843ull,
    0x3000000945267327ull, 0x4000786260680459ull, 0x4000045051673263ull, 0x5851584812786826ull,
    0x400073167161a459ull, 0x5459078701671a61ull, 0x5a737a6a305a4a04ull, 0x4000a84a458a7a67ull,
    0x300000098b9b6596ull, 0x4000590650360b63ull, 0x4000b65510b508b0ull, 0x30000001355363b6ull,
    0x400065b8b9b59a21ull, 0x5a21965690b603b0ull, 0x552025a50865b58bull, 0x400035a3a25363b6ull,
    0x4000283265825985ull, 0x3000000260069659ull, 0x5826283865081851ull, 0x2000000000612651ull,
    0x5698965683a61631ull, 0x400006505960a01aull, 0x2000000000a65830ull, 0x100000000000065aull,
    0x2000000000b57a5bull, 0x300000003857ba5bull, 0x3000000091ba57b5ull, 0x40001381897ba57aull,
    0x300000015717b21bull, 0x4000b27571721380ull, 0x40007b2209729579ull, 0x5289823295b27257ull,
    0x3000000573532a52ull, 0x400052a578258028ull, 0x40002a37353a5109ull, 0x525752a278129289ull,
    0x2000000000573531ull, 0x3000000571170780ull, 0x3000000735539309ull, 0x2000000000795789ull,
    0x30000008ba8a5485ull, 0x400003bba50b5405ull, 0x400054aba8a48910ull, 0x541314943b54a4baull,
    0x40008548b2582152ull, 0x5b151b2b543b0b40ull, 0x558b8545b2950520ull, 0x20000000003b2549ull,
    0x4000483543253a52ull, 0x30000000244252a5ull, 0x5910854583a532a3ull, 0x40002492914252a5ull,
    0x3000000153358548ull, 0x2000000000501540ull, 0x4000530509358548ull, 0x1000000000000549ull,
    0x3000000ba9b947b4ull, 0x4000ba97b9794380ull, 0x4000b470414b1ba1ull, 0x54bab474a1843413ull,
    0x4000219b294b97b4ull, 0x53801b2b197b9479ull, 0x300000004224b47bull, 0x400042343824b47bull,
    0x4000947732972a92ull, 0x570207872a4797a9ull, 0x5a040a1a472a3a73ull, 0x20000000004782a1ull,
    0x3000000317714194ull, 0x4000178180714194ull, 0x2000000000347304ull, 0x1000000000000784ull,
    0x20000000008ba8a9ull, 0x3000000a9bb93903ull, 0x3000000ba88a0a10ull, 0x2000000000a3ba13ull,
    0x30000008b99b1b21ull, 0x40009b2921b93903ull, 0x2000000000b08b20ull, 0x1000000000000b23ull,
    0x300000098aa82832ull, 0x20000000002902a9ull, 0x40008a1810a82832ull, 0x10000000000002a1ull,
    0x2000000000819831ull, 0x1000000000000190ull, 0x1000000000000830ull, 0x0000000000000000ull,
};

// corner c -> offset along axis a
__device__ __forceinline__ int mc_off(int c, int a) {
    return a == 0 ? ((c & 1) ^ ((c >> 1) & 1)) : (a == 1 ? ((c >> 1) & 1) : ((c >> 2) & 1));
}
// edge e -> its two corners (the reference's order: 0-1 1-2 2-3 3-0, 4-5 5-6
// 6-7 7-4, 0-4 1-5 2-6 3-7) and axis
__device__ __forceinline__ int mc_edge_c0(int e) { return e < 8 ? e : e - 8; }
__device__ __forceinline__ int mc_edge_c1(int e) { return e < 8 ? ((e & 3) == 3 ? e - 3 : e + 1) : e - 4; }
__device__ __forceinline__ int mc_edge_axis(int e) { return e >= 8 ? 2 : (e & 1); }
// the edge index of the lattice edge (axis, lower endpoint at offset (p, q)
// inside the cell along the two other axes, in increasing axis order)
__device__ __forceinline__ int mc_edge_of(int axis, int p, int q) {
    if (axis == 0) return q * 4 + p * 2;            // (y,z): 0, 2, 4, 6
    if (axis == 1) return q * 4 + (p ? 1 : 3);      // (x,z): 3, 1, 7, 5
    return 8 + (q ? (p ? 2 : 3) : (p ? 1 : 0));     // (x,y): 8, 9, 11, 10
}
// active edges of a case: the corners' signs differ
__device__ __forceinline__ unsigned mc_edge_mask(int ci) {
    unsigned m = 0;
#pragma unroll
    for (int e = 0; e < 12; ++e)
        if (((ci >> mc_edge_c0(e)) ^ (ci >> mc_edge_c1(e))) & 1) m |= 1u << e;
    return m;
}

struct McView {
    GridView g;
    uint16_t* cell;       // [T*4096] case index (bits 0..7) | valid (bit 8) | owned edges (bits 12..15 unused)
    uint16_t* own;        // [T*4096] edges whose vertex this cell creates
    int* vcount;          // [T*4096] owned edges, then (exclusive scan) vertex base
    int* tcount;          // [T*4096] kept triangles, then (exclusive scan) triangle base
    double* verts;        // [nv][3]
    int32_t* tris;        // [nt][3]
    double o[3];          // voxel_center(0, 0, 0)
};

// Key of the cell whose base corner is global voxel (x, y, z): tile * 4096 +
// local x-major index, or -1 when no valid cell has that base.
__device__ __forceinline__ int64_t mc_cell_key(const McView& M, int x, int y, int z) {
    const GridView& g = M.g;
    if (x < 0 || y < 0 || z < 0) return -1;
    const int t = tile_lookup(g, x >> 4, y >> 4, z >> 4);
    if (t < 0) return -1;
    const int64_t k = (int64_t)t * TV + vox_index(x & 15, y & 15, z & 15);
    return (M.cell[k] & 0x100) ? k : -1;
}

// Owner (smallest valid key) of edge e of the cell at base (x, y, z) and the
// edge's index in the owner.
__device__ __forceinline__ int64_t mc_edge_owner(const McView& M, int x, int y, int z, int e, int& e_own) {
    const int c0 = mc_edge_c0(e), c1 = mc_edge_c1(e), ax = mc_edge_axis(e);
    const int lo[3] = {x + min(mc_off(c0, 0), mc_off(c1, 0)), y + min(mc_off(c0, 1), mc_off(c1, 1)),
                       z + min(mc_off(c0, 2), mc_off(c1, 2))};
    const int a1 = ax == 0 ? 1 : 0, a2 = ax == 2 ? 1 : 2;  // the two other axes, increasing
    int64_t best = -1;
    e_own = -1;
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            int b[3] = {lo[0], lo[1], lo[2]};
            b[a1] -= p;
            b[a2] -= q;
            const int64_t k = mc_cell_key(M, b[0], b[1], b[2]);
            if (k >= 0 && (best < 0 || k < best)) {
                best = k;
                e_own = mc_edge_of(ax, p, q);
            }
        }
    return best;
}

__device__ __forceinline__ void mc_cell_coords(const McView& M, int64_t k, int& x, int& y, int& z) {
    const int4 tc = __ldg(M.g.tile_coords + (k >> 12));
    const int l = (int)(k & 4095);
    x = tc.x * TE + (l >> 8);
    y = tc.y * TE + ((l >> 4) & 15);
    z = tc.z * TE + (l & 15);
}

// mesh.cpp:363-392: the cell at each (tile, voxel); valid when inside the
// resolution and all 8 corners lie in allocated tiles.
__global__ void __launch_bounds__(256) mc_case_kernel(McView M) {
    const GridView& g = M.g;
    const int64_t n = (int64_t)g.T * TV;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        int x, y, z;
        mc_cell_coords(M, k, x, y, z);
        uint16_t out = 0;
        if (x + 1 < g.res[0] && y + 1 < g.res[1] && z + 1 < g.res[2]) {
            const int lx = x & 15, ly = y & 15, lz = z & 15;
            int ci = 0;
            bool ok = true;
            if (lx < 15 && ly < 15 && lz < 15) {  // every corner in this tile
                const float* s = g.smooth + (k >> 12) * TV;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (s[vox_index(lx + mc_off(c, 0), ly + mc_off(c, 1), lz + mc_off(c, 2))] < 0.f) ci |= 1 << c;
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int cx = x + mc_off(c, 0), cy = y + mc_off(c, 1), cz = z + mc_off(c, 2);
                    const int t = tile_lookup(g, cx >> 4, cy >> 4, cz >> 4);
                    if (t < 0) {
                        ok = false;
                        break;
                    }
                    if (__ldg(g.smooth + (int64_t)t * TV + vox_index(cx & 15, cy & 15, cz & 15)) < 0.f) ci |= 1 << c;
                }
            }
            if (ok) out = (uint16_t)(0x100 | ci);
        }
        M.cell[k] = out;
    }
}

// Edges whose vertex this cell creates (it is the first valid cell, in the
// reference's walk order, that meets the edge).
__global__ void __launch_bounds__(256) mc_own_kernel(McView M) {
    const int64_t n = (int64_t)M.g.T * TV;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned cc = M.cell[k];
        const unsigned em = (cc & 0x100) ? mc_edge_mask(cc & 0xff) : 0u;
        unsigned own = 0;
        if (em) {
            int x, y, z;
            mc_cell_coords(M, k, x, y, z);
            for (unsigned m = em; m; m &= m - 1) {
                const int e = __ffs(m) - 1;
                int eo;
                if (mc_edge_owner(M, x, y, z, e, eo) == k) own |= 1u << e;
            }
        }
        M.own[k] = (uint16_t)own;
        M.vcount[k] = __popc(own);
    }
}

__device__ __forceinline__ double mc_value(const GridView& g, int x, int y, int z) {
    const int t = tile_lookup(g, x >> 4, y >> 4, z >> 4);
    return (double)__ldg(g.smooth + (int64_t)t * TV + vox_index(x & 15, y & 15, z & 15));
}

// vertex_on_edge (mesh.cpp:322-342) for the owned edges, in edge order.
__global__ void __launch_bounds__(256) mc_vert_kernel(McView M) {
    const GridView& g = M.g;
    const int64_t n = (int64_t)g.T * TV;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned own = M.own[k];
        if (!own) continue;
        int x, y, z;
        mc_cell_coords(M, k, x, y, z);
        int vid = M.vcount[k];
        for (unsigned m = own; m; m &= m - 1, ++vid) {
            const int e = __ffs(m) - 1;
            const int c0 = mc_edge_c0(e), c1 = mc_edge_c1(e);
            const int p0i[3] = {x + mc_off(c0, 0), y + mc_off(c0, 1), z + mc_off(c0, 2)};
            const int p1i[3] = {x + mc_off(c1, 0), y + mc_off(c1, 1), z + mc_off(c1, 2)};
            const double v0 = mc_value(g, p0i[0], p0i[1], p0i[2]);
            const double v1 = mc_value(g, p1i[0], p1i[1], p1i[2]);
            double t = v0 != v1 ? ddiv(v0, dsub(v0, v1)) : 0.5;
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);  // clampd (vec.hpp:63-65)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double q0 = dadd(M.o[a], dmul((double)p0i[a], g.h));
                const double q1 = dadd(M.o[a], dmul((double)p1i[a], g.h));
                M.verts[3 * (int64_t)vid + a] = dadd(q0, dmul(dsub(q1, q0), t));
            }
        }
    }
}

// Vertex id of edge e of the cell (key k, base x, y, z).
__device__ __forceinline__ int mc_vid(const McView& M, int64_t k, unsigned own, int x, int y, int z, int e) {
    if ((own >> e) & 1u) return M.vcount[k] + __popc(own & ((1u << e) - 1u));
    int eo;
    const int64_t ko = mc_edge_owner(M, x, y, z, e, eo);
    return M.vcount[ko] + __popc((unsigned)M.own[ko] & ((1u << eo) - 1u));
}

// Triangles of the cell (mesh.cpp:353-361): WRITE = false counts the kept
// ones, WRITE = true stores them at the scanned base.
template <bool WRITE>
__global__ void __launch_bounds__(256) mc_tri_kernel(McView M) {
    const int64_t n = (int64_t)M.g.T * TV;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned cc = M.cell[k];
        const unsigned long long tw = (cc & 0x100) ? kMcTri[cc & 0xff] : 0ull;
        const int ntri = (int)(tw >> 60);
        if (!ntri) {
            if (!WRITE) M.tcount[k] = 0;
            continue;
        }
        int x, y, z;
        mc_cell_coords(M, k, x, y, z);
        const unsigned own = M.own[k];
        int kept = 0, base = WRITE ? M.tcount[k] : 0;
        for (int t = 0; t < ntri; ++t) {
            int id[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) id[j] = mc_vid(M, k, own, x, y, z, (int)((tw >> (4 * (3 * t + j))) & 15));
            if (id[0] == id[1] || id[1] == id[2] || id[0] == id[2]) continue;
            const double* a = M.verts + 3 * (int64_t)id[0];
            const double* b = M.verts + 3 * (int64_t)id[1];
            const double* c = M.verts + 3 * (int64_t)id[2];
            const double e1[3] = {dsub(b[0], a[0]), dsub(b[1], a[1]), dsub(b[2], a[2])};
            const double e2[3] = {dsub(c[0], a[0]), dsub(c[1], a[1]), dsub(c[2], a[2])};
            // vec.hpp:27-30: cross, then sqrt((x x + y y) + z z)
            const D3 cr = d3(dsub(dmul(e1[1], e2[2]), dmul(e1[2], e2[1])),
                             dsub(dmul(e1[2], e2[0]), dmul(e1[0], e2[2])),
                             dsub(dmul(e1[0], e2[1]), dmul(e1[1], e2[0])));
            if (dmul(dsqrt(ddot(cr, cr)), 0.5) <= 1e-12) continue;
            if (WRITE) {
                M.tris[3 * (int64_t)(base + kept)] = id[0];
                M.tris[3 * (int64_t)(base + kept) + 1] = id[1];
                M.tris[3 * (int64_t)(base + kept) + 2] = id[2];
            }
            ++kept;
        }
        if (!WRITE) M.tcount[k] = kept;
    }
}

}  // namespace psdf
