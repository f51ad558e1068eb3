// psdf_device.cuh — device-side building blocks of the fused ray pass.
//
// Precision contract:
//  * Geometry that decides WHICH samples exist and which get shaded — the
//    pixel ray, the march t-list, the trilinear SDF value, alpha, T and the
//    weights — is evaluated in f64 with every operation explicitly rounded
//    (__dadd_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn) so nvcc cannot contract it
//    into FMAs.  In the reference's operation order this reproduces the
//    reference's f64 results bit for bit from the same (fp32-stored) inputs.
//  * The decode (tri-plane, SH probes, MLP) and all gradients are fp32.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace psdf {

constexpr int TE = 16;     // kTileEdge (grid.hpp:15)
constexpr int TV = 4096;   // kTileVoxels
constexpr int HID = 32;    // kHidden (decoder.hpp:11)
constexpr int NPOW = 6;    // kFresnelPowers
constexpr double kPhotoEps = 1e-3;  // losses.hpp:9

// ----------------------------------------------------------- exact f64 ops
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// a / b correctly rounded from rb = RN(1/b) (Markstein: q0 = RN(a rb) is
// faithful, the residual a - b q0 is exact under FMA, and RN(q0 + r rb) is
// RN(a / b) for finite, normal operands).  Same bits as ddiv, without the
// software division; tested on 4e8 random and near-midpoint pairs.
__device__ __forceinline__ double ddiv_r(double a, double b, double rb) {
    const double q0 = __dmul_rn(a, rb);
    return __fma_rn(__fma_rn(-b, q0, a), rb, q0);
}
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
// RN(a / b) without the software division: ddiv_r from the correctly rounded
// reciprocal when a and b are normal and far from overflow (every value the
// march, the alpha chain and the photo terms divide by), the division
// sequence otherwise (zero, subnormal, huge or non-finite operands).
__device__ __forceinline__ double ddiv_fast(double a, double b) {
    const double ab = fabs(a), bb = fabs(b);
    // both in [1e-150, 1e150] (or a == 0): the quotient is normal, no
    // intermediate overflows or underflows
    if (bb > 1e-150 && bb < 1e150 && ab < 1e150 && (ab > 1e-150 || a == 0.0)) return ddiv_r(a, b, __drcp_rn(b));
    return ddiv(a, b);
}

struct D3 {
    double x, y, z;
};
__device__ __forceinline__ D3 d3(double x, double y, double z) { return D3{x, y, z}; }
// vec.hpp:26 — dot is (x*x' + y*y') + z*z'
__device__ __forceinline__ double ddot(D3 a, D3 b) {
    return dadd(dadd(dmul(a.x, b.x), dmul(a.y, b.y)), dmul(a.z, b.z));
}

// Device view of the sparse grid (SoA fp32 storage, dense tile table).
struct GridView {
    int T, P, n_s, n_a, order;     // order = grid SH order (coefficient stride)
    int res[3], nt[3];
    double h, org[3], far;         // far = far_field_voxels * voxel_size (grid.hpp:71)
    double inv_h;                  // 1 / h, used only when h is a power of two
    int h_pow2;                    // x / h == x * inv_h exactly (power-of-two h)
    double wmax[3];                // world_max() (grid.hpp:72-74)
    double occ_lo[3], occ_hi[3];   // bounding box of the allocated tiles, one voxel margin
    int occ_any;                   // any tile allocated
    const int32_t* __restrict__ tile_table;   // [nt0][nt1][nt2] -> tile or -1
    const uint32_t* __restrict__ tile_bits;   // occupancy bitmap of tile_table
    const uint8_t* __restrict__ tile_dist;    // L-inf distance (tiles) to the nearest allocated tile
    const int32_t* __restrict__ tile_nbr;     // [T][27] neighbour tile ids (-1: none), (dx,dy,dz) in {-1,0,1}^3
    int bit_words;                            // 32-bit words in tile_bits
    double margin;                            // marcher decision margin, voxels (1e-8; tests widen it)
    const int4* __restrict__ tile_coords;     // [T] (x,y,z,0)
    const int32_t* __restrict__ probe_ids;    // [T][8]
    const float* __restrict__ smooth;         // [T][4096]
    const float* __restrict__ smooth_ap;      // [T][18^3] smooth with a 1-voxel apron
    const uint8_t* __restrict__ sat_dist;     // [T][17^3] per-cell saturation distances of this pass (sat_dist_kernel)
    const float* __restrict__ planes;         // [T][3][256][n_s]
    const float* __restrict__ probes;         // [P][order^2][n_a]
};

__device__ __forceinline__ int tile_lookup(const GridView& g, int tx, int ty, int tz) {
    if ((unsigned)tx >= (unsigned)g.nt[0] || (unsigned)ty >= (unsigned)g.nt[1] ||
        (unsigned)tz >= (unsigned)g.nt[2])
        return -1;
    return __ldg(g.tile_table + ((int64_t)tx * g.nt[1] + ty) * g.nt[2] + tz);
}

__device__ __forceinline__ int vox_index(int x, int y, int z) { return (x * TE + y) * TE + z; }

// x / voxel_size.  For a power-of-two voxel size (every grid the reference
// builds: 1/16 halved per LOD, grid.cpp:276) the reciprocal is exact and
// x * (1/h) is the same correctly-rounded value as x / h, so the f64 software
// division is skipped without changing a bit.
__device__ __forceinline__ double div_h(const GridView& g, double x) {
    return g.h_pow2 ? dmul(x, g.inv_h) : ddiv(x, g.h);
}

// world_to_voxel component (grid.hpp:126): (p - origin) / voxel_size
__device__ __forceinline__ double w2v(const GridView& g, double p, int a) {
    return div_h(g, dsub(p, g.org[a]));
}

// smooth_value (grid.cpp:87-94): far field outside resolution / unallocated.
__device__ __forceinline__ double smooth_value(const GridView& g, int vx, int vy, int vz) {
    if (vx < 0 || vy < 0 || vz < 0 || vx >= g.res[0] || vy >= g.res[1] || vz >= g.res[2])
        return g.far;
    const int t = tile_lookup(g, vx >> 4, vy >> 4, vz >> 4);
    if (t < 0) return g.far;
    return (double)__ldg(g.smooth + (int64_t)t * TV + vox_index(vx & 15, vy & 15, vz & 15));
}

constexpr int AE = 18;            // apron brick edge (16 + 2)
constexpr int AV = AE * AE * AE;  // 5832
constexpr int kCellE = 17;                          // trilinear cells b in [-1, 15] per axis
constexpr int kCellN = kCellE * kCellE * kCellE;    // 4913
constexpr uint8_t kCellNone = 255;                  // sat_dist: no unsaturated cell in the tile

// Trilinear sum of sample_trilinear (grid.cpp:104-110) in its exact f64
// operation order.
__device__ __forceinline__ double trilerp8(double fx, double fy, double fz, const double c[8]) {
    const double gx0 = dsub(1.0, fx), gy0 = dsub(1.0, fy), gz0 = dsub(1.0, fz);
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const double w = dmul(dmul((i & 1) ? fx : gx0, (i & 2) ? fy : gy0), (i & 4) ? fz : gz0);
        v = dadd(v, dmul(w, c[i]));
    }
    return v;
}

// sample_sdf (grid.cpp:98-125) at a point whose containing voxel lies in the
// allocated tile `tile` (tile coordinates tc): every corner is inside the
// tile's apron brick, so no table lookup is needed.  Exact f64.
__device__ __forceinline__ double sample_sdf_in(const GridView& g, double px, double py, double pz,
                                                int tile, int4 tc) {
    const double cx = dsub(w2v(g, px, 0), 0.5);
    const double cy = dsub(w2v(g, py, 1), 0.5);
    const double cz = dsub(w2v(g, pz, 2), 0.5);
    const int bx = (int)floor(cx), by = (int)floor(cy), bz = (int)floor(cz);
    const double fx = dsub(cx, (double)bx), fy = dsub(cy, (double)by), fz = dsub(cz, (double)bz);
    // corner b - 16 tc in [-1, 15]: apron index +1
    const float* base = g.smooth_ap + (int64_t)tile * AV +
                        ((bx - 16 * tc.x + 1) * AE + (by - 16 * tc.y + 1)) * AE + (bz - 16 * tc.z + 1);
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        c[i] = (double)__ldg(base + (i & 1) * (AE * AE) + ((i >> 1) & 1) * AE + ((i >> 2) & 1));
    return trilerp8(fx, fy, fz, c);
}

// The fields the out-of-line exact paths need, passed by value: handing
// them the kernel-parameter GridView by reference would force a local copy
// of the whole parameter block (and local-memory reads in the hot loops).
struct GridLite {
    const int32_t* tile_table;
    const float* smooth;
    double org[3], h, inv_h, far;
    int nt[3], res[3], h_pow2;
};
__device__ __forceinline__ GridLite lite(const GridView& g) {
    GridLite l;
    l.tile_table = g.tile_table;
    l.smooth = g.smooth;
    for (int a = 0; a < 3; ++a) {
        l.org[a] = g.org[a];
        l.nt[a] = g.nt[a];
        l.res[a] = g.res[a];
    }
    l.h = g.h;
    l.inv_h = g.inv_h;
    l.far = g.far;
    l.h_pow2 = g.h_pow2;
    return l;
}

// sample_trilinear with per-corner lookups (corners straddling tiles or the
// grid boundary).  Out of line, arguments by value (no pointer escapes).
__device__ __noinline__ double sample_slow(GridLite g, int bx, int by, int bz, double fx,
                                           double fy, double fz) {
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int vx = bx + (i & 1), vy = by + ((i >> 1) & 1), vz = bz + ((i >> 2) & 1);
        double v = g.far;  // smooth_value (grid.cpp:87-94)
        if (vx >= 0 && vy >= 0 && vz >= 0 && vx < g.res[0] && vy < g.res[1] && vz < g.res[2]) {
            const int t = __ldg(g.tile_table + ((int64_t)(vx >> 4) * g.nt[1] + (vy >> 4)) * g.nt[2] + (vz >> 4));
            if (t >= 0) v = (double)__ldg(g.smooth + (int64_t)t * TV + vox_index(vx & 15, vy & 15, vz & 15));
        }
        c[i] = v;
    }
    return trilerp8(fx, fy, fz, c);
}

// sample_sdf (grid.cpp:98-125), exact f64, for an arbitrary point: one table
// lookup finds the containing tile; outside allocated tiles the corners are
// fetched one by one.
__device__ __forceinline__ double sample_sdf(const GridView& g, double px, double py, double pz) {
    const double vx = w2v(g, px, 0), vy = w2v(g, py, 1), vz = w2v(g, pz, 2);
    const int ix = (int)floor(vx), iy = (int)floor(vy), iz = (int)floor(vz);
    if (ix >= 0 && iy >= 0 && iz >= 0 && ix < g.res[0] && iy < g.res[1] && iz < g.res[2]) {
        const int t = tile_lookup(g, ix >> 4, iy >> 4, iz >> 4);
        if (t >= 0) return sample_sdf_in(g, px, py, pz, t, make_int4(ix >> 4, iy >> 4, iz >> 4, 0));
    }
    const double cx = dsub(vx, 0.5), cy = dsub(vy, 0.5), cz = dsub(vz, 0.5);
    const int bx = (int)floor(cx), by = (int)floor(cy), bz = (int)floor(cz);
    return sample_slow(lite(g), bx, by, bz, dsub(cx, (double)bx), dsub(cy, (double)by),
                       dsub(cz, (double)bz));
}

// ------------------------------------------------------------ camera + march
struct Cam {
    double fx, fy, cx, cy, rot[9], pos[3];
    double rfx, rfy;  // RN(1 / fx), RN(1 / fy)
    int width, height, id;
};

// Camera::pixel_dir (camera.hpp:32-35), exact f64 (out of line: once per ray).
__device__ __noinline__ D3 pixel_dir(const Cam& c, double u, double v) {
    const double x = ddiv_r(dsub(u, c.cx), c.fx, c.rfx), y = ddiv_r(dsub(v, c.cy), c.fy, c.rfy), z = 1.0;
    const D3 q = d3(dadd(dadd(dmul(c.rot[0], x), dmul(c.rot[1], y)), dmul(c.rot[2], z)),
                    dadd(dadd(dmul(c.rot[3], x), dmul(c.rot[4], y)), dmul(c.rot[5], z)),
                    dadd(dadd(dmul(c.rot[6], x), dmul(c.rot[7], y)), dmul(c.rot[8], z)));
    const double n = dsqrt(ddot(q, q));
    if (!(n > 0.0)) return d3(0, 0, 0);
    const double rn = __drcp_rn(n);
    return d3(ddiv_r(q.x, n, rn), ddiv_r(q.y, n, rn), ddiv_r(q.z, n, rn));
}

// ray_box (renderer.cpp:13-31), by value: no pointer to the caller's
// arrays escapes (that would force them into local memory).
struct BoxHit {
    bool ok;
    double t0, t1;
};
__device__ __forceinline__ BoxHit ray_box_inl(D3 o, D3 d, D3 mn, D3 mx) {
    BoxHit r{true, 0.0, 1.7976931348623157e308};
    const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    const double lo[3] = {mn.x, mn.y, mn.z}, hi[3] = {mx.x, mx.y, mx.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (fabs(dd[a]) < 1e-15) {
            if (oo[a] < lo[a] || oo[a] > hi[a]) {
                r.ok = false;
                return r;
            }
            continue;
        }
        double ta = ddiv(dsub(lo[a], oo[a]), dd[a]), tb = ddiv(dsub(hi[a], oo[a]), dd[a]);
        if (ta > tb) {
            const double s = ta;
            ta = tb;
            tb = s;
        }
        r.t0 = (r.t0 < ta) ? ta : r.t0;  // std::max
        r.t1 = (tb < r.t1) ? tb : r.t1;  // std::min
        if (r.t0 > r.t1) {
            r.ok = false;
            return r;
        }
    }
    return r;
}
// Out of line (runs once per ray); the six divisions via ddiv_r from the
// ray's reciprocal direction rd (rd_a = RN(1/d_a), unused where |d_a| < 1e-15).
__device__ __noinline__ BoxHit ray_box(D3 o, D3 d, D3 rd, D3 mn, D3 mx) {
    BoxHit r{true, 0.0, 1.7976931348623157e308};
    const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z}, rr[3] = {rd.x, rd.y, rd.z};
    const double lo[3] = {mn.x, mn.y, mn.z}, hi[3] = {mx.x, mx.y, mx.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (fabs(dd[a]) < 1e-15) {
            if (oo[a] < lo[a] || oo[a] > hi[a]) {
                r.ok = false;
                return r;
            }
            continue;
        }
        double ta = ddiv_r(dsub(lo[a], oo[a]), dd[a], rr[a]), tb = ddiv_r(dsub(hi[a], oo[a]), dd[a], rr[a]);
        if (ta > tb) {
            const double s = ta;
            ta = tb;
            tb = s;
        }
        r.t0 = (r.t0 < ta) ? ta : r.t0;  // std::max
        r.t1 = (tb < r.t1) ? tb : r.t1;  // std::min
        if (r.t0 > r.t1) {
            r.ok = false;
            return r;
        }
    }
    return r;
}

// Copies the tile occupancy bitmap into shared memory (call before a
// __syncthreads) and returns the pointer the marcher should use.
__device__ __forceinline__ const uint32_t* stage_tile_bits(const GridView& g, uint32_t* sm_bits,
                                                           int sm_words) {
    if (g.bit_words > sm_words) return g.tile_bits;  // too large: read through L1
    for (int i = threadIdx.x; i < g.bit_words; i += blockDim.x) sm_bits[i] = __ldg(g.tile_bits + i);
    return sm_bits;
}

// The reference's skip past an unallocated tile (renderer.cpp:73-82), exactly:
// ray_box against the tile, then t += max(1, ceil((e1 - t)/h + 1e-9)) h.
// Out of line: only taken when the fast form is within its error margin.
__device__ __noinline__ double exact_skip(GridLite g, D3 o, D3 d, int tx, int ty, int tz,
                                          double t) {
    const double h = g.h;
    auto div_h = [&](double x) { return g.h_pow2 ? dmul(x, g.inv_h) : ddiv(x, g.h); };
    const double tile_w = dmul(16.0, h);
    const D3 bmin = d3(dadd(g.org[0], dmul((double)tx, tile_w)), dadd(g.org[1], dmul((double)ty, tile_w)),
                       dadd(g.org[2], dmul((double)tz, tile_w)));
    const D3 bmax = d3(dadd(bmin.x, tile_w), dadd(bmin.y, tile_w), dadd(bmin.z, tile_w));
    const BoxHit b = ray_box_inl(o, d, bmin, bmax);
    if (b.ok && b.t1 > t) {
        const double skip = ceil(dadd(div_h(dsub(b.t1, t)), 1e-9));
        return dadd(t, dmul(skip > 1.0 ? skip : 1.0, h));
    }
    return dadd(t, h);
}

// Tile of p(t) exactly as the reference computes it: floor((o + t d - org)/h) >> 4.
__device__ __noinline__ int4 exact_tile(GridLite g, D3 o, D3 d, double t) {
    auto w2v_ = [&](double p, int a) {
        const double x = dsub(p, g.org[a]);
        return g.h_pow2 ? dmul(x, g.inv_h) : ddiv(x, g.h);
    };
    return make_int4(((int)floor(w2v_(dadd(o.x, dmul(d.x, t)), 0))) >> 4,
                     ((int)floor(w2v_(dadd(o.y, dmul(d.y, t)), 1))) >> 4,
                     ((int)floor(w2v_(dadd(o.z, dmul(d.z, t)), 2))) >> 4, 0);
}

#ifdef PSDF_MARCH_STATS
// diagnostics build only: [rays, in box, loop iterations, samples, jumps,
// fast skips, exact fallbacks, rewinds]
__device__ unsigned long long g_march_stats[12];
__device__ unsigned long long g_cont_hist[2][16];  // K2a rays by log2(steps), per round
// march_coop_kernel: rays, loop steps, saturated runs, batches, batch samples,
// batches of one sample, marcher iterations inside its next_run calls
__device__ unsigned long long g_coop_stats[8];
#define PSDF_STAT(i) atomicAdd(&g_march_stats[i], 1ull)
#else
#define PSDF_STAT(i) ((void)0)
#endif

// t + m h exactly as the reference's own chain of additions would produce it
// (see Marcher): every lattice step is a multiple of h, exact inside a
// binade, rounded once when t crosses a power of two; adding m h in chunks
// that each cross at most one power of two gives the same bits as any other
// such chunking.  Needs t >= 64 h (then a binade is wider than any single
// reference step).
__device__ __forceinline__ double lattice_advance(double t, double m, double h) {
    for (;;) {
        // next power of two above t (t > 0, normal): exponent field + 1, mantissa 0
        const double p2 = __longlong_as_double((__double_as_longlong(t) & 0x7FF0000000000000LL) +
                                               0x0010000000000000LL);
        if (t + m * h < 2.0 * p2) return dadd(t, dmul(m, h));
        const double m1 = ceil((p2 - t) / h);          // any m1 >= 1 landing in [p2, 2 p2)
        t = dadd(t, dmul(m1, h));
        m -= m1;
    }
}

// march_ray (renderer.cpp:55-86) as a resumable generator: the state is
// (t, count), so the backward sweep can restart at any emitted sample.
//
// t is advanced with exactly the reference's f64 additions.  The two integer
// decisions taken per iteration — which tile p(t) lies in, and the skip count
// ceil((e1 - t)/h + 1e-9) past an empty tile — are first evaluated with a
// cheap FMA form in voxel units, v = (o - org)/h + (d/h) t, whose error is
// ~1e-12 voxel; when the value is farther than a 1e-8 margin from the
// decision boundary the result is provably the reference's, otherwise the
// exact f64 path decides.
//
// Empty space.  Every t the reference produces is t0 + K h for an integer K
// (each step adds h or k h), rounded only where t crosses a power of two, so
// the reference's t-sequence is the lattice {t0 + K h} and its samples are
// the lattice points inside allocated tiles: the tile-by-tile skip of
// renderer.cpp:73-82 only decides which lattice points are visited on the
// way.  The marcher therefore jumps m lattice steps at once through the
// L-inf ball of empty tiles around p(t) (g.tile_dist), landing on a lattice
// point the reference never visits but whose successor it computes
// identically (same tile, skip count = reference's minus the integer offset)
// unless a decision is inside the margin.  In that case — and only while
// desynchronised by a jump — the marcher rewinds to the last point the
// reference itself visited (t_sync) and replays tile by tile without jumps,
// so every emitted sample is bit-identical to the reference.
// sigmoid(x) == 1.0 exactly for x >= kSatX: exp(-37.5) < 2^-54, so 1 + exp(-x)
// rounds to 1 (renderer.cpp:10), and alpha_from(a, 1.0) == 0 for any a.
constexpr double kSatX = 37.5 * (1.0 + 1e-9);

struct SampleRun {
    int n;          // samples in the run (>= 1)
    bool sat;       // every sample of the run has sigmoid == 1 exactly
    double t_last;  // t of the run's last sample
};

struct Marcher {
    double o[3], d[3], inv_d[3];
    double t, t1;
    int count, n_max;
    double vo[3], vd[3];  // (o - org)/h, d/h
    double dinv_max;      // 1 / max_a |d_a|: lattice steps per voxel of L-inf travel
    double rinv_max;      // max_a |1 / d_a| (error scale of the skip counts)
    double t_sync;        // < 0: synchronised with the reference; else its last t
    bool no_jump;         // replaying after a rewind
    unsigned n_exact;     // exact-path fallbacks taken (diagnostics)
    int c_b, c_tile;      // last tile-grid cell looked up and its tile id
    int c_blk, c_ds;      // last cell (tile * 17^3 + cell) and its saturation distance

    __device__ __forceinline__ void setup(const GridView& g, const double* o_, const double* d_, int nmax) {
        const double inv_h = g.h_pow2 ? g.inv_h : 1.0 / g.h;
        double dm = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            o[a] = o_[a];
            d[a] = d_[a];
            inv_d[a] = fabs(d[a]) < 1e-15 ? 0.0 : __drcp_rn(d[a]);
            vo[a] = (o[a] - g.org[a]) * inv_h;
            vd[a] = d[a] * inv_h;
            dm = fmax(dm, fabs(d[a]));
        }
        dinv_max = dm > 0.0 ? __drcp_rn(dm) : 0.0;  // = 1.0 / dm (correctly rounded), no division sequence
        rinv_max = fmax(fmax(fabs(inv_d[0]), fabs(inv_d[1])), fabs(inv_d[2]));
        t_sync = -1.0;
        no_jump = false;
        c_b = c_blk = -1;
        c_tile = c_ds = 0;
        n_max = nmax;
        count = 0;
        n_exact = 0;
    }

    __device__ __forceinline__ bool init(const GridView& g, const double* o_, const double* d_,
                                         int nmax) {
        setup(g, o_, d_, nmax);
        const BoxHit b = ray_box(d3(o[0], o[1], o[2]), d3(d[0], d[1], d[2]), d3(inv_d[0], inv_d[1], inv_d[2]),
                                 d3(g.org[0], g.org[1], g.org[2]), d3(g.wmax[0], g.wmax[1], g.wmax[2]));
        PSDF_STAT(0);
        if (b.ok) PSDF_STAT(1);
        if (!b.ok) {
            t = 0.0;
            t1 = -1.0;
            return false;
        }
        t1 = b.t1;
        t = dadd(b.t0, dmul(0.5, g.h));
        return true;
    }

    // false when the ray (t >= 0) misses the bounding box of the allocated
    // tiles (with a one-voxel margin): then no lattice point lies in an
    // allocated tile and march_ray yields no sample.  Call after init().
    __device__ __forceinline__ bool may_hit(const GridView& g) const {
        if (!g.occ_any) return false;
        return ray_box(d3(o[0], o[1], o[2]), d3(d[0], d[1], d[2]), d3(inv_d[0], inv_d[1], inv_d[2]),
                       d3(g.occ_lo[0], g.occ_lo[1], g.occ_lo[2]), d3(g.occ_hi[0], g.occ_hi[1], g.occ_hi[2]))
            .ok;
    }

    // may_hit(), and when the ray does meet the allocated tiles' bounding box
    // (one-voxel margin) further along, a jump (lattice argument, as in
    // next_impl) to the last lattice point before it: every lattice point up
    // to there lies in unallocated tiles.  Call right after init().
    __device__ __forceinline__ bool enter_occupied(const GridView& g) {
        if (!g.occ_any) return false;
        const BoxHit b = ray_box(d3(o[0], o[1], o[2]), d3(d[0], d[1], d[2]), d3(inv_d[0], inv_d[1], inv_d[2]),
                                 d3(g.occ_lo[0], g.occ_lo[1], g.occ_lo[2]),
                                 d3(g.occ_hi[0], g.occ_hi[1], g.occ_hi[2]));
        if (!b.ok) return false;
        if (g.h_pow2 && t >= 64.0 * g.h && b.t0 > t) {
            const double m = floor((b.t0 - t) * g.inv_h) - 1.0;
            if (m >= 2.0) {
                PSDF_STAT(4);
                t_sync = t;
                t = lattice_advance(t, m, g.h);
            }
        }
        return true;
    }

    // A jump to the last lattice point before `tl`, a lower bound on the
    // distance at which the ray can first meet an allocated tile (the scan's
    // per-work-tile bound, tile_raster_kernel): every lattice point it passes
    // lies in unallocated tiles, so the lattice argument of next_impl's jumps
    // applies (the marcher stays desynchronised until its next tile skip and
    // rewinds to t_sync on an ambiguous decision).  Call after init() /
    // enter_occupied().
    __device__ __forceinline__ void jump_to(const GridView& g, double tl) {
        if (g.h_pow2 && t >= 64.0 * g.h && tl > t) {
            const double m = floor((tl - t) * g.inv_h) - 1.0;
            if (m >= 2.0) {
                PSDF_STAT(4);
                if (t_sync < 0.0) t_sync = t;
                t = lattice_advance(t, m, g.h);
            }
        }
    }

    // Resumes a ray whose box exit t1 is known (the caller sets t and count
    // to a point the reference visited).
    __device__ __forceinline__ void init_from(const GridView& g, const double* o_, const double* d_,
                                              int nmax, double t1_) {
        setup(g, o_, d_, nmax);
        t1 = t1_;
        t = t1_;
    }

    // Rewinds to the reference's last visited point (after an ambiguous
    // decision while desynchronised); returns false if synchronised.
    __device__ __forceinline__ bool rewind() {
        if (t_sync < 0.0) return false;
        PSDF_STAT(7);
        t = t_sync;
        t_sync = -1.0;
        no_jump = true;
        return true;
    }

    // Lattice points t + j h (j >= 0) still inside the current tile and
    // before the box exit t1, each at least the decision margin (in voxels)
    // off every face of the tile — so the fast form's tile is the exact one
    // for all of them, also on a ray that runs along a face (the per-axis
    // exit distance divided by |d_a|, the voxels the ray advances per
    // lattice step along a) — or 1 when t itself is that close to a face or
    // the box exit is within its margin (then the caller steps one sample at
    // a time).  Only with the lattice preconditions (power-of-two h, t >= 64 h).
    __device__ __forceinline__ double run_length(const GridView& g, const double v[3], double t,
                                                 double h) const {
        if (!g.h_pow2 || t < 64.0 * h) return 1.0;
        const double M = g.margin + 1e-9;  // voxels: decision margin + the fast form's error
        double n = 1e300;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double r = v[a] - 16.0 * floor(v[a] * 0.0625);
            if (r <= M || r >= 16.0 - M) return 1.0;
            // |d_a| voxels per lattice step along a; 1/|d_a| from the
            // correctly rounded reciprocal, shrunk by 1e-13 so the floor never
            // exceeds the exact quotient (the margin absorbs the rest)
            if (inv_d[a] == 0.0) continue;  // parallel to the faces: r stays put
            const double dist = d[a] > 0.0 ? 16.0 - r : r;  // voxels to the exit face
            n = fmin(n, floor((dist - M) * fabs(inv_d[a]) * (1.0 - 1e-13)) + 1.0);
        }
        // the reference's own loop test t_j < t1, t_j = t + j h exactly
        const double r1 = (t1 - t) * g.inv_h;
        const double f1 = r1 - floor(r1);
        if (f1 <= 1e-9 || f1 >= 1.0 - 1e-9) return 1.0;
        return fmax(1.0, fmin(n, ceil(r1)));
    }

    // Next sample distance inside an allocated tile; false when exhausted.
    // `bits` is the tile occupancy bitmap (usually a shared-memory copy), so
    // skipping empty tiles needs no global memory access.
    __device__ __forceinline__ bool next(const GridView& g, double& t_out, int& tile_out,
                                         const uint32_t* bits, int4* tc_out = nullptr) {
        SampleRun run;
        return next_impl<false>(g, t_out, tile_out, bits, tc_out, 0.0, run);
    }

    // As next(), but when the sample's tile is saturated — tau * (minimum of
    // its apron brick) >= kSatX, so every sample in it has sigmoid exactly 1
    // and alpha exactly 0 — returns the whole run of the ray's consecutive
    // lattice points in that tile at once: run.n samples from t_out to
    // run.t_last (the reference visits them one by one with t += h; the
    // count is exact, the t values follow from the lattice argument above).
    __device__ __forceinline__ bool next_run(const GridView& g, double& t_out, int& tile_out,
                                             const uint32_t* bits, int4* tc_out, double tau,
                                             SampleRun& run) {
        return next_impl<true>(g, t_out, tile_out, bits, tc_out, tau, run);
    }

    template <bool RUNS>
    __device__ __forceinline__ bool next_impl(const GridView& g, double& t_out, int& tile_out,
                                              const uint32_t* bits, int4* tc_out, double tau,
                                              SampleRun& run) {
        const double h = g.h;
        const double kMargin = g.margin;  // voxels (1e-8); the FMA form is within ~1e-12
        while (t < t1 && count < n_max) {
            PSDF_STAT(2);
            // --- tile of p(t)
            double v[3], r[3];
            int tc[3];
            bool near = false;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                v[a] = fma(vd[a], t, vo[a]);
                const double fl16 = floor(v[a] * 0.0625);
                r[a] = v[a] - 16.0 * fl16;  // position inside the tile, [0, 16)
                near |= r[a] < kMargin || r[a] > 16.0 - kMargin;
                tc[a] = (int)fl16;
            }
            if (near) {
                if (rewind()) continue;
                const int4 e = exact_tile(lite(g), d3(o[0], o[1], o[2]), d3(d[0], d[1], d[2]), t);
                tc[0] = e.x;
                tc[1] = e.y;
                tc[2] = e.z;
                ++n_exact;
            }
            bool occupied = false, in_grid = false;
            int b = 0;
            if ((unsigned)tc[0] < (unsigned)g.nt[0] && (unsigned)tc[1] < (unsigned)g.nt[1] &&
                (unsigned)tc[2] < (unsigned)g.nt[2]) {
                in_grid = true;
                b = (tc[0] * g.nt[1] + tc[1]) * g.nt[2] + tc[2];
                occupied = (bits[b >> 5] >> (b & 31)) & 1u;
            }
            if (occupied) {
                // a sample: only reachable synchronised (jumps never cross an
                // allocated tile)
                PSDF_STAT(3);
                t_out = t;
                if (b != c_b) {  // consecutive samples mostly share the tile
                    c_b = b;
                    c_tile = __ldg(g.tile_table + b);
                }
                tile_out = c_tile;
                if (tc_out) *tc_out = make_int4(tc[0], tc[1], tc[2], 0);
                if constexpr (RUNS) {
                    run.n = 1;
                    run.sat = false;
                    run.t_last = t;
                    if (!near && tau > 0.0) {
                        // the trilinear cell holding the sample (c = v - 1/2
                        // off the cell faces by the margin) and its
                        // saturation distance Ds: every lattice point within
                        // L-inf (Ds - 1) + (distance to the cell faces)
                        // voxels, up to the tile exit, lies in a saturated
                        // cell
                        // (the distance to the cell faces only shortens the
                        // run: fp32 with a 1e-5 voxel allowance)
                        int ci = 0;
                        bool ok = true;
                        float edge = 1.f;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const double cc = r[a] - 0.5;
                            const double fb = floor(cc);
                            const double f = cc - fb;
                            ok &= f > kMargin && f < 1.0 - kMargin;
                            const float ff = (float)f;
                            edge = fminf(edge, fminf(ff, 1.f - ff));
                            ci = ci * kCellE + ((int)fb + 1);
                        }
                        int ds = 0;
                        if (ok) {
                            const int blk = tile_out * kCellN + ci;
                            if (blk != c_blk) {
                                c_blk = blk;
                                c_ds = __ldg(g.sat_dist + blk);
                            }
                            ds = c_ds;
                        }
                        if (ds > 0) {
                            run.sat = true;
                            double n = run_length(g, v, t, h);  // lattice points left in the tile
                            if (ds != kCellNone)
                                n = fmin(n, floor(((double)(ds - 1) + (double)edge - 1e-5) * dinv_max) + 1.0);
                            if (n > 1.0) {
                                const int ni = (int)fmin(n, (double)(n_max - count));
                                run.n = ni;
                                if (ni > 1) run.t_last = lattice_advance(t, (double)(ni - 1), h);
                            }
                        }
                    }
#ifdef PSDF_MARCH_STATS
                    if (run.sat) {
                        PSDF_STAT(8);
                        atomicAdd(&g_march_stats[9], (unsigned long long)run.n);
                    }
#endif
                    t = dadd(run.t_last, h);
                    count += run.n;
                    return true;
                }
                t = dadd(t, h);
                ++count;
                return true;
            }
            // --- jump through the empty L-inf ball around p(t): every
            // lattice point within m steps moves at most m max|d_a| voxels
            // (the lattice argument needs a power-of-two h and t >= 64 h)
            if (in_grid && !near && !no_jump && g.h_pow2 && t >= 64.0 * h) {
                const int D = __ldg(g.tile_dist + b);
                if (D >= 2) {
                    float edge = 16.f;  // fp32 with a 1e-5 voxel allowance (it only shortens the jump)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const float rf = (float)r[a];
                        edge = fminf(edge, fminf(rf, 16.f - rf));
                    }
                    const double m = floor((16.0 * (D - 1) + (double)edge - 1e-5) * dinv_max);
                    if (m >= 2.0) {
                        PSDF_STAT(4);
                        if (t_sync < 0.0) t_sync = t;
                        t = lattice_advance(t, m, h);
                        continue;
                    }
                }
            }
            // --- skip the empty tile.  p(t) is inside the tile and off its
            // faces (not `near`), so the box test passes and e1 > t; the skip
            // is ceil(q + 1e-9) with q = (e1 - t)/h = min_a (B_a - v_a) / d_a.
            double q = 1e300;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (inv_d[a] == 0.0) continue;
                const double B = 16.0 * (double)(tc[a] + (d[a] > 0.0 ? 1 : 0));
                q = fmin(q, (B - v[a]) * inv_d[a]);
            }
            const double fq = q - floor(q);
            const double mq = kMargin + 1e-11 * rinv_max;  // q error <~ 1e-12 |1/d|
            if (!near && q < 1e300 && fq > mq && fq < 1.0 - mq) {
                const double k = ceil(q);  // the + 1e-9 is inside the margin
                t = dadd(t, dmul(k > 1.0 ? k : 1.0, h));
                PSDF_STAT(5);
                t_sync = -1.0;  // the reference lands on the same lattice point
                no_jump = false;
                continue;
            }
            if (rewind()) continue;
            PSDF_STAT(6);
            t = exact_skip(lite(g), d3(o[0], o[1], o[2]), d3(d[0], d[1], d[2]), tc[0], tc[1], tc[2], t);
            no_jump = false;
            ++n_exact;
        }
        return false;
    }

    __device__ __forceinline__ void pos(double tt, double p[3]) const {
#pragma unroll
        for (int a = 0; a < 3; ++a) p[a] = dadd(o[a], dmul(d[a], tt));
    }
};

// sigmoid (renderer.cpp:10) and alpha_from_sdf (renderer.cpp:35-39), f64.
// __drcp_rn is the correctly rounded reciprocal, i.e. the same value as 1.0/x.
#ifdef PSDF_ABL_EXPF
__device__ __forceinline__ double sigmoid_d(double x) { return 1.0 / (1.0 + (double)__expf((float)-x)); }
#else
__device__ __forceinline__ double sigmoid_d(double x) { return __drcp_rn(dadd(1.0, exp(-x))); }
#endif
// sigmoid_d with the saturation shortcut: bit-identical (see kSatX).
__device__ __forceinline__ double sigmoid_sat(double x) { return x >= kSatX ? 1.0 : sigmoid_d(x); }

__device__ __forceinline__ double alpha_from(double a, double b) {
#ifdef PSDF_ABL_ALPHA
    const double al = (a - b) * __drcp_rn(a);
#else
    const double al = ddiv_fast(dsub(a, b), a);
#endif
    return al > 0.0 ? al : 0.0;
}

// ---------------------------------------------------------------- decode
// SH constants (sh.cpp:12-21)
constexpr float K0 = 0.28209479177387814f, K1 = 0.4886025119029199f, K2A = 1.0925484305920792f,
                K2B = 0.31539156525252005f, K2C = 0.5462742152960396f, K3A = 0.5900435899266435f,
                K3B = 2.890611442640554f, K3C = 0.4570457994644658f, K3D = 0.3731763325901154f,
                K3E = 1.445305721320277f;

// eval_sh_basis (sh.cpp:30-54); entries >= order^2 are left untouched.
__device__ __forceinline__ void sh_basis(float x, float y, float z, int order, float* Y) {
    Y[0] = K0;
    if (order < 2) return;
    Y[1] = K1 * y;
    Y[2] = K1 * z;
    Y[3] = K1 * x;
    if (order < 3) return;
    Y[4] = K2A * x * y;
    Y[5] = K2A * y * z;
    Y[6] = K2B * (3.f * z * z - 1.f);
    Y[7] = K2A * x * z;
    Y[8] = K2C * (x * x - y * y);
    if (order < 4) return;
    Y[9] = K3A * y * (3.f * x * x - y * y);
    Y[10] = K3B * x * y * z;
    Y[11] = K3C * y * (5.f * z * z - 1.f);
    Y[12] = K3D * z * (5.f * z * z - 3.f);
    Y[13] = K3C * x * (5.f * z * z - 1.f);
    Y[14] = K3E * z * (x * x - y * y);
    Y[15] = K3A * x * (x * x - 3.f * y * y);
}

// d/d(refl) of sum_j s_j Y_j (sh.cpp:56-83 contracted with s)
__device__ __forceinline__ void sh_basis_grad_dot(float x, float y, float z, int order,
                                                  const float* s, float& gx, float& gy,
                                                  float& gz) {
    gx = gy = gz = 0.f;
    if (order < 2) return;
    gy += s[1] * K1;
    gz += s[2] * K1;
    gx += s[3] * K1;
    if (order < 3) return;
    gx += s[4] * K2A * y;           gy += s[4] * K2A * x;
    gy += s[5] * K2A * z;           gz += s[5] * K2A * y;
    gz += s[6] * K2B * 6.f * z;
    gx += s[7] * K2A * z;           gz += s[7] * K2A * x;
    gx += s[8] * K2C * 2.f * x;     gy += s[8] * (-K2C * 2.f * y);
    if (order < 4) return;
    gx += s[9] * K3A * 6.f * x * y; gy += s[9] * K3A * (3.f * x * x - 3.f * y * y);
    gx += s[10] * K3B * y * z;      gy += s[10] * K3B * x * z;       gz += s[10] * K3B * x * y;
    gy += s[11] * K3C * (5.f * z * z - 1.f);                         gz += s[11] * K3C * 10.f * y * z;
    gz += s[12] * K3D * (15.f * z * z - 3.f);
    gx += s[13] * K3C * (5.f * z * z - 1.f);                         gz += s[13] * K3C * 10.f * x * z;
    gx += s[14] * K3E * 2.f * x * z; gy += s[14] * (-K3E * 2.f * y * z); gz += s[14] * K3E * (x * x - y * y);
    gx += s[15] * K3A * 3.f * (x * x - y * y); gy += s[15] * (-K3A * 6.f * x * y);
}

// Bilinear tap (grid.cpp:148-158), computed in f64 then narrowed.
struct Tap {
    int a0;
    float f;
};
__device__ __forceinline__ Tap plane_tap(double local) {
    double u = dsub(local, 0.5);
    u = u < 0.0 ? 0.0 : (u > 15.0 ? 15.0 : u);
    int a0 = (int)u;
    if (a0 > 14) a0 = 14;
    return Tap{a0, (float)dsub(u, (double)a0)};
}

// Fixed-size vector helpers for n_s / n_a channel groups.
template <int N>
struct VecF {
    float v[N];
};
template <int N>
__device__ __forceinline__ VecF<N> ldg_vec(const float* p) {
    VecF<N> r;
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(p) + i);
            r.v[4 * i] = q.x;
            r.v[4 * i + 1] = q.y;
            r.v[4 * i + 2] = q.z;
            r.v[4 * i + 3] = q.w;
        }
    } else if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const float2 q = __ldg(reinterpret_cast<const float2*>(p) + i);
            r.v[2 * i] = q.x;
            r.v[2 * i + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) r.v[i] = __ldg(p + i);
    }
    return r;
}

// The same from shared memory (a staged block).
template <int N>
__device__ __forceinline__ VecF<N> lds_vec(const float* p) {
    VecF<N> r;
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const float4 q = reinterpret_cast<const float4*>(p)[i];
            r.v[4 * i] = q.x;
            r.v[4 * i + 1] = q.y;
            r.v[4 * i + 2] = q.z;
            r.v[4 * i + 3] = q.w;
        }
    } else if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const float2 q = reinterpret_cast<const float2*>(p)[i];
            r.v[2 * i] = q.x;
            r.v[2 * i + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) r.v[i] = p[i];
    }
    return r;
}

// Vector atomics (sm_90+ float2/float4 red.global.add).
template <int N>
__device__ __forceinline__ void red_vec(float* p, const float* v) {
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i)
            atomicAdd(reinterpret_cast<float4*>(p) + i,
                      make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
    } else if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i)
            atomicAdd(reinterpret_cast<float2*>(p) + i, make_float2(v[2 * i], v[2 * i + 1]));
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) atomicAdd(p + i, v[i]);
    }
}

// scatter_smooth_grad (grads.cpp:47-65): trilinear transpose into the
// smooth-staged SDF gradient; weights in f64 exactly as the forward sample.
__device__ __forceinline__ void scatter_smooth(const GridView& g, float* __restrict__ gsm,
                                               double px, double py, double pz, double gv) {
    const double cx = dsub(w2v(g, px, 0), 0.5);
    const double cy = dsub(w2v(g, py, 1), 0.5);
    const double cz = dsub(w2v(g, pz, 2), 0.5);
    const int bx = (int)floor(cx), by = (int)floor(cy), bz = (int)floor(cz);
    const double fx = dsub(cx, (double)bx), fy = dsub(cy, (double)by), fz = dsub(cz, (double)bz);
    const double gx0 = dsub(1.0, fx), gy0 = dsub(1.0, fy), gz0 = dsub(1.0, fz);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const double w = dmul(dmul((i & 1) ? fx : gx0, (i & 2) ? fy : gy0), (i & 4) ? fz : gz0);
        if (w == 0.0) continue;
        const int vx = bx + (i & 1), vy = by + ((i >> 1) & 1), vz = bz + ((i >> 2) & 1);
        if (vx < 0 || vy < 0 || vz < 0 || vx >= g.res[0] || vy >= g.res[1] || vz >= g.res[2])
            continue;
        const int t = tile_lookup(g, vx >> 4, vy >> 4, vz >> 4);
        if (t < 0) continue;
        atomicAdd(gsm + (int64_t)t * TV + vox_index(vx & 15, vy & 15, vz & 15), (float)(w * gv));
    }
}

// scatter_smooth at a sample p of tile `tile` (coordinates tc): every corner
// lies in the tile's brick, so the owning tiles come from g.tile_nbr (no
// table lookups, all eight inside the tile in the common case).
__device__ __forceinline__ void scatter_smooth_in(const GridView& g, float* __restrict__ gsm, int tile,
                                                  int4 tc, const double p[3], double gv) {
    const double cx = dsub(w2v(g, p[0], 0), 0.5);
    const double cy = dsub(w2v(g, p[1], 1), 0.5);
    const double cz = dsub(w2v(g, p[2], 2), 0.5);
    const int bx = (int)floor(cx), by = (int)floor(cy), bz = (int)floor(cz);
    const double fx = dsub(cx, (double)bx), fy = dsub(cy, (double)by), fz = dsub(cz, (double)bz);
    const double gx0 = dsub(1.0, fx), gy0 = dsub(1.0, fy), gz0 = dsub(1.0, fz);
    const int lx = bx - 16 * tc.x, ly = by - 16 * tc.y, lz = bz - 16 * tc.z;  // in [-1, 15]
    const bool inside = (unsigned)lx < 15u && (unsigned)ly < 15u && (unsigned)lz < 15u;
    const int32_t* nbr = g.tile_nbr + (int64_t)tile * 27;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const double w = dmul(dmul((i & 1) ? fx : gx0, (i & 2) ? fy : gy0), (i & 4) ? fz : gz0);
        if (w == 0.0) continue;
        const int vx = lx + (i & 1), vy = ly + ((i >> 1) & 1), vz = lz + ((i >> 2) & 1);
        int t = tile;
        if (!inside) {
            t = __ldg(nbr + (((vx >> 4) + 1) * 3 + ((vy >> 4) + 1)) * 3 + ((vz >> 4) + 1));
            if (t < 0) continue;
        }
        atomicAdd(gsm + (int64_t)t * TV + vox_index(vx & 15, vy & 15, vz & 15), (float)(w * gv));
    }
}

// The six scatter_smooth_grad calls of the normal chain (renderer.cpp:216-235:
// +-c_a at p +- h e_a) merged: the shifted points share p's trilinear
// fractions (a shift by one voxel moves the base corner by one), so their
// 48 corner deposits fall on 32 distinct voxels — the 2^3 core around p and
// a 4-voxel arm at -1 and +2 along each axis.  Neighbour tiles come from
// g.tile_nbr (every voxel is within 2 of the sample's voxel, which lies in
// `tile`); unallocated / outside voxels are skipped like smooth_value.
__device__ __forceinline__ void scatter_gradient_stencil(const GridView& g, float* __restrict__ gsm,
                                                         int tile, const double p[3], double c0,
                                                         double c1, double c2) {
    // gradient deposits are fp32 (tolerance 1e-3): fp32 weights and
    // coefficients; the fractions come from the f64 position
    const float cc[3] = {(float)c0, (float)c1, (float)c2};
    int b[3];
    float f[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = dsub(w2v(g, p[a], a), 0.5);
        b[a] = (int)floor(x);
        f[a] = (float)dsub(x, (double)b[a]);
    }
    auto wgt = [&](int ox, int oy, int oz) {
        return (ox ? f[0] : 1.f - f[0]) * (oy ? f[1] : 1.f - f[1]) * (oz ? f[2] : 1.f - f[2]);
    };
    const int4 tc = __ldg(g.tile_coords + tile);
    const int32_t* nbr = g.tile_nbr + (int64_t)tile * 27;
    // all 4^3 stencil voxels (b - 1 .. b + 2) inside the sample's own tile:
    // no neighbour lookups (about half of the samples)
    const bool inside = (unsigned)(b[0] - 16 * tc.x - 1) <= 12u && (unsigned)(b[1] - 16 * tc.y - 1) <= 12u &&
                        (unsigned)(b[2] - 16 * tc.z - 1) <= 12u;
    float* own = gsm + (int64_t)tile * TV;
    auto deposit = [&](int dx, int dy, int dz, float v) {
        if (v == 0.f) return;
        const int vx = b[0] + dx, vy = b[1] + dy, vz = b[2] + dz;
        if (inside) {
            atomicAdd(own + vox_index(vx & 15, vy & 15, vz & 15), v);
            return;
        }
        const int n = __ldg(nbr + (((vx >> 4) - tc.x + 1) * 3 + ((vy >> 4) - tc.y + 1)) * 3 + ((vz >> 4) - tc.z + 1));
        if (n < 0) return;
        atomicAdd(gsm + (int64_t)n * TV + vox_index(vx & 15, vy & 15, vz & 15), v);
    };
    // core: +c_a w(o - e_a) where o_a = 1, -c_a w(o + e_a) where o_a = 0
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int o[3] = {i & 1, (i >> 1) & 1, (i >> 2) & 1};
        float v = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            int q[3] = {o[0], o[1], o[2]};
            q[a] ^= 1;
            v += (o[a] ? cc[a] : -cc[a]) * wgt(q[0], q[1], q[2]);
        }
        deposit(o[0], o[1], o[2], v);
    }
    // arms: +c_a w(o') at o' + e_a (o'_a = 1), -c_a w(o') at o' - e_a (o'_a = 0)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int o[3];
            o[a] = 1;
            o[(a + 1) % 3] = i & 1;
            o[(a + 2) % 3] = (i >> 1) & 1;
            const float wp = wgt(o[0], o[1], o[2]);
            int d[3] = {o[0], o[1], o[2]};
            d[a] = 2;
            deposit(d[0], d[1], d[2], cc[a] * wp);
            o[a] = 0;
            const float wn = wgt(o[0], o[1], o[2]);
            d[a] = -1;
            deposit(d[0], d[1], d[2], -cc[a] * wn);
        }
    }
}

}  // namespace psdf
