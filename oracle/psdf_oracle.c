/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C f64 restatement of the reference hot path (see psdf_oracle.h).
 * Every function cites the reference file:line it follows; operation order in
 * f64 follows the reference so that, fed the same inputs, the forward pass is
 * bit-identical to the reference (the ray t-lists are required to be).
 * Compiled WITHOUT FMA contraction (oracle/Makefile).
 */
#include "psdf_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define TE 16            /* kTileEdge, grid.hpp:15 */
#define TV 4096          /* kTileVoxels */
#define HID 32           /* kHidden, decoder.hpp:11 */
#define NPOW 6           /* kFresnelPowers */
#define MAXIN 64
#define PHOTO_EPS 1e-3   /* kPhotoEps, losses.hpp:9 */

struct OGrid {
    int T, P, n_s, n_a, order, res[3], nt[3], ncam, in_dim;
    double h, origin[3], ffv;
    int32_t *tile_table, *probe_table, *tile_coords, *probe_ids, *probe_coords;
    double *raw, *smooth, *planes, *probes, *mlp;
    int64_t mlp_size;
    /* Adam (adam.hpp:11-42); one flat state over raw|planes|probes|mlp */
    double *am, *av;
    long at;
};

typedef struct { double x, y, z; } V3;
static V3 v3(double x, double y, double z) { V3 r = {x, y, z}; return r; }
static V3 vadd(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static V3 vmul(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
static V3 vdiv(V3 a, double s) { return v3(a.x / s, a.y / s, a.z / s); }
static double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; } /* vec.hpp:26 */
static double vnorm(V3 a) { return sqrt(vdot(a, a)); }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
static double maxd(double a, double b) { return a > b ? a : b; }

static double far_field(const OGrid* g) { return g->ffv * g->h; } /* grid.hpp:71 */
static V3 world_to_voxel(const OGrid* g, V3 p) {                  /* grid.hpp:126 */
    return vdiv(vsub(p, v3(g->origin[0], g->origin[1], g->origin[2])), g->h);
}
static int64_t plane_stride(const OGrid* g) { return 256LL * g->n_s; }
static int64_t probe_stride(const OGrid* g) { return (int64_t)g->order * g->order * g->n_a; }

/* decoder.hpp:17-31 field offsets in the flat MLP buffer */
typedef struct { int64_t w1, b1, w2, b2, w3, b3, cam; } MlpOff;
static MlpOff mlp_off(const OGrid* g) {
    MlpOff o;
    o.w1 = 0;
    o.b1 = o.w1 + (int64_t)HID * g->in_dim;
    o.w2 = o.b1 + HID;
    o.b2 = o.w2 + HID * HID;
    o.w3 = o.b2 + HID;
    o.b3 = o.w3 + 3 * HID;
    o.cam = o.b3 + 3;
    return o;
}

static int tile_index(const OGrid* g, int tx, int ty, int tz) { /* grid.cpp:24-27 */
    if (tx < 0 || ty < 0 || tz < 0 || tx >= g->nt[0] || ty >= g->nt[1] || tz >= g->nt[2]) return -1;
    return g->tile_table[((int64_t)tx * g->nt[1] + ty) * g->nt[2] + tz];
}
static int probe_index(const OGrid* g, int gx, int gy, int gz) { /* grid.cpp:39-42 */
    if (gx < 0 || gy < 0 || gz < 0 || gx > g->nt[0] || gy > g->nt[1] || gz > g->nt[2]) return -1;
    return g->probe_table[((int64_t)gx * (g->nt[1] + 1) + gy) * (g->nt[2] + 1) + gz];
}
static int vidx(int x, int y, int z) { return (x * TE + y) * TE + z; } /* grid.hpp:37 */

static int in_res(const OGrid* g, int vx, int vy, int vz) {
    return vx >= 0 && vy >= 0 && vz >= 0 && vx < g->res[0] && vy < g->res[1] && vz < g->res[2];
}
static double raw_value(const OGrid* g, int vx, int vy, int vz) { /* grid.cpp:78-85 */
    if (!in_res(g, vx, vy, vz)) return far_field(g);
    int t = tile_index(g, vx >> 4, vy >> 4, vz >> 4);
    if (t < 0) return far_field(g);
    return g->raw[(int64_t)t * TV + vidx(vx & 15, vy & 15, vz & 15)];
}
static double smooth_value(const OGrid* g, int vx, int vy, int vz) { /* grid.cpp:87-94 */
    if (!in_res(g, vx, vy, vz)) return far_field(g);
    int t = tile_index(g, vx >> 4, vy >> 4, vz >> 4);
    if (t < 0) return far_field(g);
    return g->smooth[(int64_t)t * TV + vidx(vx & 15, vy & 15, vz & 15)];
}

/* grid.cpp:98-125 (sample_trilinear over the smoothed field; `inside` unused
 * on the hot path) */
static double sample_sdf(const OGrid* g, V3 p) {
    V3 c = vsub(world_to_voxel(g, p), v3(0.5, 0.5, 0.5));
    int bx = (int)floor(c.x), by = (int)floor(c.y), bz = (int)floor(c.z);
    double fx = c.x - bx, fy = c.y - by, fz = c.z - bz;
    double v = 0.0;
    for (int i = 0; i < 8; ++i) {
        double w = ((i & 1) ? fx : 1.0 - fx) * ((i & 2) ? fy : 1.0 - fy) * ((i & 4) ? fz : 1.0 - fz);
        v += w * smooth_value(g, bx + (i & 1), by + ((i >> 1) & 1), bz + ((i >> 2) & 1));
    }
    return v;
}

/* grid.cpp:10-22 */
static void gaussian_taps(double w[5]) {
    double sum = 0.0;
    for (int d = -2; d <= 2; ++d) {
        w[d + 2] = exp(-0.5 * d * d);
        sum += w[d + 2];
    }
    for (int i = 0; i < 5; ++i) w[i] /= sum;
}

/* grid.cpp:204-245 */
static void smooth_tile(OGrid* g, int t) {
    enum { E = 20 };
    static double a[E * E * E], b[E * E * E];
    double w[5];
    gaussian_taps(w);
    const int32_t* tc = g->tile_coords + 3 * t;
    int ox = tc[0] * TE - 2, oy = tc[1] * TE - 2, oz = tc[2] * TE - 2;
#define AT(buf, x, y, z) buf[((x) * E + (y)) * E + (z)]
    for (int x = 0; x < E; ++x)
        for (int y = 0; y < E; ++y)
            for (int z = 0; z < E; ++z) AT(a, x, y, z) = raw_value(g, ox + x, oy + y, oz + z);
    for (int x = 2; x < E - 2; ++x)
        for (int y = 0; y < E; ++y)
            for (int z = 0; z < E; ++z) {
                double s = 0.0;
                for (int d = -2; d <= 2; ++d) s += w[d + 2] * AT(a, x + d, y, z);
                AT(b, x, y, z) = s;
            }
    for (int x = 2; x < E - 2; ++x)
        for (int y = 2; y < E - 2; ++y)
            for (int z = 0; z < E; ++z) {
                double s = 0.0;
                for (int d = -2; d <= 2; ++d) s += w[d + 2] * AT(b, x, y + d, z);
                AT(a, x, y, z) = s;
            }
    for (int x = 0; x < TE; ++x)
        for (int y = 0; y < TE; ++y)
            for (int z = 0; z < TE; ++z) {
                double s = 0.0;
                for (int d = -2; d <= 2; ++d) s += w[d + 2] * AT(a, x + 2, y + 2, z + 2 + d);
                g->smooth[(int64_t)t * TV + vidx(x, y, z)] = s;
            }
#undef AT
}

void og_smooth_all(OGrid* g) { /* grid.cpp:247-250 */
    for (int t = 0; t < g->T; ++t) smooth_tile(g, t);
}

OGrid* og_create(int T, int P, int n_s, int n_a, int sh_order, const int32_t* res,
                 double voxel_size, const double* origin, double far_field_voxels,
                 const int32_t* tile_coords, const int32_t* probe_ids, const int32_t* probe_coords,
                 const double* raw, const double* smooth, const double* planes,
                 const double* probes, const double* mlp, int ncam) {
    OGrid* g = (OGrid*)calloc(1, sizeof(OGrid));
    g->T = T; g->P = P; g->n_s = n_s; g->n_a = n_a; g->order = sh_order; g->ncam = ncam;
    g->in_dim = n_s + n_a + NPOW;
    for (int i = 0; i < 3; ++i) {
        g->res[i] = res[i];
        g->nt[i] = res[i] / TE;
        g->origin[i] = origin[i];
    }
    g->h = voxel_size;
    g->ffv = far_field_voxels;
    int64_t ntt = (int64_t)g->nt[0] * g->nt[1] * g->nt[2];
    int64_t npt = (int64_t)(g->nt[0] + 1) * (g->nt[1] + 1) * (g->nt[2] + 1);
    g->tile_table = (int32_t*)malloc(sizeof(int32_t) * ntt);
    g->probe_table = (int32_t*)malloc(sizeof(int32_t) * npt);
    for (int64_t i = 0; i < ntt; ++i) g->tile_table[i] = -1;
    for (int64_t i = 0; i < npt; ++i) g->probe_table[i] = -1;
    g->tile_coords = (int32_t*)malloc(sizeof(int32_t) * 3 * (T > 0 ? T : 1));
    g->probe_ids = (int32_t*)malloc(sizeof(int32_t) * 8 * (T > 0 ? T : 1));
    g->probe_coords = (int32_t*)malloc(sizeof(int32_t) * 3 * (P > 0 ? P : 1));
    memcpy(g->tile_coords, tile_coords, sizeof(int32_t) * 3 * T);
    memcpy(g->probe_ids, probe_ids, sizeof(int32_t) * 8 * T);
    memcpy(g->probe_coords, probe_coords, sizeof(int32_t) * 3 * P);
    for (int t = 0; t < T; ++t) {
        const int32_t* c = tile_coords + 3 * t;
        g->tile_table[((int64_t)c[0] * g->nt[1] + c[1]) * g->nt[2] + c[2]] = t;
    }
    for (int p = 0; p < P; ++p) {
        const int32_t* c = probe_coords + 3 * p;
        g->probe_table[((int64_t)c[0] * (g->nt[1] + 1) + c[1]) * (g->nt[2] + 1) + c[2]] = p;
    }
    g->raw = (double*)malloc(sizeof(double) * TV * (T > 0 ? T : 1));
    g->smooth = (double*)malloc(sizeof(double) * TV * (T > 0 ? T : 1));
    g->planes = (double*)malloc(sizeof(double) * 3 * plane_stride(g) * (T > 0 ? T : 1));
    g->probes = (double*)malloc(sizeof(double) * probe_stride(g) * (P > 0 ? P : 1));
    memcpy(g->raw, raw, sizeof(double) * TV * T);
    memcpy(g->planes, planes, sizeof(double) * 3 * plane_stride(g) * T);
    memcpy(g->probes, probes, sizeof(double) * probe_stride(g) * P);
    g->mlp_size = mlp_off(g).cam + (int64_t)ncam * HID;
    g->mlp = (double*)malloc(sizeof(double) * g->mlp_size);
    memcpy(g->mlp, mlp, sizeof(double) * g->mlp_size);
    if (smooth)
        memcpy(g->smooth, smooth, sizeof(double) * TV * T);
    else
        og_smooth_all(g);
    return g;
}

void og_free(OGrid* g) {
    if (!g) return;
    free(g->tile_table); free(g->probe_table); free(g->tile_coords); free(g->probe_ids);
    free(g->probe_coords); free(g->raw); free(g->smooth); free(g->planes); free(g->probes);
    free(g->mlp); free(g->am); free(g->av);
    free(g);
}

int64_t og_mlp_size(const OGrid* g) { return g->mlp_size; }

void og_export(const OGrid* g, double* raw, double* smooth, double* planes, double* probes,
               double* mlp) {
    if (raw) memcpy(raw, g->raw, sizeof(double) * TV * g->T);
    if (smooth) memcpy(smooth, g->smooth, sizeof(double) * TV * g->T);
    if (planes) memcpy(planes, g->planes, sizeof(double) * 3 * plane_stride(g) * g->T);
    if (probes) memcpy(probes, g->probes, sizeof(double) * probe_stride(g) * g->P);
    if (mlp) memcpy(mlp, g->mlp, sizeof(double) * g->mlp_size);
}

/* ------------------------------------------------------------------ march */

/* renderer.cpp:13-31 */
static int ray_box(V3 o, V3 d, V3 bmin, V3 bmax, double* t0, double* t1) {
    const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    const double mn[3] = {bmin.x, bmin.y, bmin.z}, mx[3] = {bmax.x, bmax.y, bmax.z};
    *t0 = 0.0;
    *t1 = DBL_MAX;
    for (int a = 0; a < 3; ++a) {
        if (fabs(dd[a]) < 1e-15) {
            if (oo[a] < mn[a] || oo[a] > mx[a]) return 0;
            continue;
        }
        double ta = (mn[a] - oo[a]) / dd[a], tb = (mx[a] - oo[a]) / dd[a];
        if (ta > tb) { double s = ta; ta = tb; tb = s; }
        *t0 = maxd(*t0, ta);
        *t1 = *t1 < tb ? *t1 : tb; /* std::min(t1, tb) returns t1 unless tb < t1 */
        if (*t0 > *t1) return 0;
    }
    return 1;
}

static V3 grid_origin(const OGrid* g) { return v3(g->origin[0], g->origin[1], g->origin[2]); }
static V3 world_max(const OGrid* g) { /* grid.hpp:72-74 */
    return vadd(grid_origin(g), vmul(v3(g->res[0], g->res[1], g->res[2]), g->h));
}

/* renderer.cpp:55-86 */
int og_march_ray(const OGrid* g, const double* o_, const double* d_, int n_max, double* ts) {
    V3 o = v3(o_[0], o_[1], o_[2]), d = v3(d_[0], d_[1], d_[2]);
    int n = 0;
    double t0, t1;
    if (!ray_box(o, d, grid_origin(g), world_max(g), &t0, &t1)) return 0;
    const double h = g->h;
    const double tile_w = TE * h;
    double t = t0 + 0.5 * h;
    while (t < t1 && n < n_max) {
        V3 p = vadd(o, vmul(d, t));
        V3 v = world_to_voxel(g, p);
        int tx = ((int)floor(v.x)) >> 4, ty = ((int)floor(v.y)) >> 4, tz = ((int)floor(v.z)) >> 4;
        if (tile_index(g, tx, ty, tz) >= 0) {
            ts[n++] = t;
            t += h;
        } else {
            V3 bmin = vadd(grid_origin(g), vmul(v3(tx, ty, tz), tile_w));
            V3 bmax = vadd(bmin, vmul(v3(1, 1, 1), tile_w));
            double e0, e1;
            if (ray_box(o, d, bmin, bmax, &e0, &e1) && e1 > t) {
                double skip = ceil((e1 - t) / h + 1e-9);
                t += maxd(1.0, skip) * h;
            } else {
                t += h;
            }
        }
    }
    return n;
}

/* camera.hpp:14-35 */
void og_pixel_dir(const OCamera* c, double u, double v, double* out) {
    V3 d = v3((u - c->cx) / c->fx, (v - c->cy) / c->fy, 1.0);
    const double* r = c->rot;
    V3 q = v3(r[0] * d.x + r[1] * d.y + r[2] * d.z, r[3] * d.x + r[4] * d.y + r[5] * d.z,
              r[6] * d.x + r[7] * d.y + r[8] * d.z);
    double n = vnorm(q);
    V3 res = n > 0.0 ? vdiv(q, n) : v3(0, 0, 0);
    out[0] = res.x; out[1] = res.y; out[2] = res.z;
}

/* every pixel centre of a camera (test helper, batch of og_pixel_dir) */
void og_pixel_dirs(const OCamera* c, double* out) {
    for (int v = 0; v < c->height; ++v)
        for (int u = 0; u < c->width; ++u)
            og_pixel_dir(c, u + 0.5, v + 0.5, out + 3 * ((size_t)v * c->width + u));
}

/* ----------------------------------------------------------------- decode */

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); } /* renderer.cpp:10 */

/* renderer.cpp:35-39 */
static double alpha_from_sdf(double si, double sn, double tau) {
    double a = sigmoid(tau * si), b = sigmoid(tau * sn);
    return maxd((a - b) / a, 0.0);
}

/* sh.cpp:12-54 */
static const double K0 = 0.28209479177387814, K1 = 0.4886025119029199, K2A = 1.0925484305920792,
                    K2B = 0.31539156525252005, K2C = 0.5462742152960396, K3A = 0.5900435899266435,
                    K3B = 2.890611442640554, K3C = 0.4570457994644658, K3D = 0.3731763325901154,
                    K3E = 1.445305721320277;
static void sh_basis(V3 dir, int order, double* out) {
    const double x = dir.x, y = dir.y, z = dir.z;
    out[0] = K0;
    if (order == 1) return;
    out[1] = K1 * y; out[2] = K1 * z; out[3] = K1 * x;
    if (order == 2) return;
    out[4] = K2A * x * y; out[5] = K2A * y * z; out[6] = K2B * (3.0 * z * z - 1.0);
    out[7] = K2A * x * z; out[8] = K2C * (x * x - y * y);
    if (order == 3) return;
    out[9] = K3A * y * (3.0 * x * x - y * y);
    out[10] = K3B * x * y * z;
    out[11] = K3C * y * (5.0 * z * z - 1.0);
    out[12] = K3D * z * (5.0 * z * z - 3.0);
    out[13] = K3C * x * (5.0 * z * z - 1.0);
    out[14] = K3E * z * (x * x - y * y);
    out[15] = K3A * x * (x * x - 3.0 * y * y);
}
/* sh.cpp:56-83 */
static void sh_basis_grad(V3 dir, int order, double gr[16][3]) {
    const double x = dir.x, y = dir.y, z = dir.z;
#define SETG(j, a, b, c) do { gr[j][0] = (a); gr[j][1] = (b); gr[j][2] = (c); } while (0)
    SETG(0, 0, 0, 0);
    if (order == 1) return;
    SETG(1, 0, K1, 0); SETG(2, 0, 0, K1); SETG(3, K1, 0, 0);
    if (order == 2) return;
    SETG(4, K2A * y, K2A * x, 0);
    SETG(5, 0, K2A * z, K2A * y);
    SETG(6, 0, 0, K2B * 6.0 * z);
    SETG(7, K2A * z, 0, K2A * x);
    SETG(8, K2C * 2.0 * x, -K2C * 2.0 * y, 0);
    if (order == 3) return;
    SETG(9, K3A * 6.0 * x * y, K3A * (3.0 * x * x - 3.0 * y * y), 0);
    SETG(10, K3B * y * z, K3B * x * z, K3B * x * y);
    SETG(11, 0, K3C * (5.0 * z * z - 1.0), K3C * 10.0 * y * z);
    SETG(12, 0, 0, K3D * (15.0 * z * z - 3.0));
    SETG(13, K3C * (5.0 * z * z - 1.0), 0, K3C * 10.0 * x * z);
    SETG(14, K3E * 2.0 * x * z, -K3E * 2.0 * y * z, K3E * (x * x - y * y));
    SETG(15, K3A * 3.0 * (x * x - y * y), -K3A * 6.0 * x * y, 0);
#undef SETG
}

/* sh.cpp:172-181 */
static void trilinear_weights(double fx, double fy, double fz, double w[8]) {
    for (int i = 0; i < 8; ++i) {
        double wx = (i & 1) ? fx : 1.0 - fx;
        double wy = (i & 2) ? fy : 1.0 - fy;
        double wz = (i & 4) ? fz : 1.0 - fz;
        w[i] = wx * wy * wz;
    }
}

/* grid.cpp:148-175 */
typedef struct { int a0, a1; double f; } Tap;
static Tap plane_tap(double local) {
    double u = clampd(local - 0.5, 0.0, TE - 1.0);
    int a0 = (int)u;
    if (a0 > TE - 2) a0 = TE - 2;
    Tap t = {a0, a0 + 1, u - a0};
    return t;
}
static double plane_sample(const double* pl, Tap ta, Tap tb, int n_s, int k) {
    double v00 = pl[(ta.a0 * TE + tb.a0) * n_s + k], v01 = pl[(ta.a0 * TE + tb.a1) * n_s + k];
    double v10 = pl[(ta.a1 * TE + tb.a0) * n_s + k], v11 = pl[(ta.a1 * TE + tb.a1) * n_s + k];
    return (1 - ta.f) * ((1 - tb.f) * v00 + tb.f * v01) + ta.f * ((1 - tb.f) * v10 + tb.f * v11);
}
static void plane_scatter(double* gr, Tap ta, Tap tb, int n_s, int k, double gv) {
    gr[(ta.a0 * TE + tb.a0) * n_s + k] += (1 - ta.f) * (1 - tb.f) * gv;
    gr[(ta.a0 * TE + tb.a1) * n_s + k] += (1 - ta.f) * tb.f * gv;
    gr[(ta.a1 * TE + tb.a0) * n_s + k] += ta.f * (1 - tb.f) * gv;
    gr[(ta.a1 * TE + tb.a1) * n_s + k] += ta.f * tb.f * gv;
}

/* State of one shaded sample (the subset of RaySample/DecodeCache,
 * renderer.hpp:43-62, decoder.hpp:45-49, that the backward needs). */
typedef struct {
    V3 pos, local, gvec, normal, view, refl;
    double glen, n_dot_v;
    int degenerate, tile, order;
    double input[MAXIN], a1[HID], a2[HID], rgb[3];
    double f_s[MAXIN], f_a[MAXIN];
    double wts[8];
} Shade;

/* decoder.cpp:55-59 */
static void fresnel_powers(double ndv, double* out) {
    double u = 1.0 - clampd(ndv, 0.0, 1.0);
    out[0] = 1.0;
    for (int k = 1; k < NPOW; ++k) out[k] = out[k - 1] * u;
}

/* decoder.cpp:61-109 */
static void decode_color(const OGrid* g, const double* f_s, const double* f_a, double ndv,
                         int camera_id, Shade* c) {
    const MlpOff o = mlp_off(g);
    const double* m = g->mlp;
    const int in = g->in_dim;
    for (int i = 0; i < g->n_s; ++i) c->input[i] = f_s[i];
    for (int i = 0; i < g->n_a; ++i) c->input[g->n_s + i] = f_a[i];
    fresnel_powers(ndv, c->input + g->n_s + g->n_a);
    const double* cam = NULL;
    if (camera_id >= 0 && g->ncam > 0 && camera_id < g->ncam) cam = m + o.cam + (int64_t)camera_id * HID;
    for (int j = 0; j < HID; ++j) {
        double z = m[o.b1 + j] + (cam ? cam[j] : 0.0);
        const double* row = m + o.w1 + (int64_t)j * in;
        for (int i = 0; i < in; ++i) z += row[i] * c->input[i];
        c->a1[j] = z > 0.0 ? z : 0.0;
    }
    for (int j = 0; j < HID; ++j) {
        double z = m[o.b2 + j];
        const double* row = m + o.w2 + j * HID;
        for (int i = 0; i < HID; ++i) z += row[i] * c->a1[i];
        c->a2[j] = z > 0.0 ? z : 0.0;
    }
    for (int j = 0; j < 3; ++j) {
        double z = m[o.b3 + j];
        const double* row = m + o.w3 + j * HID;
        for (int i = 0; i < HID; ++i) z += row[i] * c->a2[i];
        c->rgb[j] = 1.0 / (1.0 + exp(-z));
    }
}

/* renderer.cpp:88-147 */
static void decode_fused(const OGrid* g, int tile, V3 pos, V3 view, const ORenderOpts* opt,
                         Shade* c) {
    const int order = opt->sh_order_override > 0
                          ? (opt->sh_order_override < g->order ? opt->sh_order_override : g->order)
                          : g->order;
    const double h = g->h;
    V3 gv;
    gv.x = (sample_sdf(g, vadd(pos, v3(h, 0, 0))) - sample_sdf(g, vsub(pos, v3(h, 0, 0)))) / (2 * h);
    gv.y = (sample_sdf(g, vadd(pos, v3(0, h, 0))) - sample_sdf(g, vsub(pos, v3(0, h, 0)))) / (2 * h);
    gv.z = (sample_sdf(g, vadd(pos, v3(0, 0, h))) - sample_sdf(g, vsub(pos, v3(0, 0, h)))) / (2 * h);
    const double glen = vnorm(gv);
    const int degenerate = glen < 1e-8;
    V3 normal = degenerate ? v3(0, 0, 0) : vdiv(gv, glen);
    V3 refl;
    double ndv;
    if (degenerate) {
        refl = view;
        ndv = 1.0;
    } else {
        refl = vsub(vmul(normal, 2.0 * vdot(normal, view)), view); /* vec.hpp:59-61 */
        ndv = vdot(normal, view);
    }
    double f_s[MAXIN] = {0}, f_a[MAXIN] = {0};
    const int32_t* tc = g->tile_coords + 3 * tile;
    V3 local = vsub(world_to_voxel(g, pos), vmul(v3(tc[0], tc[1], tc[2]), TE));
    const double* pl = g->planes + (int64_t)tile * 3 * plane_stride(g);
    if (!opt->no_spatial) { /* grid.cpp:179-187 */
        Tap tx = plane_tap(local.x), ty = plane_tap(local.y), tz = plane_tap(local.z);
        for (int k = 0; k < g->n_s; ++k) {
            double px = plane_sample(pl, ty, tz, g->n_s, k);
            double py = plane_sample(pl + plane_stride(g), tx, tz, g->n_s, k);
            double pz = plane_sample(pl + 2 * plane_stride(g), tx, ty, g->n_s, k);
            f_s[k] = px * py * pz;
        }
    }
    double w[8];
    trilinear_weights(local.x / TE, local.y / TE, local.z / TE, w);
    if (!opt->no_angular) { /* sh.cpp:104-123 */
        const int nc = order * order, n_a = g->n_a;
        double blended[16 * 64];
        memset(blended, 0, sizeof(double) * nc * n_a);
        for (int i = 0; i < 8; ++i) {
            if (w[i] == 0.0) continue;
            const double* cp = g->probes + (int64_t)g->probe_ids[8 * tile + i] * probe_stride(g);
            for (int t = 0; t < nc * n_a; ++t) blended[t] += w[i] * cp[t];
        }
        double basis[16];
        sh_basis(refl, order, basis);
        for (int k = 0; k < n_a; ++k) f_a[k] = 0.0;
        for (int j = 0; j < nc; ++j)
            for (int k = 0; k < n_a; ++k) f_a[k] += blended[j * n_a + k] * basis[j];
    }
    decode_color(g, f_s, f_a, opt->no_fresnel ? 1.0 : ndv, opt->camera_id, c);
    c->pos = pos; c->local = local; c->gvec = gv; c->glen = glen; c->degenerate = degenerate;
    c->normal = normal; c->view = view; c->refl = refl; c->n_dot_v = ndv; c->tile = tile;
    c->order = order;
    memcpy(c->f_s, f_s, sizeof f_s);
    memcpy(c->f_a, f_a, sizeof f_a);
    memcpy(c->wts, w, sizeof w);
}

/* --------------------------------------------------------------- render */

typedef struct {
    double t, sdf, alpha, trans, weight;
    V3 pos;
    int shaded, tile;
    double color[3];
} Sample;

typedef struct {
    Sample* s;
    int n, cap;
    double sdf_extra;
    V3 pos_extra;
    int has_extra;
    Shade* shade; /* per sample, only valid where shaded */
} Ray;

static void ray_reserve(Ray* r, int n) {
    if (n > r->cap) {
        r->s = (Sample*)realloc(r->s, sizeof(Sample) * n);
        r->shade = (Shade*)realloc(r->shade, sizeof(Shade) * n);
        r->cap = n;
    }
}

/* renderer.cpp:149-210; result = color xyz, acc, trans_end, depth */
static int render_ray(const OGrid* g, V3 o, V3 d, const ORenderOpts* opt, Ray* ws, double* result) {
    double ts_buf[4096];
    double* ts = opt->n_max <= 4096 ? ts_buf : (double*)malloc(sizeof(double) * opt->n_max);
    ws->n = 0;
    ws->has_extra = 0;
    result[0] = opt->bg[0]; result[1] = opt->bg[1]; result[2] = opt->bg[2];
    result[3] = 0.0; result[4] = 1.0; result[5] = 0.0;
    const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    int n = og_march_ray(g, oo, dd, opt->n_max, ts);
    if (n == 0) {
        if (ts != ts_buf) free(ts);
        return 0;
    }
    ray_reserve(ws, n);
    const double h = g->h;
    V3 view = v3(-d.x, -d.y, -d.z);
    for (int i = 0; i < n; ++i) {
        Sample* s = &ws->s[i];
        s->t = ts[i];
        s->pos = vadd(o, vmul(d, ts[i]));
        s->sdf = sample_sdf(g, s->pos);
        s->shaded = 0;
        s->tile = -1;
    }
    ws->pos_extra = vadd(o, vmul(d, ts[n - 1] + h));
    ws->sdf_extra = sample_sdf(g, ws->pos_extra);
    ws->has_extra = 1;
    double c[3] = {0, 0, 0}, trans = 1.0, acc = 0.0, depth = 0.0;
    int live = n;
    for (int i = 0; i < n; ++i) {
        Sample* s = &ws->s[i];
        double s_next = (i + 1 < n) ? ws->s[i + 1].sdf : ws->sdf_extra;
        s->alpha = alpha_from_sdf(s->sdf, s_next, opt->tau);
        s->trans = trans;
        s->weight = trans * s->alpha;
        if (opt->need_colors && s->weight > 0.0) {
            V3 v = world_to_voxel(g, s->pos);
            int tx = ((int)floor(v.x)) >> 4, ty = ((int)floor(v.y)) >> 4, tz = ((int)floor(v.z)) >> 4;
            s->tile = tile_index(g, tx, ty, tz);
            if (s->tile >= 0) {
                Shade* sh = &ws->shade[i];
                decode_fused(g, s->tile, s->pos, view, opt, sh);
                s->shaded = 1;
                for (int k = 0; k < 3; ++k) {
                    s->color[k] = sh->rgb[k];
                    c[k] += sh->rgb[k] * s->weight;
                }
            }
        }
        acc += s->weight;
        depth += s->weight * s->t;
        trans *= 1.0 - s->alpha;
        if (opt->early_stop > 0.0 && trans < opt->early_stop) {
            live = i + 1;
            if (live < n) {
                ws->sdf_extra = ws->s[live].sdf;
                ws->pos_extra = ws->s[live].pos;
            }
            break;
        }
    }
    ws->n = live;
    for (int k = 0; k < 3; ++k) result[k] = c[k] + opt->bg[k] * (1.0 - acc);
    result[3] = acc;
    result[4] = trans;
    result[5] = depth;
    if (ts != ts_buf) free(ts);
    return live;
}

int og_render_ray(const OGrid* g, const double* o, const double* d, const ORenderOpts* opt,
                  double* result) {
    Ray ws = {0};
    int n = render_ray(g, v3(o[0], o[1], o[2]), v3(d[0], d[1], d[2]), opt, &ws, result);
    free(ws.s);
    free(ws.shade);
    return n;
}

/* renderer.cpp:321-337 (+ counts and the depth extension) */
void og_render_image(const OGrid* g, const OCamera* cam, const ORenderOpts* opt, double* rgb,
                     double* alpha, double* depth, int64_t* counts) {
    int64_t n_m = 0, n_x = 0, n_sh = 0, n_al = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : n_m, n_x, n_sh, n_al)
    for (int v = 0; v < cam->height; ++v) {
        Ray ws = {0};
        for (int u = 0; u < cam->width; ++u) {
            double d[3], res[6];
            og_pixel_dir(cam, u + 0.5, v + 0.5, d);
            int n = render_ray(g, v3(cam->pos[0], cam->pos[1], cam->pos[2]), v3(d[0], d[1], d[2]),
                               opt, &ws, res);
            int64_t px = (int64_t)v * cam->width + u;
            for (int k = 0; k < 3; ++k) rgb[3 * px + k] = res[k];
            alpha[px] = res[3];
            if (depth) depth[px] = res[5];
            n_m += n;
            n_x += n > 0;
            for (int i = 0; i < n; ++i) {
                n_sh += ws.s[i].shaded;
                n_al += ws.s[i].alpha > 0.0;
            }
        }
        free(ws.s);
        free(ws.shade);
    }
    if (counts) {
        counts[0] = (int64_t)cam->width * cam->height;
        counts[1] = n_m; counts[2] = n_x; counts[3] = n_sh; counts[4] = n_al;
    }
}

/* --------------------------------------------------------------- backward */

OGrads* og_grads_new(const OGrid* g) {
    OGrads* gb = (OGrads*)calloc(1, sizeof(OGrads));
    gb->raw = (double*)calloc((size_t)TV * (g->T ? g->T : 1), sizeof(double));
    gb->smooth = (double*)calloc((size_t)TV * (g->T ? g->T : 1), sizeof(double));
    gb->planes = (double*)calloc((size_t)3 * plane_stride(g) * (g->T ? g->T : 1), sizeof(double));
    gb->probes = (double*)calloc((size_t)probe_stride(g) * (g->P ? g->P : 1), sizeof(double));
    gb->mlp = (double*)calloc((size_t)g->mlp_size, sizeof(double));
    return gb;
}
void og_grads_free(OGrads* gb) {
    if (!gb) return;
    free(gb->raw); free(gb->smooth); free(gb->planes); free(gb->probes); free(gb->mlp);
    free(gb);
}
void og_grads_clear(const OGrid* g, OGrads* gb) {
    memset(gb->raw, 0, sizeof(double) * TV * g->T);
    memset(gb->smooth, 0, sizeof(double) * TV * g->T);
    memset(gb->planes, 0, sizeof(double) * 3 * plane_stride(g) * g->T);
    memset(gb->probes, 0, sizeof(double) * probe_stride(g) * g->P);
    memset(gb->mlp, 0, sizeof(double) * g->mlp_size);
}
void og_grads_export(const OGrid* g, const OGrads* gb, double* raw, double* smooth, double* planes,
                     double* probes, double* mlp) {
    if (raw) memcpy(raw, gb->raw, sizeof(double) * TV * g->T);
    if (smooth) memcpy(smooth, gb->smooth, sizeof(double) * TV * g->T);
    if (planes) memcpy(planes, gb->planes, sizeof(double) * 3 * plane_stride(g) * g->T);
    if (probes) memcpy(probes, gb->probes, sizeof(double) * probe_stride(g) * g->P);
    if (mlp) memcpy(mlp, gb->mlp, sizeof(double) * g->mlp_size);
}

/* grads.cpp:47-65 */
static void scatter_smooth_grad(const OGrid* g, OGrads* gb, V3 p, double gv) {
    V3 c = vsub(world_to_voxel(g, p), v3(0.5, 0.5, 0.5));
    int bx = (int)floor(c.x), by = (int)floor(c.y), bz = (int)floor(c.z);
    double fx = c.x - bx, fy = c.y - by, fz = c.z - bz;
    for (int i = 0; i < 8; ++i) {
        double w = ((i & 1) ? fx : 1.0 - fx) * ((i & 2) ? fy : 1.0 - fy) * ((i & 4) ? fz : 1.0 - fz);
        if (w == 0.0) continue;
        int vx = bx + (i & 1), vy = by + ((i >> 1) & 1), vz = bz + ((i >> 2) & 1);
        if (!in_res(g, vx, vy, vz)) continue;
        int ti = tile_index(g, vx >> 4, vy >> 4, vz >> 4);
        if (ti < 0) continue;
        gb->smooth[(int64_t)ti * TV + vidx(vx & 15, vy & 15, vz & 15)] += w * gv;
    }
}

/* decoder.cpp:111-176 */
static void decode_backward(const OGrid* g, const Shade* c, double ndv, int camera_id,
                            const double up[3], OGrads* gb, double* grad_fs, double* grad_fa,
                            double* grad_ndotv) {
    const MlpOff o = mlp_off(g);
    const double* m = g->mlp;
    double* gm = gb->mlp;
    const int in = g->in_dim;
    double dz3[3];
    for (int j = 0; j < 3; ++j) dz3[j] = up[j] * c->rgb[j] * (1.0 - c->rgb[j]);
    double da2[HID] = {0};
    for (int j = 0; j < 3; ++j) {
        const double* row = m + o.w3 + j * HID;
        double* grow = gm + o.w3 + j * HID;
        for (int i = 0; i < HID; ++i) {
            grow[i] += dz3[j] * c->a2[i];
            da2[i] += dz3[j] * row[i];
        }
        gm[o.b3 + j] += dz3[j];
    }
    double da1[HID] = {0};
    for (int j = 0; j < HID; ++j) {
        if (c->a2[j] <= 0.0) continue;
        const double dz = da2[j];
        const double* row = m + o.w2 + j * HID;
        double* grow = gm + o.w2 + j * HID;
        for (int i = 0; i < HID; ++i) {
            grow[i] += dz * c->a1[i];
            da1[i] += dz * row[i];
        }
        gm[o.b2 + j] += dz;
    }
    double din[MAXIN] = {0};
    double* gcam = NULL;
    if (camera_id >= 0 && g->ncam > 0 && camera_id < g->ncam) gcam = gm + o.cam + (int64_t)camera_id * HID;
    for (int j = 0; j < HID; ++j) {
        if (c->a1[j] <= 0.0) continue;
        const double dz = da1[j];
        const double* row = m + o.w1 + (int64_t)j * in;
        double* grow = gm + o.w1 + (int64_t)j * in;
        for (int i = 0; i < in; ++i) {
            grow[i] += dz * c->input[i];
            din[i] += dz * row[i];
        }
        gm[o.b1 + j] += dz;
        if (gcam) gcam[j] += dz;
    }
    for (int i = 0; i < g->n_s; ++i) grad_fs[i] += din[i];
    for (int i = 0; i < g->n_a; ++i) grad_fa[i] += din[g->n_s + i];
    if (ndv >= 0.0 && ndv <= 1.0) {
        const double u = 1.0 - ndv;
        double du = 0.0, upw = 1.0;
        for (int k = 1; k < NPOW; ++k) {
            du += din[g->n_s + g->n_a + k] * k * upw;
            upw *= u;
        }
        *grad_ndotv += -du;
    }
}

/* renderer.cpp:216-235 */
static void normal_chain_backward(const OGrid* g, OGrads* gb, const Shade* s, V3 d_refl,
                                  double d_ndotv) {
    if (s->degenerate) return;
    V3 n = s->normal, v = s->view;
    V3 dn = vadd(vmul(v, 2.0 * vdot(d_refl, n)), vmul(d_refl, 2.0 * vdot(n, v)));
    dn = vadd(dn, vmul(v, d_ndotv));
    V3 dg = vdiv(vsub(dn, vmul(n, vdot(dn, n))), s->glen);
    const double h = g->h, inv2h = 1.0 / (2.0 * h);
    const V3 axes[3] = {{h, 0, 0}, {0, h, 0}, {0, 0, h}};
    const double comp[3] = {dg.x, dg.y, dg.z};
    for (int a = 0; a < 3; ++a) {
        if (comp[a] == 0.0) continue;
        scatter_smooth_grad(g, gb, vadd(s->pos, axes[a]), comp[a] * inv2h);
        scatter_smooth_grad(g, gb, vsub(s->pos, axes[a]), -comp[a] * inv2h);
    }
}

/* renderer.cpp:239-319 */
static void ray_backward(const OGrid* g, const ORenderOpts* opt, const Ray* ws, const double* upc,
                         double upa, OGrads* gb) {
    const int n = ws->n;
    if (n == 0) return;
    double* dw = (double*)malloc(sizeof(double) * n);
    double* dalpha = (double*)malloc(sizeof(double) * n);
    double* ds = (double*)calloc(n + 1, sizeof(double));
    for (int i = 0; i < n; ++i) {
        const Sample* s = &ws->s[i];
        double ci[3] = {0, 0, 0};
        if (s->shaded) { ci[0] = s->color[0]; ci[1] = s->color[1]; ci[2] = s->color[2]; }
        dw[i] = upc[0] * (ci[0] - opt->bg[0]) + upc[1] * (ci[1] - opt->bg[1]) +
                upc[2] * (ci[2] - opt->bg[2]) + upa;
    }
    double suffix = 0.0;
    for (int ii = n; ii-- > 0;) {
        const Sample* s = &ws->s[ii];
        double term = 0.0;
        if (1.0 - s->alpha > 1e-12) term = suffix / (1.0 - s->alpha);
        dalpha[ii] = dw[ii] * s->trans - term;
        suffix += dw[ii] * s->weight;
    }
    const double tau = opt->tau;
    for (int i = 0; i < n; ++i) {
        const Sample* s = &ws->s[i];
        if (s->alpha <= 0.0 || dalpha[i] == 0.0) continue;
        double s_next = (i + 1 < n) ? ws->s[i + 1].sdf : ws->sdf_extra;
        double a = sigmoid(tau * s->sdf), b = sigmoid(tau * s_next);
        double da = tau * a * (1.0 - a), db = tau * b * (1.0 - b);
        ds[i] += dalpha[i] * b * da / (a * a);
        ds[i + 1] += dalpha[i] * (-db / a);
    }
    if (opt->need_colors) {
        for (int i = 0; i < n; ++i) {
            const Sample* s = &ws->s[i];
            if (!s->shaded || s->tile < 0) continue;
            const Shade* c = &ws->shade[i];
            double up[3] = {upc[0] * s->weight, upc[1] * s->weight, upc[2] * s->weight};
            double gfs[MAXIN] = {0}, gfa[MAXIN] = {0}, dndv_in = 0.0;
            decode_backward(g, c, opt->no_fresnel ? 1.0 : c->n_dot_v, opt->camera_id, up, gb, gfs,
                            gfa, &dndv_in);
            const int n_s = g->n_s, n_a = g->n_a;
            if (!opt->no_spatial) { /* grid.cpp:189-202 */
                const double* pl = g->planes + (int64_t)c->tile * 3 * plane_stride(g);
                double* gp = gb->planes + (int64_t)c->tile * 3 * plane_stride(g);
                Tap tx = plane_tap(c->local.x), ty = plane_tap(c->local.y), tz = plane_tap(c->local.z);
                for (int k = 0; k < n_s; ++k) {
                    double px = plane_sample(pl, ty, tz, n_s, k);
                    double py = plane_sample(pl + plane_stride(g), tx, tz, n_s, k);
                    double pz = plane_sample(pl + 2 * plane_stride(g), tx, ty, n_s, k);
                    double gk = gfs[k];
                    plane_scatter(gp, ty, tz, n_s, k, gk * py * pz);
                    plane_scatter(gp + plane_stride(g), tx, tz, n_s, k, gk * px * pz);
                    plane_scatter(gp + 2 * plane_stride(g), tx, ty, n_s, k, gk * px * py);
                }
            }
            V3 d_refl = v3(0, 0, 0);
            if (!opt->no_angular) { /* sh.cpp:138-170 */
                const int nc = c->order * c->order;
                double basis[16];
                sh_basis(c->refl, c->order, basis);
                for (int i8 = 0; i8 < 8; ++i8) {
                    const double w = c->wts[i8];
                    if (w == 0.0) continue;
                    double* cg = gb->probes + (int64_t)g->probe_ids[8 * c->tile + i8] * probe_stride(g);
                    for (int j = 0; j < nc; ++j) {
                        const double wy = w * basis[j];
                        for (int k = 0; k < n_a; ++k) cg[j * n_a + k] += gfa[k] * wy;
                    }
                }
                double bg[16][3];
                sh_basis_grad(c->refl, c->order, bg);
                V3 gr = v3(0, 0, 0);
                for (int j = 0; j < nc; ++j) {
                    double sacc = 0.0;
                    for (int i8 = 0; i8 < 8; ++i8) {
                        const double w = c->wts[i8];
                        if (w == 0.0) continue;
                        const double* row = g->probes +
                                            (int64_t)g->probe_ids[8 * c->tile + i8] * probe_stride(g) +
                                            (int64_t)j * n_a;
                        for (int k = 0; k < n_a; ++k) sacc += w * row[k] * gfa[k];
                    }
                    gr.x += sacc * bg[j][0];
                    gr.y += sacc * bg[j][1];
                    gr.z += sacc * bg[j][2];
                }
                d_refl = vadd(d_refl, gr);
            }
            const double d_ndotv = opt->no_fresnel ? 0.0 : dndv_in;
            normal_chain_backward(g, gb, c, d_refl, d_ndotv);
        }
    }
    for (int i = 0; i < n; ++i)
        if (ds[i] != 0.0) scatter_smooth_grad(g, gb, ws->s[i].pos, ds[i]);
    if (ds[n] != 0.0 && ws->has_extra) scatter_smooth_grad(g, gb, ws->pos_extra, ds[n]);
    free(dw);
    free(dalpha);
    free(ds);
}

void og_ray_backward(const OGrid* g, const double* o, const double* d, const ORenderOpts* opt,
                     const double* up_color, double up_alpha, OGrads* gb) {
    Ray ws = {0};
    double res[6];
    render_ray(g, v3(o[0], o[1], o[2]), v3(d[0], d[1], d[2]), opt, &ws, res);
    ray_backward(g, opt, &ws, up_color, up_alpha, gb);
    free(ws.s);
    free(ws.shade);
}

/* losses.hpp:11-20 */
static double relative_weight(double a, double b, double eps) { return 1.0 / (maxd(a, b) + eps); }
static double proximity_weight(double s) { return 1.0 / (1.0 + fabs(s) * 5.0); }

/* losses.cpp:8-38 */
void og_photo_pixel(const double* c, const double* gt, int in_mask, double acc, double scale,
                    double* out) {
    for (int i = 0; i < 6; ++i) out[i] = 0.0;
    if (in_mask) {
        for (int k = 0; k < 3; ++k) {
            double d = c[k] - gt[k];
            double w = relative_weight(c[k], gt[k], PHOTO_EPS);
            out[0] += scale * d * d;
            out[1] += scale * w * d * d;
            out[2 + k] = scale * 2.0 * w * d;
        }
    } else {
        double wa = relative_weight(maxd(acc, 0.0), 0.0, PHOTO_EPS);
        out[0] = scale * acc * acc;
        out[1] = scale * wa * acc * acc;
        out[5] = scale * 2.0 * wa * acc;
    }
}

/* ------------------------------------------------------------ regularizers */

/* losses.cpp:61-117 (TileHalo) */
enum { HE = 20 };
typedef struct {
    int ox, oy, oz;
    double val[HE * HE * HE];
    unsigned char alloc[HE * HE * HE];
    double grad[HE * HE * HE];
} Halo;
static int hidx(int x, int y, int z) { return (x * HE + y) * HE + z; }
static void halo_load(const OGrid* g, int t, Halo* hl) {
    const int32_t* tc = g->tile_coords + 3 * t;
    hl->ox = tc[0] * TE - 2; hl->oy = tc[1] * TE - 2; hl->oz = tc[2] * TE - 2;
    for (int x = 0; x < HE; ++x)
        for (int y = 0; y < HE; ++y)
            for (int z = 0; z < HE; ++z) {
                int vx = hl->ox + x, vy = hl->oy + y, vz = hl->oz + z;
                int in = in_res(g, vx, vy, vz) && tile_index(g, vx >> 4, vy >> 4, vz >> 4) >= 0;
                hl->alloc[hidx(x, y, z)] = (unsigned char)in;
                hl->val[hidx(x, y, z)] = in ? smooth_value(g, vx, vy, vz) : far_field(g);
                hl->grad[hidx(x, y, z)] = 0.0;
            }
}
static void halo_flush(const OGrid* g, const Halo* hl, OGrads* gb) {
    for (int x = 0; x < HE; ++x)
        for (int y = 0; y < HE; ++y)
            for (int z = 0; z < HE; ++z) {
                double gv = hl->grad[hidx(x, y, z)];
                if (gv == 0.0 || !hl->alloc[hidx(x, y, z)]) continue;
                int vx = hl->ox + x, vy = hl->oy + y, vz = hl->oz + z;
                int ti = tile_index(g, vx >> 4, vy >> 4, vz >> 4);
                gb->smooth[(int64_t)ti * TV + vidx(vx & 15, vy & 15, vz & 15)] += gv;
            }
}
static V3 halo_grad(const Halo* hl, int x, int y, int z, double inv2h) {
    return v3((hl->val[hidx(x + 1, y, z)] - hl->val[hidx(x - 1, y, z)]) * inv2h,
              (hl->val[hidx(x, y + 1, z)] - hl->val[hidx(x, y - 1, z)]) * inv2h,
              (hl->val[hidx(x, y, z + 1)] - hl->val[hidx(x, y, z - 1)]) * inv2h);
}
static void halo_stencil(Halo* hl, int x, int y, int z, V3 dg, double inv2h) {
    hl->grad[hidx(x + 1, y, z)] += dg.x * inv2h;
    hl->grad[hidx(x - 1, y, z)] -= dg.x * inv2h;
    hl->grad[hidx(x, y + 1, z)] += dg.y * inv2h;
    hl->grad[hidx(x, y - 1, z)] -= dg.y * inv2h;
    hl->grad[hidx(x, y, z + 1)] += dg.z * inv2h;
    hl->grad[hidx(x, y, z - 1)] -= dg.z * inv2h;
}

void og_regularizer_range(const OGrid* g, int which, double lambda, int begin, int end, OGrads* gb,
                          double* out) {
    double plain = 0.0, weighted = 0.0;
    const double inv2h = 1.0 / (2.0 * g->h);
    static Halo hl;
    if (which == 0) { /* loss_sdf, losses.cpp:121-142 */
        for (int t = begin; t < end; ++t)
            for (int v = 0; v < TV; ++v) {
                const double sm = g->smooth[(int64_t)t * TV + v], rw = g->raw[(int64_t)t * TV + v];
                const double r = sm - rw;
                const double w = relative_weight(fabs(sm), fabs(rw), PHOTO_EPS) * proximity_weight(sm);
                plain += lambda * r * r;
                weighted += lambda * w * r * r;
                if (gb) {
                    const double gg = 2.0 * lambda * w * r;
                    gb->smooth[(int64_t)t * TV + v] += gg;
                    gb->raw[(int64_t)t * TV + v] -= gg;
                }
            }
    } else if (which == 1) { /* loss_eikonal, losses.cpp:144-171 */
        for (int t = begin; t < end; ++t) {
            halo_load(g, t, &hl);
            for (int x = 0; x < TE; ++x)
                for (int y = 0; y < TE; ++y)
                    for (int z = 0; z < TE; ++z) {
                        V3 gr = halo_grad(&hl, x + 2, y + 2, z + 2, inv2h);
                        double len = vnorm(gr), e = len - 1.0;
                        double w = proximity_weight(g->smooth[(int64_t)t * TV + vidx(x, y, z)]);
                        plain += lambda * e * e;
                        weighted += lambda * w * e * e;
                        if (gb && len > 1e-12)
                            halo_stencil(&hl, x + 2, y + 2, z + 2, vmul(gr, 2.0 * lambda * w * e / len),
                                         inv2h);
                    }
            if (gb) halo_flush(g, &hl, gb);
        }
    } else if (which == 2) { /* loss_normal, losses.cpp:173-220 */
        for (int t = begin; t < end; ++t) {
            halo_load(g, t, &hl);
            for (int x = 0; x < TE; ++x)
                for (int y = 0; y < TE; ++y)
                    for (int z = 0; z < TE; ++z) {
                        int bx = x + 2, by = y + 2, bz = z + 2;
                        V3 g1 = halo_grad(&hl, bx, by, bz, inv2h);
                        double l1 = vnorm(g1);
                        if (l1 < 1e-8) continue;
                        V3 n1 = vdiv(g1, l1);
                        double w = proximity_weight(g->smooth[(int64_t)t * TV + vidx(x, y, z)]);
                        static const int off[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
                        for (int a = 0; a < 3; ++a) {
                            int nx = bx + off[a][0], ny = by + off[a][1], nz = bz + off[a][2];
                            if (!hl.alloc[hidx(nx, ny, nz)]) continue;
                            V3 g2 = halo_grad(&hl, nx, ny, nz, inv2h);
                            double l2 = vnorm(g2);
                            if (l2 < 1e-8) continue;
                            V3 n2 = vdiv(g2, l2);
                            V3 d = vsub(n2, n1);
                            double vv = vdot(d, d);
                            plain += lambda * vv;
                            weighted += lambda * w * vv;
                            if (gb) {
                                V3 dn2 = vmul(d, 2.0 * lambda * w);
                                V3 dn1 = v3(-dn2.x, -dn2.y, -dn2.z);
                                V3 dg2 = vdiv(vsub(dn2, vmul(n2, vdot(dn2, n2))), l2);
                                V3 dg1 = vdiv(vsub(dn1, vmul(n1, vdot(dn1, n1))), l1);
                                halo_stencil(&hl, nx, ny, nz, dg2, inv2h);
                                halo_stencil(&hl, bx, by, bz, dg1, inv2h);
                            }
                        }
                    }
            if (gb) halo_flush(g, &hl, gb);
        }
    } else if (which == 3) { /* loss_features, losses.cpp:222-257 */
        const int n_s = g->n_s;
        for (int t = begin; t < end; ++t)
            for (int pp = 0; pp < 3; ++pp) {
                const double* p = g->planes + ((int64_t)t * 3 + pp) * plane_stride(g);
                double* gp = gb ? gb->planes + ((int64_t)t * 3 + pp) * plane_stride(g) : NULL;
                for (int a = 0; a < TE; ++a)
                    for (int b = 0; b < TE; ++b)
                        for (int k = 0; k < n_s; ++k) {
                            const int i0 = (a * TE + b) * n_s + k;
                            const int nb[2] = {a + 1 < TE ? ((a + 1) * TE + b) * n_s + k : -1,
                                               b + 1 < TE ? (a * TE + b + 1) * n_s + k : -1};
                            for (int q = 0; q < 2; ++q) {
                                const int i1 = nb[q];
                                if (i1 < 0) continue;
                                const double d = p[i1] - p[i0];
                                const double w = relative_weight(fabs(p[i0]), fabs(p[i1]), PHOTO_EPS);
                                plain += lambda * d * d;
                                weighted += lambda * w * d * d;
                                if (gp) {
                                    const double gg = 2.0 * lambda * w * d;
                                    gp[i1] += gg;
                                    gp[i0] -= gg;
                                }
                            }
                        }
            }
    } else if (which == 4) { /* loss_probes, losses.cpp:259-283 */
        const int64_t stride = probe_stride(g);
        for (int pi = begin; pi < end; ++pi) {
            const int32_t* c = g->probe_coords + 3 * pi;
            static const int off[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
            for (int a = 0; a < 3; ++a) {
                int qi = probe_index(g, c[0] + off[a][0], c[1] + off[a][1], c[2] + off[a][2]);
                if (qi < 0) continue;
                const double* b1 = g->probes + (int64_t)pi * stride;
                const double* b2 = g->probes + (int64_t)qi * stride;
                for (int64_t t = 0; t < stride; ++t) {
                    const double d = b1[t] - b2[t];
                    plain += lambda * d * d;
                    if (gb) {
                        const double gg = 2.0 * lambda * d;
                        gb->probes[(int64_t)pi * stride + t] += gg;
                        gb->probes[(int64_t)qi * stride + t] -= gg;
                    }
                }
            }
        }
        weighted = plain;
    }
    out[0] = plain;
    out[1] = weighted;
}

void og_regularizer(const OGrid* g, int which, double lambda, OGrads* gb, double* out) {
    og_regularizer_range(g, which, lambda, 0, which == 4 ? g->P : g->T, gb, out);
}

/* grads.cpp:67-96 */
void og_gt_fold(const OGrid* g, OGrads* gb) {
    double w[5];
    gaussian_taps(w);
    for (int t = 0; t < g->T; ++t) {
        const int32_t* tc = g->tile_coords + 3 * t;
        const int ox = tc[0] * TE, oy = tc[1] * TE, oz = tc[2] * TE;
        for (int x = 0; x < TE; ++x)
            for (int y = 0; y < TE; ++y)
                for (int z = 0; z < TE; ++z) {
                    double acc = 0.0;
                    for (int dx = -2; dx <= 2; ++dx)
                        for (int dy = -2; dy <= 2; ++dy)
                            for (int dz = -2; dz <= 2; ++dz) {
                                int vx = ox + x + dx, vy = oy + y + dy, vz = oz + z + dz;
                                if (!in_res(g, vx, vy, vz)) continue;
                                int nti = tile_index(g, vx >> 4, vy >> 4, vz >> 4);
                                if (nti < 0) continue;
                                double sw = w[dx + 2] * w[dy + 2] * w[dz + 2];
                                acc += sw * gb->smooth[(int64_t)nti * TV + vidx(vx & 15, vy & 15, vz & 15)];
                            }
                    gb->raw[(int64_t)t * TV + vidx(x, y, z)] += acc;
                }
    }
}

/* ------------------------------------------------------------------ train */

void og_train_reset(OGrid* g) {
    int64_t n = (int64_t)TV * g->T + 3 * plane_stride(g) * g->T + probe_stride(g) * g->P + g->mlp_size;
    free(g->am);
    free(g->av);
    g->am = (double*)calloc((size_t)n, sizeof(double));
    g->av = (double*)calloc((size_t)n, sizeof(double));
    g->at = 0;
}

/* adam.hpp:28-37 on one contiguous range */
static void adam_range(double* p, const double* gr, double* m, double* v, int64_t n, double lr,
                       long t) {
    const double b1 = 0.9, b2 = 0.995, eps = 1e-8;
    const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * gr[i];
        v[i] = b2 * v[i] + (1.0 - b2) * gr[i] * gr[i];
        p[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
    }
}

/* trainer.cpp:136-195 for one explicit batch */
void og_train_step(OGrid* g, int n_views, const OCamera* cams, const double* const* gt_rgb,
                   const double* const* mask, const OStepParams* hp, double* losses,
                   int64_t* counts, OGrads* raypass_out, OGrads* gb) {
    if (!g->am) og_train_reset(g);
    og_grads_clear(g, gb);
    double photo_plain = 0.0, sq_err = 0.0;
    long mask_px = 0;
    int64_t n_rays = 0, n_m = 0, n_x = 0, n_sh = 0, n_al = 0, n_bwd = 0;
    Ray ws = {0};
    for (int vi = 0; vi < n_views; ++vi) {
        const OCamera* cam = &cams[vi];
        ORenderOpts ro;
        memset(&ro, 0, sizeof ro);
        ro.tau = hp->tau;
        ro.n_max = 512;
        ro.early_stop = 1e-4;
        ro.camera_id = hp->use_camera_bias ? cam->id : -1;
        ro.sh_order_override = -1;
        const int w = cam->width, h = cam->height;
        n_rays += (int64_t)w * h;
        for (int px = 0; px < w * h; ++px) {
            const int u = px % w, v = px / w;
            const int in_mask = mask[vi][px] > 0.5;
            ro.need_colors = in_mask;
            double d[3], res[6], pp[6];
            og_pixel_dir(cam, u + 0.5, v + 0.5, d);
            int n = render_ray(g, v3(cam->pos[0], cam->pos[1], cam->pos[2]), v3(d[0], d[1], d[2]),
                               &ro, &ws, res);
            const double* gt = gt_rgb[vi] + 3 * (int64_t)px;
            og_photo_pixel(res, gt, in_mask, res[3], hp->photo_scale, pp);
            photo_plain += pp[0];
            if (in_mask) {
                const double e0 = res[0] - gt[0], e1 = res[1] - gt[1], e2 = res[2] - gt[2];
                sq_err += e0 * e0 + e1 * e1 + e2 * e2;
                mask_px += 3;
            }
            n_m += n;
            n_x += n > 0;
            for (int i = 0; i < n; ++i) n_sh += ws.s[i].shaded;
            if (pp[2] * pp[2] + pp[3] * pp[3] + pp[4] * pp[4] > 0.0 || pp[5] != 0.0) {
                ++n_bwd;
                for (int i = 0; i < n; ++i) n_al += ws.s[i].alpha > 0.0;
                ray_backward(g, &ro, &ws, pp + 2, pp[5], gb);
            }
        }
    }
    free(ws.s);
    free(ws.shade);
    if (raypass_out) {
        og_grads_clear(g, raypass_out);
        og_grads_export(g, gb, raypass_out->raw, raypass_out->smooth, raypass_out->planes,
                        raypass_out->probes, raypass_out->mlp);
    }
    double r[5][2];
    og_regularizer(g, 0, hp->l_sdf, gb, r[0]);
    og_regularizer(g, 1, hp->l_eik, gb, r[1]);
    og_regularizer(g, 2, hp->l_norm, gb, r[2]);
    og_regularizer(g, 3, hp->l_feat, gb, r[3]);
    og_regularizer(g, 4, hp->l_probe, gb, r[4]);
    og_gt_fold(g, gb);
    /* trainer.cpp:53-70 (Optimizer::step): lr_vox for raw SDF and planes,
     * lr_mlp for probes, MLP and camera bias; one shared step count. */
    g->at += 1;
    const int64_t n_raw = (int64_t)TV * g->T, n_pl = 3 * plane_stride(g) * g->T;
    const int64_t n_pr = probe_stride(g) * g->P;
    adam_range(g->raw, gb->raw, g->am, g->av, n_raw, hp->lr_vox, g->at);
    adam_range(g->planes, gb->planes, g->am + n_raw, g->av + n_raw, n_pl, hp->lr_vox, g->at);
    adam_range(g->probes, gb->probes, g->am + n_raw + n_pl, g->av + n_raw + n_pl, n_pr, hp->lr_mlp,
               g->at);
    adam_range(g->mlp, gb->mlp, g->am + n_raw + n_pl + n_pr, g->av + n_raw + n_pl + n_pr,
               g->mlp_size, hp->lr_mlp, g->at);
    og_smooth_all(g);
    const double mse = mask_px > 0 ? sq_err / mask_px : 0.0;
    const double psnr = mse > 1e-10 ? 10.0 * log10(1.0 / mse) : 99.0;
    if (losses) {
        losses[0] = photo_plain;
        for (int i = 0; i < 5; ++i) losses[1 + i] = r[i][0];
        losses[6] = photo_plain + r[0][0] + r[1][0] + r[2][0] + r[3][0] + r[4][0];
        losses[7] = psnr;
        losses[8] = sq_err;
        losses[9] = (double)mask_px;
    }
    if (counts) {
        counts[0] = n_rays; counts[1] = n_m; counts[2] = n_x; counts[3] = n_sh; counts[4] = n_al;
        counts[5] = n_bwd;
    }
}

/* ---------------------------------------------------- known-answer hooks */
double og_alpha_from_sdf(double si, double sn, double tau) { return alpha_from_sdf(si, sn, tau); }
void og_sh_basis(const double* dir, int order, double* out) { sh_basis(v3(dir[0], dir[1], dir[2]), order, out); }
void og_fresnel_powers(double ndv, double* out) { fresnel_powers(ndv, out); }
void og_gaussian_taps(double* out) { gaussian_taps(out); }
void og_adam_steps(int n, double* params, const double* grads_seq, int steps, const double* lrs) {
    double* m = (double*)calloc((size_t)n, sizeof(double));
    double* v = (double*)calloc((size_t)n, sizeof(double));
    for (int t = 0; t < steps; ++t) adam_range(params, grads_seq + (size_t)t * n, m, v, n, lrs[t], t + 1);
    free(m);
    free(v);
}

/* The ray pass of trainer.cpp:149-182 restricted to the 8x4-pixel work tiles
 * [tile_begin, tile_end) of the batch (views concatenated, tiles row-major per
 * view): the data-parallel partition the CUDA path gives each rank
 * (psdf.cu do_train_step).  Accumulates into gb; losses[3] = photo plain,
 * sq_err, mask_px. */
void og_raypass_tiles(const OGrid* g, int n_views, const OCamera* cams, const double* const* gt_rgb,
                      const double* const* mask, const OStepParams* hp, int64_t tile_begin,
                      int64_t tile_end, OGrads* gb, double* losses) {
    double photo_plain = 0.0, sq_err = 0.0, mask_px = 0.0;
    Ray ws = {0};
    int64_t tile0 = 0;
    for (int vi = 0; vi < n_views; ++vi) {
        const OCamera* cam = &cams[vi];
        const int w = cam->width, h = cam->height;
        const int tx = (w + 7) / 8, ty = (h + 3) / 4;
        ORenderOpts ro;
        memset(&ro, 0, sizeof ro);
        ro.tau = hp->tau;
        ro.n_max = 512;
        ro.early_stop = 1e-4;
        ro.camera_id = hp->use_camera_bias ? cam->id : -1;
        ro.sh_order_override = -1;
        for (int64_t lt = 0; lt < (int64_t)tx * ty; ++lt) {
            const int64_t tile = tile0 + lt;
            if (tile < tile_begin || tile >= tile_end) continue;
            for (int lane = 0; lane < 32; ++lane) {
                const int u = (int)(lt % tx) * 8 + (lane & 7), v = (int)(lt / tx) * 4 + (lane >> 3);
                if (u >= w || v >= h) continue;
                const int64_t px = (int64_t)v * w + u;
                const int in_mask = mask[vi][px] > 0.5;
                ro.need_colors = in_mask;
                double d[3], res[6], pp[6];
                og_pixel_dir(cam, u + 0.5, v + 0.5, d);
                render_ray(g, v3(cam->pos[0], cam->pos[1], cam->pos[2]), v3(d[0], d[1], d[2]), &ro,
                           &ws, res);
                const double* gt = gt_rgb[vi] + 3 * px;
                og_photo_pixel(res, gt, in_mask, res[3], hp->photo_scale, pp);
                photo_plain += pp[0];
                if (in_mask) {
                    const double e0 = res[0] - gt[0], e1 = res[1] - gt[1], e2 = res[2] - gt[2];
                    sq_err += e0 * e0 + e1 * e1 + e2 * e2;
                    mask_px += 3;
                }
                if (pp[2] * pp[2] + pp[3] * pp[3] + pp[4] * pp[4] > 0.0 || pp[5] != 0.0)
                    ray_backward(g, &ro, &ws, pp + 2, pp[5], gb);
            }
        }
        tile0 += (int64_t)tx * ty;
    }
    free(ws.s);
    free(ws.shade);
    losses[0] = photo_plain;
    losses[1] = sq_err;
    losses[2] = mask_px;
}
