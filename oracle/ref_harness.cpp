// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// Thin extern "C" harness over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libsdfrecon_ref.so).  It is used only by tests/ (to pin the C
// restatement in oracle/psdf_oracle.c and to generate golden fixtures) and by
// bench.py's cpu_baseline / --impl reference leg (to time the reference's own
// CPU path).  Nothing in the product links it.
//
// Every function goes through the reference's public C++ API.  The train-step
// harness mirrors the loop body of trainer.cpp:125-209 because the reference
// exports no single-step entry (its Optimizer lives in an anonymous namespace,
// trainer.cpp:32); ref_train_full() calls the real train() so the mirror can be
// pinned against it.

#include <cmath>
#include <cstdint>
#include <chrono>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "sdfrecon/adam.hpp"
#include "sdfrecon/checkpoint.hpp"
#include "sdfrecon/dataset.hpp"
#include "sdfrecon/gradcheck.hpp"
#include "sdfrecon/grads.hpp"
#include "sdfrecon/grid.hpp"
#include "sdfrecon/losses.hpp"
#include "sdfrecon/mesh.hpp"
#include "sdfrecon/metrics.hpp"
#include "sdfrecon/renderer.hpp"
#include "sdfrecon/schedule.hpp"
#include "sdfrecon/synth.hpp"
#include "sdfrecon/trainer.hpp"

using namespace sdfrecon;

namespace {

thread_local std::string g_err;

struct OptimizerMirror {
    // trainer.cpp:32-71 (one AdamState per tensor, lr_vox for SDF+planes,
    // lr_mlp for probes, MLP and camera bias).
    std::vector<AdamState> raw_sdf, plane_x, plane_y, plane_z, probes;
    AdamState w1, b1, w2, b2, w3, b3, camera_bias;

    void init(const SparseGrid& g, const DecoderMlp& m) {
        raw_sdf.assign(g.tiles.size(), AdamState(kTileVoxels));
        const size_t plane_sz = static_cast<size_t>(kTileEdge) * kTileEdge * g.n_s;
        plane_x.assign(g.tiles.size(), AdamState(plane_sz));
        plane_y.assign(g.tiles.size(), AdamState(plane_sz));
        plane_z.assign(g.tiles.size(), AdamState(plane_sz));
        const size_t probe_sz = static_cast<size_t>(g.sh_order) * g.sh_order * g.n_a;
        probes.assign(g.probes.size(), AdamState(probe_sz));
        w1 = AdamState(m.w1.size());
        b1 = AdamState(m.b1.size());
        w2 = AdamState(m.w2.size());
        b2 = AdamState(m.b2.size());
        w3 = AdamState(m.w3.size());
        b3 = AdamState(m.b3.size());
        camera_bias = AdamState(m.camera_bias.size());
    }

    void step(SparseGrid& g, DecoderMlp& m, const GradBuffers& gb, double lr_vox, double lr_mlp) {
        for (size_t t = 0; t < g.tiles.size(); ++t) {
            raw_sdf[t].step(g.tiles[t].raw_sdf.data(), gb.raw_sdf[t].data(), lr_vox);
            plane_x[t].step(g.tiles[t].plane_x.data(), gb.plane_x[t].data(), lr_vox);
            plane_y[t].step(g.tiles[t].plane_y.data(), gb.plane_y[t].data(), lr_vox);
            plane_z[t].step(g.tiles[t].plane_z.data(), gb.plane_z[t].data(), lr_vox);
        }
        for (size_t p = 0; p < g.probes.size(); ++p)
            probes[p].step(g.probes[p].coeffs.data(), gb.probes[p].data(), lr_mlp);
        w1.step(m.w1.data(), gb.mlp.w1.data(), lr_mlp);
        b1.step(m.b1.data(), gb.mlp.b1.data(), lr_mlp);
        w2.step(m.w2.data(), gb.mlp.w2.data(), lr_mlp);
        b2.step(m.b2.data(), gb.mlp.b2.data(), lr_mlp);
        w3.step(m.w3.data(), gb.mlp.w3.data(), lr_mlp);
        b3.step(m.b3.data(), gb.mlp.b3.data(), lr_mlp);
        if (!m.camera_bias.empty())
            camera_bias.step(m.camera_bias.data(), gb.mlp.camera_bias.data(), lr_mlp);
    }
};

} // namespace

struct RefScene {
    SparseGrid grid;
    DecoderMlp mlp;
    OptimizerMirror opt;
    bool opt_ready = false;
    GradBuffers gb_raypass; // gradients after the ray pass (before regularizers)
    GradBuffers gb_final;   // gradients handed to Adam
    // per-thread gradient replicas kept across steps and cleared per step, as
    // train() keeps them per LOD (trainer.cpp:115-117, 136)
    std::vector<GradBuffers> gbs;
    bool keep_grads = true; // copy gb_raypass / gb_final (parity tests; off when timing)
    double phase_ms[3] = {0, 0, 0}; // last step: clear + ray pass + reduce | regularizers + fold | Adam + smoothing
};

extern "C" {

struct RefCamera {
    double fx, fy, cx, cy;
    int32_t width, height;
    double rot[9];
    double pos[3];
    int32_t id;
    int32_t pad_;
};

struct RefRenderOpts {
    double tau;
    double early_stop;
    double bg[3];
    int32_t n_max;
    int32_t camera_id;
    int32_t no_spatial, no_angular, no_fresnel, sh_order_override, need_colors;
};

struct RefStepParams {
    double tau, lr_vox, lr_mlp, l_sdf, l_eik, l_norm, l_feat, l_probe, photo_scale;
    int32_t use_camera_bias;
    int32_t pad_;
};

const char* ref_last_error() { return g_err.c_str(); }

static Camera to_cam(const RefCamera* c) {
    Camera cam;
    cam.id = c->id;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    cam.width = c->width;
    cam.height = c->height;
    for (int i = 0; i < 9; ++i) cam.rot[i] = c->rot[i];
    cam.pos = {c->pos[0], c->pos[1], c->pos[2]};
    return cam;
}

static RenderOptions to_opts(const RefRenderOpts* o) {
    RenderOptions r;
    r.tau = o->tau;
    r.n_max = o->n_max;
    r.early_stop_transmittance = o->early_stop;
    r.background = {o->bg[0], o->bg[1], o->bg[2]};
    r.camera_id = o->camera_id;
    r.no_spatial = o->no_spatial != 0;
    r.no_angular = o->no_angular != 0;
    r.no_fresnel = o->no_fresnel != 0;
    r.sh_order_override = o->sh_order_override;
    r.need_colors = o->need_colors != 0;
    return r;
}

// camera.cpp:5-23
void ref_make_lookat_camera(int id, const double* eye, const double* target, const double* up,
                            double fx, double fy, int width, int height, RefCamera* out) {
    Camera c = make_lookat_camera(id, {eye[0], eye[1], eye[2]}, {target[0], target[1], target[2]},
                                  {up[0], up[1], up[2]}, fx, fy, width, height);
    out->fx = c.fx;
    out->fy = c.fy;
    out->cx = c.cx;
    out->cy = c.cy;
    out->width = c.width;
    out->height = c.height;
    for (int i = 0; i < 9; ++i) out->rot[i] = c.rot[i];
    out->pos[0] = c.pos.x;
    out->pos[1] = c.pos.y;
    out->pos[2] = c.pos.z;
    out->id = c.id;
    out->pad_ = 0;
}

// synth.cpp:238-255
int ref_make_ring_cameras(int n_views, int resolution, double radius, double elevation,
                          uint64_t seed, RefCamera* out) {
    auto cams = make_ring_cameras(n_views, resolution, radius, elevation, seed);
    for (size_t i = 0; i < cams.size(); ++i) {
        const Camera& c = cams[i];
        double eye[3] = {c.pos.x, c.pos.y, c.pos.z};
        RefCamera& o = out[i];
        o.fx = c.fx; o.fy = c.fy; o.cx = c.cx; o.cy = c.cy;
        o.width = c.width; o.height = c.height;
        for (int k = 0; k < 9; ++k) o.rot[k] = c.rot[k];
        for (int k = 0; k < 3; ++k) o.pos[k] = eye[k];
        o.id = c.id;
        o.pad_ = 0;
    }
    return static_cast<int>(cams.size());
}

// Sphere-initialised scene (grid.cpp:462-467) plus a Glorot MLP
// (decoder.cpp:9-30).
RefScene* ref_scene_sphere(int res, double voxel_size, double ox, double oy, double oz, int n_s,
                           int n_a, int sh_order, int band_voxels, double far_field_voxels,
                           double cx, double cy, double cz, double radius, int ncam,
                           uint64_t mlp_seed) {
    try {
        GridConfig cfg;
        cfg.resolution = {res, res, res};
        cfg.voxel_size = voxel_size;
        cfg.origin = {ox, oy, oz};
        cfg.n_s = n_s;
        cfg.n_a = n_a;
        cfg.sh_order = sh_order;
        cfg.band_voxels = band_voxels;
        cfg.far_field_voxels = far_field_voxels;
        auto* s = new RefScene;
        s->grid = init_grid_sphere(cfg, {cx, cy, cz}, radius);
        s->mlp = DecoderMlp::glorot_init(n_s, n_a, ncam, mlp_seed);
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Analytic union scene written into an allocated grid: tiles whose 16^3 block
// is within band of the zero crossing are allocated (the init_common rule,
// grid.cpp:359-398) and filled from AnalyticScene::sdf (synth.cpp:142-154).
RefScene* ref_scene_analytic(int res, double voxel_size, double ox, double oy, double oz, int n_s,
                             int n_a, int sh_order, int band_voxels, double far_field_voxels,
                             int n_prims, const int32_t* kinds, const double* centers,
                             const double* extents, int ncam, uint64_t mlp_seed) {
    try {
        AnalyticScene sc;
        for (int i = 0; i < n_prims; ++i) {
            Primitive p;
            p.kind = kinds[i] == 0 ? Primitive::Kind::Sphere
                     : kinds[i] == 1 ? Primitive::Kind::Box
                                     : Primitive::Kind::Torus;
            p.center = {centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]};
            p.extent = {extents[3 * i], extents[3 * i + 1], extents[3 * i + 2]};
            sc.primitives.push_back(p);
        }
        GridConfig cfg;
        cfg.resolution = {res, res, res};
        cfg.voxel_size = voxel_size;
        cfg.origin = {ox, oy, oz};
        cfg.n_s = n_s;
        cfg.n_a = n_a;
        cfg.sh_order = sh_order;
        cfg.band_voxels = band_voxels;
        cfg.far_field_voxels = far_field_voxels;
        // init_grid_sphere with a huge radius gives an empty grid with the
        // right metadata; tiles are then allocated in init_common order.
        auto* s = new RefScene;
        SparseGrid g = init_grid_sphere(cfg, {0, 0, 0}, 1e6);
        const double band = band_voxels * voxel_size;
        const int nt = res / kTileEdge;
        std::vector<double> vals(kTileVoxels);
        for (int tx = 0; tx < nt; ++tx)
            for (int ty = 0; ty < nt; ++ty)
                for (int tz = 0; tz < nt; ++tz) {
                    double min_abs = 1e300;
                    bool pos = false, neg = false;
                    for (int x = 0; x < kTileEdge; ++x)
                        for (int y = 0; y < kTileEdge; ++y)
                            for (int z = 0; z < kTileEdge; ++z) {
                                double v = sc.sdf(g.voxel_center(tx * 16 + x, ty * 16 + y, tz * 16 + z));
                                vals[voxel_index(x, y, z)] = v;
                                min_abs = std::min(min_abs, std::abs(v));
                                (v >= 0 ? pos : neg) = true;
                            }
                    if (min_abs > band && !(pos && neg)) continue;
                    int ti = g.allocate_tile(tx, ty, tz);
                    g.tiles[ti].raw_sdf = vals;
                }
        g.smooth_all();
        s->grid = std::move(g);
        s->mlp = DecoderMlp::glorot_init(n_s, n_a, ncam, mlp_seed);
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_scene_free(RefScene* s) { delete s; }

// init_grid_visual_hull (grid.cpp:470-504) through the reference's own code.
RefScene* ref_scene_hull(int res, double voxel_size, double ox, double oy, double oz, int n_s, int n_a,
                         int sh_order, int band_voxels, double far_field_voxels, int n_cams,
                         const RefCamera* cams, const uint8_t* const* masks, int ncam_bias,
                         uint64_t mlp_seed) {
    try {
        GridConfig cfg;
        cfg.resolution = {res, res, res};
        cfg.voxel_size = voxel_size;
        cfg.origin = {ox, oy, oz};
        cfg.n_s = n_s;
        cfg.n_a = n_a;
        cfg.sh_order = sh_order;
        cfg.band_voxels = band_voxels;
        cfg.far_field_voxels = far_field_voxels;
        std::vector<Camera> cv;
        std::vector<MaskImage> mv;
        for (int i = 0; i < n_cams; ++i) {
            cv.push_back(to_cam(cams + i));
            MaskImage m;
            m.width = cams[i].width;
            m.height = cams[i].height;
            m.data.assign(masks[i], masks[i] + (size_t)m.width * m.height);
            mv.push_back(std::move(m));
        }
        auto* s = new RefScene;
        s->grid = init_grid_visual_hull(cfg, cv, mv);
        s->mlp = DecoderMlp::glorot_init(n_s, n_a, ncam_bias, mlp_seed);
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Seeded "trained-like" parameters: the pattern of test_renderer.cpp:32-43 and
// gradcheck.cpp:40-53 (raw jitter, planes 0.5 +- plane_amp, probes +- probe_amp,
// camera bias +- bias_amp), then smooth_all.
void ref_scene_randomize(RefScene* s, uint64_t seed, double sdf_jitter, double plane_amp,
                         double probe_amp, double bias_amp) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    for (Tile& t : s->grid.tiles) {
        if (sdf_jitter != 0.0)
            for (double& v : t.raw_sdf) v += sdf_jitter * uni(rng);
        for (double& v : t.plane_x) v = 0.5 + plane_amp * uni(rng);
        for (double& v : t.plane_y) v = 0.5 + plane_amp * uni(rng);
        for (double& v : t.plane_z) v = 0.5 + plane_amp * uni(rng);
    }
    for (ProbeSH& p : s->grid.probes)
        for (double& c : p.coeffs) c = probe_amp * uni(rng);
    s->grid.smooth_all();
    for (double& b : s->mlp.camera_bias) b = bias_amp * uni(rng);
}

// info: T, P, n_s, n_a, sh_order, res_x, res_y, res_z, mlp_size, ncam
void ref_scene_info(const RefScene* s, int64_t* info, double* geom) {
    const SparseGrid& g = s->grid;
    info[0] = static_cast<int64_t>(g.tiles.size());
    info[1] = static_cast<int64_t>(g.probes.size());
    info[2] = g.n_s;
    info[3] = g.n_a;
    info[4] = g.sh_order;
    info[5] = g.resolution.x;
    info[6] = g.resolution.y;
    info[7] = g.resolution.z;
    const DecoderMlp& m = s->mlp;
    info[8] = static_cast<int64_t>(m.w1.size() + m.b1.size() + m.w2.size() + m.b2.size() +
                                   m.w3.size() + m.b3.size() + m.camera_bias.size());
    info[9] = m.num_cameras();
    geom[0] = g.voxel_size;
    geom[1] = g.origin.x;
    geom[2] = g.origin.y;
    geom[3] = g.origin.z;
    geom[4] = g.far_field_voxels;
}

// Flat layouts (shared with the CUDA path's upload format):
//   tile_coords [T][3], probe_ids [T][8], probe_coords [P][3]
//   raw/smooth  [T][4096]    planes [T][3][256][n_s] (plane_x, plane_y, plane_z)
//   probes      [P][l^2][n_a]
void ref_scene_export(const RefScene* s, int32_t* tile_coords, int32_t* probe_ids,
                      int32_t* probe_coords, double* raw, double* smooth, double* planes,
                      double* probes) {
    const SparseGrid& g = s->grid;
    const size_t ps = static_cast<size_t>(kTileEdge) * kTileEdge * g.n_s;
    for (size_t t = 0; t < g.tiles.size(); ++t) {
        const Tile& tile = g.tiles[t];
        if (tile_coords) {
            tile_coords[3 * t] = tile.coords.x;
            tile_coords[3 * t + 1] = tile.coords.y;
            tile_coords[3 * t + 2] = tile.coords.z;
        }
        if (probe_ids)
            for (int i = 0; i < 8; ++i) probe_ids[8 * t + i] = tile.probe_ids[i];
        if (raw) std::memcpy(raw + t * kTileVoxels, tile.raw_sdf.data(), kTileVoxels * sizeof(double));
        if (smooth)
            std::memcpy(smooth + t * kTileVoxels, tile.smooth_sdf.data(), kTileVoxels * sizeof(double));
        if (planes) {
            std::memcpy(planes + (3 * t + 0) * ps, tile.plane_x.data(), ps * sizeof(double));
            std::memcpy(planes + (3 * t + 1) * ps, tile.plane_y.data(), ps * sizeof(double));
            std::memcpy(planes + (3 * t + 2) * ps, tile.plane_z.data(), ps * sizeof(double));
        }
    }
    const size_t pc = static_cast<size_t>(g.sh_order) * g.sh_order * g.n_a;
    for (size_t p = 0; p < g.probes.size(); ++p) {
        if (probe_coords) {
            probe_coords[3 * p] = g.probe_coords[p].x;
            probe_coords[3 * p + 1] = g.probe_coords[p].y;
            probe_coords[3 * p + 2] = g.probe_coords[p].z;
        }
        if (probes) std::memcpy(probes + p * pc, g.probes[p].coeffs.data(), pc * sizeof(double));
    }
}

// Overwrites parameter values.  smooth == nullptr re-smooths (grid.cpp:247-250);
// otherwise the given smoothed SDF is installed verbatim (used to feed both
// sides bit-identical fp32-representable inputs).
void ref_scene_import(RefScene* s, const double* raw, const double* smooth, const double* planes,
                      const double* probes) {
    SparseGrid& g = s->grid;
    const size_t ps = static_cast<size_t>(kTileEdge) * kTileEdge * g.n_s;
    for (size_t t = 0; t < g.tiles.size(); ++t) {
        Tile& tile = g.tiles[t];
        if (raw) std::memcpy(tile.raw_sdf.data(), raw + t * kTileVoxels, kTileVoxels * sizeof(double));
        if (planes) {
            std::memcpy(tile.plane_x.data(), planes + (3 * t + 0) * ps, ps * sizeof(double));
            std::memcpy(tile.plane_y.data(), planes + (3 * t + 1) * ps, ps * sizeof(double));
            std::memcpy(tile.plane_z.data(), planes + (3 * t + 2) * ps, ps * sizeof(double));
        }
    }
    const size_t pc = static_cast<size_t>(g.sh_order) * g.sh_order * g.n_a;
    if (probes)
        for (size_t p = 0; p < g.probes.size(); ++p)
            std::memcpy(g.probes[p].coeffs.data(), probes + p * pc, pc * sizeof(double));
    if (smooth) {
        for (size_t t = 0; t < g.tiles.size(); ++t)
            std::memcpy(g.tiles[t].smooth_sdf.data(), smooth + t * kTileVoxels,
                        kTileVoxels * sizeof(double));
    } else {
        g.smooth_all();
    }
}

void ref_smooth_all(RefScene* s) { s->grid.smooth_all(); }

// SDFC checkpoints through the reference's own save / load (checkpoint.cpp).
int ref_save_checkpoint(const RefScene* s, const char* path, int lod_cursor, int64_t iteration, uint64_t seed) {
    try {
        Checkpoint ck;
        ck.grid = s->grid;
        ck.mlp = s->mlp;
        ck.lod_cursor = lod_cursor;
        ck.iteration = iteration;
        ck.seed = seed;
        save_checkpoint(path, ck);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
RefScene* ref_load_checkpoint(const char* path, int64_t* cursor_iter_seed) {
    try {
        Checkpoint ck = load_checkpoint(path);
        auto* s = new RefScene;
        s->grid = ck.grid;
        s->mlp = ck.mlp;
        cursor_iter_seed[0] = ck.lod_cursor;
        cursor_iter_seed[1] = ck.iteration;
        cursor_iter_seed[2] = (int64_t)ck.seed;
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// LOD transitions through the reference's own members (grid.cpp:252-345).
int ref_subdivide(RefScene* s) {
    try {
        s->grid = s->grid.subdivide();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
int ref_raise_sh_order(RefScene* s, int order) {
    try {
        s->grid.raise_sh_order(order);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// MLP flat layout: w1 [32][in], b1 [32], w2 [32][32], b2 [32], w3 [3][32],
// b3 [3], camera_bias [ncam][32]  (decoder.hpp:17-31 field order).
static void mlp_copy(DecoderMlp& m, double* out, const double* in) {
    std::vector<double>* parts[7] = {&m.w1, &m.b1, &m.w2, &m.b2, &m.w3, &m.b3, &m.camera_bias};
    size_t off = 0;
    for (auto* p : parts) {
        if (out) std::memcpy(out + off, p->data(), p->size() * sizeof(double));
        if (in) std::memcpy(p->data(), in + off, p->size() * sizeof(double));
        off += p->size();
    }
}
void ref_mlp_export(RefScene* s, double* out) { mlp_copy(s->mlp, out, nullptr); }
void ref_mlp_import(RefScene* s, const double* in) { mlp_copy(s->mlp, nullptr, in); }

// renderer.cpp:55-86
int ref_march_ray(const RefScene* s, const double* o, const double* d, int n_max, double* ts) {
    auto v = march_ray(s->grid, {o[0], o[1], o[2]}, {d[0], d[1], d[2]}, n_max);
    for (size_t i = 0; i < v.size(); ++i) ts[i] = v[i];
    return static_cast<int>(v.size());
}

// camera.hpp:32-35
void ref_pixel_dir(const RefCamera* c, double u, double v, double* d) {
    Vec3 r = to_cam(c).pixel_dir(u, v);
    d[0] = r.x;
    d[1] = r.y;
    d[2] = r.z;
}

// renderer.cpp:149-210 for one ray, exposing the RayWorkspace.
// sample_out [n][8]: t, sdf, alpha, trans, weight, shaded, tile, pad
// color_out [n][3]; result [6]: color xyz, acc_alpha, trans_end, sdf_extra
int ref_render_ray(const RefScene* s, const double* o, const double* d, const RefRenderOpts* opt,
                   int max_n, double* sample_out, double* color_out, double* result) {
    try {
        RayWorkspace ws;
        RayResult r = render_ray(s->grid, s->mlp, {o[0], o[1], o[2]}, {d[0], d[1], d[2]},
                                 to_opts(opt), ws);
        const int n = static_cast<int>(ws.samples.size());
        for (int i = 0; i < n && i < max_n; ++i) {
            const RaySample& rs = ws.samples[i];
            double* so = sample_out + 8 * i;
            so[0] = rs.t;
            so[1] = rs.sdf;
            so[2] = rs.alpha;
            so[3] = rs.trans;
            so[4] = rs.weight;
            so[5] = rs.shaded ? 1.0 : 0.0;
            so[6] = rs.tile;
            so[7] = 0.0;
            if (color_out) {
                color_out[3 * i] = rs.shaded ? rs.color.x : 0.0;
                color_out[3 * i + 1] = rs.shaded ? rs.color.y : 0.0;
                color_out[3 * i + 2] = rs.shaded ? rs.color.z : 0.0;
            }
        }
        result[0] = r.color.x;
        result[1] = r.color.y;
        result[2] = r.color.z;
        result[3] = r.acc_alpha;
        result[4] = r.trans_end;
        result[5] = ws.has_extra ? ws.sdf_extra : 0.0;
        return n;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// render_image (renderer.cpp:321-337) re-expressed per ray so the per-ray
// counts and the depth extension D = sum_i w_i t_i can be read from the
// RayWorkspace.  counts: [N_rays, N_m (marched, after early stop), N_x (rays
// with >=1 sample), N_sh (shaded samples), N_alpha (samples with alpha > 0)].
int ref_render_image(const RefScene* s, const RefCamera* cam, const RefRenderOpts* opt,
                     double* rgb, double* alpha, double* depth, int64_t* counts, int threads) {
    try {
        const Camera c = to_cam(cam);
        const RenderOptions ro = to_opts(opt);
        int64_t n_m = 0, n_x = 0, n_sh = 0, n_a = 0;
#ifdef _OPENMP
        if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : n_m, n_x, n_sh, n_a)
        for (int v = 0; v < c.height; ++v) {
            RayWorkspace ws;
            for (int u = 0; u < c.width; ++u) {
                const Vec3 dir = c.pixel_dir(u + 0.5, v + 0.5);
                RayResult r = render_ray(s->grid, s->mlp, c.pos, dir, ro, ws);
                const size_t px = static_cast<size_t>(v) * c.width + u;
                rgb[3 * px] = r.color.x;
                rgb[3 * px + 1] = r.color.y;
                rgb[3 * px + 2] = r.color.z;
                alpha[px] = r.acc_alpha;
                double dsum = 0.0;
                for (const RaySample& rs : ws.samples) {
                    dsum += rs.weight * rs.t;
                    n_sh += rs.shaded ? 1 : 0;
                    n_a += rs.alpha > 0.0 ? 1 : 0;
                }
                if (depth) depth[px] = dsum;
                n_m += static_cast<int64_t>(ws.samples.size());
                n_x += ws.samples.empty() ? 0 : 1;
            }
        }
        if (counts) {
            counts[0] = static_cast<int64_t>(c.width) * c.height;
            counts[1] = n_m;
            counts[2] = n_x;
            counts[3] = n_sh;
            counts[4] = n_a;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The reference's own public entry, unchanged (renderer.cpp:321-337): used to
// time the CPU baseline.
int ref_render_image_api(const RefScene* s, const RefCamera* cam, const RefRenderOpts* opt,
                         double* rgb, double* alpha, int threads) {
    try {
#ifdef _OPENMP
        if (threads > 0) omp_set_num_threads(threads);
#endif
        RenderedImage im = render_image(s->grid, s->mlp, to_cam(cam), to_opts(opt));
        if (rgb) std::memcpy(rgb, im.color.data.data(), im.color.data.size() * sizeof(double));
        if (alpha) std::memcpy(alpha, im.alpha.data.data(), im.alpha.data.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Single-ray backward into fresh buffers (renderer.cpp:239-319 then
// grads.cpp:67-96 when fold != 0).  Gradients are exported in the flat layout.
int ref_ray_backward(const RefScene* s, const double* o, const double* d, const RefRenderOpts* opt,
                     const double* up_color, double up_alpha, int fold, double* g_raw,
                     double* g_smooth, double* g_planes, double* g_probes, double* g_mlp) {
    try {
        RayWorkspace ws;
        const RenderOptions ro = to_opts(opt);
        render_ray(s->grid, s->mlp, {o[0], o[1], o[2]}, {d[0], d[1], d[2]}, ro, ws);
        GradBuffers gb;
        gb.init(s->grid, s->mlp);
        render_ray_backward(s->grid, s->mlp, ro, ws, {up_color[0], up_color[1], up_color[2]},
                            up_alpha, gb);
        if (fold) finalize_smooth_grads(s->grid, gb);
        const SparseGrid& g = s->grid;
        const size_t ps = static_cast<size_t>(kTileEdge) * kTileEdge * g.n_s;
        for (size_t t = 0; t < g.tiles.size(); ++t) {
            if (g_raw) std::memcpy(g_raw + t * kTileVoxels, gb.raw_sdf[t].data(), kTileVoxels * 8);
            if (g_smooth)
                std::memcpy(g_smooth + t * kTileVoxels, gb.smooth_sdf[t].data(), kTileVoxels * 8);
            if (g_planes) {
                std::memcpy(g_planes + (3 * t) * ps, gb.plane_x[t].data(), ps * 8);
                std::memcpy(g_planes + (3 * t + 1) * ps, gb.plane_y[t].data(), ps * 8);
                std::memcpy(g_planes + (3 * t + 2) * ps, gb.plane_z[t].data(), ps * 8);
            }
        }
        const size_t pc = static_cast<size_t>(g.sh_order) * g.sh_order * g.n_a;
        if (g_probes)
            for (size_t p = 0; p < g.probes.size(); ++p)
                std::memcpy(g_probes + p * pc, gb.probes[p].data(), pc * 8);
        if (g_mlp) {
            DecoderMlp tmp = s->mlp;
            tmp.w1 = gb.mlp.w1; tmp.b1 = gb.mlp.b1; tmp.w2 = gb.mlp.w2; tmp.b2 = gb.mlp.b2;
            tmp.w3 = gb.mlp.w3; tmp.b3 = gb.mlp.b3; tmp.camera_bias = gb.mlp.camera_bias;
            mlp_copy(tmp, g_mlp, nullptr);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// losses.cpp:8-38
void ref_photo_pixel(const double* c, const double* gt, int in_mask, double acc, double scale,
                     double* out /* plain, weighted, dcx, dcy, dcz, dalpha */) {
    PhotoPixel p = photo_pixel({c[0], c[1], c[2]}, {gt[0], gt[1], gt[2]}, in_mask != 0, acc, scale);
    out[0] = p.plain;
    out[1] = p.weighted;
    out[2] = p.d_color.x;
    out[3] = p.d_color.y;
    out[4] = p.d_color.z;
    out[5] = p.d_alpha;
}

static void export_gb(const SparseGrid& g, const GradBuffers& gb, double* g_raw, double* g_smooth,
                      double* g_planes, double* g_probes, double* g_mlp, const DecoderMlp& m) {
    const size_t ps = static_cast<size_t>(kTileEdge) * kTileEdge * g.n_s;
    for (size_t t = 0; t < g.tiles.size(); ++t) {
        if (g_raw) std::memcpy(g_raw + t * kTileVoxels, gb.raw_sdf[t].data(), kTileVoxels * 8);
        if (g_smooth) std::memcpy(g_smooth + t * kTileVoxels, gb.smooth_sdf[t].data(), kTileVoxels * 8);
        if (g_planes) {
            std::memcpy(g_planes + (3 * t) * ps, gb.plane_x[t].data(), ps * 8);
            std::memcpy(g_planes + (3 * t + 1) * ps, gb.plane_y[t].data(), ps * 8);
            std::memcpy(g_planes + (3 * t + 2) * ps, gb.plane_z[t].data(), ps * 8);
        }
    }
    const size_t pc = static_cast<size_t>(g.sh_order) * g.sh_order * g.n_a;
    if (g_probes)
        for (size_t p = 0; p < g.probes.size(); ++p)
            std::memcpy(g_probes + p * pc, gb.probes[p].data(), pc * 8);
    if (g_mlp) {
        DecoderMlp tmp = m;
        tmp.w1 = gb.mlp.w1; tmp.b1 = gb.mlp.b1; tmp.w2 = gb.mlp.w2; tmp.b2 = gb.mlp.b2;
        tmp.w3 = gb.mlp.w3; tmp.b3 = gb.mlp.b3; tmp.camera_bias = gb.mlp.camera_bias;
        mlp_copy(tmp, g_mlp, nullptr);
    }
}

// Each regularizer separately into a fresh buffer (losses.cpp:121-283), with
// wsrc = grid (trainer.cpp:187-191).  which: 0 sdf, 1 eik, 2 normal,
// 3 features, 4 probes.  out: plain, weighted.
int ref_regularizer(const RefScene* s, int which, double lambda, double* out, double* g_raw,
                    double* g_smooth, double* g_planes, double* g_probes) {
    GradBuffers gb;
    gb.init(s->grid, s->mlp);
    LossResult r;
    switch (which) {
        case 0: r = loss_sdf(s->grid, s->grid, lambda, &gb); break;
        case 1: r = loss_eikonal(s->grid, s->grid, lambda, &gb); break;
        case 2: r = loss_normal(s->grid, s->grid, lambda, &gb); break;
        case 3: r = loss_features(s->grid, s->grid, lambda, &gb); break;
        case 4: r = loss_probes(s->grid, lambda, &gb); break;
        default: g_err = "bad regularizer id"; return -1;
    }
    out[0] = r.plain;
    out[1] = r.weighted;
    export_gb(s->grid, gb, g_raw, g_smooth, g_planes, g_probes, nullptr, s->mlp);
    return 0;
}

// finalize_smooth_grads (grads.cpp:67-96) on a given staged buffer:
// raw_out = raw_in + G^T staged.
void ref_gt_fold(const RefScene* s, const double* staged, const double* raw_in, double* raw_out) {
    GradBuffers gb;
    gb.init(s->grid, s->mlp);
    const size_t T = s->grid.tiles.size();
    for (size_t t = 0; t < T; ++t) {
        std::memcpy(gb.smooth_sdf[t].data(), staged + t * kTileVoxels, kTileVoxels * 8);
        if (raw_in) std::memcpy(gb.raw_sdf[t].data(), raw_in + t * kTileVoxels, kTileVoxels * 8);
    }
    finalize_smooth_grads(s->grid, gb);
    for (size_t t = 0; t < T; ++t)
        std::memcpy(raw_out + t * kTileVoxels, gb.raw_sdf[t].data(), kTileVoxels * 8);
}

// Timing runs: skip the per-step copies of the gradient buffers (parity
// tests read them through ref_grads).
void ref_set_keep_grads(RefScene* s, int keep) { s->keep_grads = keep != 0; }

// Phase times of the last ref_train_step (ms): [clear + ray pass + replica
// reduction, regularizers + G^T fold, Adam + smoothing].
void ref_last_phase_ms(const RefScene* s, double* out) {
    for (int i = 0; i < 3; ++i) out[i] = s->phase_ms[i];
}

void ref_train_reset(RefScene* s) {
    s->opt.init(s->grid, s->mlp);
    s->opt_ready = true;
}

// One training step: the loop body of trainer.cpp:136-195 for an explicit
// batch of views.  gt_rgb[i] is [h][w][3], mask[i] is [h][w] (>0.5 = in).
// losses out: photo_plain, sdf, eik, normal, features, probes, total, psnr,
//             sq_err, mask_px
// counts out: N_rays, N_m, N_x, N_sh, N_alpha(backward rays), N_bwd_rays
int ref_train_step(RefScene* s, int n_views, const RefCamera* cams, const double* const* gt_rgb,
                   const double* const* mask, const RefStepParams* hp, int threads,
                   double* losses, int64_t* counts) {
    try {
        SparseGrid& grid = s->grid;
        DecoderMlp& mlp = s->mlp;
        if (!s->opt_ready) ref_train_reset(s);
        int n_threads = 1;
#ifdef _OPENMP
        if (threads > 0) omp_set_num_threads(threads);
        n_threads = omp_get_max_threads();
#endif
        // replicas allocated once per thread count / grid (train() allocates
        // them per LOD, outside its step loop); the per-step clear is timed
        std::vector<GradBuffers>& gbs = s->gbs;
        const bool fresh = (int)gbs.size() != n_threads || gbs[0].raw_sdf.size() != grid.tiles.size() ||
                           gbs[0].probes.size() != grid.probes.size();
        if (fresh) {
            gbs.assign(n_threads, GradBuffers{});
            for (GradBuffers& gb : gbs) gb.init(grid, mlp);
        }
        const auto t_begin = std::chrono::steady_clock::now();
        if (!fresh)
            for (GradBuffers& gb : gbs) gb.clear();

        double photo_plain = 0.0, sq_err = 0.0;
        long mask_px = 0;
        int64_t n_rays = 0, n_m = 0, n_x = 0, n_sh = 0, n_al = 0, n_bwd = 0;
        for (int vi = 0; vi < n_views; ++vi) {
            const Camera cam = to_cam(&cams[vi]);
            RenderOptions ropt;
            ropt.tau = hp->tau;
            ropt.camera_id = hp->use_camera_bias ? cam.id : -1;
            const int w = cam.width, h = cam.height;
            const double* img = gt_rgb[vi];
            const double* msk = mask[vi];
            n_rays += static_cast<int64_t>(w) * h;
#pragma omp parallel for schedule(static) reduction(+ : photo_plain, sq_err, mask_px, n_m, n_x, n_sh, n_al, n_bwd)
            for (int px = 0; px < w * h; ++px) {
                const int u = px % w, v = px / w;
#ifdef _OPENMP
                GradBuffers& gb = gbs[omp_get_thread_num()];
#else
                GradBuffers& gb = gbs[0];
#endif
                const bool in_mask = msk[px] > 0.5;
                RenderOptions popt = ropt;
                popt.need_colors = in_mask;
                thread_local RayWorkspace ws;
                RayResult rr = render_ray(grid, mlp, cam.pos, cam.pixel_dir(u + 0.5, v + 0.5), popt, ws);
                const Vec3 gt{img[3 * px], img[3 * px + 1], img[3 * px + 2]};
                PhotoPixel pp = photo_pixel(rr.color, gt, in_mask, rr.acc_alpha, hp->photo_scale);
                photo_plain += pp.plain;
                if (in_mask) {
                    sq_err += (rr.color - gt).norm2();
                    mask_px += 3;
                }
                n_m += static_cast<int64_t>(ws.samples.size());
                n_x += ws.samples.empty() ? 0 : 1;
                for (const RaySample& rs : ws.samples) n_sh += rs.shaded ? 1 : 0;
                if (pp.d_color.norm2() > 0.0 || pp.d_alpha != 0.0) {
                    ++n_bwd;
                    for (const RaySample& rs : ws.samples) n_al += rs.alpha > 0.0 ? 1 : 0;
                    render_ray_backward(grid, mlp, popt, ws, pp.d_color, pp.d_alpha, gb);
                }
            }
        }
        GradBuffers& gb = gbs[0];
        for (int t = 1; t < n_threads; ++t) gb.add(gbs[t]);
        if (s->keep_grads) s->gb_raypass = gb;
        const auto t_ray = std::chrono::steady_clock::now();

        const LossResult r_sdf = loss_sdf(grid, grid, hp->l_sdf, &gb);
        const LossResult r_eik = loss_eikonal(grid, grid, hp->l_eik, &gb);
        const LossResult r_norm = loss_normal(grid, grid, hp->l_norm, &gb);
        const LossResult r_feat = loss_features(grid, grid, hp->l_feat, &gb);
        const LossResult r_probe = loss_probes(grid, hp->l_probe, &gb);
        finalize_smooth_grads(grid, gb);
        const auto t_reg = std::chrono::steady_clock::now();
        if (s->keep_grads) s->gb_final = gb;
        const auto t_opt = std::chrono::steady_clock::now();
        s->opt.step(grid, mlp, gb, hp->lr_vox, hp->lr_mlp);
        grid.smooth_all();
        const auto t_end = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        s->phase_ms[0] = ms(t_begin, t_ray);
        s->phase_ms[1] = ms(t_ray, t_reg);
        s->phase_ms[2] = ms(t_opt, t_end);

        const double mse = mask_px > 0 ? sq_err / mask_px : 0.0;
        const double psnr = mse > 1e-10 ? 10.0 * std::log10(1.0 / mse) : 99.0;
        if (losses) {
            losses[0] = photo_plain;
            losses[1] = r_sdf.plain;
            losses[2] = r_eik.plain;
            losses[3] = r_norm.plain;
            losses[4] = r_feat.plain;
            losses[5] = r_probe.plain;
            losses[6] = photo_plain + r_sdf.plain + r_eik.plain + r_norm.plain + r_feat.plain +
                        r_probe.plain;
            losses[7] = psnr;
            losses[8] = sq_err;
            losses[9] = static_cast<double>(mask_px);
        }
        if (counts) {
            counts[0] = n_rays;
            counts[1] = n_m;
            counts[2] = n_x;
            counts[3] = n_sh;
            counts[4] = n_al;
            counts[5] = n_bwd;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// stage 0: after the ray pass; stage 1: final (after regularizers + G^T).
void ref_grads_export(const RefScene* s, int stage, double* g_raw, double* g_smooth,
                      double* g_planes, double* g_probes, double* g_mlp) {
    const GradBuffers& gb = stage == 0 ? s->gb_raypass : s->gb_final;
    export_gb(s->grid, gb, g_raw, g_smooth, g_planes, g_probes, g_mlp, s->mlp);
}

// The real train() (trainer.cpp:81-220) for a single-LOD schedule with no
// subdivision, on a dataset whose views are given explicitly.  Used to pin the
// step mirror above (batch order from mt19937_64(seed), trainer.cpp:98,119-145).
int ref_train_full(RefScene* s, int n_views, const RefCamera* cams, const double* const* gt_rgb,
                   const double* const* mask, int iterations, int images_per_batch,
                   const double* brackets /* lr_vox a,b lr_mlp a,b eik a,b sdf a,b feat a,b
                                             normal a,b probes a,b tau a,b */,
                   double lambda_photo, int camera_bias, uint64_t seed, int threads,
                   double* final_psnr) {
    try {
#ifdef _OPENMP
        if (threads > 0) omp_set_num_threads(threads);
#endif
        Dataset ds;
        for (int i = 0; i < n_views; ++i) {
            DatasetView v;
            v.camera = to_cam(&cams[i]);
            const int w = cams[i].width, h = cams[i].height;
            v.image = ImageRGB(w, h);
            v.mask = ImageGray(w, h);
            std::memcpy(v.image.data.data(), gt_rgb[i], sizeof(double) * w * h * 3);
            std::memcpy(v.mask.data.data(), mask[i], sizeof(double) * w * h);
            ds.views.push_back(std::move(v));
        }
        TrainSchedule sched;
        sched.lambda_photo = lambda_photo;
        sched.camera_bias = camera_bias != 0;
        LodSchedule l;
        l.iterations = iterations;
        l.images_per_batch = images_per_batch;
        l.sh_order = s->grid.sh_order;
        l.image_divisor = 1;
        l.lr_voxels = Bracket{brackets[0], brackets[1]};
        l.lr_mlp = Bracket{brackets[2], brackets[3]};
        l.lambda_eik = Bracket{brackets[4], brackets[5]};
        l.lambda_sdf = Bracket{brackets[6], brackets[7]};
        l.lambda_features = Bracket{brackets[8], brackets[9]};
        l.lambda_normal = Bracket{brackets[10], brackets[11]};
        l.lambda_probes = Bracket{brackets[12], brackets[13]};
        l.tau = Bracket{brackets[14], brackets[15]};
        sched.lods = {l};
        Checkpoint ck;
        ck.grid = s->grid;
        ck.mlp = s->mlp;
        ck.seed = seed;
        TrainStats st = train(ds, sched, ck, nullptr);
        s->grid = ck.grid;
        s->mlp = ck.mlp;
        if (final_psnr) *final_psnr = st.final_psnr;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// synth.cpp:204-236: analytic ground truth for a scene of primitives with the
// acceptance lights (acceptance.cpp:54-74).
int ref_raytrace(int n_prims, const int32_t* kinds, const double* centers, const double* extents,
                 const double* albedo, const double* r0, const double* spec_exp, int n_lights,
                 const double* light_pos, const double* light_int, const RefCamera* cam,
                 double* rgb, double* mask) {
    try {
        AnalyticScene sc;
        for (int i = 0; i < n_prims; ++i) {
            Primitive p;
            p.kind = kinds[i] == 0 ? Primitive::Kind::Sphere
                     : kinds[i] == 1 ? Primitive::Kind::Box
                                     : Primitive::Kind::Torus;
            p.center = {centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]};
            p.extent = {extents[3 * i], extents[3 * i + 1], extents[3 * i + 2]};
            p.material.albedo = {albedo[3 * i], albedo[3 * i + 1], albedo[3 * i + 2]};
            p.material.r0 = r0[i];
            p.material.spec_exp = spec_exp[i];
            sc.primitives.push_back(p);
        }
        for (int i = 0; i < n_lights; ++i) {
            Light l;
            l.kind = Light::Kind::Point;
            l.pos_or_dir = {light_pos[3 * i], light_pos[3 * i + 1], light_pos[3 * i + 2]};
            l.intensity = {light_int[3 * i], light_int[3 * i + 1], light_int[3 * i + 2]};
            sc.lights.push_back(l);
        }
        RaytraceResult rt = raytrace(sc, to_cam(cam));
        std::memcpy(rgb, rt.image.data.data(), rt.image.data.size() * sizeof(double));
        std::memcpy(mask, rt.mask.data.data(), rt.mask.data.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// gradcheck.cpp:163-219 (the reference's own FD audit).
int ref_gradcheck(uint64_t seed, double h, double tol, int samples, double* max_rel, int* pass) {
    GradCheckReport r = run_gradcheck(seed, h, tol, samples);
    for (size_t i = 0; i < r.classes.size() && i < 5; ++i) max_rel[i] = r.classes[i].max_rel_err;
    *pass = r.pass ? 1 : 0;
    return static_cast<int>(r.classes.size());
}

// Known-answer helpers from the reference unit tests.
double ref_alpha_from_sdf(double a, double b, double tau) { return alpha_from_sdf(a, b, tau); }
void ref_eval_sh_basis(const double* dir, int order, double* out) {
    eval_sh_basis({dir[0], dir[1], dir[2]}, order, out);
}
void ref_fresnel_powers(double ndv, double* out) { fresnel_powers(ndv, out); }
void ref_gaussian_kernel(double* out) {
    const auto& w = gaussian_kernel_1d();
    for (int i = 0; i < 5; ++i) out[i] = w[i];
}
void ref_adam_steps(int n, double* params, const double* grads_seq, int steps, const double* lrs) {
    AdamState a(n);
    for (int t = 0; t < steps; ++t) a.step(params, grads_seq + static_cast<size_t>(t) * n, lrs[t]);
}

// metrics.cpp:196-211 psnr_masked (evaluation of a rendered view).
int ref_psnr_masked(const double* img, const double* gt, const double* mask, int w, int h, double* out) {
    try {
        ImageRGB a(w, h), b(w, h);
        ImageGray m(w, h);
        std::memcpy(a.data.data(), img, a.data.size() * sizeof(double));
        std::memcpy(b.data.data(), gt, b.data.size() * sizeof(double));
        std::memcpy(m.data.data(), mask, m.data.size() * sizeof(double));
        *out = psnr_masked(a, b, m);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// mesh.cpp:363 marching_cubes of the scene's smoothed grid; call with zero
// capacities for the sizes, then again with buffers.
int ref_marching_cubes(RefScene* s, double* verts, int64_t vcap, int32_t* tris, int64_t tcap, int64_t* nv,
                       int64_t* nt) {
    try {
        const TriMesh m = marching_cubes(s->grid);
        *nv = static_cast<int64_t>(m.vertices.size());
        *nt = static_cast<int64_t>(m.triangles.size());
        if (verts && tris && vcap >= *nv && tcap >= *nt) {
            for (int64_t i = 0; i < *nv; ++i) {
                verts[3 * i] = m.vertices[i].x;
                verts[3 * i + 1] = m.vertices[i].y;
                verts[3 * i + 2] = m.vertices[i].z;
            }
            for (int64_t i = 0; i < *nt; ++i)
                for (int k = 0; k < 3; ++k) tris[3 * i + k] = m.triangles[i][k];
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// mesh.cpp:396 marching_cubes_field over a dense field (x-major), same
// two-call protocol as ref_marching_cubes.
int ref_marching_cubes_field(const double* values, int nx, int ny, int nz, const double origin[3],
                             double spacing, double* verts, int64_t vcap, int32_t* tris, int64_t tcap,
                             int64_t* nv, int64_t* nt) {
    try {
        std::vector<double> vals(values, values + static_cast<size_t>(nx) * ny * nz);
        const TriMesh m = marching_cubes_field(vals, nx, ny, nz, Vec3(origin[0], origin[1], origin[2]), spacing);
        *nv = static_cast<int64_t>(m.vertices.size());
        *nt = static_cast<int64_t>(m.triangles.size());
        if (verts && tris && vcap >= *nv && tcap >= *nt) {
            for (int64_t i = 0; i < *nv; ++i) {
                verts[3 * i] = m.vertices[i].x;
                verts[3 * i + 1] = m.vertices[i].y;
                verts[3 * i + 2] = m.vertices[i].z;
            }
            for (int64_t i = 0; i < *nt; ++i)
                for (int k = 0; k < 3; ++k) tris[3 * i + k] = m.triangles[i][k];
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

static TriMesh to_mesh(const double* verts, int64_t nv, const int32_t* tris, int64_t nt) {
    TriMesh m;
    m.vertices.resize(nv);
    for (int64_t i = 0; i < nv; ++i) m.vertices[i] = {verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]};
    m.triangles.resize(nt);
    for (int64_t i = 0; i < nt; ++i) m.triangles[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    return m;
}

static std::vector<Vec3> to_points(const double* p, int64_t n) {
    std::vector<Vec3> v(n);
    for (int64_t i = 0; i < n; ++i) v[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
    return v;
}

// metrics.cpp:131-135 MeshDistance::distance for each point.
int ref_point_mesh_distance(const double* pts, int64_t n, const double* verts, int64_t nv, const int32_t* tris,
                            int64_t nt, double* out) {
    try {
        const TriMesh m = to_mesh(verts, nv, tris, nt);
        const MeshDistance md(m);
        for (int64_t i = 0; i < n; ++i) out[i] = md.distance({pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// metrics.cpp:137-166 sample_mesh_points.
int ref_sample_mesh_points(const double* verts, int64_t nv, const int32_t* tris, int64_t nt, int n, uint64_t seed,
                           double* out) {
    try {
        const auto pts = sample_mesh_points(to_mesh(verts, nv, tris, nt), n, seed);
        for (int i = 0; i < n; ++i) {
            out[3 * i] = pts[i].x;
            out[3 * i + 1] = pts[i].y;
            out[3 * i + 2] = pts[i].z;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// metrics.cpp:182-194 chamfer; out = {accuracy, completeness, mean}.
int ref_chamfer(const double* pp, int64_t np, const double* pv, int64_t pnv, const int32_t* pt, int64_t pnt,
                const double* gp, int64_t ng, const double* gv, int64_t gnv, const int32_t* gt, int64_t gnt,
                double max_dist, double* out) {
    try {
        const ChamferResult r = chamfer(to_points(pp, np), to_mesh(pv, pnv, pt, pnt), to_points(gp, ng),
                                        to_mesh(gv, gnv, gt, gnt), max_dist);
        out[0] = r.accuracy;
        out[1] = r.completeness;
        out[2] = r.mean;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

} // extern "C"

