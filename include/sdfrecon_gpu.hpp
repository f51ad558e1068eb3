// sdfrecon_gpu.hpp — C++ drop-in for the reference's hot-path entry points,
// implemented over the C ABI of psdf.h (libpsdf.so, sm_100a kernels).
//
// A maintainer of /root/reference/proj adds this header and links libpsdf.so;
// callers switch by replacing
//     sdfrecon::render_image(grid, mlp, cam, opt)        (renderer.hpp:98-99)
//     sdfrecon::train(ds, sched, ckpt, log)              (trainer.hpp:20-21)
// with sdfrecon_gpu::render_image / sdfrecon_gpu::train (same arguments,
// same return types, same exceptions).  The reference's own types
// (SparseGrid, DecoderMlp, Camera, RenderOptions, Dataset, TrainSchedule,
// Checkpoint) are used unchanged.  Inside train() the grid stays resident on
// the device across LODs: raise_sh_order and subdivide run there
// (psdf_raise_sh_order / psdf_subdivide, same tile and probe order as the
// reference); only the per-LOD image downscaling stays host code.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <numeric>
#include <ostream>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "psdf.h"
#include "sdfrecon/checkpoint.hpp"
#include "sdfrecon/dataset.hpp"
#include "sdfrecon/mesh.hpp"
#include "sdfrecon/metrics.hpp"
#include "sdfrecon/renderer.hpp"
#include "sdfrecon/schedule.hpp"
#include "sdfrecon/trainer.hpp"

namespace sdfrecon_gpu {

// Status codes -> the reference's exception types.
inline void check(int rc, psdf_ctx* ctx) {
    if (rc == PSDF_OK) return;
    const std::string msg = psdf_last_error(ctx);
    if (rc == PSDF_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == PSDF_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

inline psdf_camera to_c(const sdfrecon::Camera& c) {
    psdf_camera o{};
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    o.width = c.width;
    o.height = c.height;
    for (int i = 0; i < 9; ++i) o.rot[i] = c.rot[i];
    o.pos[0] = c.pos.x;
    o.pos[1] = c.pos.y;
    o.pos[2] = c.pos.z;
    o.id = c.id;
    return o;
}

inline psdf_render_opts to_c(const sdfrecon::RenderOptions& r) {
    psdf_render_opts o{};
    o.tau = r.tau;
    o.early_stop = r.early_stop_transmittance;
    o.bg[0] = r.background.x;
    o.bg[1] = r.background.y;
    o.bg[2] = r.background.z;
    o.n_max = r.n_max;
    o.camera_id = r.camera_id;
    o.no_spatial = r.no_spatial;
    o.no_angular = r.no_angular;
    o.no_fresnel = r.no_fresnel;
    o.sh_order_override = r.sh_order_override;
    o.need_colors = r.need_colors;
    return o;
}

// One GPU context holding a grid + decoder in HBM.
class Device {
public:
    explicit Device(int device = 0) { check(psdf_create(device, &ctx_), nullptr); }
    ~Device() { psdf_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    psdf_ctx* ctx() const { return ctx_; }

    // SparseGrid (grid.hpp:57-132) + DecoderMlp (decoder.hpp:17-31) -> HBM.
    // The smoothed SDF is uploaded as is (the reference keeps it in sync with
    // the raw SDF after every mutation).
    void upload(const sdfrecon::SparseGrid& g, const sdfrecon::DecoderMlp& m) {
        const int T = (int)g.tiles.size(), P = (int)g.probes.size();
        const size_t ps = 256u * g.n_s, pc = (size_t)g.sh_order * g.sh_order * g.n_a;
        std::vector<int32_t> tc(3 * T), pid(8 * T), pco(3 * P);
        std::vector<float> raw((size_t)T * 4096), sm((size_t)T * 4096), planes(3 * ps * T),
            probes(pc * P);
        for (int t = 0; t < T; ++t) {
            const sdfrecon::Tile& tile = g.tiles[t];
            tc[3 * t] = tile.coords.x;
            tc[3 * t + 1] = tile.coords.y;
            tc[3 * t + 2] = tile.coords.z;
            for (int i = 0; i < 8; ++i) pid[8 * t + i] = tile.probe_ids[i];
            for (int v = 0; v < 4096; ++v) {
                raw[(size_t)t * 4096 + v] = (float)tile.raw_sdf[v];
                sm[(size_t)t * 4096 + v] = (float)tile.smooth_sdf[v];
            }
            for (size_t i = 0; i < ps; ++i) {
                planes[(3 * t + 0) * ps + i] = (float)tile.plane_x[i];
                planes[(3 * t + 1) * ps + i] = (float)tile.plane_y[i];
                planes[(3 * t + 2) * ps + i] = (float)tile.plane_z[i];
            }
        }
        for (int p = 0; p < P; ++p) {
            pco[3 * p] = g.probe_coords[p].x;
            pco[3 * p + 1] = g.probe_coords[p].y;
            pco[3 * p + 2] = g.probe_coords[p].z;
            for (size_t i = 0; i < pc; ++i) probes[p * pc + i] = (float)g.probes[p].coeffs[i];
        }
        psdf_grid_desc d{};
        d.T = T;
        d.P = P;
        d.n_s = g.n_s;
        d.n_a = g.n_a;
        d.sh_order = g.sh_order;
        d.res[0] = g.resolution.x;
        d.res[1] = g.resolution.y;
        d.res[2] = g.resolution.z;
        d.voxel_size = g.voxel_size;
        d.origin[0] = g.origin.x;
        d.origin[1] = g.origin.y;
        d.origin[2] = g.origin.z;
        d.far_field_voxels = g.far_field_voxels;
        d.ncam = m.num_cameras();
        check(psdf_upload_grid(ctx_, &d, tc.data(), pid.data(), pco.data(), raw.data(), sm.data(),
                               planes.data(), probes.data()),
              ctx_);
        std::vector<float> w;
        for (const std::vector<double>* part : {&m.w1, &m.b1, &m.w2, &m.b2, &m.w3, &m.b3, &m.camera_bias})
            for (double x : *part) w.push_back((float)x);
        check(psdf_upload_mlp(ctx_, w.data(), (int64_t)w.size()), ctx_);
    }

    // HBM -> SparseGrid / DecoderMlp values (same topology as uploaded).
    void download(sdfrecon::SparseGrid& g, sdfrecon::DecoderMlp& m) const {
        const int T = (int)g.tiles.size(), P = (int)g.probes.size();
        const size_t ps = 256u * g.n_s, pc = (size_t)g.sh_order * g.sh_order * g.n_a;
        std::vector<float> raw((size_t)T * 4096), sm((size_t)T * 4096), planes(3 * ps * T),
            probes(pc * P);
        size_t nm = m.w1.size() + m.b1.size() + m.w2.size() + m.b2.size() + m.w3.size() +
                    m.b3.size() + m.camera_bias.size();
        std::vector<float> w(nm);
        check(psdf_download_params(ctx_, raw.data(), sm.data(), planes.data(), probes.data(), w.data()),
              ctx_);
        for (int t = 0; t < T; ++t) {
            sdfrecon::Tile& tile = g.tiles[t];
            for (int v = 0; v < 4096; ++v) {
                tile.raw_sdf[v] = raw[(size_t)t * 4096 + v];
                tile.smooth_sdf[v] = sm[(size_t)t * 4096 + v];
            }
            for (size_t i = 0; i < ps; ++i) {
                tile.plane_x[i] = planes[(3 * t + 0) * ps + i];
                tile.plane_y[i] = planes[(3 * t + 1) * ps + i];
                tile.plane_z[i] = planes[(3 * t + 2) * ps + i];
            }
        }
        for (int p = 0; p < P; ++p)
            for (size_t i = 0; i < pc; ++i) g.probes[p].coeffs[i] = probes[p * pc + i];
        size_t off = 0;
        for (std::vector<double>* part : {&m.w1, &m.b1, &m.w2, &m.b2, &m.w3, &m.b3, &m.camera_bias})
            for (double& x : *part) x = w[off++];
    }

private:
    psdf_ctx* ctx_ = nullptr;
};

// render_image (renderer.hpp:98-99) on a grid already resident on `dev`.
inline sdfrecon::RenderedImage render_image(Device& dev, const sdfrecon::Camera& camera,
                                            const sdfrecon::RenderOptions& opt) {
    const psdf_camera c = to_c(camera);
    const psdf_render_opts o = to_c(opt);
    const size_t n = (size_t)camera.width * camera.height;
    std::vector<float> rgb(3 * n), alpha(n);
    check(psdf_render(dev.ctx(), &c, &o, rgb.data(), alpha.data(), nullptr, nullptr), dev.ctx());
    sdfrecon::RenderedImage out;
    out.color = sdfrecon::ImageRGB(camera.width, camera.height);
    out.alpha = sdfrecon::ImageGray(camera.width, camera.height);
    for (size_t i = 0; i < 3 * n; ++i) out.color.data[i] = rgb[i];
    for (size_t i = 0; i < n; ++i) out.alpha.data[i] = alpha[i];
    return out;
}

// Same signature as sdfrecon::render_image: uploads, renders.
inline sdfrecon::RenderedImage render_image(const sdfrecon::SparseGrid& grid,
                                            const sdfrecon::DecoderMlp& mlp,
                                            const sdfrecon::Camera& camera,
                                            const sdfrecon::RenderOptions& opt) {
    Device dev(0);
    dev.upload(grid, mlp);
    return render_image(dev, camera, opt);
}

// The device grid's structure as a host SparseGrid (allocate_tile in the
// device's tile order reproduces the probe pool order, grid.cpp:44-72), with
// its values downloaded.
inline void sync_grid_from_device(const Device& dev, const sdfrecon::SparseGrid& like, int lod,
                                  sdfrecon::SparseGrid& out, sdfrecon::DecoderMlp& mlp) {
    psdf_grid_desc d{};
    check(psdf_grid_info(dev.ctx(), &d), dev.ctx());
    std::vector<int32_t> tc(3 * (size_t)d.T), pid(8 * (size_t)d.T), pco(3 * (size_t)d.P);
    check(psdf_download_structure(dev.ctx(), tc.data(), pid.data(), pco.data()), dev.ctx());
    sdfrecon::SparseGrid g;
    g.voxel_size = d.voxel_size;
    g.origin = sdfrecon::Vec3(d.origin[0], d.origin[1], d.origin[2]);
    g.resolution = {d.res[0], d.res[1], d.res[2]};
    g.n_s = d.n_s;
    g.n_a = d.n_a;
    g.sh_order = d.sh_order;
    g.lod = lod;
    g.far_field_voxels = d.far_field_voxels;
    g.band_voxels = like.band_voxels;
    for (int t = 0; t < d.T; ++t) {
        const int ti = g.allocate_tile(tc[3 * t], tc[3 * t + 1], tc[3 * t + 2]);
        for (int i = 0; i < 8; ++i)
            if (ti != t || g.tiles[t].probe_ids[i] != pid[8 * t + i])
                throw std::runtime_error("sync_grid_from_device: tile / probe order mismatch");
    }
    dev.download(g, mlp);
    out = std::move(g);
}

// train (trainer.cpp:81-220) with the step body and the LOD transitions on
// the GPU.  Identical schedule arithmetic, batch order (mt19937_64 shuffle,
// trainer.cpp:98, 119-145), per-LOD Adam reset, log line and checkpoint
// cursor handling.  The grid stays resident across LODs: raise_sh_order and
// subdivide run on the device (psdf_raise_sh_order / psdf_subdivide, same
// tile and probe order as the reference); only the per-LOD image downscale
// (image.cpp:110-137) is host code; the trained grid is synchronised back
// into ckpt.grid at the end.
inline sdfrecon::TrainStats train(const sdfrecon::Dataset& ds, const sdfrecon::TrainSchedule& sched,
                                  sdfrecon::Checkpoint& ckpt, std::ostream* log = nullptr,
                                  int device = 0) {
    using namespace sdfrecon;
    if (ds.views.empty()) throw std::runtime_error("train: empty dataset");
    if (ckpt.lod_cursor < 0 || ckpt.lod_cursor >= static_cast<int>(sched.lods.size()))
        throw std::runtime_error("train: checkpoint LOD cursor outside the schedule");
    if (ckpt.grid.sh_order > sched.lods[ckpt.lod_cursor].sh_order)
        throw std::runtime_error("train: grid SH order exceeds the schedule's");
    SparseGrid& grid = ckpt.grid;
    DecoderMlp& mlp = ckpt.mlp;
    if (sched.camera_bias && mlp.camera_bias.empty())
        mlp.camera_bias.assign(ds.views.size() * kHidden, 0.0);
    if (sched.camera_bias)
        for (const DatasetView& v : ds.views)
            if (v.camera.id < 0 || v.camera.id >= mlp.num_cameras())
                throw std::runtime_error("train: camera id outside the bias table");
    std::mt19937_64 rng(ckpt.seed);
    TrainStats stats;
    long global_step = 0;
    Device dev(device);
    dev.upload(grid, mlp);
    int lod = grid.lod;
    psdf_grid_desc cur{};
    for (; ckpt.lod_cursor < static_cast<int>(sched.lods.size()); ++ckpt.lod_cursor) {
        const LodSchedule& ls = sched.lods[ckpt.lod_cursor];
        check(psdf_grid_info(dev.ctx(), &cur), dev.ctx());
        if (cur.sh_order < ls.sh_order) {
            check(psdf_raise_sh_order(dev.ctx(), ls.sh_order), dev.ctx());
            check(psdf_grid_info(dev.ctx(), &cur), dev.ctx());
        }
        // per-LOD views, resident in HBM for the whole LOD
        std::vector<psdf_camera> cams;
        std::vector<std::vector<float>> rgb;
        std::vector<std::vector<uint8_t>> msk;
        for (const DatasetView& v : ds.views) {
            const Camera c = v.camera.downscaled(ls.image_divisor);
            const ImageRGB im = downscale(v.image, ls.image_divisor);
            const ImageGray mk = downscale_mask(v.mask, ls.image_divisor);
            cams.push_back(to_c(c));
            rgb.emplace_back(im.data.begin(), im.data.end());
            std::vector<uint8_t> m8(mk.data.size());
            for (size_t i = 0; i < m8.size(); ++i) m8[i] = mk.data[i] > 0.5 ? 1 : 0;
            msk.push_back(std::move(m8));
        }
        std::vector<const float*> rp;
        std::vector<const uint8_t*> mp;
        for (size_t i = 0; i < rgb.size(); ++i) {
            rp.push_back(rgb[i].data());
            mp.push_back(msk[i].data());
        }
        check(psdf_train_reset(dev.ctx()), dev.ctx());  // per-LOD optimizer (trainer.cpp:115)
        check(psdf_upload_views(dev.ctx(), (int)cams.size(), cams.data(), rp.data(), mp.data()), dev.ctx());
        std::vector<int> order(ds.views.size());
        std::iota(order.begin(), order.end(), 0);
        std::shuffle(order.begin(), order.end(), rng);
        size_t order_pos = 0;
        const int total = ls.iterations;
        for (int it = static_cast<int>(ckpt.iteration); it < total; ++it) {
            psdf_step_params hp{};
            hp.lr_vox = ls.lr_voxels.at(it, total) * warmup_scale(it);
            hp.lr_mlp = ls.lr_mlp.at(it, total) * warmup_scale(it);
            hp.l_sdf = ls.lambda_sdf.at(it, total);
            hp.l_eik = ls.lambda_eik.at(it, total);
            hp.l_norm = ls.lambda_normal.at(it, total);
            hp.l_feat = ls.lambda_features.at(it, total);
            hp.l_probe = ls.lambda_probes.at(it, total);
            hp.tau = ls.tau.at_geometric(it, total) / cur.voxel_size;
            hp.photo_scale = sched.lambda_photo / ls.images_per_batch;
            hp.use_camera_bias = sched.camera_bias;
            std::vector<int32_t> batch(ls.images_per_batch);
            for (int32_t& b : batch) {
                if (order_pos == order.size()) {
                    std::shuffle(order.begin(), order.end(), rng);
                    order_pos = 0;
                }
                b = order[order_pos++];
            }
            psdf_losses L{};
            check(psdf_train_step_views(dev.ctx(), (int)batch.size(), batch.data(), &hp, &L, nullptr),
                  dev.ctx());
            stats.final_psnr = L.psnr;
            ++stats.steps_run;
            if (log)
                (*log) << "step " << global_step + it << " lod " << ckpt.lod_cursor << " photo "
                       << L.photo << " sdf " << L.sdf << " eik " << L.eik << " normal " << L.normal
                       << " features " << L.features << " probes " << L.probes << " total "
                       << L.total << " psnr " << L.psnr << '\n';
        }
        global_step += total;
        ckpt.iteration = 0;
        if (ckpt.lod_cursor + 1 < static_cast<int>(sched.lods.size())) {
            check(psdf_subdivide(dev.ctx(), (double)grid.band_voxels, nullptr, nullptr), dev.ctx());
            ++lod;
        }
    }
    sync_grid_from_device(dev, grid, lod, grid, mlp);
    ckpt.lod_cursor = static_cast<int>(sched.lods.size()) - 1;
    ckpt.iteration = sched.lods.back().iterations;
    return stats;
}

// psnr_masked (metrics.cpp:196-211) of a render of the resident grid against
// a ground-truth view, render and reduction on the device.
inline double psnr_masked_render(Device& dev, const sdfrecon::Camera& camera, const sdfrecon::RenderOptions& opt,
                                 const sdfrecon::ImageRGB& gt, const sdfrecon::ImageGray& mask) {
    if (gt.width != camera.width || gt.height != camera.height || mask.width != gt.width ||
        mask.height != gt.height)
        throw std::invalid_argument("psnr_masked: image shape mismatch");
    const psdf_camera c = to_c(camera);
    const psdf_render_opts o = to_c(opt);
    std::vector<float> g(gt.data.begin(), gt.data.end());
    std::vector<uint8_t> m(mask.data.size());
    for (size_t i = 0; i < m.size(); ++i) m[i] = mask.data[i] > 0.5 ? 1 : 0;
    double psnr = 0.0;
    check(psdf_eval_psnr(dev.ctx(), &c, &o, g.data(), m.data(), &psnr, nullptr), dev.ctx());
    return psnr;
}

// marching_cubes (mesh.hpp:24, mesh.cpp:363-394) of the grid resident on
// `dev`: the reference's mesh exactly (same vertices, same triangle order).
inline sdfrecon::TriMesh marching_cubes(Device& dev) {
    int64_t nv = 0, nt = 0;
    check(psdf_marching_cubes(dev.ctx(), &nv, &nt), dev.ctx());
    std::vector<double> v(3 * (size_t)nv);
    std::vector<int32_t> t(3 * (size_t)nt);
    check(psdf_download_mesh(dev.ctx(), v.data(), t.data()), dev.ctx());
    sdfrecon::TriMesh m;
    m.vertices.resize((size_t)nv);
    for (int64_t i = 0; i < nv; ++i) m.vertices[i] = sdfrecon::Vec3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    m.triangles.resize((size_t)nt);
    for (int64_t i = 0; i < nt; ++i) m.triangles[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
    return m;
}

// Same signature as sdfrecon::chamfer (metrics.hpp:46-48); the point-to-mesh
// distances run on `dev`, bit-identical to MeshDistance.
inline sdfrecon::ChamferResult chamfer(Device& dev, const std::vector<sdfrecon::Vec3>& pred_points,
                                       const sdfrecon::TriMesh& pred_mesh,
                                       const std::vector<sdfrecon::Vec3>& gt_points,
                                       const sdfrecon::TriMesh& gt_mesh, double max_dist) {
    auto flat_pts = [](const std::vector<sdfrecon::Vec3>& p) {
        std::vector<double> f(3 * p.size());
        for (size_t i = 0; i < p.size(); ++i) {
            f[3 * i] = p[i].x;
            f[3 * i + 1] = p[i].y;
            f[3 * i + 2] = p[i].z;
        }
        return f;
    };
    auto flat_tris = [](const sdfrecon::TriMesh& m) {
        std::vector<int32_t> t(3 * m.triangles.size());
        for (size_t i = 0; i < m.triangles.size(); ++i)
            for (int k = 0; k < 3; ++k) t[3 * i + k] = m.triangles[i][k];
        return t;
    };
    const auto pp = flat_pts(pred_points), gp = flat_pts(gt_points);
    const auto pv = flat_pts(pred_mesh.vertices), gv = flat_pts(gt_mesh.vertices);
    const auto pt = flat_tris(pred_mesh), gt = flat_tris(gt_mesh);
    double out[3];
    check(psdf_chamfer(dev.ctx(), pp.data(), (int64_t)pred_points.size(), pv.data(),
                       (int64_t)pred_mesh.vertices.size(), pt.data(), (int64_t)pred_mesh.triangles.size(),
                       gp.data(), (int64_t)gt_points.size(), gv.data(), (int64_t)gt_mesh.vertices.size(),
                       gt.data(), (int64_t)gt_mesh.triangles.size(), max_dist, out),
          dev.ctx());
    sdfrecon::ChamferResult r;
    r.accuracy = out[0];
    r.completeness = out[1];
    r.mean = out[2];
    return r;
}

}  // namespace sdfrecon_gpu
