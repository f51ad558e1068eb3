// TEST INFRASTRUCTURE: exercises include/sdfrecon_gpu.hpp exactly as a
// reference maintainer would — the reference's own types and entry points on
// the CPU (sdfrecon::render_image / sdfrecon::train) against the drop-ins on
// the GPU (sdfrecon_gpu::render_image / sdfrecon_gpu::train), same inputs.
// Built by oracle/Makefile (needs the reference headers); run by
// tests/test_gpu_dropin.py.  Prints one "key value" line per metric.
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>

#include "sdfrecon/synth.hpp"
#include "sdfrecon_gpu.hpp"

using namespace sdfrecon;

static double maxdiff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

static void round_f32(std::vector<double>& v) {
    for (double& x : v) x = (double)(float)x;
}

int main() {
    // a seeded scene in the pattern of test_renderer.cpp:21-45, values
    // fp32-representable so both sides see identical inputs
    GridConfig cfg;
    cfg.resolution = {32, 32, 32};
    cfg.voxel_size = 1.0 / 32.0;
    cfg.n_s = cfg.n_a = 4;
    cfg.sh_order = 3;
    cfg.band_voxels = 32;
    SparseGrid grid = init_grid_sphere(cfg, {0, 0, 0}, 0.3);
    std::mt19937_64 rng(6);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    for (Tile& t : grid.tiles) {
        for (double& v : t.plane_x) v = 0.5 + 0.2 * uni(rng);
        for (double& v : t.plane_y) v = 0.5 + 0.2 * uni(rng);
        for (double& v : t.plane_z) v = 0.5 + 0.2 * uni(rng);
        round_f32(t.raw_sdf);
        round_f32(t.plane_x);
        round_f32(t.plane_y);
        round_f32(t.plane_z);
    }
    for (ProbeSH& p : grid.probes) {
        for (double& c : p.coeffs) c = 0.3 * uni(rng);
        round_f32(p.coeffs);
    }
    grid.smooth_all();
    for (Tile& t : grid.tiles) round_f32(t.smooth_sdf);
    DecoderMlp mlp = DecoderMlp::glorot_init(4, 4, 0, 7);
    for (auto* w : {&mlp.w1, &mlp.w2, &mlp.w3}) round_f32(*w);

    const Camera cam = make_lookat_camera(0, {1.3, 0.2, 0.4}, {0, 0, 0}, {0, 1, 0}, 57.6, 57.6, 48, 48);
    RenderOptions opt;
    opt.tau = 2000.0;
    const RenderedImage a = render_image(grid, mlp, cam, opt);
    const RenderedImage b = sdfrecon_gpu::render_image(grid, mlp, cam, opt);
    std::printf("render_color_maxdiff %.3e\n", maxdiff(a.color.data, b.color.data));
    std::printf("render_alpha_maxdiff %.3e\n", maxdiff(a.alpha.data, b.alpha.data));

    // exceptions map to the reference's types
    try {
        RenderOptions bad = opt;
        DecoderMlp m2 = DecoderMlp::glorot_init(4, 4, 2, 7);
        bad.camera_id = 5;
        sdfrecon_gpu::render_image(grid, m2, cam, bad);
        std::printf("out_of_range_thrown 0\n");
    } catch (const std::out_of_range&) {
        std::printf("out_of_range_thrown 1\n");
    }

    // train(): two LODs (32^3 -> 64^3 subdivide on the host), 8 ring views
    AnalyticScene sc;
    Primitive p;
    p.extent = {0.3, 0.3, 0.3};
    p.material.albedo = {0.55, 0.3, 0.2};
    p.material.r0 = 0.08;
    sc.primitives.push_back(p);
    Light l1;
    l1.pos_or_dir = {1.5, 2.0, 1.0};
    l1.intensity = {6.0, 6.0, 5.5};
    sc.lights = {l1};
    const Dataset ds = make_dataset(sc, 8, 32, 2.0, 0);
    TrainSchedule sched;
    LodSchedule l;
    l.iterations = 20;
    l.images_per_batch = 2;
    l.sh_order = 3;
    l.lr_voxels = Bracket{2e-3, 1e-3};
    l.lr_mlp = Bracket{2e-3, 1e-3};
    l.tau = Bracket{30.0, 60.0};
    sched.lods = {l, l};
    GridConfig c16 = cfg;
    c16.resolution = {16, 16, 16};
    c16.voxel_size = 1.0 / 16.0;
    Checkpoint ck_cpu;
    ck_cpu.grid = init_grid_sphere(c16, {0, 0, 0}, 0.32);
    ck_cpu.mlp = DecoderMlp::glorot_init(4, 4, 0, 3);
    for (auto* w : {&ck_cpu.mlp.w1, &ck_cpu.mlp.w2, &ck_cpu.mlp.w3}) round_f32(*w);
    for (Tile& t : ck_cpu.grid.tiles) round_f32(t.raw_sdf);
    ck_cpu.grid.smooth_all();
    for (Tile& t : ck_cpu.grid.tiles) round_f32(t.smooth_sdf);
    Checkpoint ck_gpu = ck_cpu;
    std::ostringstream log_cpu, log_gpu;
    const TrainStats sa = train(ds, sched, ck_cpu, &log_cpu);
    const TrainStats sb = sdfrecon_gpu::train(ds, sched, ck_gpu, &log_gpu);
    std::printf("train_steps %ld %ld\n", sa.steps_run, sb.steps_run);
    std::printf("train_psnr %.6f %.6f\n", sa.final_psnr, sb.final_psnr);
    std::printf("train_tiles %zu %zu\n", ck_cpu.grid.tiles.size(), ck_gpu.grid.tiles.size());
    double dr = 0.0, mr = 0.0;
    for (size_t t = 0; t < std::min(ck_cpu.grid.tiles.size(), ck_gpu.grid.tiles.size()); ++t)
        for (int v = 0; v < 4096; ++v) {
            dr = std::max(dr, std::abs(ck_cpu.grid.tiles[t].raw_sdf[v] - ck_gpu.grid.tiles[t].raw_sdf[v]));
            mr = std::max(mr, std::abs(ck_cpu.grid.tiles[t].raw_sdf[v]));
        }
    std::printf("train_raw_maxdiff %.3e of %.3e\n", dr, mr);
    std::printf("train_cursor %d %d\n", ck_cpu.lod_cursor, ck_gpu.lod_cursor);
    const std::string lc = log_cpu.str(), lg = log_gpu.str();
    std::printf("log_lines %zu %zu\n", (size_t)std::count(lc.begin(), lc.end(), '\n'),
                (size_t)std::count(lg.begin(), lg.end(), '\n'));

    // evaluation (acceptance.cpp:266-300 pattern): chamfer of the two trained
    // grids' marching-cubes meshes, and psnr_masked of a render of view 0
    const TriMesh ma = marching_cubes(ck_cpu.grid), mb = marching_cubes(ck_gpu.grid);
    const auto pa = sample_mesh_points(ma, 3000, 1), pb = sample_mesh_points(mb, 3000, 2);
    sdfrecon_gpu::Device dev(0);
    for (double md : {0.0, 0.01}) {
        const ChamferResult ca = chamfer(pa, ma, pb, mb, md);
        const ChamferResult cb = sdfrecon_gpu::chamfer(dev, pa, ma, pb, mb, md);
        std::printf("chamfer_equal %d\n", ca.accuracy == cb.accuracy && ca.completeness == cb.completeness &&
                                               ca.mean == cb.mean ? 1 : 0);
    }
    dev.upload(ck_gpu.grid, ck_gpu.mlp);
    RenderOptions eo;
    eo.tau = 60.0 / ck_gpu.grid.voxel_size;
    const RenderedImage ri = render_image(ck_gpu.grid, ck_gpu.mlp, ds.views[0].camera, eo);
    const double psnr_cpu = psnr_masked(ri.color, ds.views[0].image, ds.views[0].mask);
    const double psnr_gpu = sdfrecon_gpu::psnr_masked_render(dev, ds.views[0].camera, eo, ds.views[0].image,
                                                             ds.views[0].mask);
    std::printf("eval_psnr %.6f %.6f\n", psnr_cpu, psnr_gpu);
    return 0;
}
