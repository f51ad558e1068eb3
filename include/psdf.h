/* psdf.h — C ABI of the B200-native ProbeSDF fused render + train hot path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj).  The reference exposes it as a C++ static-library
 * API with no FFI; each entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only: no C++ or
 * torch types cross this boundary.  All functions return a status code
 * (PSDF_OK == 0); psdf_last_error() gives the message.  The C++ drop-in shim
 * (include/sdfrecon_gpu.hpp) maps the codes back to the reference's exception
 * types (std::invalid_argument / std::out_of_range / std::runtime_error).
 *
 * Threading: one host thread and one CUDA stream per context; one context per
 * GPU (rank).  Device memory is owned by the context; host buffers are
 * borrowed for the duration of the call.
 *
 * Flat layouts (identical to the reference's storage order):
 *   tile_coords [T][3] int32          tile lattice coordinates (grid.hpp:25)
 *   probe_ids   [T][8] int32          corner probes, bit0->x bit1->y bit2->z
 *                                     (grid.cpp:70-71)
 *   probe_coords[P][3] int32          probe lattice coordinates (grid.hpp:86)
 *   raw, smooth [T][4096] f32         x-major (x*16+y)*16+z (grid.hpp:26-27)
 *   planes      [T][3][256][n_s] f32  plane_x (y,z), plane_y (x,z),
 *                                     plane_z (x,y) (grid.hpp:28-35)
 *   probes      [P][l*l][n_a] f32     band-major coefficient blocks (sh.hpp:15-23)
 *   mlp         f32 w1[32][in] b1[32] w2[32][32] b2[32] w3[3][32] b3[3]
 *               camera_bias[ncam][32], in = n_s + n_a + 6 (decoder.hpp:17-31)
 *   images      rgb [h][w][3] f32 row-major, mask [h][w] uint8 (!=0 = in)
 */
#ifndef PSDF_H
#define PSDF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSDF_ABI_VERSION 1

enum {
    PSDF_OK = 0,
    PSDF_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    PSDF_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range */
    PSDF_ERR_RUNTIME = 3,          /* std::runtime_error */
    PSDF_ERR_CUDA = 4,
    PSDF_ERR_NCCL = 5,
};

typedef struct psdf_ctx psdf_ctx;

/* Camera (camera.hpp:12-17): pinhole, world-from-camera rotation row-major. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double rot[9];
    double pos[3];
    int32_t id, pad_;
} psdf_camera;

/* RenderOptions (renderer.hpp:13-27). */
typedef struct {
    double tau;
    double early_stop;   /* early_stop_transmittance; 0 disables */
    double bg[3];        /* background */
    int32_t n_max;
    int32_t camera_id;   /* -1 omits the per-camera bias */
    int32_t no_spatial, no_angular, no_fresnel, sh_order_override, need_colors;
} psdf_render_opts;

/* Per-step hyper-parameters, already evaluated for this iteration exactly as
 * trainer.cpp:126-134 does (brackets, warm-up, tau / voxel_size,
 * photo_scale = lambda_photo / images_per_batch). */
typedef struct {
    double tau, lr_vox, lr_mlp, l_sdf, l_eik, l_norm, l_feat, l_probe, photo_scale;
    int32_t use_camera_bias; /* TrainSchedule::camera_bias (trainer.cpp:153) */
    int32_t pad_;
} psdf_step_params;

/* SparseGrid metadata (grid.hpp:57-70). */
typedef struct {
    int32_t T, P;              /* allocated tiles, pool probes */
    int32_t n_s, n_a, sh_order; /* channel widths, any pair in [1, 8] x [1, 8] (the
                                  reference's DecoderMlp takes any width,
                                  decoder.hpp:17-31).  The kernels are
                                  instantiated for (2,2), (4,4), (8,8), (4,8),
                                  (8,4); another pair runs on the smallest of
                                  those that holds it, its extra channels zero
                                  planes / probes / W1 columns (results
                                  unchanged), and every array crossing this ABI
                                  stays at the caller's widths.  Wider pairs are
                                  PSDF_ERR_INVALID_ARGUMENT ("unsupported (n_s,
                                  n_a)") before any work */
    int32_t res[3];            /* voxels per axis, multiples of 16 */
    double voxel_size;
    double origin[3];
    double far_field_voxels;
    int32_t ncam;              /* camera-bias rows in the MLP (0 = disabled) */
    int32_t pad_;
} psdf_grid_desc;

/* Statistics of one render / train pass (the oracle's RayWorkspace counts). */
typedef struct {
    int64_t n_rays;     /* rays traced */
    int64_t n_marched;  /* samples kept after early termination (N_m) */
    int64_t n_extra;    /* rays with >= 1 sample (N_x) */
    int64_t n_shaded;   /* decoded samples (N_sh) */
    int64_t n_alpha;    /* samples with alpha > 0 on rays run backward (N_alpha) */
    int64_t n_bwd_rays; /* rays with a non-zero loss gradient */
} psdf_counts;

/* Losses of one step — the trainer.cpp:201-207 log line. */
typedef struct {
    double photo, sdf, eik, normal, features, probes, total, psnr;
    double sq_err, mask_px;
} psdf_losses;

/* ---- context ----------------------------------------------------------- */
int psdf_abi_version(void);
int psdf_create(int device, psdf_ctx** out);
int psdf_destroy(psdf_ctx* ctx);
/* Message of the last failed call on this thread (ctx may be NULL). */
const char* psdf_last_error(psdf_ctx* ctx);

/* ---- scene state ---------------------------------------------------------
 * Replaces constructing a sdfrecon::SparseGrid / DecoderMlp in host memory
 * (grid.hpp:57-132, decoder.hpp:17-31); uploaded once per LOD.  smooth may be
 * NULL, in which case it is recomputed on the device (SparseGrid::smooth_all,
 * grid.cpp:247-250).  Uploading a grid resets the optimizer state. */
int psdf_upload_grid(psdf_ctx* ctx, const psdf_grid_desc* desc, const int32_t* tile_coords,
                     const int32_t* probe_ids, const int32_t* probe_coords, const float* raw,
                     const float* smooth, const float* planes, const float* probes);
int psdf_upload_mlp(psdf_ctx* ctx, const float* mlp, int64_t n);
int64_t psdf_mlp_size(int n_s, int n_a, int ncam);
/* Copies parameters device -> host (any pointer may be NULL). */
int psdf_download_params(psdf_ctx* ctx, float* raw, float* smooth, float* planes, float* probes,
                         float* mlp);
/* Gradient buffers of the last train step (parity / debugging).
 * stage 0: after the ray pass (GradBuffers after trainer.cpp:184-185);
 * stage 1: what Adam consumed (after regularizers + G^T fold, trainer.cpp:193).
 * smooth = the smooth-staged SDF gradient (grads.hpp:15). */
/* ---- LOD transitions ---------------------------------
 * The current grid's description and its tile / probe structure (the order
 * of SparseGrid::tiles / probes, grid.hpp:103-107; arrays of 3 T, 8 T and
 * 3 P ints; any pointer may be NULL). */
int psdf_grid_info(psdf_ctx* ctx, psdf_grid_desc* out);
int psdf_download_structure(psdf_ctx* ctx, int32_t* tile_coords, int32_t* probe_ids, int32_t* probe_coords);
/* Replaces grid = grid.subdivide() (SparseGrid::subdivide, grid.cpp:271-345;
 * called at trainer.cpp:213): the device grid becomes its 2x subdivision —
 * children kept unless min |raw| > band_voxels * h_new with no sign change,
 * planes upsampled, probes re-interpolated on the doubled lattice, smoothed;
 * same tile / probe order as the reference.  Optimizer state is reset.
 * out_T / out_P (may be NULL) receive the new counts. */
int psdf_subdivide(psdf_ctx* ctx, double band_voxels, int32_t* out_T, int32_t* out_P);
/* Replaces SparseGrid::raise_sh_order (grid.cpp:252-262, trainer.cpp:105):
 * std::invalid_argument (PSDF_ERR_INVALID_ARGUMENT) if the order decreases or
 * exceeds 4; new bands start at zero.  Optimizer state is reset. */
int psdf_raise_sh_order(psdf_ctx* ctx, int new_order);

/* Replaces init_grid_visual_hull(cfg, cameras, masks) (grid.cpp:470-504,
 * SURVEY.md 8f row 3; the CLI default init, main.cpp:188-192): the context's
 * grid becomes the visual-hull initialisation — occupancy by projection into
 * every mask (uint8, > 127 = foreground), squared EDTs to the occupied and the
 * free set, seed SDF, tiles within band_voxels — with the reference's tile /
 * probe order and defaults (planes 0.5, probes 0, smoothed).  desc gives the
 * configuration (res, voxel_size, origin, n_s, n_a, sh_order,
 * far_field_voxels, ncam; T / P ignored); the MLP is zero until
 * psdf_upload_mlp.  out_T / out_P may be NULL. */
int psdf_init_visual_hull(psdf_ctx* ctx, const psdf_grid_desc* desc, int band_voxels, int n_cams,
                          const psdf_camera* cams, const uint8_t* const* masks, int32_t* out_T, int32_t* out_P);

/* ---- SDFC v1 checkpoints -------------------------------
 * Replace save_checkpoint / load_checkpoint (checkpoint.cpp:54-181): the same
 * file layout (little-endian f32 tensors, tile / probe order, decoder, LOD
 * cursor), read into / written from the device grid; the grid description has
 * no lod / band_voxels, so they travel as arguments.  Errors are
 * PSDF_ERR_RUNTIME (std::runtime_error) with the reference's messages.  A
 * load re-smooths on the device and resets the optimizer. */
int psdf_save_checkpoint(psdf_ctx* ctx, const char* path, int32_t lod, int32_t band_voxels, int32_t lod_cursor,
                         int64_t iteration, uint64_t seed);
int psdf_load_checkpoint(psdf_ctx* ctx, const char* path, int32_t* lod, int32_t* band_voxels, int32_t* lod_cursor,
                         int64_t* iteration, uint64_t* seed);

/* Keep a copy of the stage-0 (post ray pass) gradients on every step. */
int psdf_set_keep_raypass_grads(psdf_ctx* ctx, int keep);
int psdf_download_grads(psdf_ctx* ctx, int stage, float* raw, float* smooth, float* planes,
                        float* probes, float* mlp);
/* SparseGrid::smooth_all (grid.cpp:247-250) on the device. */
int psdf_smooth_all(psdf_ctx* ctx);

/* ---- render ----------------------------------------------------------------
 * render_image (renderer.cpp:321-337 / renderer.hpp:98-99).  Host outputs:
 * rgb [h][w][3], alpha [h][w] (RenderedImage), depth [h][w] = sum_i w_i t_i
 * (extension; NULL to skip).  counts may be NULL. */
int psdf_render(psdf_ctx* ctx, const psdf_camera* cam, const psdf_render_opts* opt, float* rgb,
                float* alpha, float* depth, psdf_counts* counts);
/* Same, device-resident outputs (pointers into device memory). */
int psdf_render_device(psdf_ctx* ctx, const psdf_camera* cam, const psdf_render_opts* opt,
                       float* d_rgb, float* d_alpha, float* d_depth, psdf_counts* counts);
/* Evaluation: psnr_masked (metrics.cpp:196-211, metrics.hpp:51) of this
   context's render of `cam` (with `opt`) against a host ground-truth view.
   gt_rgb: H*W*3 f32 row-major; mask: H*W u8, nonzero = inside (the reference's
   mask > 0.5, as psdf_train_step).  Squared error summed in f64 on the device;
   99 dB when the mask is empty or the error is 0, capped at 99. */
int psdf_eval_psnr(psdf_ctx* ctx, const psdf_camera* cam, const psdf_render_opts* opt,
                   const float* gt_rgb, const uint8_t* mask, double* psnr, psdf_counts* counts);
/* Evaluation geometry (metrics.cpp, metrics.hpp:15-48).  Meshes are host
   TriMesh arrays: verts nv x 3 f64, tris nt x 3 i32; points n x 3 f64.
   psdf_point_mesh_distance = MeshDistance(mesh).distance(p) per point
   (metrics.cpp:131-135), exact minimum over the triangles on the device.
   psdf_chamfer = chamfer(pred_points, pred_mesh, gt_points, gt_mesh, max_dist)
   (metrics.cpp:182-194): out[3] = {accuracy, completeness, mean}, x1000.
   Errors as the reference: empty mesh / empty input -> INVALID_ARGUMENT; a
   triangle index outside the vertex array -> OUT_OF_RANGE. */
int psdf_point_mesh_distance(psdf_ctx* ctx, const double* points, int64_t n, const double* verts, int64_t nv,
                             const int32_t* tris, int64_t nt, double* out_dist);
int psdf_chamfer(psdf_ctx* ctx, const double* pred_pts, int64_t n_pred, const double* pred_verts,
                 int64_t pred_nv, const int32_t* pred_tris, int64_t pred_nt, const double* gt_pts,
                 int64_t n_gt, const double* gt_verts, int64_t gt_nv, const int32_t* gt_tris, int64_t gt_nt,
                 double max_dist, double* out);

/* Marching cubes (mesh.cpp:305-394, marching_cubes(grid)) of the context's
   smoothed SDF on the device: the reference's mesh exactly (same vertex ids
   and f64 positions, same triangles in the same order; cells with a corner in
   an unallocated tile vetoed, zero-area triangles dropped).  The mesh stays in
   the context; psdf_download_mesh copies it out (verts nv x 3 f64, tris nt x 3
   i32).  An empty grid gives an empty mesh. */
int psdf_marching_cubes(psdf_ctx* ctx, int64_t* nv, int64_t* nt);
int psdf_download_mesh(psdf_ctx* ctx, double* verts, int32_t* tris);

/* ---- train ------------------------------------------------------------------
 * One iteration of the train() loop body (trainer.cpp:136-195): clear
 * gradients, ray pass over every pixel of the batch views (render_ray +
 * photo_pixel + render_ray_backward), regularizers, G^T fold, Adam, re-smooth.
 * Host images: gt_rgb[i] [h][w][3] f32, mask[i] [h][w] u8 (nonzero = in
 * mask); colours are read only at in-mask pixels, and only the rows between a
 * view's first and last mask row are copied to the device.  With a
 * communicator (psdf_comm_init) each rank processes its contiguous 1/N slice
 * of the batch's pixels and the gradients are all-reduced before Adam. */
int psdf_train_reset(psdf_ctx* ctx); /* fresh Adam state (trainer.cpp:115) */
int psdf_train_step(psdf_ctx* ctx, int n_views, const psdf_camera* cams,
                    const float* const* gt_rgb, const uint8_t* const* mask,
                    const psdf_step_params* hp, psdf_losses* losses, psdf_counts* counts);
/* Dataset kept resident in HBM: upload once, then step by view index. */
int psdf_upload_views(psdf_ctx* ctx, int n_views, const psdf_camera* cams,
                      const float* const* gt_rgb, const uint8_t* const* mask);
int psdf_train_step_views(psdf_ctx* ctx, int n_batch, const int32_t* view_ids,
                          const psdf_step_params* hp, psdf_losses* losses, psdf_counts* counts);

/* ---- test hooks for the bit-exact indexing contract ------------------------
 * march_ray (renderer.cpp:55-86 / renderer.hpp:39-40) for n explicit rays:
 * ts [n][n_max] (row-major), counts [n] = samples of each ray. */
int psdf_march_rays(psdf_ctx* ctx, int n, const double* origins, const double* dirs, int n_max,
                    double* ts, int32_t* counts);
/* Camera::pixel_dir (camera.hpp:32-35) at every pixel centre: out [h][w][3]. */
int psdf_pixel_dirs(const psdf_camera* cam, double* out);

/* ---- multi-GPU (ray-batch data parallel) ------------ */
#define PSDF_UNIQUE_ID_BYTES 128
int psdf_comm_unique_id(void* out /* PSDF_UNIQUE_ID_BYTES */);
int psdf_comm_init(psdf_ctx* ctx, const void* unique_id, int rank, int world_size);
/* Test hook: act as `rank` of `world_size` WITHOUT a communicator — the
 * step processes only this rank's slice (work tiles, regularizer tiles /
 * probes, and psdf_train_step copies only the slice's pixel rows) and skips
 * the all-reduce, so the stage-1 gradients of the N slices sum to the
 * one-rank gradients (tests/test_gpu_shard.py). */
int psdf_debug_set_shard(psdf_ctx* ctx, int rank, int world_size);
/* How the ranks combine gradients each step (effective with a communicator):
   ALLREDUCE (default): G^T fold, then one all-reduce of the flat gradient;
   BUCKETED: the [planes | probes | mlp] bucket all-reduced on a second stream
     under the fold, then the raw-SDF bucket;
   SHARDED: fold, reduce-scatter into world-size chunks, Adam on this rank's
     chunk, all-gather of the updated parameters (same bytes as an
     all-reduce, 1/N of the Adam work per rank).
   All three give every rank the same parameters as the single-rank step
   (with SHARDED, psdf_download_grads(stage 1) holds the summed gradient only
   on this rank's chunk). */
enum { PSDF_EXCHANGE_ALLREDUCE = 0, PSDF_EXCHANGE_BUCKETED = 1, PSDF_EXCHANGE_SHARDED = 2 };
int psdf_set_grad_exchange(psdf_ctx* ctx, int mode);
/* Diagnostics: raw copy of n items of one ray-pass queue of the last pass
   (psdf.cu psdf_debug_wave lists the queues and item sizes). */
int psdf_debug_wave(psdf_ctx* ctx, int which, void* out, int64_t n);

/* ---- timing / introspection ------------------------------------------------ */
/* Device time (ms) of the last call's dominant kernel (the fused ray-pass
 * kernel), measured with CUDA events on the context's stream, and the number
 * of kernels the last call launched. */
int psdf_last_timing(psdf_ctx* ctx, double* ray_kernel_ms, double* step_ms, int* launches);
/* Device time (ms) of the four K2 kernels of the last train step (march_fwd,
 * shade_fwd, alpha_bwd, shade_bwd) and the ray-entry / shading-record counts. */
int psdf_last_k2_breakdown(psdf_ctx* ctx, double* ms4, int64_t* entries, int64_t* records);
/* Queue sizes of the last train step's ray pass: ray entries, shading
   records, scan hand-overs, round-1 continuations, alpha samples.  Records
   are the valid ones; the entry and alpha-sample counts include the holes
   of the march's abandoned allocation chunks (slots never written). */
int psdf_last_wave_counts(psdf_ctx* ctx, int64_t* out5);
/* Raw CUDA stream of the context (cudaStream_t), for callers that time or
 * overlap work around the context. */
void* psdf_stream(psdf_ctx* ctx);
/* Host -> device bytes the last psdf_train_step copied (images + masks). */
int64_t psdf_last_h2d_bytes(psdf_ctx* ctx);
/* Page-locked host memory for staging images (cudaMallocHost). */
void* psdf_host_alloc(size_t bytes);
void psdf_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* PSDF_H */
