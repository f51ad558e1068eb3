/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * psdf_oracle: a plain-C, f64, single-threaded restatement of the reference's
 * fused render + train hot path (/root/reference/proj/src), used only as the
 * parity checker for the CUDA path (tests/, __graft_entry__.smoke()) and as a
 * "port" CPU baseline.  Each function cites the reference file:line it
 * restates.  It is pinned against the compiled reference in
 * tests/test_oracle_vs_reference.py and against tests/golden/.
 *
 * Layouts are the CUDA path's upload layouts (include/psdf.h), in f64:
 *   tile_coords [T][3] int32, probe_ids [T][8] int32, probe_coords [P][3]
 *   raw, smooth [T][4096] (x-major (x*16+y)*16+z, grid.hpp:23-34)
 *   planes      [T][3][256][n_s] (plane_x (y,z), plane_y (x,z), plane_z (x,y))
 *   probes      [P][l*l][n_a]
 *   mlp         w1[32][in] b1[32] w2[32][32] b2[32] w3[3][32] b3[3] cam[ncam][32]
 */
#ifndef PSDF_ORACLE_H
#define PSDF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct OGrid OGrid;

typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double rot[9];
    double pos[3];
    int32_t id, pad_;
} OCamera; /* same memory layout as RefCamera / psdf_camera */

typedef struct {
    double tau, early_stop, bg[3];
    int32_t n_max, camera_id, no_spatial, no_angular, no_fresnel, sh_order_override, need_colors;
} ORenderOpts;

typedef struct {
    double tau, lr_vox, lr_mlp, l_sdf, l_eik, l_norm, l_feat, l_probe, photo_scale;
    int32_t use_camera_bias, pad_;
} OStepParams;

OGrid* og_create(int T, int P, int n_s, int n_a, int sh_order, const int32_t* res,
                 double voxel_size, const double* origin, double far_field_voxels,
                 const int32_t* tile_coords, const int32_t* probe_ids, const int32_t* probe_coords,
                 const double* raw, const double* smooth /* NULL: smooth here */,
                 const double* planes, const double* probes, const double* mlp, int ncam);
void og_free(OGrid* g);
int64_t og_mlp_size(const OGrid* g);
void og_export(const OGrid* g, double* raw, double* smooth, double* planes, double* probes,
               double* mlp);
void og_smooth_all(OGrid* g);

int og_march_ray(const OGrid* g, const double* o, const double* d, int n_max, double* ts);
void og_pixel_dir(const OCamera* c, double u, double v, double* d);
void og_pixel_dirs(const OCamera* c, double* out);
/* per-ray: result[6] = color xyz, acc, trans_end, depth; returns #samples */
int og_render_ray(const OGrid* g, const double* o, const double* d, const ORenderOpts* opt,
                  double* result);
/* counts [5] = N_rays, N_m, N_x, N_sh, N_alpha */
void og_render_image(const OGrid* g, const OCamera* cam, const ORenderOpts* opt, double* rgb,
                     double* alpha, double* depth, int64_t* counts);

/* Gradient buffers in the same flat layouts. */
typedef struct {
    double *raw, *smooth, *planes, *probes, *mlp;
} OGrads;
OGrads* og_grads_new(const OGrid* g);
void og_grads_free(OGrads* gb);
void og_grads_clear(const OGrid* g, OGrads* gb);
void og_grads_export(const OGrid* g, const OGrads* gb, double* raw, double* smooth, double* planes,
                     double* probes, double* mlp);

void og_ray_backward(const OGrid* g, const double* o, const double* d, const ORenderOpts* opt,
                     const double* up_color, double up_alpha, OGrads* gb);
void og_photo_pixel(const double* c, const double* gt, int in_mask, double acc, double scale,
                    double* out /* plain, weighted, dc xyz, dalpha */);
/* which: 0 sdf, 1 eik, 2 normal, 3 features, 4 probes; out: plain, weighted */
void og_regularizer(const OGrid* g, int which, double lambda, OGrads* gb, double* out);
void og_gt_fold(const OGrid* g, OGrads* gb);
/* loss over tiles [begin, end) (which 0..3) or probes [begin, end) (which 4) */
void og_regularizer_range(const OGrid* g, int which, double lambda, int begin, int end, OGrads* gb,
                          double* out);
/* ray pass over the 8x4 work tiles [tile_begin, tile_end) of the batch */
void og_raypass_tiles(const OGrid* g, int n_views, const OCamera* cams, const double* const* gt_rgb,
                      const double* const* mask, const OStepParams* hp, int64_t tile_begin,
                      int64_t tile_end, OGrads* gb, double* losses);

/* known-answer hooks (the reference's unit-test constants) */
double og_alpha_from_sdf(double si, double sn, double tau);
void og_sh_basis(const double* dir, int order, double* out);
void og_fresnel_powers(double ndv, double* out);
void og_gaussian_taps(double* out);
void og_adam_steps(int n, double* params, const double* grads_seq, int steps, const double* lrs);

/* Training: Adam state lives in the grid object. */
void og_train_reset(OGrid* g);
/* losses[10] as ref_train_step; counts[6] as ref_train_step */
void og_train_step(OGrid* g, int n_views, const OCamera* cams, const double* const* gt_rgb,
                   const double* const* mask, const OStepParams* hp, double* losses,
                   int64_t* counts, OGrads* raypass_out /* nullable */, OGrads* final_out);

#ifdef __cplusplus
}
#endif
#endif
