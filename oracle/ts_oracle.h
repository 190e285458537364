/*
 * ts_oracle.h — CPU restatement of the reference's 3DGS training hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the timed
 * CPU baseline.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product
 * (paper_2602_09999_b200/, libtilesplat_b200.so) never links or calls it.
 *
 * Every function restates an operation of /root/reference/SPEC.md (cited per
 * function in ts_oracle.cpp).  The reference ships no implementation and no
 * test vectors beyond the SPEC's per-op examples, so the oracle is pinned by
 * those examples (tests/test_oracle_spec.py), by central finite differences in
 * 64-bit mode, by brute-force culling / sorting / Adam cross-checks, and by
 * compiling the reference's own vecmath.hpp beside our header (oracle/_ref).
 *
 * Layout conventions:
 *   params: one flat fp32 array of 59*N floats, attribute blocks in order
 *     means[N][3] | log_scales[N][3] | quats[N][4] (w,x,y,z) | opacity_logits[N]
 *     | sh_dc[N][3] | sh_rest[N][15][3]
 *   images: H*W*3 interleaved (row-major), T and contributor count H*W.
 */
#ifndef TS_ORACLE_H
#define TS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field layout as ts_camera / ts_render_config in include/tilesplat_c.h,
 * redeclared so the oracle has no include dependency on the product. */
typedef struct {
    float W[16]; /* world->camera, row-major 4x4 */
    float fx, fy, cx, cy, near_plane;
    int32_t width, height;
} tso_camera;

typedef struct {
    int32_t sh_degree;        /* active SH degree 0..3 */
    int32_t bound_mode;       /* 0 square, 1 rect, 2 rect_opacity */
    int32_t cull_mode;        /* 0 none, 1 exact */
    int32_t truncation;       /* 0 classic, 1 response */
    int32_t early_stop_compat;/* 0 blend-then-stop, 1 skip-before-blend */
    int32_t backward_mode;    /* 0 per-pixel, 1 per-gaussian buckets */
    float tau_alpha;          /* 1/255 */
    float dilation;           /* 0.3 when AA off */
    float sigma_cut;          /* response truncation cutoff (sigmas) */
    float bg[3];
    int32_t aa_mode;          /* 0 off, 1 filter3d_original, 2 filter3d_clip, 3 full = clip + mip */
    float kappa3d;            /* 3D filter variance kappa_3D = 0.2 */
} tso_render_config;

/* ---- antialias ---- */
/* compute_sampling_rates: nu[g] = max over cameras where the mean passes frustum culling
 * (z > near, |x/z| <= 1.3 tan(fov_x/2), |y/z| <= 1.3 tan(fov_y/2)) of max(fx, fy) / z;
 * 1 / extent when visible in none. */
void tso_compute_sampling_rates(int64_t n, const float* params, const tso_camera* cams, int32_t ncams, float extent,
                                float* nu);
/* sampling rates used by preprocess / backward in aa_mode 1 (filter3d_original) */
void tso_set_sampling_rates(int64_t n, const float* nu);
/* apply_3d_filter_clip: log_scales <- max(log_scales, log(sqrt(kappa) / nu)), in place */
void tso_apply_3d_filter_clip(int64_t n, float* params, const float* nu, float kappa3d);

/* worker threads used by every parallel loop (0 = hardware_concurrency) */
void tso_set_workers(int n);
int tso_get_workers(void);

/* deterministic scalar math shared with the product's numerics contract */
float tso_cos2pi(float u);
float tso_expf(float x);
float tso_logf(float x);

/* ---- per-Gaussian ops (SPEC core/camera), exposed for the SPEC golden tests ---- */
/* rotation_from_quaternion: returns 0 if degenerate (||q||<1e-4), R row-major 3x3 */
int tso_rotation_from_quaternion_f64(const double q[4], double R[9]);
void tso_build_covariance3d_f64(const double R[9], const double s[3], double cov6[6]);
void tso_eval_sh_f64(const double* coeffs48 /*[16][3]*/, const double dir[3], int deg, double rgb[3]);
/* returns 0 if out of frustum */
int tso_project_mean_f64(const tso_camera* cam, const double mean[3], double mean2d[2], double cam_pt[3]);
void tso_project_covariance_f64(const tso_camera* cam, const double cam_pt[3], const double cov6[6], double cov2d[3]);
/* returns 0 if degenerate */
int tso_invert_cov2d_f64(const double cov2d[3], double dilation, double conic[3], double* det);

/* ---- forward ---- */
/* preprocess (K1 restatement).  splat: N*12 floats {mx,my,k2,o, A,B,C,depth, r,g,b,det};
 * rect: N*4 int32 tile rect (tx0,ty0,tx1,ty1) (tx0>tx1 when empty);
 * tile_count: N; depth_key: N (0xFFFFFFFF when count==0). */
void tso_preprocess(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg,
                    float* splat, int32_t* rect, uint32_t* tile_count, uint32_t* depth_key);
/* Gaussian-major instance list; keys = tile<<32 | depthkey, vals = gaussian.
 * offsets: N+1 exclusive scan of tile_count.  Returns I. */
int64_t tso_build_instances(int64_t n, const float* splat, const int32_t* rect, const uint32_t* tile_count,
                            const uint32_t* depth_key, const tso_camera* cam, const tso_render_config* cfg,
                            uint64_t* keys, uint32_t* vals);
/* single stable sort on the packed 64-bit key (SPEC.md:247 oracle) */
void tso_sort_combined(int64_t I, uint64_t* keys, uint32_t* vals);
/* two-stage LSD radix: stable 32-bit depth sort then stable tile sort.
 * Returns key bytes touched (bench metric). */
int64_t tso_sort_two_stage(int64_t I, int tile_bits, uint64_t* keys, uint32_t* vals);
void tso_tile_ranges(int64_t I, const uint64_t* sorted_keys, int32_t n_tiles, uint32_t* ranges /*2*Tn*/);

/* full render.  rgb H*W*3, T H*W, count H*W (each may be NULL).
 * Returns I (instances) or -1 on validation error. */
int64_t tso_render(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg,
                   float* rgb, float* T, uint32_t* count);
int64_t tso_render_f64(int64_t n, const double* params, const tso_camera* cam, const tso_render_config* cfg,
                       double* rgb, double* T, uint32_t* count);
/* blend weights sum check: out[p] = sum_i alpha_i T_i + T_final */
void tso_render_weight_sum(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg,
                           double* out);

/* ---- loss : returns loss, writes dL/dC (H*W*3) ---- */
double tso_training_loss(int32_t H, int32_t W, const float* rgb, const float* target, float* dL_dC);
double tso_training_loss_f64(int32_t H, int32_t W, const double* rgb, const double* target, double* dL_dC);

/* ---- backward ----
 * grads: 59*N (accumulated: +=), grad2d: N*9 optional (+=) {dmx,dmy,dA,dB,dC,do,dr,dg,db},
 * accum/count: N densify stats (+=). */
void tso_backward(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg,
                  const float* dL_dC, float* grads, float* grad2d, float* accum, float* vcount);
void tso_backward_f64(int64_t n, const double* params, const tso_camera* cam, const tso_render_config* cfg,
                      const double* dL_dC, double* grads, double* grad2d, double* accum, double* vcount);

/* ---- optimizer ----
 * lr[6] per group (means, log_scales, quats, opacity, sh_dc, sh_rest); mode 0 reference, 1 fused,
 * 2 skip-invisible (visible mask per Gaussian).  bc1 = 1-b1^t, bc2 = 1-b2^t (host double->float). */
void tso_adam_step(int64_t n, float* params, const float* grads, float* m, float* v, const float lr[6],
                   float beta1, float beta2, float eps, float bc1, float bc2, int32_t mode,
                   const uint8_t* visible);
void tso_adam_step_f64(int64_t n, double* params, const double* grads, double* m, double* v,
                       const double lr[6], double beta1, double beta2, double eps, double bc1, double bc2);
double tso_mean_lr(int64_t step, double extent);

/* ---- densify ----
 * Inputs n rows of params/m/v/accum/count; outputs up to 3n rows (caller allocates 3n).
 * Returns n_after and fills out_stats[3] = {clones, splits, pruned}. */
int64_t tso_densify_and_prune(int64_t n, const float* params, const float* m, const float* v,
                              const float* accum, const float* vcount, float grad_thresh, float extent,
                              uint64_t seed, int64_t iter, float* out_params, float* out_m, float* out_v,
                              int64_t* out_stats);
void tso_opacity_reset(int64_t n, float* params);
/* ---- morton_reorder ----
 * interleave: bits per axis, x in the least significant position of each triple. */
uint64_t tso_morton_interleave(uint32_t qx, uint32_t qy, uint32_t qz, int bits);
/* 63-bit codes of the means quantised to 21 bits over the AABB inflated by 1e-6 */
void tso_morton_codes(int64_t n, const float* params, uint64_t* codes);
/* stable sort by code; permutes params/m/v (59n each, may be NULL) and accum/vcount (n, may be NULL)
 * in place; perm[new] = old. */
void tso_morton_reorder(int64_t n, float* params, float* m, float* v, float* accum, float* vcount, uint32_t* perm);
/* full single-view training step (render, loss vs target HWC, backward, fused Adam);
 * stage_seconds[8] = {preprocess, binning, blend, loss, raster_bwd, project_bwd, adam, I}. */
double tso_train_step(int64_t n, float* params, float* m, float* v, const tso_camera* cam,
                      const tso_render_config* cfg, const float* target, const float lr[6], float beta1,
                      float beta2, float eps, float bc1, float bc2, float* accum, float* vcount,
                      double* stage_seconds);
int32_t tso_sh_active_degree(int64_t iter);
double tso_scene_extent(int32_t n_cams, const double* centers /*n*3*/);

#ifdef __cplusplus
}
#endif
#endif
