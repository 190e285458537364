/*
 * tilesplat_c.h — C-ABI of the B200-native Faster-GS training hot path
 * (libtilesplat_b200.so, sm_100a).
 *
 * The reference (arxiv 2602.09999 artifact, /root/reference) ships its API as
 * the C++ namespace `tilesplat` (proj/include/tilesplat/vecmath.hpp:11-245) plus
 * the typed operation list of SPEC.md; it has no FFI of its own.  Each entry
 * point below replaces one SPEC operation (cited); the C++ wrapper
 * include/tilesplat/tilesplat.hpp and the Python mirror
 * paper_2602_09999_b200/tilesplat.py sit on top of it.  INTEGRATION.md shows
 * the ctypes / C++ bindings.
 *
 * Conventions:
 *  - plain pointers and sizes only; host buffers are borrowed for the call;
 *    the context owns all device memory;
 *  - every call returns ts_status and never throws; ts_last_error() explains;
 *  - a context is bound to one device and one CUDA stream and is not
 *    thread-safe (one host thread per GPU);
 *  - calls are stream-ordered; calls that return host data synchronize;
 *  - there is no CPU fallback: without a usable sm_100 device every call that
 *    needs one returns TS_ERR_CUDA.
 *
 * Data layouts:
 *  - parameters / gradients / Adam moments: one flat fp32 buffer of 59*N,
 *    blocks means[N][3] | log_scales[N][3] | quats[N][4] (w,x,y,z)
 *    | opacity_logits[N] | sh_dc[N][3] | sh_rest[N][15][3]
 *  - host images: H*W*3 interleaved fp32; T and contributor
 *    count H*W.
 */
#ifndef TILESPLAT_C_H
#define TILESPLAT_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ts_ctx ts_ctx;

/* 0/1/2 mirror the reference CLI exit codes. */
typedef enum {
    TS_OK = 0,
    TS_ERR_VALIDATION = 1,
    TS_ERR_CHECK = 2,
    TS_ERR_CUDA = 3,
    TS_ERR_OOM = 4,
    TS_ERR_STATE = 5
} ts_status;

/* Camera: world->camera W (row-major 4x4), intrinsics, size. */
typedef struct {
    float W[16];
    float fx, fy, cx, cy, near_plane;
    int32_t width, height;
} ts_camera;

/* Per-view render flags (TrainConfig subset). */
typedef struct {
    int32_t sh_degree;         /* active degree 0..3                    */
    int32_t bound_mode;        /* 0 square, 1 rect, 2 rect_opacity     */
    int32_t cull_mode;         /* 0 none, 1 exact tile culling         */
    int32_t truncation;        /* 0 classic, 1 response: keep iff Q <= sigma_cut^2       */
                               /*                                       */
    int32_t early_stop_compat; /* 0 blend-then-stop, 1 skip-before-blend   */
    int32_t backward_mode;     /* 0 per-pixel replay + reduction,     */
                               /* 1 per-Gaussian buckets; the forward then records the  */
                               /* BlendCheckpoint            */
    float tau_alpha;           /* 1/255                                                  */
    float dilation;            /* 0.3 with AA off (DESIGN.md App. A.1)                   */
    float sigma_cut;           /* response truncation cutoff in sigmas (3.33)            */
    float bg[3];               /* background colour c_bg                                 */
    int32_t aa_mode;           /* 0 off, 1 filter3d_original, 2 filter3d_clip, 3 full    */
                               /* (clip + Mip 2D filter, dilation 0.1) */
    float kappa3d;             /* 3D filter variance kappa_3D, 0.2         */
} ts_render_config;

/* Adam: per-group lr (means, log_scales, quats, opacity,
 * sh_dc, sh_rest), betas, eps, host-computed bias corrections 1-b^t, mode
 * (0 reference, 1 fused, 2 skip-invisible, 3 fused_backward,
 * 4 fused_backward_skip_invisible; modes 3/4 only in ts_backward_adam /
 * ts_train_step), zero_grads (1: clear the gradient buffer in the same sweep). */
typedef struct {
    float lr[6];
    float beta1, beta2, eps, bc1, bc2;
    int32_t mode;
    int32_t zero_grads;
} ts_adam_config;

/* ---- lifetime ---- */
ts_status ts_create(int32_t device, void* cuda_stream /* NULL: own stream */, ts_ctx** out);
ts_status ts_destroy(ts_ctx* ctx);
const char* ts_last_error(const ts_ctx* ctx);
const char* ts_version(void);
ts_status ts_synchronize(ts_ctx* ctx);

/* ---- ParameterStore ---- */
ts_status ts_set_params(ts_ctx* ctx, int64_t n, const float* means, const float* log_scales, const float* quats,
                        const float* opacity_logits, const float* sh_dc, const float* sh_rest);
ts_status ts_set_params_flat(ts_ctx* ctx, int64_t n, const float* flat /* 59*n host */);
ts_status ts_get_params_flat(ts_ctx* ctx, float* flat /* 59*n host */);
ts_status ts_num_gaussians(const ts_ctx* ctx, int64_t* n);

/* ---- render: preprocess, bin, sort, blend ---- */
ts_status ts_forward(ts_ctx* ctx, const ts_camera* cam, const ts_render_config* cfg, float* out_rgb /* H*W*3 */,
                     float* out_T /* H*W */, uint32_t* out_count /* H*W */);

/* ---- training_loss on the last forward; writes dL/dC on device ---- */
ts_status ts_set_target(ts_ctx* ctx, int32_t slot, int32_t width, int32_t height, const float* target_hwc);
ts_status ts_loss(ts_ctx* ctx, const float* target_hwc /* host, or NULL to use slot */, int32_t slot,
                  float* out_loss);

/* ---- backward: accumulates into the gradient buffer ---- */
ts_status ts_backward(ts_ctx* ctx, const float* dL_dC_hwc /* host, or NULL: use ts_loss result */);
ts_status ts_zero_grads(ts_ctx* ctx);
/* mark the gradient buffer consumed without clearing it (data-parallel sharded optimizer:
 * each rank's Adam consumed only its own slice): the next backward overwrites every row
 * (zeros for Gaussians it does not see) instead of accumulating. */
ts_status ts_mark_grads_consumed(ts_ctx* ctx);
ts_status ts_grad_buffer(ts_ctx* ctx, float** dev_ptr, int64_t* count); /* 59*N device fp32 (for NCCL) */
ts_status ts_param_buffer(ts_ctx* ctx, float** dev_ptr, int64_t* count);
ts_status ts_stats_buffer(ts_ctx* ctx, float** dev_accum, float** dev_count);
/* grow the parameter / gradient buffers to >= min_len floats (zero-filled pad
 * beyond 59*N) so collectives can use equal-sized shards */
ts_status ts_reserve_flat(ts_ctx* ctx, int64_t min_len);

/* ---- optimizer ---- */
ts_status ts_adam_step(ts_ctx* ctx, const ts_adam_config* cfg);
/* Adam over [begin, end) of the flat buffer only (sharded optimizer for data parallel). */
ts_status ts_adam_step_range(ts_ctx* ctx, const ts_adam_config* cfg, int64_t begin, int64_t end);

/* fused_backward_update: backward of the last forward with the Adam
 * update applied to each Gaussian's gradient row in place (modes 3/4); the end state
 * equals ts_backward + ts_adam_step(mode 1/2) bitwise.  Only for single-view steps
 * (the gradient buffer is neither read nor written). */
ts_status ts_backward_adam(ts_ctx* ctx, const float* dL_dC_hwc /* or NULL: ts_loss result */,
                           const ts_adam_config* adam);

/* ---- one training step on one view: forward, loss, backward, Adam ---- */
ts_status ts_train_step(ts_ctx* ctx, const ts_camera* cam, const ts_render_config* cfg,
                        const float* target_hwc /* host (pinned preferred) or NULL: slot */, int32_t target_slot,
                        const ts_adam_config* adam, float* out_loss /* may be NULL: no D2H */);

/* CUDA-graph mode of ts_train_step (default off): each (view, render config, target slot or host
 * target address, optimizer mode) is captured once into a CUDA graph -- forward, loss, backward,
 * Adam, the host-target upload as a parallel branch -- and relaunched per step with no host round
 * trip inside the step; the per-step optimizer arguments enter through device memory.  The first
 * step of a view runs on the host path (sizes the buffers), the second captures.  A graph step
 * that outgrows its buffers is voided on the device and replayed on the host path before any
 * other call observes state, so results equal the host-driven path.  A host target must stay
 * valid (and unchanged) until the next synchronising call.  Modes 3/4, the radix binning path,
 * antialias mode 1 and profiling run host-driven. */
ts_status ts_set_graph(ts_ctx* ctx, int32_t on);
/* {graph launches, captures, replayed (voided) steps, live graphs} */
ts_status ts_graph_stats(ts_ctx* ctx, int64_t out[4]);

/* ---- densification ---- */
ts_status ts_densify(ts_ctx* ctx, float grad_thresh, float extent, uint64_t seed, int64_t iter,
                     int64_t* n_after, int64_t stats[3] /* clones, splits, pruned */);
ts_status ts_opacity_reset(ts_ctx* ctx);
/* morton_reorder: permute params, Adam moments and densify statistics into
 * 63-bit Morton order of the means; perm (N, may be NULL) receives old index per new row. */
ts_status ts_morton_reorder(ts_ctx* ctx, uint32_t* perm);

/* ---- antialias ---- */
/* compute_sampling_rates: nu[g] = max over the cameras whose frustum (z > near, |x/z|, |y/z| within
 * the 1.3 tan(fov/2) J-clamp limits) contains the mean of max(fx, fy) / z; 1 / extent if none.
 * Kept by the context for aa_mode 1 and the 3D-filter clip; invalidated by densify / reorder. */
ts_status ts_compute_sampling_rates(ts_ctx* ctx, const ts_camera* cams, int32_t n_cams, float extent);
ts_status ts_set_sampling_rates(ts_ctx* ctx, const float* nu /* N host */);
ts_status ts_get_sampling_rates(ts_ctx* ctx, float* nu /* N host */);
/* apply_3d_filter_clip: log_scales <- max(log_scales, log(sqrt(kappa3d) / nu)) (after an optimizer step) */
ts_status ts_apply_3d_filter_clip(ts_ctx* ctx, float kappa3d);

/* ---- state access for tests / checkpointing ---- */
ts_status ts_set_state(ts_ctx* ctx, const float* grads, const float* m, const float* v, const float* accum,
                       const float* vcount); /* each may be NULL */
ts_status ts_get_state(ts_ctx* ctx, float* grads, float* m, float* v, float* accum, float* vcount);

/* ---- binning path: 0 auto = bucketed binning + per-tile sort (lists up to
 * 65536 instances, frames up to 51200 tiles), falling back to the two-stage radix sort (depth
 * sort over N, tile sort over I) beyond that; 1 = always the radix path.  Both give
 * bit-identical tile lists. ---- */
ts_status ts_set_binning(ts_ctx* ctx, int32_t mode);
ts_status ts_binning_path(ts_ctx* ctx, int32_t* radix /* 1 if the last forward used the radix path */);

/* ---- parity / debug hooks (bit-exact contract) ---- */
ts_status ts_debug_preprocess(ts_ctx* ctx, float* splat12 /* N*12 */, int32_t* rect4 /* N*4 */,
                              uint32_t* tile_count /* N */, uint32_t* depth_key /* N */);
ts_status ts_debug_instances(ts_ctx* ctx, int64_t* n_inst, uint64_t* keys /* I */, uint32_t* vals /* I */,
                             uint32_t* ranges /* 2*Tn */);
/* dL/dC of the last ts_loss (H*W*3 interleaved, host) */
ts_status ts_debug_loss_grad(ts_ctx* ctx, float* dLdC_hwc);
/* per-Gaussian 2D gradients {dmx,dmy,dA,dB,dC,do,dr,dg,db} of the blend backward (K8 only) of the
 * last forward for the given dL/dC; does not touch the parameter gradients. */
ts_status ts_debug_grad2d(ts_ctx* ctx, const float* dL_dC_hwc, float* g2d9 /* N*9 */);
/* counters of the last view: {V visible, I instances, Ip processed instances, P pixels} */
ts_status ts_view_stats(ts_ctx* ctx, int64_t out[4]);
/* per-stage device times: while profiling is on, every stage of every call is
 * bracketed by CUDA events on the context stream; ts_stage_times returns the
 * summed milliseconds and call counts per stage since ts_set_profiling(1):
 * {preprocess, depth_sort, scan, duplicate, tile_sort, ranges, blend, loss, blend_bwd, project_bwd, adam} */
ts_status ts_set_profiling(ts_ctx* ctx, int32_t on);
ts_status ts_stage_times(ts_ctx* ctx, float* ms, int32_t* counts /* may be NULL */, int32_t n);
/* number of kernels this context has launched (evidence counter) */
ts_status ts_launch_count(ts_ctx* ctx, int64_t* n);

/* pinned host memory for e2e staging */
ts_status ts_host_alloc(size_t bytes, void** out);
ts_status ts_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* TILESPLAT_C_H */
