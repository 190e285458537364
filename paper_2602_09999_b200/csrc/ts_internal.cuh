// ts_internal.cuh — device buffers, context and kernel launcher declarations.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tilesplat_c.h"

namespace ts {

constexpr int kTile = 16;
constexpr int kParams = 59;
constexpr int kG2D = 12;  // floats per Gaussian in the 2D-gradient accumulator (9 used, 16B aligned)
constexpr int kNumStages = 11;
constexpr int kGraphFlag = 12;  // counters[kGraphFlag]: sticky overflow flag of graph-captured steps
// Largest store: the flat 59*N sweeps (Adam, densify, Morton) index in 32 bits, so
// 59*N (+ float4 padding) must stay below 2^32.  ~72M Gaussians = ~85 GB of store +
// moments + gradients, within a 180 GB B200; ts_set_params* and ts_densify reject more.
constexpr int64_t kMaxGaussians = (int64_t(0xFFFFFFFFu) - 64) / 59;

// flat 59*N buffer block offsets
struct Off {
    int64_t means, ls, q, op, dc, rest;
    __host__ __device__ explicit Off(int64_t n)
        : means(0), ls(3 * n), q(6 * n), op(10 * n), dc(11 * n), rest(14 * n) {}
};

// Device-side camera with derived constants (computed in-kernel from ts_camera
// fields so the float op sequence matches the oracle's Cam<float>).
struct DevCam {
    float W[16];
    float fx, fy, cx, cy, nearp;
    int w, h, tiles_x, tiles_y;
    float limx, limy;  // J ratio clamps 1.3 * (0.5 w / fx), 1.3 * (0.5 h / fy) (host float, the oracle's Cam op order)
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
};

// CUDA-graph mode of ts_train_step: one instantiated graph per (view, config, target, mode)
struct GraphEntry {
    ts_camera cam;
    ts_render_config cfg;
    const float* target;  // host target (pinned, fixed address) or nullptr (slot)
    int32_t slot, want_loss, mode;
    int64_t N;
    uint64_t gen;
    cudaGraphExec_t exec;
    int64_t kernels;     // kernel nodes of the graph (launch-count evidence)
    uint32_t cls[7];     // size-class tile counts of the view's host-path step (sort grid hints)
    int64_t I;           // its instance count (list capacity of the capture)
};
// a graph step launched but not yet known to have passed its capacity check
struct GraphStep {
    ts_camera cam;
    ts_render_config cfg;
    const float* target;
    int32_t slot;
    ts_adam_config adam;
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    int sm_count = 148;
    int64_t launches = 0;

    // ParameterStore + optimizer state + gradients (59*N each)
    int64_t N = 0;
    DevBuf<float> params, grads, m, v, accum, vcount;
    int64_t step = 0;
    // gradient buffer state: ZERO (all zero), STALE (consumed by the optimizer, not
    // cleared: the next backward overwrites every row), LIVE (holds gradients of
    // >= 1 view not yet consumed: the next backward accumulates)
    enum GradState { kGradZero, kGradStale, kGradLive } grad_state = kGradZero;

    // per-view (sized by N)
    DevBuf<float4> splat;        // 3 float4 per Gaussian: (mx,my,k2,o) (A,B,C,depth) (r,g,b,det)
    DevBuf<float> ryv;           // per Gaussian: half-height of the keep ellipse for the blend row cull
    DevBuf<uint4> rect;          // {tx0|tx1<<16, ty0|ty1<<16 (bit31: >64 tiles), kept-tile mask lo, hi}
    DevBuf<uint32_t> tcount;     // tiles per Gaussian
    DevBuf<uint32_t> dkey[2];    // depth keys (radix double buffer)
    DevBuf<uint32_t> dperm[2];   // gaussian indices (radix double buffer)
    DevBuf<uint32_t> offsets;    // N+1 exclusive scan (depth-sorted order)
    DevBuf<float4> g2d;          // 3 float4 per Gaussian, 2D grad accumulator
    DevBuf<uint8_t> vis;         // visible in any view since the last optimizer step
    // instances
    int64_t I = 0;
    DevBuf<uint16_t> tkey[2];    // 16-bit tile keys (radix path, < 2^16 tiles)
    DevBuf<uint32_t> tkey32[2];  // 32-bit tile keys (radix path, >= 2^16 tiles)
    DevBuf<uint32_t> ival[2];
    DevBuf<uint32_t> starts;     // Tn+1
    // radix scratch
    DevBuf<uint32_t> rhist;      // 256 * blocks
    DevBuf<unsigned long long> scan_state;
    DevBuf<uint32_t> scan_tmp;
    DevBuf<uint32_t> counters;   // [0] scan tile ticket, [1] visible V, [2] Ip, [3..] spare
    // frame (planar CHW)
    int fw = 0, fh = 0;
    DevBuf<float> rgb, Tfin, dLdC, hwc_stage, tgt;
    DevBuf<uint32_t> pcount;
    DevBuf<double> loss_acc;     // [0] L1 sum, [1] SSIM sum
    DevBuf<float> targets;       // target slots, CHW planar
    int n_target_slots = 0, target_w = 0, target_h = 0;

    // last view (forward -> backward contract)
    bool view_valid = false;
    bool loss_valid = false;
    ts_camera cam{};
    ts_render_config cfg{};
    int64_t last_V = 0, last_Ip = 0;
    bool stats_valid = false;

    // profiling
    bool profiling = false;
    std::vector<cudaEvent_t> ev_b, ev_e;
    std::vector<int> ev_stage;
    size_t ev_cursor = 0;

    DevBuf<uint32_t> dens;       // densify scratch
    DevBuf<DevCam> cams;         // camera set of compute_sampling_rates
    DevBuf<float> spare;         // a second 59*N store: densify / Morton write into it and swap it in
    DevBuf<unsigned long long> mcode[2];  // Morton codes (radix double buffer)
    DevBuf<uint32_t> midx[2];             // Morton permutation (radix double buffer)

    // binning (k_bin.cu): per-chunk tile histograms, tile totals (+ max list length)
    DevBuf<uint32_t> binH, bintot;
    DevBuf<uint32_t> tile_order;   // blend order of the tiles (longest lists first)
    bool order_ok = false;         // tile_order is valid for the current view
    DevBuf<uint32_t> tile_proc;    // per tile: list positions the forward processed (its max contributor count)
    DevBuf<uint32_t> bwd_order;    // blend-backward order: tiles by descending processed length
    DevBuf<float4> ckpt;           // BlendCheckpoint: (T, C) per pixel at every 32-entry bucket start
    bool ckpt_valid = false;       // the last forward wrote checkpoints
    bool bwd_order_ok = false;
    uint32_t* bin_host = nullptr;  // pinned read-back of (I, class counts, longest list)
    cudaEvent_t bin_ev = nullptr;
    cudaEvent_t bin_fork = nullptr;  // counts ready on the engine stream (read back on side[1])
    DevBuf<float> nu_hat;        // sampling rates (antialias), N floats
    bool nu_valid = false;       // computed for the current ParameterStore rows
    uint32_t bin_class[7] = {0, 0, 0, 0, 0, 0, 0};  // tiles per per-tile sort size class (last view)
    DevBuf<uint32_t> sortmp;     // merge scratch of the long-list class (I entries)
    cudaStream_t side[2] = {nullptr, nullptr};  // fork streams for independent launches
    cudaEvent_t fork_ev = nullptr, join_ev[2] = {nullptr, nullptr};
    // host path: the two tile-order kernels run on side[1] (the forward order beside the scatter,
    // the backward order beside the loss), joined before their consumers
    cudaEvent_t ord_fork = nullptr, ord_join = nullptr, bwd_fork = nullptr, bwd_join = nullptr;
    bool bwd_order_pending = false;
    // the 2D-gradient accumulator is all zero (cleared by each forward's K6; a backward accumulates
    // into it and K9 consumes it without clearing)
    bool g2d_clean = true;
    // ts_train_step's host-target upload, overlapped with the forward
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_fork = nullptr, copy_join = nullptr;
    DevBuf<float> tgt_stage;
    double* loss_host = nullptr;  // pinned (L1 sum, SSIM sum) of the last train_step
    cudaEvent_t loss_ev = nullptr;
    int binning_mode = 0;        // 0 auto (bucket + per-tile sort), 1 force the two-stage radix path
    // CUDA-graph mode of ts_train_step (ts_capi.cu graph_step)
    bool graph_on = false;       // ts_set_graph
    bool gmode = false;          // the step being captured: no host reads, device-side counts and checks
    bool capturing = false;      // stream capture active: ensure() must not allocate
    uint64_t gen = 1;            // bumped by every device (re)allocation / buffer swap (graphs embed pointers)
    std::vector<GraphEntry> graphs;
    std::vector<GraphEntry> graph_seen;  // views run once on the host path (buffers sized), exec unused
    std::vector<GraphStep> glog;         // launched graph steps not yet verified
    cudaEvent_t gstep_ev = nullptr;      // recorded after each graph launch
    // events used inside captures (fork / join dependencies, the loss read-back node): an event
    // recorded in a capturing stream may not be waited on outside the graph, so the host path
    // keeps its own set (swapped in and out around each capture)
    cudaEvent_t cap_fork = nullptr, cap_join[2] = {nullptr, nullptr}, cap_copy_fork = nullptr,
                cap_copy_join = nullptr, cap_loss = nullptr;
    uint32_t* gflag_host = nullptr;      // pinned copy of the sticky flag (written inside each graph)
    bool I_on_device = false;            // the last view ran in a graph: c.I is read back lazily
    int64_t graph_launches = 0, graph_captures = 0, graph_replays = 0;
    int cur_tn = 0;              // tiles of the view being binned
    void* adam_dev = nullptr;    // device copy of the per-step Adam arguments (graph mode)
    unsigned char adam_dev_bytes[128] = {};  // host staging of those arguments (size bound)
    bool last_view_radix = false;
};

// ---- kernels / launchers (each returns cudaError_t of the launch) ----
void launch_preprocess(Context& c, const DevCam& cam, const ts_render_config& cfg);
void launch_depth_sort(Context& c);                 // sorts (dkey, perm) for N entries
int64_t launch_scan_counts(Context& c);             // offsets in depth order; returns I (syncs)
void launch_duplicate(Context& c, const DevCam& cam, const ts_render_config& cfg);
void launch_tile_sort(Context& c, int tile_bits, bool key32);
void launch_ranges(Context& c, int n_tiles, bool key32);
// bucketed binning (k_bin.cu): returns I (syncs) and the longest tile list, -1 on OOM
#ifndef TS_BIN_CHUNK
#define TS_BIN_CHUNK 6144  // measured: 6144 beats 8192 (fewer same-address histogram REDs, fuller scatter waves)
#endif
constexpr int kBinChunk = TS_BIN_CHUNK;  // largest chunk of the bucketed binning (Gaussians per histogram row)
// chunk size for N Gaussians: the largest of 6144 / 3072 / 1536 that still gives >= 2 chunk
// CTAs per SM for the scatter (small stores would otherwise leave SMs idle).  Every size is a
// multiple of the scatter's 512 threads (whole rects per thread) and of a warp (K1's per-warp row).
inline int bin_chunk_for(int64_t N, int sm_count) {
    int ch = kBinChunk;
    while (ch > 2048 && (N + ch - 1) / ch < 2 * int64_t(sm_count)) ch >>= 1;
    static_assert(kBinChunk % 2048 == 0, "chunk halvings must stay multiples of 512");
    return ch;
}
bool bin_supported(int Tn);
int bin_sort_cap();
// enqueue the column scan, the tile ranges and the read-back of (I, class counts, longest list)
bool launch_bin_count(Context& c, const DevCam& cam, const ts_render_config& cfg);
// wait for that read-back; returns I (-1 on error)
int64_t finish_bin_count(Context& c, uint32_t* max_len);
// c.tile_order = tiles by descending list length (from the tile ranges; both binning paths)
void launch_tile_order(Context& c, int Tn, cudaStream_t st = nullptr);
// c.bwd_order from the forward's processed lengths (the backward's per-tile work)
void launch_bwd_tile_order(Context& c, int Tn, cudaStream_t st = nullptr);
void launch_bin_scatter(Context& c, const DevCam& cam, const ts_render_config& cfg);
void launch_tile_depth_sort(Context& c, int Tn, uint32_t max_len);
void launch_blend_fwd(Context& c, const DevCam& cam, const ts_render_config& cfg);
void launch_loss(Context& c, const float* target_chw);
void launch_blend_bwd(Context& c, const DevCam& cam, const ts_render_config& cfg);
void launch_project_bwd(Context& c, const DevCam& cam, const ts_render_config& cfg, bool accumulate,
                        bool zero_inactive);
void launch_project_bwd_adam(Context& c, const DevCam& cam, const ts_render_config& cfg, const ts_adam_config& a);
void launch_adam(Context& c, const ts_adam_config& a, int64_t begin, int64_t end);
size_t adam_args_bytes(const ts_adam_config& a, void* out);  // the kernel's argument block of a (<= 128 B)
void launch_hwc_to_chw(Context& c, const float* hwc, float* chw, int P, cudaStream_t st = nullptr);
void launch_chw_to_hwc(Context& c, const float* chw, float* hwc, int P);
void launch_opacity_reset(Context& c, float logit_max);
bool launch_sampling_rates(Context& c, const DevCam* cams_host, int ncams, float extent);
void launch_filter3d_clip(Context& c, float kappa3d);
bool launch_morton_reorder(Context& c, uint32_t* perm_host);
int64_t launch_densify(Context& c, float grad_thresh, float log_small, float log_big, float logit_min,
                       uint64_t seed, int64_t iter, int64_t stats[3]);

// generic device-wide exclusive scan of u32 (decoupled look-back); in may be
// gathered through perm (in[perm[i]]) when perm != nullptr.  out has n+1 entries.
void launch_exclusive_scan(Context& c, const uint32_t* in, const uint32_t* perm, uint32_t* out, int64_t n);


template <class T>
bool ensure(Context& c, DevBuf<T>& b, size_t n, bool keep = false);

// Function attributes and __constant__ tables belong to a device context, and one
// host thread per GPU may drive its own context concurrently: both helpers keep a
// mutex-protected record per (key, device) instead of process-global flags.
// set_func_attr: cudaFuncSetAttribute(fn, attr, value) once per device (retried
// until it succeeds); first_on_device: true exactly once per (key, device).
bool set_func_attr(const Context& c, const void* fn, cudaFuncAttribute attr, int value);
bool first_on_device(const Context& c, const void* key);

// ensure with 25% slack when the buffer has to grow (stores that grow step by step, e.g. by
// densification, reallocate rarely)
template <class T>
bool ensure_grow(Context& c, DevBuf<T>& b, size_t n) {
    if (n <= b.cap && b.p) return true;
    return ensure(c, b, n + n / 4);
}

#define TS_LAUNCHED(c) ((c).launches++)

template <class T>
__host__ __device__ __forceinline__ T tmin(T a, T b) {
    return a < b ? a : b;
}
template <class T>
__host__ __device__ __forceinline__ T tmax(T a, T b) {
    return a < b ? b : a;
}

}  // namespace ts
