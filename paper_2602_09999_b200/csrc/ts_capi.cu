// ts_capi.cu — C-ABI entry points (include/tilesplat_c.h) and the host runtime:
// context, grow-only device buffers, the per-view pipeline and stage timing.
// Every entry point is noexcept-by-construction (no C++ exceptions cross the
// ABI) and maps CUDA failures to TS_ERR_CUDA with ts_last_error() text.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <set>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ts_internal.cuh"

using namespace ts;

struct ts_ctx {
    Context c;
};

namespace ts {

template <class T>
bool ensure(Context& c, DevBuf<T>& b, size_t n, bool keep) {
    if (n <= b.cap && b.p) return true;
    if (c.capturing) {  // a captured graph may not allocate (buffers are sized before the capture)
        c.err = "buffer growth during graph capture";
        return false;
    }
    ++c.gen;  // captured graphs embed buffer addresses
    size_t cap = std::max<size_t>(n, 1);
    T* p = nullptr;
    if (cudaMalloc(&p, cap * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        c.err = "cudaMalloc failed (" + std::to_string(cap * sizeof(T)) + " bytes)";
        return false;
    }
    if (keep && b.p && b.cap) cudaMemcpyAsync(p, b.p, b.cap * sizeof(T), cudaMemcpyDeviceToDevice, c.stream);
    if (b.p) {
        cudaStreamSynchronize(c.stream);
        cudaFree(b.p);
    }
    b.p = p;
    b.cap = cap;
    return true;
}

namespace {
std::mutex g_dev_mu;
std::map<std::tuple<const void*, int, int>, int> g_attr;  // (fn, device, attribute) -> value set
std::set<std::pair<const void*, int>> g_first;              // (key, device) already initialised
}  // namespace

bool set_func_attr(const Context& c, const void* fn, cudaFuncAttribute attr, int value) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    const auto key = std::make_tuple(fn, c.device, int(attr));
    auto it = g_attr.find(key);
    if (it != g_attr.end() && it->second == value) return true;
    if (cudaFuncSetAttribute(fn, attr, value) != cudaSuccess) return false;  // the launch reports it
    g_attr[key] = value;
    return true;
}

bool first_on_device(const Context& c, const void* key) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    return g_first.insert(std::make_pair(key, c.device)).second;
}

template bool ensure<float>(Context&, DevBuf<float>&, size_t, bool);
template bool ensure<float4>(Context&, DevBuf<float4>&, size_t, bool);
template bool ensure<uint2>(Context&, DevBuf<uint2>&, size_t, bool);
template bool ensure<uint4>(Context&, DevBuf<uint4>&, size_t, bool);
template bool ensure<DevCam>(Context&, DevBuf<DevCam>&, size_t, bool);
template bool ensure<uint8_t>(Context&, DevBuf<uint8_t>&, size_t, bool);
template bool ensure<uint16_t>(Context&, DevBuf<uint16_t>&, size_t, bool);
template bool ensure<uint32_t>(Context&, DevBuf<uint32_t>&, size_t, bool);
template bool ensure<double>(Context&, DevBuf<double>&, size_t, bool);
template bool ensure<unsigned long long>(Context&, DevBuf<unsigned long long>&, size_t, bool);

}  // namespace ts

namespace {

template <class T>
void release(DevBuf<T>& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
}

#define TS_CHECK_CTX(ctx)                          \
    do {                                           \
        if (!(ctx)) return TS_ERR_VALIDATION;      \
    } while (0)

ts_status cuda_fail(Context& c, cudaError_t e, const char* where) {
    c.err = std::string(where) + ": " + cudaGetErrorString(e);
    return TS_ERR_CUDA;
}

#define CK(expr)                                              \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_fail(c, _e, #expr); \
    } while (0)

ts_status last_launch(Context& c, const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, where);
    return TS_OK;
}

ts_status validation(Context& c, const char* msg) {
    c.err = msg;
    return TS_ERR_VALIDATION;
}


// stage names of the NVTX ranges (nsys / ncu --nvtx) and of ts_stage_times
const char* const kStageName[kNumStages] = {"preprocess", "depth_sort", "scan",      "duplicate",
                                            "tile_sort",  "ranges",     "blend",     "loss",
                                            "blend_bwd",  "project_bwd", "adam"};

// Every stage is an NVTX range (header-only NVTX3: a no-op unless a tool is attached); with
// profiling on it is also bracketed by CUDA events on the context stream.
void stage_begin(Context& c, int k) {
    nvtxRangePushA(kStageName[k]);
    if (!c.profiling) return;
    if (c.ev_cursor == c.ev_b.size()) {
        cudaEvent_t b, e;
        cudaEventCreate(&b);
        cudaEventCreate(&e);
        c.ev_b.push_back(b);
        c.ev_e.push_back(e);
        c.ev_stage.push_back(k);
    }
    c.ev_stage[c.ev_cursor] = k;
    cudaEventRecord(c.ev_b[c.ev_cursor], c.stream);
}
void stage_end(Context& c, int k) {
    (void)k;
    nvtxRangePop();
    if (!c.profiling) return;
    cudaEventRecord(c.ev_e[c.ev_cursor], c.stream);
    ++c.ev_cursor;
}

bool valid_camera(const ts_camera* cam, std::string* why) {
    if (!cam) return *why = "camera is NULL", false;
    if (cam->width < 6 || cam->height < 6) return *why = "image must be at least 6x6", false;
    if (!(cam->fx > 0.f) || !(cam->fy > 0.f)) return *why = "fx, fy must be > 0", false;
    // TileGrid: 16-bit tile keys below 2^16 tiles, 32-bit keys above (selected
    // in launch_duplicate / launch_tile_sort); rect fields hold 15-bit tile coordinates
    int64_t tn = int64_t((cam->width + 15) / 16) * ((cam->height + 15) / 16);
    if (tn >= (int64_t(1) << 24) || cam->width > 32767 * 16 || cam->height > 32767 * 16)
        return *why = "frame too large (>= 2^24 tiles)", false;
    return true;
}

bool valid_config(const ts_render_config* cfg, std::string* why) {
    if (!cfg) return *why = "render config is NULL", false;
    if (cfg->sh_degree < 0 || cfg->sh_degree > 3) return *why = "sh_degree must be 0..3", false;
    if (cfg->bound_mode < 0 || cfg->bound_mode > 2) return *why = "bound_mode must be 0..2", false;
    if (cfg->cull_mode < 0 || cfg->cull_mode > 1) return *why = "cull_mode must be 0..1", false;
    if (cfg->truncation < 0 || cfg->truncation > 1) return *why = "truncation must be 0 (classic) or 1 (response)", false;
    if (cfg->truncation == 1 && !(cfg->sigma_cut > 0.f && cfg->sigma_cut < 1e3f))
        return *why = "response truncation needs sigma_cut in (0, 1000)", false;
    if (cfg->backward_mode < 0 || cfg->backward_mode > 1) return *why = "backward_mode must be 0 (per-pixel) or 1 (per-Gaussian)", false;
    if (cfg->backward_mode == 1 && cfg->early_stop_compat)
        return *why = "the per-Gaussian backward needs the standard early stop (early_stop_compat = 0)", false;
    if (!(cfg->tau_alpha > 0.f && cfg->tau_alpha < 1.f)) return *why = "tau_alpha must be in (0,1)", false;
    if (!(cfg->dilation >= 0.f)) return *why = "dilation must be >= 0", false;
    if (cfg->aa_mode < 0 || cfg->aa_mode > 3) return *why = "aa_mode must be 0..3", false;
    if (cfg->aa_mode != 0 && !(cfg->kappa3d > 0.f)) return *why = "kappa3d must be > 0", false;
    return true;
}

DevCam make_devcam(const ts_camera& cam) {
    DevCam d;
    for (int i = 0; i < 16; ++i) d.W[i] = cam.W[i];
    d.fx = cam.fx;
    d.fy = cam.fy;
    d.cx = cam.cx;
    d.cy = cam.cy;
    d.nearp = cam.near_plane;
    d.w = cam.width;
    d.h = cam.height;
    d.tiles_x = (cam.width + 15) / 16;
    d.tiles_y = (cam.height + 15) / 16;
    // SPEC.md:169 clamp limits, once per camera; volatile keeps each fp32 op separately rounded
    // in this order (the oracle's Cam: 1.3f * ((0.5f * w) / fx))
    volatile float hw = 0.5f * float(cam.width), hh = 0.5f * float(cam.height);
    volatile float qx = hw / cam.fx, qy = hh / cam.fy;
    d.limx = 1.3f * qx;
    d.limy = 1.3f * qy;
    return d;
}

ts_status ensure_gaussian_buffers(Context& c, int64_t n) {
    const size_t N = size_t(std::max<int64_t>(n, 1));
    const size_t L = (59 * N + 7) & ~size_t(3);  // float4 sweeps read whole quads
    bool ok = ensure(c, c.params, L) && ensure(c, c.grads, L) && ensure(c, c.m, L) &&
              ensure(c, c.v, L) && ensure(c, c.accum, N + 4) && ensure(c, c.vcount, N + 4) &&
              ensure(c, c.splat, 3 * N) && ensure(c, c.rect, N) && ensure(c, c.tcount, N) &&
              ensure(c, c.dkey[0], N) && ensure(c, c.dkey[1], N) && ensure(c, c.dperm[0], N) &&
              ensure(c, c.dperm[1], N) && ensure(c, c.offsets, N + 1) && ensure(c, c.g2d, 3 * N + 1) &&
              ensure(c, c.vis, N) && ensure(c, c.nu_hat, N) && ensure(c, c.ryv, N);
    return ok ? TS_OK : TS_ERR_OOM;
}

ts_status zero_state(Context& c) {
    const size_t N = size_t(c.N);
    if (N == 0) return TS_OK;
    CK(cudaMemsetAsync(c.grads.p, 0, c.grads.cap * 4, c.stream));
    CK(cudaMemsetAsync(c.m.p, 0, c.m.cap * 4, c.stream));
    CK(cudaMemsetAsync(c.v.p, 0, c.v.cap * 4, c.stream));
    CK(cudaMemsetAsync(c.accum.p, 0, N * 4, c.stream));
    CK(cudaMemsetAsync(c.vcount.p, 0, N * 4, c.stream));
    CK(cudaMemsetAsync(c.g2d.p, 0, 3 * N * 16, c.stream));
    c.g2d_clean = true;
    CK(cudaMemsetAsync(c.vis.p, 0, N, c.stream));
    return TS_OK;
}

ts_status ensure_frame(Context& c, int w, int h) {
    const size_t P = size_t(w) * h;
    bool ok = ensure(c, c.rgb, 3 * P) && ensure(c, c.Tfin, P) && ensure(c, c.pcount, P) && ensure(c, c.dLdC, 3 * P) &&
              ensure(c, c.hwc_stage, 3 * P) && ensure(c, c.tgt, 3 * P);
    c.fw = w;
    c.fh = h;
    return ok ? TS_OK : TS_ERR_OOM;
}

int tile_bits_for(int tn) {
    int b = 1;
    while ((1 << b) < tn) ++b;
    return b;
}

// the forward pipeline of one view
bool ensure_order_events(Context& c) {
    if (c.ord_fork) return true;
    return cudaEventCreateWithFlags(&c.ord_fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&c.ord_join, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&c.bwd_fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&c.bwd_join, cudaEventDisableTiming) == cudaSuccess;
}

ts_status run_forward(Context& c, const ts_camera& cam, const ts_render_config& cfg) {
    if (cfg.aa_mode == 1 && !c.nu_valid)
        return validation(c, "aa_mode filter3d_original needs ts_compute_sampling_rates (or ts_set_sampling_rates)");
    DevCam dc = make_devcam(cam);
    const int Tn = dc.tiles_x * dc.tiles_y;
    if (ensure_frame(c, cam.width, cam.height) != TS_OK) return TS_ERR_OOM;
    if (!ensure(c, c.starts, size_t(Tn) + 1)) return TS_ERR_OOM;
    CK(cudaMemsetAsync(c.counters.p + 1, 0, 2 * sizeof(uint32_t), c.stream));
    stage_begin(c, 0);
    launch_preprocess(c, dc, cfg);
    stage_end(c, 0);
    // binning: bucketed path (k_bin.cu) unless a tile list exceeds the per-tile sort
    // capacity (or the radix path is forced); both give the identical sorted lists
    bool radix = c.binning_mode == 1 || !bin_supported(Tn);
    uint32_t max_len = 0;
    int64_t I = 0;
    bool scattered = false;
    if (!radix) {
        stage_begin(c, 1);
        if (!launch_bin_count(c, dc, cfg)) return c.err.empty() ? TS_ERR_OOM : TS_ERR_CUDA;
        stage_end(c, 1);
        if (!ensure_order_events(c)) return cuda_fail(c, cudaGetLastError(), "order events");
        CK(cudaEventRecord(c.ord_fork, c.stream));  // the tile order needs only the ranges
        // the scatter does not need I on the host: launch it into the current list buffer
        // (bounds-checked) while the host waits for I; relaunched below if the buffer was short
        if (c.ival[1].p && c.ival[1].cap > 0) {
            stage_begin(c, 3);
            launch_bin_scatter(c, dc, cfg);
            stage_end(c, 3);
            scattered = true;
        }
        I = finish_bin_count(c, &max_len);
        if (I < 0) return TS_ERR_CUDA;
        if (ts_status s = last_launch(c, "preprocess/bin_count"); s != TS_OK) return s;
        radix = max_len > uint32_t(bin_sort_cap());
        if (scattered && c.ival[1].cap < size_t(I)) scattered = false;
    }
    if (radix) {
        stage_begin(c, 1);
        launch_depth_sort(c);
        stage_end(c, 1);
        stage_begin(c, 2);
        I = launch_scan_counts(c);
        stage_end(c, 2);
        if (ts_status s = last_launch(c, "preprocess/sort/scan"); s != TS_OK) return s;
    }
    c.last_view_radix = radix;
    if (I > int64_t(0xFFFFFFF0u)) return validation(c, "instance count exceeds 2^32");
    const size_t capI = size_t(I) + size_t(I) / 4 + 1024;
    for (int k = 0; k < 2; ++k) {
        if (c.ival[k].cap < size_t(I)) {
            release(c.ival[k]);
            if (!ensure(c, c.ival[k], capI)) return TS_ERR_OOM;
        }
        if (radix && Tn < 65536 && c.tkey[k].cap < size_t(I)) {
            release(c.tkey[k]);
            if (!ensure(c, c.tkey[k], capI)) return TS_ERR_OOM;
        }
        if (radix && Tn >= 65536 && c.tkey32[k].cap < size_t(I)) {  // 32-bit tile keys
            release(c.tkey32[k]);
            if (!ensure(c, c.tkey32[k], capI)) return TS_ERR_OOM;
        }
    }
    if (!radix && c.bin_class[6] && !ensure_grow(c, c.sortmp, size_t(I))) return TS_ERR_OOM;  // long-list merges
    c.I = I;
    if (radix) {
        stage_begin(c, 3);
        launch_duplicate(c, dc, cfg);
        stage_end(c, 3);
        stage_begin(c, 4);
        launch_tile_sort(c, tile_bits_for(Tn), Tn >= 65536);
        stage_end(c, 4);
        stage_begin(c, 5);
        launch_ranges(c, Tn, Tn >= 65536);
        stage_end(c, 5);
        launch_tile_order(c, Tn);
    } else {
        if (!scattered) {
            stage_begin(c, 3);
            launch_bin_scatter(c, dc, cfg);
            stage_end(c, 3);
        }
        // the tile order (also the per-class tile lists of the sorts, longest first) runs on a side
        // stream beside the scatter
        CK(cudaStreamWaitEvent(c.side[1], c.ord_fork, 0));
        launch_tile_order(c, Tn, c.side[1]);
        if (!c.tile_order.p) return TS_ERR_OOM;
        CK(cudaEventRecord(c.ord_join, c.side[1]));
        CK(cudaStreamWaitEvent(c.stream, c.ord_join, 0));
        stage_begin(c, 4);
        launch_tile_depth_sort(c, Tn, max_len);
        stage_end(c, 4);
    }
    c.order_ok = c.tile_order.p != nullptr;
    c.bwd_order_ok = false;  // rebuilt from this view's processed lengths by the backward
    stage_begin(c, 6);
    launch_blend_fwd(c, dc, cfg);
    stage_end(c, 6);
    // the backward's tile order (by this view's processed lengths) beside the loss
    if (ensure_order_events(c)) {
        CK(cudaEventRecord(c.bwd_fork, c.stream));
        CK(cudaStreamWaitEvent(c.side[1], c.bwd_fork, 0));
        launch_bwd_tile_order(c, Tn, c.side[1]);
        CK(cudaEventRecord(c.bwd_join, c.side[1]));
        c.bwd_order_pending = c.bwd_order.p != nullptr;
    }
    if (ts_status s = last_launch(c, "forward"); s != TS_OK) return s;
    c.cam = cam;
    c.cfg = cfg;
    c.view_valid = true;
    c.loss_valid = false;
    return TS_OK;
}

// The forward of a graph-captured step (bucketed binning only): no host reads.  The tile order
// runs before the scatter and performs the step's capacity check (tile_order_kernel); the size
// classes are launched on resident grids that read the device-side class counts.
ts_status run_forward_graph(Context& c, const ts_camera& cam, const ts_render_config& cfg) {
    c.bwd_order_pending = false;  // the captured backward builds its order in-line
    DevCam dc = make_devcam(cam);
    const int Tn = dc.tiles_x * dc.tiles_y;
    if (ensure_frame(c, cam.width, cam.height) != TS_OK) return TS_ERR_OOM;
    if (!ensure(c, c.starts, size_t(Tn) + 1)) return TS_ERR_OOM;
    CK(cudaMemsetAsync(c.counters.p + 1, 0, 2 * sizeof(uint32_t), c.stream));
    stage_begin(c, 0);
    launch_preprocess(c, dc, cfg);
    stage_end(c, 0);
    stage_begin(c, 1);
    if (!launch_bin_count(c, dc, cfg)) return c.err.empty() ? TS_ERR_OOM : TS_ERR_CUDA;
    stage_end(c, 1);
    launch_tile_order(c, Tn);
    stage_begin(c, 3);
    launch_bin_scatter(c, dc, cfg);
    stage_end(c, 3);
    stage_begin(c, 4);
    launch_tile_depth_sort(c, Tn, 0);
    stage_end(c, 4);
    c.order_ok = true;
    c.bwd_order_ok = false;
    stage_begin(c, 6);
    launch_blend_fwd(c, dc, cfg);
    stage_end(c, 6);
    if (ts_status s = last_launch(c, "forward (graph)"); s != TS_OK) return s;
    c.last_view_radix = false;
    c.I_on_device = true;
    c.cam = cam;
    c.cfg = cfg;
    c.view_valid = true;
    c.loss_valid = false;
    return TS_OK;
}

ts_status upload_image_chw(Context& c, const float* hwc, float* dst_chw) {
    const size_t P = size_t(c.fw) * c.fh;
    CK(cudaMemcpyAsync(c.hwc_stage.p, hwc, 3 * P * 4, cudaMemcpyHostToDevice, c.stream));
    launch_hwc_to_chw(c, c.hwc_stage.p, dst_chw, int(P));
    return last_launch(c, "hwc_to_chw");
}

ts_status run_loss(Context& c, const float* target_hwc, int32_t slot, float* out_loss,
                   const float* target_chw_dev = nullptr) {
    if (!c.view_valid) return validation(c, "ts_loss needs a preceding ts_forward");
    const size_t P = size_t(c.fw) * c.fh;
    const float* tgt = nullptr;
    if (target_chw_dev) {
        tgt = target_chw_dev;
    } else if (target_hwc) {
        if (ts_status s = upload_image_chw(c, target_hwc, c.tgt.p); s != TS_OK) return s;
        tgt = c.tgt.p;
    } else {
        if (slot < 0 || slot >= c.n_target_slots) return validation(c, "target slot out of range");
        if (c.target_w != c.fw || c.target_h != c.fh) return validation(c, "target slot size != view size");
        tgt = c.targets.p + size_t(slot) * 3 * P;
    }
    stage_begin(c, 7);
    launch_loss(c, tgt);
    stage_end(c, 7);
    if (ts_status s = last_launch(c, "loss"); s != TS_OK) return s;
    c.loss_valid = true;
    if (out_loss) {
        double acc[2];
        CK(cudaMemcpyAsync(acc, c.loss_acc.p, sizeof(acc), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        const double M = 3.0 * double(P);
        *out_loss = float(0.8 * acc[0] / M + 0.2 * (1.0 - acc[1] / M));
    }
    return TS_OK;
}

ts_status run_backward(Context& c, const float* dLdC_hwc) {
    if (!c.view_valid) return validation(c, "ts_backward needs a preceding ts_forward");
    if (dLdC_hwc) {
        if (ts_status s = upload_image_chw(c, dLdC_hwc, c.dLdC.p); s != TS_OK) return s;
    } else if (!c.loss_valid) {
        return validation(c, "ts_backward(NULL) needs a preceding ts_loss");
    }
    DevCam dc = make_devcam(c.cam);
    // vis = visible in any view since the last optimizer step: a new accumulation starts empty
    // (cleared here rather than after Adam, so a range-chunked optimizer sweep sees it whole)
    if (c.grad_state != Context::kGradLive)
        CK(cudaMemsetAsync(c.vis.p, 0, size_t(std::max<int64_t>(c.N, 1)), c.stream));
    if (!c.g2d_clean) CK(cudaMemsetAsync(c.g2d.p, 0, size_t(c.N) * 48, c.stream));  // a second backward of a view
    stage_begin(c, 8);
    // backward order: tiles by the forward's processed length (the backward's per-tile work),
    // built beside the loss by the host-path forward
    if (c.bwd_order_pending) CK(cudaStreamWaitEvent(c.stream, c.bwd_join, 0));
    else launch_bwd_tile_order(c, dc.tiles_x * dc.tiles_y);
    c.bwd_order_ok = c.bwd_order.p != nullptr && c.tile_proc.p != nullptr;
    launch_blend_bwd(c, dc, c.cfg);
    stage_end(c, 8);
    stage_begin(c, 9);
    launch_project_bwd(c, dc, c.cfg, c.grad_state == Context::kGradLive, c.grad_state == Context::kGradStale);
    c.grad_state = Context::kGradLive;
    stage_end(c, 9);
    return last_launch(c, "backward");
}

ts_status run_backward_adam(Context& c, const float* dLdC_hwc, const ts_adam_config& a) {
    if (!c.view_valid) return validation(c, "ts_backward_adam needs a preceding ts_forward");
    if (a.mode != 3 && a.mode != 4) return validation(c, "fused backward Adam needs mode 3 or 4");
    if (!(a.bc1 > 0.f) || !(a.bc2 > 0.f)) return validation(c, "bias corrections must be > 0 (step >= 1)");
    if (c.grad_state == Context::kGradLive)
        return validation(c, "fused backward Adam needs a consumed gradient buffer (single-view step)");
    if (dLdC_hwc) {
        if (ts_status s = upload_image_chw(c, dLdC_hwc, c.dLdC.p); s != TS_OK) return s;
    } else if (!c.loss_valid) {
        return validation(c, "ts_backward_adam(NULL) needs a preceding ts_loss");
    }
    DevCam dc = make_devcam(c.cam);
    CK(cudaMemsetAsync(c.vis.p, 0, size_t(std::max<int64_t>(c.N, 1)), c.stream));  // new accumulation
    if (!c.g2d_clean) CK(cudaMemsetAsync(c.g2d.p, 0, size_t(c.N) * 48, c.stream));
    stage_begin(c, 8);
    launch_blend_bwd(c, dc, c.cfg);
    stage_end(c, 8);
    stage_begin(c, 9);
    launch_project_bwd_adam(c, dc, c.cfg, a);
    stage_end(c, 9);
    c.view_valid = false;
    c.loss_valid = false;
    return last_launch(c, "backward_adam");
}

ts_status run_adam(Context& c, const ts_adam_config& a, int64_t begin, int64_t end) {
    if (!(a.bc1 > 0.f) || !(a.bc2 > 0.f)) return validation(c, "bias corrections must be > 0 (step >= 1)");
    if (a.mode < 0 || a.mode > 2) return validation(c, "adam mode must be 0..2 (3/4 run inside the backward)");
    stage_begin(c, 10);
    launch_adam(c, a, begin, end);
    stage_end(c, 10);
    // the sweep that reaches the end of the buffer completes the step (a full sweep, or the
    // last of in-order range chunks, dp.py "chunked"): the gradient buffer is consumed
    if (end == 59 * c.N) c.grad_state = a.zero_grads ? Context::kGradZero : Context::kGradStale;
    c.view_valid = false;
    c.loss_valid = false;
    return last_launch(c, "adam");
}

// one training step on the host-driven path (ts_train_step without a graph; graph replays)
ts_status run_train_step(Context& c, const ts_camera& camr, const ts_render_config& cfgr, const float* target_hwc,
                         int32_t slot, const ts_adam_config& adamr, float* out_loss) {
    const ts_camera* cam = &camr;
    const ts_render_config* cfg = &cfgr;
    const ts_adam_config* adam = &adamr;
    // a host target is uploaded on a copy stream while the forward runs (the loss waits for it)
    const size_t P = size_t(cam->width) * cam->height;
    if (target_hwc) {
        if (ensure_frame(c, cam->width, cam->height) != TS_OK || !ensure(c, c.tgt_stage, 3 * P)) return TS_ERR_OOM;
        if (!c.copy_stream) {
            CK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c.copy_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c.copy_join, cudaEventDisableTiming));
        }
        // upload and layout conversion both on the copy stream, off the engine stream: the upload
        // at once (tgt_stage was last read by the previous conversion, earlier on this stream),
        // the conversion once the previous step's loss has consumed tgt (copy_fork; never
        // recorded yet: the wait is a no-op)
        CK(cudaMemcpyAsync(c.tgt_stage.p, target_hwc, 3 * P * 4, cudaMemcpyHostToDevice, c.copy_stream));
        CK(cudaStreamWaitEvent(c.copy_stream, c.copy_fork, 0));
        launch_hwc_to_chw(c, c.tgt_stage.p, c.tgt.p, int(P), c.copy_stream);
        CK(cudaEventRecord(c.copy_join, c.copy_stream));
    }
    if (ts_status s = run_forward(c, *cam, *cfg); s != TS_OK) return s;
    if (target_hwc) {
        CK(cudaStreamWaitEvent(c.stream, c.copy_join, 0));
        if (ts_status s = run_loss(c, nullptr, slot, nullptr, c.tgt.p); s != TS_OK) return s;
        CK(cudaEventRecord(c.copy_fork, c.stream));  // tgt consumed: the next conversion may overwrite it
    } else {
        if (ts_status s = run_loss(c, nullptr, slot, nullptr); s != TS_OK) return s;
    }
    // the loss sums go to pinned host memory right behind the loss kernel; the host
    // waits for that event only, so backward + Adam keep the GPU busy while the caller
    // prepares the next step
    if (out_loss) {
        if (!c.loss_host) {
            CK(cudaMallocHost(reinterpret_cast<void**>(&c.loss_host), 2 * sizeof(double)));
            CK(cudaEventCreateWithFlags(&c.loss_ev, cudaEventDisableTiming));
        }
        CK(cudaMemcpyAsync(c.loss_host, c.loss_acc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaEventRecord(c.loss_ev, c.stream));
    }
    if (adam->mode >= 3) {
        if (ts_status s = run_backward_adam(c, nullptr, *adam); s != TS_OK) return s;
    } else {
        if (ts_status s = run_backward(c, nullptr); s != TS_OK) return s;
        // the gradient buffer is internal to the step: skip the clear (the next
        // backward overwrites every row); ts_get_state then shows this step's gradient
        ts_adam_config a = *adam;
        a.zero_grads = 0;
        if (ts_status s = run_adam(c, a, 0, 59 * c.N); s != TS_OK) return s;
    }
    if (out_loss) {
        CK(cudaEventSynchronize(c.loss_ev));
        const double M = 3.0 * double(cam->width) * cam->height;
        *out_loss = float(0.8 * c.loss_host[0] / M + 0.2 * (1.0 - c.loss_host[1] / M));
    }
    return TS_OK;
}

// ---------------------------------------------------------------------------
// CUDA-graph mode of ts_train_step (ts_set_graph).  A training step on a given view, render
// config, target and optimizer mode is captured once into a CUDA graph (forward, loss,
// backward, Adam; the host-target upload as a parallel branch) and relaunched each step:
// no host round trip inside the step (the host-driven path waits for the instance count
// before sizing the sort launches).  Per-step inputs enter through device memory (the Adam
// argument block, written before each launch); the per-view camera, config and target address
// are part of the graph key.  A captured step cannot grow buffers: its capacity check
// (tile_order_kernel) voids the step (sticky device flag; K9 and Adam skip) when the instance
// count outgrows the lists or a list needs the radix path, and the host replays every voided
// step in order on the host path (graph_settle), so the result equals host-driven training.
// ---------------------------------------------------------------------------
bool same_view(const GraphEntry& e, const ts_camera& cam, const ts_render_config& cfg, const float* target,
               int32_t slot, int32_t want_loss, int32_t mode, int64_t N) {
    return std::memcmp(&e.cam, &cam, sizeof(cam)) == 0 && std::memcmp(&e.cfg, &cfg, sizeof(cfg)) == 0 &&
           e.target == target && e.slot == (target ? -1 : slot) && e.want_loss == want_loss && e.mode == mode &&
           e.N == N;
}

void drop_graphs(Context& c) {
    for (GraphEntry& e : c.graphs)
        if (e.exec) cudaGraphExecDestroy(e.exec);
    c.graphs.clear();
    c.graph_seen.clear();
}

bool graph_eligible(const Context& c, const ts_camera& cam, const ts_render_config& cfg, const ts_adam_config& a) {
    const int Tn = ((cam.width + 15) / 16) * ((cam.height + 15) / 16);
    // (a live gradient buffer would be accumulated into by the host path; the graph overwrites)
    return c.graph_on && !c.profiling && c.binning_mode == 0 && bin_supported(Tn) && a.mode >= 0 && a.mode <= 2 &&
           cfg.aa_mode != 1 && c.N > 0 && c.grad_state != Context::kGradLive && cfg.backward_mode == 0;
}

// every launched graph step verified; voided steps replayed on the host path.  block: wait for the
// last launch (else only look if it has completed)
ts_status graph_check(Context& c, bool block) {
    if (c.glog.empty()) return TS_OK;
    if (block) {
        CK(cudaEventSynchronize(c.gstep_ev));
    } else {
        const cudaError_t q = cudaEventQuery(c.gstep_ev);
        if (q == cudaErrorNotReady) return TS_OK;
        if (q != cudaSuccess) return cuda_fail(c, q, "graph step");
    }
    if (*c.gflag_host == 0u) {
        c.glog.clear();
        return TS_OK;
    }
    // a step outgrew its captured buffers: it and every later graph step were no-ops
    CK(cudaStreamSynchronize(c.stream));
    CK(cudaMemsetAsync(c.counters.p + kGraphFlag, 0, sizeof(uint32_t), c.stream));
    *c.gflag_host = 0u;
    drop_graphs(c);
    std::vector<GraphStep> steps;
    steps.swap(c.glog);
    for (const GraphStep& st : steps) {
        if (ts_status s = run_train_step(c, st.cam, st.cfg, st.target, st.slot, st.adam, nullptr); s != TS_OK) return s;
        ++c.graph_replays;
    }
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status graph_settle(Context& c) {
    if (c.glog.empty() && !c.I_on_device) return TS_OK;
    if (ts_status s = graph_check(c, true); s != TS_OK) return s;
    if (c.I_on_device && c.view_valid) {  // instance count of the last graph-rendered view
        const int Tn = ((c.cam.width + 15) / 16) * ((c.cam.height + 15) / 16);
        uint32_t I = 0;
        CK(cudaMemcpy(&I, c.starts.p + Tn, sizeof(I), cudaMemcpyDeviceToHost));
        c.I = I;
    }
    c.I_on_device = false;
    return TS_OK;
}

#define TS_SETTLE(c)                                             \
    do {                                                         \
        if (ts_status s_ = graph_settle(c); s_ != TS_OK) return s_; \
    } while (0)

ts_status graph_capture(Context& c, const ts_camera& cam, const ts_render_config& cfg, const float* target_hwc,
                        int32_t slot, int want_loss, const ts_adam_config& adam, cudaGraphExec_t* out,
                        int64_t* kernels) {
    // buffers sized by the view's host-path step; the lists get 25% headroom (growth beyond it
    // voids a step and is replayed)
    const size_t capI = size_t(c.I) + size_t(c.I) / 4 + 4096;
    for (int k = 0; k < 2; ++k)
        if (c.ival[k].cap < capI && !ensure(c, c.ival[k], capI)) return TS_ERR_OOM;
    if (!ensure_grow(c, c.sortmp, capI)) return TS_ERR_OOM;
    const size_t P = size_t(cam.width) * cam.height;
    if (target_hwc && !ensure(c, c.tgt_stage, 3 * P)) return TS_ERR_OOM;
    CK(cudaStreamSynchronize(c.stream));
    const int64_t launches0 = c.launches;  // captured launches are counted when the graph runs
    auto swap_events = [&c] {
        std::swap(c.fork_ev, c.cap_fork);
        std::swap(c.join_ev[0], c.cap_join[0]);
        std::swap(c.join_ev[1], c.cap_join[1]);
        std::swap(c.copy_fork, c.cap_copy_fork);
        std::swap(c.copy_join, c.cap_copy_join);
        std::swap(c.loss_ev, c.cap_loss);
    };
    swap_events();  // the capture records its own events (see Context::cap_fork)
    c.capturing = c.gmode = true;
    cudaError_t e = cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        c.capturing = c.gmode = false;
        return cuda_fail(c, e, "cudaStreamBeginCapture");
    }
    ts_status st = TS_OK;
    do {
        if (target_hwc) {  // host target: a parallel branch of the graph (copy node + layout kernel)
            if ((e = cudaEventRecord(c.copy_fork, c.stream)) != cudaSuccess) break;
            if ((e = cudaStreamWaitEvent(c.copy_stream, c.copy_fork, 0)) != cudaSuccess) break;
            if ((e = cudaMemcpyAsync(c.tgt_stage.p, target_hwc, 3 * P * 4, cudaMemcpyHostToDevice, c.copy_stream)) !=
                cudaSuccess)
                break;
            if ((e = cudaEventRecord(c.copy_join, c.copy_stream)) != cudaSuccess) break;
        }
        if ((st = run_forward_graph(c, cam, cfg)) != TS_OK) break;
        if (target_hwc) {
            if ((e = cudaStreamWaitEvent(c.stream, c.copy_join, 0)) != cudaSuccess) break;
            launch_hwc_to_chw(c, c.tgt_stage.p, c.tgt.p, int(P));
            if ((st = run_loss(c, nullptr, slot, nullptr, c.tgt.p)) != TS_OK) break;
        } else if ((st = run_loss(c, nullptr, slot, nullptr)) != TS_OK) {
            break;
        }
        // the step's capacity verdict (set by the tile order) and the loss sums to pinned memory
        if ((e = cudaMemcpyAsync(c.gflag_host, c.counters.p + kGraphFlag, 4, cudaMemcpyDeviceToHost, c.stream)) !=
            cudaSuccess)
            break;
        if (want_loss) {
            if ((e = cudaMemcpyAsync(c.loss_host, c.loss_acc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                     c.stream)) != cudaSuccess)
                break;
            // an external event node: the host waits on it after each launch (a plain record in a
            // capturing stream would only be a fork/join dependency)
            if ((e = cudaEventRecordWithFlags(c.loss_ev, c.stream, cudaEventRecordExternal)) != cudaSuccess) break;
        }
        c.grad_state = Context::kGradStale;  // the captured backward overwrites every row
        if ((st = run_backward(c, nullptr)) != TS_OK) break;
        ts_adam_config a = adam;
        a.zero_grads = 0;
        stage_begin(c, 10);
        launch_adam(c, a, 0, 59 * c.N);
        stage_end(c, 10);
    } while (false);
    cudaGraph_t g = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(c.stream, &g);
    c.capturing = c.gmode = false;
    swap_events();
    *kernels = c.launches - launches0;
    c.launches = launches0;
    if (st == TS_OK && e != cudaSuccess) st = cuda_fail(c, e, "graph capture");
    if (st == TS_OK && e2 != cudaSuccess) st = cuda_fail(c, e2, "cudaStreamEndCapture");
    if (st == TS_OK) {
        e = cudaGraphInstantiate(out, g, 0);
        if (e != cudaSuccess) st = cuda_fail(c, e, "cudaGraphInstantiate");
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    c.view_valid = c.loss_valid = false;
    ++c.graph_captures;
    return st;
}

ts_status graph_step(Context& c, const ts_camera& cam, const ts_render_config& cfg, const float* target_hwc,
                     int32_t slot, const ts_adam_config& adam, float* out_loss) {
    if (!(adam.bc1 > 0.f) || !(adam.bc2 > 0.f)) return validation(c, "bias corrections must be > 0 (step >= 1)");
    if (!target_hwc && (slot < 0 || slot >= c.n_target_slots || c.target_w != cam.width || c.target_h != cam.height))
        return validation(c, "target slot out of range / size != view size");
    if (c.glog.size() > 32) {
        if (ts_status s = graph_check(c, true); s != TS_OK) return s;
    } else if (ts_status s = graph_check(c, false); s != TS_OK) {
        return s;
    }
    const int want = out_loss ? 1 : 0;
    GraphEntry* ent = nullptr;
    for (GraphEntry& e : c.graphs)
        if (e.gen == c.gen && same_view(e, cam, cfg, target_hwc, slot, want, adam.mode, c.N)) ent = &e;
    if (!ent) {
        bool seen = false;
        const GraphEntry* sv = nullptr;
        for (const GraphEntry& e : c.graph_seen)
            if (e.gen == c.gen && same_view(e, cam, cfg, target_hwc, slot, want, adam.mode, c.N)) sv = &e;
        seen = sv != nullptr;
        if (sv) {  // the view's own host-path sizes: sort grid hints and list capacity
            std::memcpy(c.bin_class, sv->cls, sizeof(c.bin_class));
            c.I = sv->I;
        }
        if (!seen) {
            // first time for this view (or buffers changed): a host-path step sizes the buffers
            if (ts_status s = graph_settle(c); s != TS_OK) return s;
            if (ts_status s = run_train_step(c, cam, cfg, target_hwc, slot, adam, out_loss); s != TS_OK) return s;
            if (c.graph_seen.size() >= 64) c.graph_seen.erase(c.graph_seen.begin());  // bounded
            GraphEntry seen{cam, cfg, target_hwc, target_hwc ? -1 : slot, want, adam.mode, c.N, c.gen, nullptr, 0,
                            {0, 0, 0, 0, 0, 0, 0}, c.I};
            std::memcpy(seen.cls, c.bin_class, sizeof(seen.cls));
            c.graph_seen.push_back(seen);
            return TS_OK;
        }
        if (ts_status s = graph_settle(c); s != TS_OK) return s;
        cudaGraphExec_t exec = nullptr;
        int64_t kernels = 0;
        if (ts_status s = graph_capture(c, cam, cfg, target_hwc, slot, want, adam, &exec, &kernels); s != TS_OK) {
            c.err = "graph capture failed (" + c.err + ")";
            return s;
        }
        if (c.graphs.size() >= 32) {  // bounded cache: drop the oldest graph
            cudaGraphExecDestroy(c.graphs.front().exec);
            c.graphs.erase(c.graphs.begin());
        }
        c.graphs.push_back(GraphEntry{cam, cfg, target_hwc, target_hwc ? -1 : slot, want, adam.mode, c.N, c.gen, exec,
                                      kernels, {0, 0, 0, 0, 0, 0, 0}, c.I});
        ent = &c.graphs.back();
    }
    const size_t nb = adam_args_bytes(adam, c.adam_dev_bytes);
    CK(cudaMemcpyAsync(c.adam_dev, c.adam_dev_bytes, nb, cudaMemcpyHostToDevice, c.stream));
    CK(cudaGraphLaunch(ent->exec, c.stream));
    CK(cudaEventRecord(c.gstep_ev, c.stream));
    c.glog.push_back(GraphStep{cam, cfg, target_hwc, slot, adam});
    ++c.graph_launches;
    c.launches += ent->kernels;
    c.grad_state = Context::kGradStale;
    c.cam = cam;
    c.cfg = cfg;
    c.view_valid = true;  // the view's buffers (frame, lists) hold this step's forward
    c.loss_valid = false;
    c.I_on_device = true;
    if (out_loss) {
        CK(cudaEventSynchronize(c.cap_loss));  // the graph's external loss event node
        if (*c.gflag_host) {  // voided: replay now and report the replayed loss
            CK(cudaEventSynchronize(c.gstep_ev));
            c.glog.pop_back();
            if (ts_status s = graph_check(c, true); s != TS_OK) return s;  // earlier voided steps
            *c.gflag_host = 0u;
            CK(cudaMemsetAsync(c.counters.p + kGraphFlag, 0, sizeof(uint32_t), c.stream));
            drop_graphs(c);
            ++c.graph_replays;
            return run_train_step(c, cam, cfg, target_hwc, slot, adam, out_loss);
        }
        const double M = 3.0 * double(cam.width) * cam.height;
        *out_loss = float(0.8 * c.loss_host[0] / M + 0.2 * (1.0 - c.loss_host[1] / M));
    }
    return TS_OK;
}

}  // namespace

extern "C" {

const char* ts_version(void) { return "tilesplat-b200 0.1 (sm_100a)"; }

ts_status ts_create(int32_t device, void* stream, ts_ctx** out) {
    if (!out) return TS_ERR_VALIDATION;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return TS_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) return TS_ERR_VALIDATION;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return TS_ERR_CUDA;
    if (prop.major < 10) return TS_ERR_CUDA;  // built for sm_100a only; no fallback
    ts_ctx* x = new (std::nothrow) ts_ctx();
    if (!x) return TS_ERR_OOM;
    Context& c = x->c;
    c.device = device;
    c.sm_count = prop.multiProcessorCount;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete x;
        return TS_ERR_CUDA;
    }
    if (stream) {
        c.stream = static_cast<cudaStream_t>(stream);
    } else {
        if (cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete x;
            return TS_ERR_CUDA;
        }
        c.own_stream = true;
    }
    if (!ensure(c, c.counters, 16) || !ensure(c, c.loss_acc, 2)) {
        delete x;
        return TS_ERR_OOM;
    }
    cudaMemsetAsync(c.counters.p, 0, 16 * 4, c.stream);
    // per-step plumbing created once here, never inside a timed step: the host-target copy
    // stream, the pinned loss / graph-flag slots, the graph-step event and the device block of
    // the per-step Adam arguments (graph mode)
    if (cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.copy_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.copy_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.loss_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.gstep_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.join_ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.join_ev[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c.side[0], cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c.side[1], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.cap_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.cap_join[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.cap_join[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.cap_copy_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.cap_copy_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.cap_loss, cudaEventDisableTiming) != cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void**>(&c.loss_host), 2 * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void**>(&c.gflag_host), sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&c.adam_dev, sizeof(c.adam_dev_bytes)) != cudaSuccess) {
        cudaGetLastError();
        delete x;
        return TS_ERR_CUDA;
    }
    *c.gflag_host = 0u;
    if (ensure_gaussian_buffers(c, 1) != TS_OK) {
        delete x;
        return TS_ERR_OOM;
    }
    if (cudaStreamSynchronize(c.stream) != cudaSuccess) {
        delete x;
        return TS_ERR_CUDA;
    }
    *out = x;
    return TS_OK;
}

ts_status ts_destroy(ts_ctx* x) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    cudaSetDevice(c.device);
    cudaStreamSynchronize(c.stream);
    drop_graphs(c);
    if (c.gstep_ev) cudaEventDestroy(c.gstep_ev);
    for (cudaEvent_t ev : {c.cap_fork, c.cap_join[0], c.cap_join[1], c.cap_copy_fork, c.cap_copy_join, c.cap_loss})
        if (ev) cudaEventDestroy(ev);
    if (c.gflag_host) cudaFreeHost(c.gflag_host);
    if (c.adam_dev) cudaFree(c.adam_dev);
    release(c.params), release(c.grads), release(c.m), release(c.v), release(c.accum), release(c.vcount);
    release(c.splat), release(c.ryv), release(c.rect), release(c.tcount), release(c.offsets), release(c.g2d), release(c.vis);
    for (int k = 0; k < 2; ++k) {
        release(c.dkey[k]), release(c.dperm[k]), release(c.tkey[k]), release(c.tkey32[k]), release(c.ival[k]);
    }
    release(c.starts), release(c.rhist), release(c.scan_state), release(c.scan_tmp), release(c.counters);
    release(c.rgb), release(c.Tfin), release(c.dLdC), release(c.hwc_stage), release(c.tgt), release(c.pcount);
    release(c.loss_acc), release(c.targets), release(c.dens);
    release(c.binH), release(c.bintot), release(c.tile_order), release(c.tile_proc), release(c.bwd_order), release(c.sortmp), release(c.spare), release(c.cams), release(c.mcode[0]), release(c.mcode[1]),
        release(c.midx[0]), release(c.midx[1]), release(c.tgt_stage), release(c.nu_hat);
    for (size_t k = 0; k < c.ev_b.size(); ++k) {
        cudaEventDestroy(c.ev_b[k]);
        cudaEventDestroy(c.ev_e[k]);
    }
    for (int k = 0; k < 2; ++k) {
        if (c.side[k]) cudaStreamDestroy(c.side[k]);
        if (c.join_ev[k]) cudaEventDestroy(c.join_ev[k]);
    }
    if (c.fork_ev) cudaEventDestroy(c.fork_ev);
    for (cudaEvent_t e : {c.ord_fork, c.ord_join, c.bwd_fork, c.bwd_join})
        if (e) cudaEventDestroy(e);
    if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
    if (c.bin_host) cudaFreeHost(c.bin_host);
    if (c.bin_ev) cudaEventDestroy(c.bin_ev);
    if (c.bin_fork) cudaEventDestroy(c.bin_fork);
    if (c.loss_host) cudaFreeHost(c.loss_host);
    if (c.loss_ev) cudaEventDestroy(c.loss_ev);
    if (c.copy_fork) cudaEventDestroy(c.copy_fork);
    if (c.copy_join) cudaEventDestroy(c.copy_join);
    if (c.own_stream) cudaStreamDestroy(c.stream);
    delete x;
    return TS_OK;
}

const char* ts_last_error(const ts_ctx* x) { return x ? x->c.err.c_str() : "null context"; }

ts_status ts_synchronize(ts_ctx* x) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_set_params_flat(ts_ctx* x, int64_t n, const float* flat) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (n < 0 || (n > 0 && !flat)) return validation(c, "bad parameter array");
    if (n > kMaxGaussians) return validation(c, "N exceeds the 32-bit flat-index limit (~72.8M Gaussians)");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (ensure_gaussian_buffers(c, n) != TS_OK) return TS_ERR_OOM;
    if (n != c.N) c.nu_valid = false;  // sampling rates are per row (kept across same-size updates)
    c.N = n;
    if (n) CK(cudaMemcpyAsync(c.params.p, flat, size_t(59) * n * 4, cudaMemcpyHostToDevice, c.stream));
    if (ts_status s = zero_state(c); s != TS_OK) return s;
    c.grad_state = Context::kGradZero;
    c.view_valid = c.loss_valid = false;
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_set_params(ts_ctx* x, int64_t n, const float* means, const float* ls, const float* q, const float* op,
                        const float* dc, const float* rest) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (n < 0) return validation(c, "n < 0");
    if (n > 0 && (!means || !ls || !q || !op || !dc || !rest)) return validation(c, "NULL parameter array");
    std::vector<float> flat(size_t(59) * n);
    const Off o(n);
    std::memcpy(flat.data() + o.means, means, size_t(3) * n * 4);
    std::memcpy(flat.data() + o.ls, ls, size_t(3) * n * 4);
    std::memcpy(flat.data() + o.q, q, size_t(4) * n * 4);
    std::memcpy(flat.data() + o.op, op, size_t(1) * n * 4);
    std::memcpy(flat.data() + o.dc, dc, size_t(3) * n * 4);
    std::memcpy(flat.data() + o.rest, rest, size_t(45) * n * 4);
    return ts_set_params_flat(x, n, flat.data());
}

ts_status ts_get_params_flat(ts_ctx* x, float* flat) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (c.N && !flat) return validation(c, "NULL output");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (c.N) CK(cudaMemcpyAsync(flat, c.params.p, size_t(59) * c.N * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_num_gaussians(const ts_ctx* x, int64_t* n) {
    if (!x || !n) return TS_ERR_VALIDATION;
    *n = x->c.N;
    return TS_OK;
}

ts_status ts_forward(ts_ctx* x, const ts_camera* cam, const ts_render_config* cfg, float* out_rgb, float* out_T,
                     uint32_t* out_count) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    std::string why;
    if (!valid_camera(cam, &why) || !valid_config(cfg, &why)) return validation(c, why.c_str());
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (ts_status s = run_forward(c, *cam, *cfg); s != TS_OK) return s;
    const size_t P = size_t(cam->width) * cam->height;
    if (out_rgb) {
        launch_chw_to_hwc(c, c.rgb.p, c.hwc_stage.p, int(P));
        CK(cudaMemcpyAsync(out_rgb, c.hwc_stage.p, 3 * P * 4, cudaMemcpyDeviceToHost, c.stream));
    }
    if (out_T) CK(cudaMemcpyAsync(out_T, c.Tfin.p, P * 4, cudaMemcpyDeviceToHost, c.stream));
    if (out_count) CK(cudaMemcpyAsync(out_count, c.pcount.p, P * 4, cudaMemcpyDeviceToHost, c.stream));
    if (out_rgb || out_T || out_count) CK(cudaStreamSynchronize(c.stream));
    return last_launch(c, "ts_forward");
}

ts_status ts_set_target(ts_ctx* x, int32_t slot, int32_t w, int32_t h, const float* hwc) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (slot < 0 || slot > 4096 || w < 6 || h < 6 || !hwc) return validation(c, "bad target");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t P = size_t(w) * h;
    if (c.target_w != w || c.target_h != h) {
        release(c.targets);
        c.n_target_slots = 0;
        c.target_w = w;
        c.target_h = h;
    }
    if (slot >= c.n_target_slots) {
        if (!ensure(c, c.targets, size_t(slot + 1) * 3 * P, true)) return TS_ERR_OOM;
        c.n_target_slots = slot + 1;
    }
    if (ensure_frame(c, std::max(c.fw, w), std::max(c.fh, h)) != TS_OK) return TS_ERR_OOM;
    CK(cudaMemcpyAsync(c.hwc_stage.p, hwc, 3 * P * 4, cudaMemcpyHostToDevice, c.stream));
    launch_hwc_to_chw(c, c.hwc_stage.p, c.targets.p + size_t(slot) * 3 * P, int(P));
    CK(cudaStreamSynchronize(c.stream));
    return last_launch(c, "ts_set_target");
}

ts_status ts_loss(ts_ctx* x, const float* target_hwc, int32_t slot, float* out_loss) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    return run_loss(c, target_hwc, slot, out_loss);
}

ts_status ts_backward(ts_ctx* x, const float* dLdC_hwc) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    return run_backward(c, dLdC_hwc);
}

ts_status ts_backward_adam(ts_ctx* x, const float* dLdC_hwc, const ts_adam_config* a) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!a) return validation(c, "adam config is NULL");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    return run_backward_adam(c, dLdC_hwc, *a);
}

ts_status ts_zero_grads(ts_ctx* x) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (c.N) CK(cudaMemsetAsync(c.grads.p, 0, size_t(59) * c.N * 4, c.stream));
    c.grad_state = Context::kGradZero;
    return TS_OK;
}

ts_status ts_mark_grads_consumed(ts_ctx* x) {
    TS_CHECK_CTX(x);
    TS_SETTLE(x->c);
    Context& c = x->c;
    if (c.grad_state == Context::kGradLive) c.grad_state = Context::kGradStale;
    c.view_valid = c.loss_valid = false;
    return TS_OK;
}

ts_status ts_grad_buffer(ts_ctx* x, float** p, int64_t* n) {
    TS_CHECK_CTX(x);
    TS_SETTLE(x->c);
    if (p) *p = x->c.grads.p;
    if (n) *n = 59 * x->c.N;
    return TS_OK;
}

ts_status ts_param_buffer(ts_ctx* x, float** p, int64_t* n) {
    TS_CHECK_CTX(x);
    TS_SETTLE(x->c);
    if (p) *p = x->c.params.p;
    if (n) *n = 59 * x->c.N;
    return TS_OK;
}

ts_status ts_stats_buffer(ts_ctx* x, float** a, float** cnt) {
    TS_CHECK_CTX(x);
    TS_SETTLE(x->c);
    if (a) *a = x->c.accum.p;
    if (cnt) *cnt = x->c.vcount.p;
    return TS_OK;
}

ts_status ts_reserve_flat(ts_ctx* x, int64_t min_len) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t L = size_t(59) * c.N;
    if (min_len < 0) return validation(c, "min_len < 0");
    if (size_t(min_len) > c.params.cap || size_t(min_len) > c.grads.cap) {
        if (!ensure(c, c.params, size_t(min_len), true) || !ensure(c, c.grads, size_t(min_len), true))
            return TS_ERR_OOM;
    }
    if (c.params.cap > L) CK(cudaMemsetAsync(c.params.p + L, 0, (c.params.cap - L) * 4, c.stream));
    if (c.grads.cap > L) CK(cudaMemsetAsync(c.grads.p + L, 0, (c.grads.cap - L) * 4, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_adam_step(ts_ctx* x, const ts_adam_config* a) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!a) return validation(c, "adam config is NULL");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    return run_adam(c, *a, 0, 59 * c.N);
}

ts_status ts_adam_step_range(ts_ctx* x, const ts_adam_config* a, int64_t begin, int64_t end) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!a) return validation(c, "adam config is NULL");
    if (begin < 0 || end > 59 * c.N || begin > end) return validation(c, "bad range");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    return run_adam(c, *a, begin, end);
}

ts_status ts_train_step(ts_ctx* x, const ts_camera* cam, const ts_render_config* cfg, const float* target_hwc,
                        int32_t slot, const ts_adam_config* adam, float* out_loss) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    std::string why;
    if (!valid_camera(cam, &why) || !valid_config(cfg, &why)) return validation(c, why.c_str());
    if (!adam) return validation(c, "adam config is NULL");
    CK(cudaSetDevice(c.device));
    if (graph_eligible(c, *cam, *cfg, *adam)) return graph_step(c, *cam, *cfg, target_hwc, slot, *adam, out_loss);
    TS_SETTLE(c);
    return run_train_step(c, *cam, *cfg, target_hwc, slot, *adam, out_loss);
}

ts_status ts_set_graph(ts_ctx* x, int32_t on) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    c.graph_on = on != 0;
    if (!c.graph_on) drop_graphs(c);
    return TS_OK;
}

ts_status ts_graph_stats(ts_ctx* x, int64_t out[4]) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!out) return validation(c, "NULL output");
    out[0] = c.graph_launches;
    out[1] = c.graph_captures;
    out[2] = c.graph_replays;
    out[3] = int64_t(c.graphs.size());
    return TS_OK;
}

ts_status ts_opacity_reset(ts_ctx* x) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    launch_opacity_reset(c, float(std::log(0.01 / 0.99)));
    c.view_valid = c.loss_valid = false;
    return last_launch(c, "opacity_reset");
}

ts_status ts_densify(ts_ctx* x, float grad_thresh, float extent, uint64_t seed, int64_t iter, int64_t* n_after,
                     int64_t stats[3]) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!(extent > 0.f)) return validation(c, "extent must be > 0");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    int64_t st[3] = {0, 0, 0};
    const float log_small = float(std::log(0.01 * double(extent)));
    const float log_big = float(std::log(0.1 * double(extent)));
    const float logit_min = float(std::log(0.05 / 0.95));
    const int64_t na = launch_densify(c, grad_thresh, log_small, log_big, logit_min, seed, iter, st);
    if (na == -2) return TS_ERR_VALIDATION;  // store unchanged
    if (na < 0) return c.err.empty() ? TS_ERR_CUDA : TS_ERR_OOM;
    if (n_after) *n_after = na;
    c.grad_state = Context::kGradZero;
    if (stats) std::memcpy(stats, st, sizeof(st));
    c.view_valid = c.loss_valid = false;
    return last_launch(c, "densify");
}

ts_status ts_morton_reorder(ts_ctx* x, uint32_t* perm) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (c.grad_state == Context::kGradLive) return validation(c, "morton_reorder between backward and optimizer step");
    if (!launch_morton_reorder(c, perm)) return c.err.empty() ? TS_ERR_CUDA : TS_ERR_OOM;
    c.view_valid = c.loss_valid = false;
    return last_launch(c, "morton_reorder");
}

ts_status ts_set_state(ts_ctx* x, const float* grads, const float* m, const float* v, const float* accum,
                       const float* vcount) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t L = size_t(59) * c.N, N = size_t(c.N);
    if (grads) {
        CK(cudaMemcpyAsync(c.grads.p, grads, L * 4, cudaMemcpyHostToDevice, c.stream));
        c.grad_state = Context::kGradLive;
    }
    if (m) CK(cudaMemcpyAsync(c.m.p, m, L * 4, cudaMemcpyHostToDevice, c.stream));
    if (v) CK(cudaMemcpyAsync(c.v.p, v, L * 4, cudaMemcpyHostToDevice, c.stream));
    if (accum) CK(cudaMemcpyAsync(c.accum.p, accum, N * 4, cudaMemcpyHostToDevice, c.stream));
    if (vcount) CK(cudaMemcpyAsync(c.vcount.p, vcount, N * 4, cudaMemcpyHostToDevice, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_get_state(ts_ctx* x, float* grads, float* m, float* v, float* accum, float* vcount) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t L = size_t(59) * c.N, N = size_t(c.N);
    if (grads) CK(cudaMemcpyAsync(grads, c.grads.p, L * 4, cudaMemcpyDeviceToHost, c.stream));
    if (m) CK(cudaMemcpyAsync(m, c.m.p, L * 4, cudaMemcpyDeviceToHost, c.stream));
    if (v) CK(cudaMemcpyAsync(v, c.v.p, L * 4, cudaMemcpyDeviceToHost, c.stream));
    if (accum) CK(cudaMemcpyAsync(accum, c.accum.p, N * 4, cudaMemcpyDeviceToHost, c.stream));
    if (vcount) CK(cudaMemcpyAsync(vcount, c.vcount.p, N * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_compute_sampling_rates(ts_ctx* x, const ts_camera* cams, int32_t n_cams, float extent) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!cams || n_cams < 1) return validation(c, "need >= 1 camera");
    if (!(extent > 0.f)) return validation(c, "extent must be > 0");
    std::string why;
    std::vector<DevCam> dc(static_cast<size_t>(n_cams));
    for (int k = 0; k < n_cams; ++k) {
        if (!valid_camera(cams + k, &why)) return validation(c, why.c_str());
        dc[size_t(k)] = make_devcam(cams[k]);
    }
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (!launch_sampling_rates(c, dc.data(), n_cams, extent)) return c.err.empty() ? TS_ERR_CUDA : TS_ERR_OOM;
    c.nu_valid = true;
    return last_launch(c, "compute_sampling_rates");
}

ts_status ts_set_sampling_rates(ts_ctx* x, const float* nu) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!nu) return validation(c, "NULL sampling rates");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (c.N) CK(cudaMemcpyAsync(c.nu_hat.p, nu, size_t(c.N) * 4, cudaMemcpyHostToDevice, c.stream));
    c.nu_valid = true;
    return TS_OK;
}

ts_status ts_get_sampling_rates(ts_ctx* x, float* nu) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!nu) return validation(c, "NULL output");
    if (!c.nu_valid) return validation(c, "sampling rates not computed for the current store");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (c.N) CK(cudaMemcpyAsync(nu, c.nu_hat.p, size_t(c.N) * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return TS_OK;
}

ts_status ts_apply_3d_filter_clip(ts_ctx* x, float kappa3d) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!(kappa3d > 0.f)) return validation(c, "kappa3d must be > 0");
    if (!c.nu_valid) return validation(c, "apply_3d_filter_clip needs ts_compute_sampling_rates");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    launch_filter3d_clip(c, kappa3d);
    c.view_valid = c.loss_valid = false;
    return last_launch(c, "apply_3d_filter_clip");
}

ts_status ts_set_binning(ts_ctx* x, int32_t mode) {
    TS_CHECK_CTX(x);
    TS_SETTLE(x->c);
    Context& c = x->c;
    if (mode < 0 || mode > 1) return validation(c, "binning mode must be 0 (auto) or 1 (radix)");
    c.binning_mode = mode;
    return TS_OK;
}

ts_status ts_binning_path(ts_ctx* x, int32_t* radix) {
    TS_CHECK_CTX(x);
    if (radix) *radix = x->c.last_view_radix ? 1 : 0;
    return TS_OK;
}

ts_status ts_debug_loss_grad(ts_ctx* x, float* dLdC_hwc) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!c.loss_valid) return validation(c, "no training_loss state");
    if (!dLdC_hwc) return validation(c, "NULL output");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t P = size_t(c.fw) * c.fh;
    launch_chw_to_hwc(c, c.dLdC.p, c.hwc_stage.p, int(P));
    CK(cudaMemcpyAsync(dLdC_hwc, c.hwc_stage.p, 3 * P * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return last_launch(c, "debug_loss_grad");
}

ts_status ts_debug_preprocess(ts_ctx* x, float* splat12, int32_t* rect4, uint32_t* tile_count, uint32_t* depth_key) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!c.view_valid) return validation(c, "no forward state");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t N = size_t(c.N);
    std::vector<float4> sp(3 * N);
    std::vector<uint4> rc(N);
    std::vector<uint32_t> cnt(N);
    if (N) {
        CK(cudaMemcpyAsync(sp.data(), c.splat.p, 3 * N * 16, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(rc.data(), c.rect.p, N * 16, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(cnt.data(), c.tcount.p, N * 4, cudaMemcpyDeviceToHost, c.stream));
    }
    CK(cudaStreamSynchronize(c.stream));
    for (size_t g = 0; g < N; ++g) {
        if (splat12) std::memcpy(splat12 + 12 * g, &sp[3 * g], 48);
        if (rect4) {
            rect4[4 * g] = int32_t(rc[g].x & 0xFFFF);
            rect4[4 * g + 1] = int32_t(rc[g].y & 0xFFFF);
            rect4[4 * g + 2] = int32_t((rc[g].x >> 16) & 0x7FFF);
            rect4[4 * g + 3] = int32_t((rc[g].y >> 16) & 0x7FFF);
        }
        if (tile_count) tile_count[g] = cnt[g];
        if (depth_key) {
            uint32_t bits;
            std::memcpy(&bits, &sp[3 * g + 1].w, 4);
            depth_key[g] = cnt[g] ? (bits ^ 0x80000000u) : 0xFFFFFFFFu;
        }
    }
    return TS_OK;
}

ts_status ts_debug_instances(ts_ctx* x, int64_t* n_inst, uint64_t* keys, uint32_t* vals, uint32_t* ranges) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!c.view_valid) return validation(c, "no forward state");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    if (n_inst) *n_inst = c.I;
    if (!keys && !vals && !ranges) return TS_OK;
    const size_t I = size_t(c.I), N = size_t(c.N);
    const int Tn = ((c.cam.width + 15) / 16) * ((c.cam.height + 15) / 16);
    std::vector<uint32_t> iv(I), st(size_t(Tn) + 1);
    std::vector<float4> sp(3 * N);
    if (I) CK(cudaMemcpyAsync(iv.data(), c.ival[0].p, I * 4, cudaMemcpyDeviceToHost, c.stream));
    if (N) CK(cudaMemcpyAsync(sp.data(), c.splat.p, 3 * N * 16, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(st.data(), c.starts.p, (size_t(Tn) + 1) * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    // tile of instance i from the ranges (both binning paths produce the ranges)
    int tile = 0;
    for (size_t i = 0; i < I; ++i) {
        while (tile < Tn && size_t(st[tile + 1]) <= i) ++tile;
        if (vals) vals[i] = iv[i];
        if (keys) {
            uint32_t bits;
            std::memcpy(&bits, &sp[3 * size_t(iv[i]) + 1].w, 4);
            keys[i] = (uint64_t(uint32_t(tile)) << 32) | uint64_t(bits ^ 0x80000000u);
        }
    }
    if (ranges)
        for (int t = 0; t < Tn; ++t) {
            ranges[2 * t] = st[t];
            ranges[2 * t + 1] = st[t + 1];
        }
    return TS_OK;
}

ts_status ts_debug_grad2d(ts_ctx* x, const float* dLdC_hwc, float* g2d9) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!c.view_valid) return validation(c, "no forward state");
    if (!dLdC_hwc || !g2d9) return validation(c, "NULL argument");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    const size_t N = size_t(c.N);
    if (ts_status s = upload_image_chw(c, dLdC_hwc, c.dLdC.p); s != TS_OK) return s;
    CK(cudaMemsetAsync(c.g2d.p, 0, 3 * N * 16, c.stream));
    DevCam dc = make_devcam(c.cam);
    launch_blend_bwd(c, dc, c.cfg);
    std::vector<float4> g(3 * N);
    if (N) CK(cudaMemcpyAsync(g.data(), c.g2d.p, 3 * N * 16, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemsetAsync(c.g2d.p, 0, 3 * N * 16, c.stream));
    c.g2d_clean = true;
    CK(cudaStreamSynchronize(c.stream));
    for (size_t k = 0; k < N; ++k) {
        const float* s = reinterpret_cast<const float*>(&g[3 * k]);
        std::memcpy(g2d9 + 9 * k, s, 9 * 4);
    }
    return last_launch(c, "debug_grad2d");
}

ts_status ts_view_stats(ts_ctx* x, int64_t out[4]) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!out) return validation(c, "NULL output");
    CK(cudaSetDevice(c.device));
    TS_SETTLE(c);
    uint32_t cnt[3];
    CK(cudaMemcpyAsync(cnt, c.counters.p, sizeof(cnt), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    out[0] = cnt[1];
    out[1] = c.I;
    out[2] = cnt[2];
    out[3] = int64_t(c.cam.width) * c.cam.height;
    return TS_OK;
}

ts_status ts_set_profiling(ts_ctx* x, int32_t on) {
    TS_CHECK_CTX(x);
    TS_SETTLE(x->c);
    Context& c = x->c;
    if (c.profiling || on) cudaStreamSynchronize(c.stream);
    c.profiling = on != 0;
    if (on) c.ev_cursor = 0;
    return TS_OK;
}

ts_status ts_stage_times(ts_ctx* x, float* ms, int32_t* counts, int32_t n) {
    TS_CHECK_CTX(x);
    Context& c = x->c;
    if (!ms) return validation(c, "NULL output");
    CK(cudaStreamSynchronize(c.stream));
    for (int k = 0; k < n; ++k) {
        ms[k] = 0.f;
        if (counts) counts[k] = 0;
    }
    for (size_t i = 0; i < c.ev_cursor; ++i) {
        const int k = c.ev_stage[i];
        if (k >= n) continue;
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, c.ev_b[i], c.ev_e[i]));
        ms[k] += t;
        if (counts) counts[k] += 1;
    }
    return TS_OK;
}

ts_status ts_launch_count(ts_ctx* x, int64_t* n) {
    TS_CHECK_CTX(x);
    if (n) *n = x->c.launches;
    return TS_OK;
}

ts_status ts_host_alloc(size_t bytes, void** out) {
    if (!out) return TS_ERR_VALIDATION;
    if (cudaMallocHost(out, bytes) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return TS_ERR_OOM;
    }
    return TS_OK;
}

ts_status ts_host_free(void* p) {
    if (p) cudaFreeHost(p);
    return TS_OK;
}

}  // extern "C"
