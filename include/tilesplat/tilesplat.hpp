// tilesplat/tilesplat.hpp — C++ host API of the B200 hot path over the C-ABI
// (include/tilesplat_c.h).  Mirrors the reference's SPEC.md operation set on
// the reference's value types (tilesplat/vecmath.hpp): ParameterStore
// (SPEC.md:23-29), Camera (:119-123), render (:336-344), training_loss
// (:767-775), backward (:382-420), adam_step_* (:463-490), densify_and_prune
// (:545-553), opacity_reset (:555-563), mean_lr (:502-510),
// sh_active_degree (:575-580).  Errors raise tilesplat::Error carrying the
// C-ABI status (1 = validation, mirroring the reference CLI exit code).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../tilesplat_c.h"
#include "vecmath.hpp"

namespace tilesplat {

class Error : public std::runtime_error {
   public:
    Error(ts_status s, const std::string& what) : std::runtime_error(what), status(s) {}
    ts_status status;
};

// Column-oriented raw parameters; 59 floats per Gaussian.
struct ParameterStore {
    std::vector<float> means, log_scales, quaternions, opacity_logits, sh_dc, sh_rest;
    int64_t size() const { return int64_t(opacity_logits.size()); }
    void resize(int64_t n) {
        means.resize(3 * n), log_scales.resize(3 * n), quaternions.resize(4 * n);
        opacity_logits.resize(n), sh_dc.resize(3 * n), sh_rest.resize(45 * n);
    }
    // flat 59*N layout of the C-ABI
    std::vector<float> flat() const {
        std::vector<float> f;
        f.reserve(size_t(59) * size());
        for (const auto* v : {&means, &log_scales, &quaternions, &opacity_logits, &sh_dc, &sh_rest})
            f.insert(f.end(), v->begin(), v->end());
        return f;
    }
    void from_flat(const std::vector<float>& f, int64_t n) {
        resize(n);
        size_t o = 0;
        for (auto* v : {&means, &log_scales, &quaternions, &opacity_logits, &sh_dc, &sh_rest}) {
            std::copy(f.begin() + o, f.begin() + o + v->size(), v->begin());
            o += v->size();
        }
    }
};

struct Camera {
    Mat4<float> world_to_camera = Mat4<float>::identity();
    float fx = 1, fy = 1, cx = 0, cy = 0, near_plane = 0.2f;
    int32_t width = 0, height = 0;

    ts_camera abi() const {
        ts_camera c{};
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) c.W[4 * i + j] = world_to_camera.m[i][j];
        c.fx = fx, c.fy = fy, c.cx = cx, c.cy = cy, c.near_plane = near_plane;
        c.width = width, c.height = height;
        return c;
    }
    // camera centre -R^T t
    Vec3<float> center() const {
        const Mat3<float> R = world_to_camera.upper3x3();
        const Vec3<float> t{world_to_camera.m[0][3], world_to_camera.m[1][3], world_to_camera.m[2][3]};
        return R.transposed_mul(t) * -1.0f;
    }
};

// antialias config block: aa = off | filter3d_original | filter3d_clip | full (clip + mip)
enum class AntiAlias : int32_t { off = 0, filter3d_original = 1, filter3d_clip = 2, full = 3 };

struct RenderConfig {
    int32_t sh_degree = 3;
    int32_t bound_mode = 2;  // rect_opacity
    int32_t cull_mode = 1;   // exact
    int32_t early_stop_compat = 0;
    int32_t truncation = 0;     // 0 classic, 1 response (keep iff the Mahalanobis distance <= sigma_cut)
    float sigma_cut = 3.33f;
    int32_t backward_mode = 0;  // 0 per-pixel, 1 per-Gaussian buckets
    float tau_alpha = 1.0f / 255.0f;
    float dilation = 0.3f;   // classic 0.3; the Mip 2D filter variance 0.1 with AntiAlias::full
    Vec3<float> background{0.f, 0.f, 0.f};
    AntiAlias aa = AntiAlias::off;
    float kappa3d = 0.2f;

    ts_render_config abi() const {
        ts_render_config c{};
        c.sh_degree = sh_degree, c.bound_mode = bound_mode, c.cull_mode = cull_mode;
        c.truncation = truncation, c.early_stop_compat = early_stop_compat, c.backward_mode = backward_mode;
        c.tau_alpha = tau_alpha, c.dilation = dilation, c.sigma_cut = sigma_cut;
        c.bg[0] = background.x, c.bg[1] = background.y, c.bg[2] = background.z;
        c.aa_mode = static_cast<int32_t>(aa), c.kappa3d = kappa3d;
        return c;
    }
};

inline double mean_lr(int64_t step, double extent) { return extent * 1.6e-4 * std::pow(1e-2, double(step) / 30000.0); }
inline int sh_active_degree(int64_t iter) { return int(iter / 1000 < 3 ? iter / 1000 : 3); }

enum class OptimizerMode : int32_t { reference = 0, fused = 1, skip_invisible = 2 };

// Adam hyper-parameters and LR schedule for 1-based step t.
inline ts_adam_config adam_config(int64_t t, double extent, OptimizerMode mode = OptimizerMode::fused) {
    ts_adam_config a{};
    const double lrs[6] = {mean_lr(t - 1, extent), 0.005, 0.001, 0.025, 2.5e-3, 1.25e-4};
    for (int k = 0; k < 6; ++k) a.lr[k] = float(lrs[k]);
    a.beta1 = 0.9f, a.beta2 = 0.999f, a.eps = 1e-15f;
    a.bc1 = float(1.0 - std::pow(0.9, double(t)));
    a.bc2 = float(1.0 - std::pow(0.999, double(t)));
    a.mode = int32_t(mode);
    a.zero_grads = 1;
    return a;
}

struct FrameBuffers {
    int32_t width = 0, height = 0;
    std::vector<float> color, final_transmittance;  // H*W*3, H*W
    std::vector<uint32_t> contributor_count;         // H*W
};

// One device context: ParameterStore + AdamState + GradientStore on the GPU.
class Engine {
   public:
    explicit Engine(int device = 0, void* stream = nullptr) {
        check(ts_create(device, stream, &ctx_), "ts_create");
    }
    ~Engine() {
        if (ctx_) ts_destroy(ctx_);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void set_params(const ParameterStore& s) {
        check(ts_set_params(ctx_, s.size(), s.means.data(), s.log_scales.data(), s.quaternions.data(),
                            s.opacity_logits.data(), s.sh_dc.data(), s.sh_rest.data()),
              "ts_set_params");
    }
    ParameterStore params() {
        int64_t n = 0;
        ts_num_gaussians(ctx_, &n);
        std::vector<float> f(size_t(59) * n);
        check(ts_get_params_flat(ctx_, f.data()), "ts_get_params_flat");
        ParameterStore s;
        s.from_flat(f, n);
        return s;
    }
    int64_t size() const {
        int64_t n = 0;
        ts_num_gaussians(ctx_, &n);
        return n;
    }

    FrameBuffers render(const Camera& cam, const RenderConfig& cfg) {
        const ts_camera c = cam.abi();
        const ts_render_config r = cfg.abi();
        FrameBuffers fb;
        fb.width = cam.width, fb.height = cam.height;
        const size_t P = size_t(cam.width) * cam.height;
        fb.color.resize(3 * P), fb.final_transmittance.resize(P), fb.contributor_count.resize(P);
        check(ts_forward(ctx_, &c, &r, fb.color.data(), fb.final_transmittance.data(), fb.contributor_count.data()),
              "ts_forward");
        return fb;
    }
    float training_loss(const std::vector<float>& target_hwc) {
        float l = 0.f;
        check(ts_loss(ctx_, target_hwc.data(), 0, &l), "ts_loss");
        return l;
    }
    void backward() { check(ts_backward(ctx_, nullptr), "ts_backward"); }
    void adam_step(const ts_adam_config& a) { check(ts_adam_step(ctx_, &a), "ts_adam_step"); }
    float train_step(const Camera& cam, const RenderConfig& cfg, const float* target_hwc, const ts_adam_config& a) {
        const ts_camera c = cam.abi();
        const ts_render_config r = cfg.abi();
        float l = 0.f;
        check(ts_train_step(ctx_, &c, &r, target_hwc, 0, &a, &l), "ts_train_step");
        return l;
    }
    // returns N after; stats = {clones, splits, pruned}
    int64_t densify_and_prune(float grad_thresh, float extent, uint64_t seed, int64_t iter, int64_t stats[3]) {
        int64_t n = 0;
        check(ts_densify(ctx_, grad_thresh, extent, seed, iter, &n, stats), "ts_densify");
        return n;
    }
    void opacity_reset() { check(ts_opacity_reset(ctx_), "ts_opacity_reset"); }
    // antialias: sampling rates over the training views, post-step 3D-filter clip
    void compute_sampling_rates(const std::vector<Camera>& cams, float extent) {
        std::vector<ts_camera> c;
        for (const auto& k : cams) c.push_back(k.abi());
        check(ts_compute_sampling_rates(ctx_, c.data(), int32_t(c.size()), extent), "ts_compute_sampling_rates");
    }
    void apply_3d_filter_clip(float kappa3d = 0.2f) { check(ts_apply_3d_filter_clip(ctx_, kappa3d), "ts_apply_3d_filter_clip"); }
    // morton_reorder: returns perm[new] = old
    std::vector<uint32_t> morton_reorder() {
        std::vector<uint32_t> perm(static_cast<size_t>(size()));
        check(ts_morton_reorder(ctx_, perm.data()), "ts_morton_reorder");
        return perm;
    }
    ts_ctx* handle() { return ctx_; }

   private:
    void check(ts_status s, const char* what) {
        if (s == TS_OK) return;
        throw Error(s, std::string(what) + ": " + (ctx_ ? ts_last_error(ctx_) : "no context"));
    }
    ts_ctx* ctx_ = nullptr;
};

}  // namespace tilesplat
