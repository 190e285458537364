// ts_train — C++ host driver of the B200 hot path through tilesplat.hpp (the
// reference's C++ API surface): synth_scene in C++, render
// the ground truth, then train a perturbed store with the full schedule
// (SH ramp, mean-LR decay, densify/prune and opacity reset).
// Prints one JSON line with the loss trajectory.  Exit codes: 0 ok,
// 1 validation error, 2 check failure.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "tilesplat/tilesplat.hpp"

using namespace tilesplat;

static Camera look_at(Vec3<float> eye, int w, int h) {
    Vec3<float> z = (Vec3<float>{0, 0, 0} - eye).normalized();
    Vec3<float> down{0, -1, 0};
    Vec3<float> x{down.y * z.z - down.z * z.y, down.z * z.x - down.x * z.z, down.x * z.y - down.y * z.x};
    x = x.normalized();
    Vec3<float> y{z.y * x.z - z.z * x.y, z.z * x.x - z.x * x.z, z.x * x.y - z.y * x.x};
    Camera c;
    const Vec3<float> rows[3] = {x, y, z};
    for (int i = 0; i < 3; ++i) {
        c.world_to_camera.m[i][0] = rows[i].x, c.world_to_camera.m[i][1] = rows[i].y;
        c.world_to_camera.m[i][2] = rows[i].z, c.world_to_camera.m[i][3] = -rows[i].dot(eye);
    }
    c.fx = c.fy = float(w / (2.0 * std::tan(M_PI / 6.0)));
    c.cx = w / 2.0f, c.cy = h / 2.0f, c.width = w, c.height = h;
    return c;
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? std::atoll(argv[1]) : 20000;
    const int iters = argc > 2 ? std::atoi(argv[2]) : 300;
    const int W = 256, H = 192;
    try {
        std::mt19937_64 rng(7);
        std::uniform_real_distribution<float> U(-1.f, 1.f);
        std::normal_distribution<float> Nn(0.f, 1.f);
        ParameterStore gt;
        gt.resize(n);
        for (int64_t g = 0; g < n; ++g) {
            for (int k = 0; k < 3; ++k) gt.means[3 * g + k] = U(rng);
            for (int k = 0; k < 3; ++k) gt.log_scales[3 * g + k] = std::log(0.02f) + 0.3f * Nn(rng);
            for (int k = 0; k < 4; ++k) gt.quaternions[4 * g + k] = Nn(rng);
            gt.opacity_logits[g] = Nn(rng);
            for (int k = 0; k < 3; ++k) gt.sh_dc[3 * g + k] = 1.5f * U(rng);
            for (int k = 0; k < 45; ++k) gt.sh_rest[45 * g + k] = 0.05f * Nn(rng);
        }
        std::vector<Camera> cams;
        for (int i = 0; i < 8; ++i) {
            const float a = float(i) * 0.785398f;
            cams.push_back(look_at({3.5f * std::sin(a), -0.5f, -3.5f * std::cos(a)}, W, H));
        }
        RenderConfig cfg;
        Engine e(0);
        e.set_params(gt);
        std::vector<std::vector<float>> targets;
        for (const auto& c : cams) targets.push_back(e.render(c, cfg).color);
        ParameterStore p = gt;
        for (auto& v : p.means) v += 0.02f * Nn(rng);
        for (auto& v : p.log_scales) v += 0.2f * Nn(rng);
        e.set_params(p);
        double extent = 0;
        {
            Vec3<float> m{0, 0, 0};
            for (auto& c : cams) m += c.center() * (1.0f / cams.size());
            for (auto& c : cams) extent = std::max(extent, double((c.center() - m).norm()));
            extent *= 1.1;
        }
        float first = 0, last = 0;
        const auto t0 = std::chrono::steady_clock::now();
        for (int it = 0; it < iters; ++it) {
            cfg.sh_degree = std::min(3, sh_active_degree(int64_t(it) * 10));
            const size_t v = size_t(it) % cams.size();
            last = e.train_step(cams[v], cfg, targets[v].data(), adam_config(it + 1, extent));
            if (it == 0) first = last;
            if (it > 0 && it % 100 == 0) {
                int64_t st[3];
                e.densify_and_prune(2e-4f, float(extent), 42, it, st);
            }
            // Morton reindexing while densification is active (cadence scaled 5000 -> 250)
            if (it > 0 && it % 250 == 0) e.morton_reorder();
        }
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"n_initial\": %lld, \"n_final\": %lld, \"iters\": %d, \"loss_first\": %.6f, "
                    "\"loss_last\": %.6f, \"seconds\": %.3f}\n",
                    (long long)n, (long long)e.size(), iters, first, last, secs);
        return last < first ? 0 : 2;
    } catch (const Error& err) {
        std::fprintf(stderr, "ts_train: %s\n", err.what());
        return err.status == TS_ERR_VALIDATION ? 1 : 3;
    }
}
