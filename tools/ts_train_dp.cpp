// ts_train_dp — the C++ multi-GPU host path of the training step:
// one process, one host thread per GPU, one NCCL communicator per GPU
// (ncclCommInitAll), each GPU driving its own tilesplat context (C-ABI,
// include/tilesplat_c.h) on its own CUDA stream.  Gaussians, Adam moments and
// densify statistics are replicated; rank r renders views {r, r+G, ...} of each
// step's batch and accumulates their gradients in its flat 59N buffer
// (ts_grad_buffer; batch gradient = sum over views); one exchange
// per step then runs on the context stream, ordered behind the backward without
// a host wait:
//   allreduce : ncclAllReduce(grads, sum) + replicated fused Adam (ts_adam_step)
//   sharded   : ncclReduceScatter(grads) -> Adam on this rank's 1/G slice
//               (ts_adam_step_range) -> ncclAllGather(params), both in place in the
//               padded flat buffers (ts_reserve_flat once); the gradient buffer is then
//               marked consumed (ts_mark_grads_consumed: the next backward overwrites)
//   chunked   : K in-order ncclAllReduce chunks, each followed by the Adam sweep of
//               its range, so the optimizer of chunk k overlaps the sum of chunk k+1
// These mirror paper_2602_09999_b200/dp.py (torch.distributed) one for one.
//
// usage: ts_train_dp <gpus> <allreduce|sharded|chunked> [n=20000] [iters=6] [views_per_step=4] [--check]
// --check: every step, the exchange + optimizer is re-run in a separate single
// context on GPU 0 from host snapshots: the pre-step parameters and moments, and
// the batch gradient = sum of the ranks' accumulated gradient buffers (summed in
// rank order; for G <= 2 that is NCCL's sum bit for bit, fp32 addition commutes).
// The data-parallel step must leave rank 0's parameters and moments bitwise where
// ts_adam_step over the whole buffer does (the rendering gradients themselves use
// fp32 atomics and are not run-to-run deterministic, so they are snapshotted, not
// recomputed).  Every replica must equal rank 0 bit for bit.  One JSON line; exit
// codes 0 ok, 1 validation, 2 check failure, 3 CUDA / NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "tilesplat/tilesplat.hpp"

using namespace tilesplat;

namespace {

constexpr int W = 256, H = 192, kViews = 8;

Camera look_at(Vec3<float> eye, int w, int h) {
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

struct Failure {
    int code;
    std::string what;
};

#define NCCL_OK(x)                                                                          \
    do {                                                                                    \
        ncclResult_t r_ = (x);                                                              \
        if (r_ != ncclSuccess) throw Failure{3, std::string(#x) + ": " + ncclGetErrorString(r_)}; \
    } while (0)
#define CUDA_OK(x)                                                                          \
    do {                                                                                    \
        cudaError_t r_ = (x);                                                               \
        if (r_ != cudaSuccess) throw Failure{3, std::string(#x) + ": " + cudaGetErrorString(r_)}; \
    } while (0)
#define TS_OK_(x)                                                                           \
    do {                                                                                    \
        ts_status s_ = (x);                                                                 \
        if (s_ != TS_OK) throw Failure{s_ == TS_ERR_VALIDATION ? 1 : 3, std::string(#x)};    \
    } while (0)

// [begin, end) of rank's slice of a flat buffer of L floats, 16-byte aligned slices (dp.py shard_bounds)
void shard_bounds(int64_t L, int world, int rank, int64_t* b, int64_t* e, int64_t* per) {
    int64_t p = (L + world - 1) / world;
    p = (p + 3) / 4 * 4;
    *per = p;
    *b = std::min(L, int64_t(rank) * p);
    *e = std::min(L, *b + p);
}

std::vector<float> flat_of(const ParameterStore& s) {
    const int64_t n = s.size();
    std::vector<float> f(size_t(59) * n);
    size_t o = 0;
    for (const auto* v : {&s.means, &s.log_scales, &s.quaternions, &s.opacity_logits, &s.sh_dc, &s.sh_rest}) {
        std::memcpy(f.data() + o, v->data(), v->size() * 4);
        o += v->size();
    }
    return f;
}

ts_camera to_c(const Camera& c) { return c.abi(); }

// reusable barrier of the G rank threads (C++17)
class Barrier {
  public:
    explicit Barrier(int n) : n_(n) {}
    void wait() {
        std::unique_lock<std::mutex> lk(mu_);
        const int gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
        } else {
            cv_.wait(lk, [&] { return gen != gen_; });
        }
    }

  private:
    std::mutex mu_;
    std::condition_variable cv_;
    int n_, count_ = 0, gen_ = 0;
};

struct Rank {
    int dev = 0;
    cudaStream_t stream = nullptr;
    ts_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    std::vector<float> final_params, gsnap;
    double ms = 0;
    std::string err;
    int code = 0;
};

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ts_train_dp <gpus> <allreduce|sharded|chunked> [n] [iters] [views] [--check]\n");
        return 1;
    }
    const int G = std::atoi(argv[1]);
    const std::string mode = argv[2];
    const int64_t n = argc > 3 ? std::atoll(argv[3]) : 20000;
    const int iters = argc > 4 ? std::atoi(argv[4]) : 6;
    const int vps = argc > 5 ? std::atoi(argv[5]) : 4;
    bool check = false;
    for (int i = 1; i < argc; ++i) check |= std::strcmp(argv[i], "--check") == 0;
    if (G < 1 || vps < 1 || (mode != "allreduce" && mode != "sharded" && mode != "chunked")) {
        std::fprintf(stderr, "ts_train_dp: bad arguments\n");
        return 1;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < G) {
        std::fprintf(stderr, "ts_train_dp: %d GPUs requested, %d present\n", G, ndev);
        return 3;
    }
    // synth_scene: seeded GT store, 8 inward cameras, perturbed start
    std::mt19937_64 rng(11);
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
    for (int i = 0; i < kViews; ++i) {
        const float a = float(i) * 0.785398f;
        cams.push_back(look_at({3.5f * std::sin(a), -0.5f, -3.5f * std::cos(a)}, W, H));
    }
    RenderConfig rcfg;
    rcfg.sh_degree = 3;
    const ts_render_config cfg = rcfg.abi();
    ParameterStore p0 = gt;
    for (auto& v : p0.means) v += 0.02f * Nn(rng);
    for (auto& v : p0.log_scales) v += 0.2f * Nn(rng);
    const std::vector<float> gt_flat = flat_of(gt), p0_flat = flat_of(p0);
    const int64_t L = 59 * n;
    auto views_of = [&](int step, int world, int rank) {  // the step's batch: global views step*vps + k
        std::vector<int> v;
        for (int k = rank; k < vps; k += world) v.push_back((step * vps + k) % kViews);
        return v;
    };

    std::vector<Rank> ranks(static_cast<size_t>(G));
    Barrier bar(G);
    int64_t mismatches = check ? 0 : -1;
    double max_rel = 0;
    ts_ctx* ref = nullptr;  // the single-context reference of --check (GPU 0)
    std::vector<float> pre_p, pre_m, pre_v, post_p, post_m, post_v, gsum, rp, rm, rv;
    std::vector<int> devs(static_cast<size_t>(G));
    for (int r = 0; r < G; ++r) devs[size_t(r)] = r;
    std::vector<ncclComm_t> comms(static_cast<size_t>(G));
    if (ncclCommInitAll(comms.data(), G, devs.data()) != ncclSuccess) {
        std::fprintf(stderr, "ts_train_dp: ncclCommInitAll failed\n");
        return 3;
    }
    auto rank_main = [&](int r) {
        Rank& R = ranks[size_t(r)];
        try {
            R.dev = r;
            R.comm = comms[size_t(r)];
            CUDA_OK(cudaSetDevice(r));
            CUDA_OK(cudaStreamCreateWithFlags(&R.stream, cudaStreamNonBlocking));
            TS_OK_(ts_create(r, R.stream, &R.ctx));
            ts_ctx* c = R.ctx;
            // targets of this rank's views: rendered from the GT store, kept in device slots
            TS_OK_(ts_set_params_flat(c, n, gt_flat.data()));
            std::vector<float> img(size_t(W) * H * 3);
            for (int v = 0; v < kViews; ++v) {
                const ts_camera cc = to_c(cams[size_t(v)]);
                TS_OK_(ts_forward(c, &cc, &cfg, img.data(), nullptr, nullptr));
                TS_OK_(ts_set_target(c, v, W, H, img.data()));
            }
            TS_OK_(ts_set_params_flat(c, n, p0_flat.data()));
            int64_t b = 0, e = L, per = L;
            shard_bounds(L, G, r, &b, &e, &per);
            if (mode == "sharded") TS_OK_(ts_reserve_flat(c, per * G));  // once, not per step
            const auto t0 = std::chrono::steady_clock::now();
            for (int it = 0; it < iters; ++it) {
                for (int v : views_of(it, G, r)) {
                    const ts_camera cc = to_c(cams[size_t(v)]);
                    TS_OK_(ts_forward(c, &cc, &cfg, nullptr, nullptr, nullptr));
                    TS_OK_(ts_loss(c, nullptr, v, nullptr));
                    TS_OK_(ts_backward(c, nullptr));
                }
                ts_adam_config a = adam_config(it + 1, 1.0);
                if (check) {  // snapshots before the exchange (every rank its gradient, rank 0 the state)
                    R.gsnap.resize(size_t(L));
                    TS_OK_(ts_get_state(c, R.gsnap.data(), nullptr, nullptr, nullptr, nullptr));
                    if (r == 0) {
                        pre_p.resize(size_t(L)), pre_m.resize(size_t(L)), pre_v.resize(size_t(L));
                        TS_OK_(ts_get_params_flat(c, pre_p.data()));
                        TS_OK_(ts_get_state(c, nullptr, pre_m.data(), pre_v.data(), nullptr, nullptr));
                    }
                }
                float* gp = nullptr;
                float* pp = nullptr;
                int64_t cnt = 0;
                TS_OK_(ts_grad_buffer(c, &gp, &cnt));
                TS_OK_(ts_param_buffer(c, &pp, &cnt));
                if (mode == "allreduce") {
                    NCCL_OK(ncclAllReduce(gp, gp, size_t(L), ncclFloat, ncclSum, R.comm, R.stream));
                    TS_OK_(ts_adam_step(c, &a));
                } else if (mode == "chunked") {
                    const int K = 8;
                    for (int k = 0; k < K; ++k) {
                        int64_t cb, ce, cp;
                        shard_bounds(L, K, k, &cb, &ce, &cp);
                        if (ce <= cb) continue;
                        NCCL_OK(ncclAllReduce(gp + cb, gp + cb, size_t(ce - cb), ncclFloat, ncclSum, R.comm,
                                              R.stream));
                        TS_OK_(ts_adam_step_range(c, &a, cb, ce));
                    }
                } else {
                    // in place: this rank's slot of the padded buffer is the receive / send buffer
                    NCCL_OK(ncclReduceScatter(gp, gp + int64_t(r) * per, size_t(per), ncclFloat, ncclSum, R.comm,
                                              R.stream));
                    a.zero_grads = 0;
                    if (e > b) TS_OK_(ts_adam_step_range(c, &a, b, e));
                    NCCL_OK(ncclAllGather(pp + int64_t(r) * per, pp, size_t(per), ncclFloat, R.comm, R.stream));
                    TS_OK_(ts_mark_grads_consumed(c));
                }
                if (check) {
                    if (r == 0) {
                        post_p.resize(size_t(L)), post_m.resize(size_t(L)), post_v.resize(size_t(L));
                        TS_OK_(ts_get_params_flat(c, post_p.data()));
                        TS_OK_(ts_get_state(c, nullptr, post_m.data(), post_v.data(), nullptr, nullptr));
                    }
                    bar.wait();  // every rank's gradient snapshot is in
                    if (r == 0) {
                        gsum = ranks[0].gsnap;
                        for (int q = 1; q < G; ++q)
                            for (int64_t i = 0; i < L; ++i) gsum[size_t(i)] += ranks[size_t(q)].gsnap[size_t(i)];
                        const ts_adam_config a_ref = adam_config(it + 1, 1.0);
                        TS_OK_(ts_set_params_flat(ref, n, pre_p.data()));
                        TS_OK_(ts_set_state(ref, gsum.data(), pre_m.data(), pre_v.data(), nullptr, nullptr));
                        TS_OK_(ts_adam_step(ref, &a_ref));
                        rp.resize(size_t(L)), rm.resize(size_t(L)), rv.resize(size_t(L));
                        TS_OK_(ts_get_params_flat(ref, rp.data()));
                        TS_OK_(ts_get_state(ref, nullptr, rm.data(), rv.data(), nullptr, nullptr));
                        for (int64_t i = 0; i < L; ++i) {
                            const size_t u = size_t(i);
                            const bool same = std::memcmp(&rp[u], &post_p[u], 4) == 0 &&
                                              std::memcmp(&rm[u], &post_m[u], 4) == 0 &&
                                              std::memcmp(&rv[u], &post_v[u], 4) == 0;
                            if (!same) ++mismatches;
                            max_rel = std::max(max_rel, double(std::fabs(rp[u] - post_p[u])) /
                                                            std::max(1e-6, double(std::fabs(rp[u]))));
                        }
                    }
                    bar.wait();  // snapshots consumed before the next step overwrites them
                }
            }
            CUDA_OK(cudaStreamSynchronize(R.stream));
            R.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / iters;
            R.final_params.resize(size_t(L));
            TS_OK_(ts_get_params_flat(c, R.final_params.data()));
        } catch (const Failure& f) {
            R.code = f.code;
            R.err = f.what + (R.ctx ? std::string(" (") + ts_last_error(R.ctx) + ")" : "");
        }
    };
    if (check && (cudaSetDevice(0) != cudaSuccess || ts_create(0, nullptr, &ref) != TS_OK)) {
        std::fprintf(stderr, "ts_train_dp: reference context\n");
        return 3;
    }
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r) th.emplace_back(rank_main, r);
    for (auto& t : th) t.join();
    int rc = 0;
    for (const Rank& R : ranks)
        if (R.code) {
            std::fprintf(stderr, "ts_train_dp rank %d: %s\n", R.dev, R.err.c_str());
            rc = std::max(rc, R.code);
        }
    bool replicas_equal = rc == 0;
    for (int r = 1; r < G && rc == 0; ++r)
        replicas_equal &= std::memcmp(ranks[size_t(r)].final_params.data(), ranks[0].final_params.data(),
                                      size_t(L) * 4) == 0;
    if (check && rc == 0 && G <= 2 && mismatches != 0) rc = 2;  // G > 2: ring sum order (reported only)
    if (ref) ts_destroy(ref);
    if (!replicas_equal && rc == 0) rc = 2;
    double ms = 0;
    for (const Rank& R : ranks) ms = std::max(ms, R.ms);
    std::printf("{\"gpus\": %d, \"mode\": \"%s\", \"n\": %lld, \"iters\": %d, \"views_per_step\": %d, "
                "\"ms_per_step_host\": %.3f, \"replicas_bitwise_equal\": %s, \"check_mismatches\": %lld, "
                "\"check_max_rel\": %.3g, \"nccl_version\": %d}\n",
                G, mode.c_str(), (long long)n, iters, vps, ms, replicas_equal ? "true" : "false",
                (long long)mismatches, max_rel, NCCL_VERSION_CODE);
    for (Rank& R : ranks) {
        if (R.ctx) ts_destroy(R.ctx);
        if (R.comm) ncclCommDestroy(R.comm);
        if (R.stream) cudaStreamDestroy(R.stream);
    }
    return rc;
}
