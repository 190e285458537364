// ts_oracle.cpp — CPU restatement of the reference 3DGS training hot path.
//
// TEST INFRASTRUCTURE ONLY (see ts_oracle.h).  Build: oracle/Makefile with
// -O3 -ffp-contract=off (no FMA contraction: the float binning path must be
// bit-identical to the CUDA kernels, which use explicit __f*_rn intrinsics for
// the same operation sequence — DESIGN.md §4 "numerics contract").
//
// Templated on the scalar type: float = production mirror, double = the SPEC's
// 64-bit oracle mode.
#include "ts_oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// ----------------------------------------------------------------------------
// worker pool: contiguous static chunks (deterministic outputs)
// ----------------------------------------------------------------------------
int g_workers = 0;
int workers() {
    if (g_workers > 0) return g_workers;
    const char* e = std::getenv("TS_WORKERS");
    if (e && std::atoi(e) > 0) return std::atoi(e);
    unsigned h = std::thread::hardware_concurrency();
    return h ? int(h) : 1;
}

template <class F>
void pfor(int64_t n, F&& f) {  // f(begin, end)
    int nw = workers();
    if (nw <= 1 || n < 2048) {
        if (n > 0) f(int64_t(0), n);
        return;
    }
    if (int64_t(nw) > n / 1024) nw = int(std::max<int64_t>(1, n / 1024));
    std::vector<std::thread> th;
    int64_t chunk = (n + nw - 1) / nw;
    for (int w = 0; w < nw; ++w) {
        int64_t b = w * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        th.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& t : th) t.join();
}

// dynamic scheduling for uneven work items (tiles); per-item outputs are disjoint
template <class F>
void pfor_dyn(int64_t n, F&& f) {  // f(item)
    int nw = workers();
    if (nw <= 1 || n < 4) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> th;
    for (int w = 0; w < nw; ++w)
        th.emplace_back([&] {
            for (;;) {
                int64_t i = next.fetch_add(1);
                if (i >= n) break;
                f(i);
            }
        });
    for (auto& t : th) t.join();
}

inline float f_from_bits(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
inline uint32_t bits_of(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

// ----------------------------------------------------------------------------
// Deterministic exp/log (numerics contract).  Only IEEE +,-,*,/
// and bit operations, evaluated strictly in the written order, so the CUDA
// restatement (csrc/ts_math.cuh) produces the same bits.  Cody-Waite reduction +
// degree-6 polynomial (Cephes expf coefficients); log per the fdlibm/musl logf
// reduction.  Accuracy ~1-2 ulp; only reproducibility matters for binning.
// ----------------------------------------------------------------------------
float soft_expf(float x) {
    if (x != x) return x;
    if (x > 88.72283935546875f) return INFINITY;
    if (x < -103.972084045410156f) return 0.0f;
    const float magic = 12582912.0f;  // 1.5 * 2^23
    const float t = std::fma(x, 0x1.715476p+0f, magic);
    const float n = t - magic;
    float r = std::fma(n, -0x1.63p-1f, x);
    r = std::fma(n, 0x1.bd0106p-13f, r);
    float p = 0x1.a0d2cep-13f;
    p = std::fma(p, r, 0x1.6e879cp-10f);
    p = std::fma(p, r, 0x1.111210p-7f);
    p = std::fma(p, r, 0x1.555382p-5f);
    p = std::fma(p, r, 0x1.555554p-3f);
    p = std::fma(p, r, 0x1.0p-1f);
    p = std::fma(p, r * r, r);
    p = p + 1.0f;
    int ni = int(n);
    if (ni > 127) {
        p = p * f_from_bits(0x7f000000u);
        ni -= 127;
    }
    if (ni < -126) {
        p = p * f_from_bits(0x00800000u);
        ni += 126;
    }
    return p * f_from_bits(uint32_t(ni + 127) << 23);
}

float soft_logf(float x) {
    uint32_t ix = bits_of(x);
    int k = 0;
    if (ix < 0x00800000u || (ix >> 31)) {
        if ((ix << 1) == 0) return -INFINITY;
        if (ix >> 31) return NAN;
        k -= 25;
        x = x * 33554432.0f;
        ix = bits_of(x);
    } else if (ix >= 0x7f800000u) {
        return x;
    } else if (ix == 0x3f800000u) {
        return 0.0f;
    }
    ix += 0x3f800000u - 0x3f3504f3u;
    k += int(ix >> 23) - 0x7f;
    ix = (ix & 0x007fffffu) + 0x3f3504f3u;
    x = f_from_bits(ix);
    const float f = x - 1.0f;
    const float s = f / (2.0f + f);
    const float z = s * s;
    const float w = z * z;
    const float t1 = w * std::fma(w, 0x1.f13c4cp-3f, 0x1.999c26p-2f);
    const float t2 = z * std::fma(w, 0x1.23d3dcp-2f, 0x1.555554p-1f);
    const float R = t2 + t1;
    const float hfsq = 0.5f * f * f;
    const float dk = float(k);
    float acc = std::fma(dk, 0x1.2fefa2p-17f, s * (hfsq + R));
    acc = acc - hfsq;
    acc = acc + f;
    return std::fma(dk, 0x1.62e3p-1f, acc);
}

// scalar-type traits: float uses the deterministic soft exp/log on the binning path
template <class T>
struct M;
template <>
struct M<float> {
    static float exp_(float x) { return soft_expf(x); }
    static float log_(float x) { return soft_logf(x); }
    static float exp_blend(float x) { return std::exp(x); }
};
template <>
struct M<double> {
    static double exp_(double x) { return std::exp(x); }
    static double log_(double x) { return std::log(x); }
    static double exp_blend(double x) { return std::exp(x); }
};

constexpr int TILE = 16;
constexpr int NPARAM = 59;
std::vector<float> g_nu;  // sampling rates for aa_mode 1 (tso_set_sampling_rates)
struct Off {
    int64_t means, ls, q, op, dc, rest;
    explicit Off(int64_t n) : means(0), ls(3 * n), q(6 * n), op(10 * n), dc(11 * n), rest(14 * n) {}
};

// 3DGS real SH basis constants
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
constexpr double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                             0.5462742152960396};
constexpr double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                             -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

// SH basis values Y[16] at unit dir (SPEC.md:79-87 eval_sh)
template <class T>
void sh_basis(T x, T y, T z, int deg, T* Y) {
    Y[0] = T(SH_C0);
    if (deg < 1) return;
    Y[1] = -T(SH_C1) * y;
    Y[2] = T(SH_C1) * z;
    Y[3] = -T(SH_C1) * x;
    if (deg < 2) return;
    T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = T(SH_C2[0]) * xy;
    Y[5] = T(SH_C2[1]) * yz;
    Y[6] = T(SH_C2[2]) * (T(2) * zz - xx - yy);
    Y[7] = T(SH_C2[3]) * xz;
    Y[8] = T(SH_C2[4]) * (xx - yy);
    if (deg < 3) return;
    Y[9] = T(SH_C3[0]) * y * (T(3) * xx - yy);
    Y[10] = T(SH_C3[1]) * xy * z;
    Y[11] = T(SH_C3[2]) * y * (T(4) * zz - xx - yy);
    Y[12] = T(SH_C3[3]) * z * (T(2) * zz - T(3) * xx - T(3) * yy);
    Y[13] = T(SH_C3[4]) * x * (T(4) * zz - xx - yy);
    Y[14] = T(SH_C3[5]) * z * (xx - yy);
    Y[15] = T(SH_C3[6]) * x * (xx - T(3) * yy);
}

// d Y_k / d(x,y,z) for k < (deg+1)^2
template <class T>
void sh_basis_grad(T x, T y, T z, int deg, T (*dY)[3]) {
    for (int k = 0; k < 16; ++k) dY[k][0] = dY[k][1] = dY[k][2] = T(0);
    if (deg < 1) return;
    dY[1][1] = -T(SH_C1);
    dY[2][2] = T(SH_C1);
    dY[3][0] = -T(SH_C1);
    if (deg < 2) return;
    T xx = x * x, yy = y * y, zz = z * z;
    dY[4][0] = T(SH_C2[0]) * y;
    dY[4][1] = T(SH_C2[0]) * x;
    dY[5][1] = T(SH_C2[1]) * z;
    dY[5][2] = T(SH_C2[1]) * y;
    dY[6][0] = T(-2) * T(SH_C2[2]) * x;
    dY[6][1] = T(-2) * T(SH_C2[2]) * y;
    dY[6][2] = T(4) * T(SH_C2[2]) * z;
    dY[7][0] = T(SH_C2[3]) * z;
    dY[7][2] = T(SH_C2[3]) * x;
    dY[8][0] = T(2) * T(SH_C2[4]) * x;
    dY[8][1] = T(-2) * T(SH_C2[4]) * y;
    if (deg < 3) return;
    dY[9][0] = T(SH_C3[0]) * T(6) * x * y;
    dY[9][1] = T(SH_C3[0]) * (T(3) * xx - T(3) * yy);
    dY[10][0] = T(SH_C3[1]) * y * z;
    dY[10][1] = T(SH_C3[1]) * x * z;
    dY[10][2] = T(SH_C3[1]) * x * y;
    dY[11][0] = T(-2) * T(SH_C3[2]) * x * y;
    dY[11][1] = T(SH_C3[2]) * (T(4) * zz - xx - T(3) * yy);
    dY[11][2] = T(8) * T(SH_C3[2]) * y * z;
    dY[12][0] = T(-6) * T(SH_C3[3]) * x * z;
    dY[12][1] = T(-6) * T(SH_C3[3]) * y * z;
    dY[12][2] = T(SH_C3[3]) * (T(6) * zz - T(3) * xx - T(3) * yy);
    dY[13][0] = T(SH_C3[4]) * (T(4) * zz - T(3) * xx - yy);
    dY[13][1] = T(-2) * T(SH_C3[4]) * x * y;
    dY[13][2] = T(8) * T(SH_C3[4]) * x * z;
    dY[14][0] = T(2) * T(SH_C3[5]) * x * z;
    dY[14][1] = T(-2) * T(SH_C3[5]) * y * z;
    dY[14][2] = T(SH_C3[5]) * (xx - yy);
    dY[15][0] = T(SH_C3[6]) * (T(3) * xx - T(3) * yy);
    dY[15][1] = T(-6) * T(SH_C3[6]) * x * y;
}

// camera in scalar T (values are the float camera fields, widened exactly)
template <class T>
struct Cam {
    T W[16];
    T fx, fy, cx, cy, nearp;
    int w, h;
    T limx, limy;      // 1.3 * tan(fov/2), SURVEY App. A.11
    T pos[3];          // camera centre = -R^T t
    int tiles_x, tiles_y;
    explicit Cam(const tso_camera& c) {
        for (int i = 0; i < 16; ++i) W[i] = T(c.W[i]);
        fx = T(c.fx);
        fy = T(c.fy);
        cx = T(c.cx);
        cy = T(c.cy);
        nearp = T(c.near_plane);
        w = c.width;
        h = c.height;
        limx = T(1.3f) * ((T(0.5f) * T(w)) / fx);
        limy = T(1.3f) * ((T(0.5f) * T(h)) / fy);
        pos[0] = -((W[0] * W[3] + W[4] * W[7]) + W[8] * W[11]);
        pos[1] = -((W[1] * W[3] + W[5] * W[7]) + W[9] * W[11]);
        pos[2] = -((W[2] * W[3] + W[6] * W[7]) + W[10] * W[11]);
        tiles_x = (w + TILE - 1) / TILE;
        tiles_y = (h + TILE - 1) / TILE;
    }
};

// All per-Gaussian forward quantities (recomputed identically by the backward).
template <class T>
struct GFwd {
    bool ok = false;           // passed frustum + degeneracy gating
    T xh, yh, zh;              // camera point
    T qn, qw, qx, qy, qz;      // norm and normalized quaternion
    T s[3];                    // activated scales
    T R[9];                    // rotation (row-major)
    T Mm[9];                   // R * diag(s)
    T S[6];                    // cov3d upper triangle xx,xy,xz,yy,yz,zz
    T txz, tyz;                // unclamped ratios
    bool clx, cly;             // ratio clamp active
    T ux, uy;                  // clamped ratios
    T J00, J02, J11, J12;
    T Tm[6];                   // J * W3 (2x3)
    T a, b, c, det;            // dilated cov2d and its determinant
    T A, B, C;                 // conic
    T mx, my;                  // mean2d
    T o;                       // effective opacity (after the AA compensation factor)
    T o_raw;                   // sigmoid(logit)
    T ofac;                    // o = o_raw * ofac (3D filter ratio or Mip compensation; 1 when AA off)
    T s_raw[3], s_h[3];        // aa_mode 1: activated scales before the 3D filter, s^2 + kappa/nu^2
    T aaf;                     // aa_mode 1: kappa / nu^2
    T k2;                      // alpha level set: Q <= k2  <=>  o*exp(-Q/2) >= tau
    bool has_bound;            // o > tau
    T dir[3], dlen;            // unit view direction, |mu - campos|
    T raw[3];                  // SH sum + 0.5 before clamp
    T rgb[3];
};

// SPEC core + camera: activate_* :39-57, rotation_from_quaternion :59-67,
// build_covariance3d :69-77, project_mean :132-140, project_covariance :142-150,
// invert_cov2d :152-160, eval_sh :79-87, bound k :214-222.
template <class T>
GFwd<T> gaussian_forward(const T* P, int64_t N, int64_t g, const Cam<T>& cam, const tso_render_config& cfg) {
    Off off(N);
    GFwd<T> F;
    const T* mu = P + off.means + 3 * g;
    const T* ls = P + off.ls + 3 * g;
    const T* q = P + off.q + 4 * g;
    const T* W = cam.W;
    // project_mean (fixed order, no contraction)
    // project_mean: FMA chains, one rounding per step (the kernels' fma_ order)
    F.xh = std::fma(W[2], mu[2], std::fma(W[1], mu[1], W[0] * mu[0])) + W[3];
    F.yh = std::fma(W[6], mu[2], std::fma(W[5], mu[1], W[4] * mu[0])) + W[7];
    F.zh = std::fma(W[10], mu[2], std::fma(W[9], mu[1], W[8] * mu[0])) + W[11];
    if (!(F.zh > cam.nearp)) return F;
    // rotation_from_quaternion (degenerate if ||q|| < 1e-4)
    T qq = std::fma(q[3], q[3], std::fma(q[2], q[2], std::fma(q[1], q[1], q[0] * q[0])));
    F.qn = std::sqrt(qq);
    if (!(F.qn >= T(1e-4f))) return F;
    const T rq = T(1) / F.qn;
    F.qw = q[0] * rq;
    F.qx = q[1] * rq;
    F.qy = q[2] * rq;
    F.qz = q[3] * rq;
    {
        T w = F.qw, x = F.qx, y = F.qy, z = F.qz;
        T xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z, wx = w * x, wy = w * y,
          wz = w * z;
        F.R[0] = T(1) - T(2) * (yy + zz);
        F.R[1] = T(2) * (xy - wz);
        F.R[2] = T(2) * (xz + wy);
        F.R[3] = T(2) * (xy + wz);
        F.R[4] = T(1) - T(2) * (xx + zz);
        F.R[5] = T(2) * (yz - wx);
        F.R[6] = T(2) * (xz - wy);
        F.R[7] = T(2) * (yz + wx);
        F.R[8] = T(1) - T(2) * (xx + yy);
    }
    // activate_scales, build_covariance3d: Sigma = (R S)(R S)^T
    for (int k = 0; k < 3; ++k) F.s[k] = M<T>::exp_(ls[k]);
    F.ofac = T(1);
    if (cfg.aa_mode == 1) {
        // apply_3d_filter_original: s_hat = sqrt(s^2 + kappa/nu^2),
        // opacity factor sqrt(prod s^2 / prod s_hat^2)
        const T nu = T(g_nu.empty() ? 1.0f : g_nu[size_t(g)]);
        F.aaf = T(cfg.kappa3d) / (nu * nu);
        T q[3];
        for (int k = 0; k < 3; ++k) {
            F.s_raw[k] = F.s[k];
            q[k] = F.s[k] * F.s[k];
            F.s_h[k] = q[k] + F.aaf;
            F.s[k] = std::sqrt(F.s_h[k]);
        }
        F.ofac = std::sqrt(((q[0] * q[1]) * q[2]) / ((F.s_h[0] * F.s_h[1]) * F.s_h[2]));
    }
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) F.Mm[3 * i + k] = F.R[3 * i + k] * F.s[k];
    const T* Mm = F.Mm;
    auto sdot = [&](int i, int j) {
        return std::fma(Mm[3 * i + 2], Mm[3 * j + 2], std::fma(Mm[3 * i + 1], Mm[3 * j + 1], Mm[3 * i] * Mm[3 * j]));
    };
    F.S[0] = sdot(0, 0);
    F.S[1] = sdot(0, 1);
    F.S[2] = sdot(0, 2);
    F.S[3] = sdot(1, 1);
    F.S[4] = sdot(1, 2);
    F.S[5] = sdot(2, 2);
    // project_covariance with clamped ratios
    const T rz = T(1) / F.zh;
    F.txz = F.xh * rz;
    F.tyz = F.yh * rz;
    F.clx = (F.txz < -cam.limx) || (F.txz > cam.limx);
    F.cly = (F.tyz < -cam.limy) || (F.tyz > cam.limy);
    F.ux = F.txz < -cam.limx ? -cam.limx : (F.txz > cam.limx ? cam.limx : F.txz);
    F.uy = F.tyz < -cam.limy ? -cam.limy : (F.tyz > cam.limy ? cam.limy : F.tyz);
    // J = [[fx/z, 0, -fx u_x / z], [0, fy/z, -fy u_y / z]] (u = clamped x/z, y/z)
    F.J00 = cam.fx * rz;
    F.J02 = (-(cam.fx * F.ux)) * rz;
    F.J11 = cam.fy * rz;
    F.J12 = (-(cam.fy * F.uy)) * rz;
    for (int j = 0; j < 3; ++j) {
        F.Tm[j] = std::fma(F.J02, W[8 + j], F.J00 * W[j]);
        F.Tm[3 + j] = std::fma(F.J12, W[8 + j], F.J11 * W[4 + j]);
    }
    T Sf[9] = {F.S[0], F.S[1], F.S[2], F.S[1], F.S[3], F.S[4], F.S[2], F.S[4], F.S[5]};
    T U[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            U[3 * i + j] = std::fma(F.Tm[3 * i + 2], Sf[6 + j], std::fma(F.Tm[3 * i + 1], Sf[3 + j], F.Tm[3 * i] * Sf[j]));
    T a = std::fma(U[2], F.Tm[2], std::fma(U[1], F.Tm[1], U[0] * F.Tm[0]));
    T b = std::fma(U[2], F.Tm[5], std::fma(U[1], F.Tm[4], U[0] * F.Tm[3]));
    T c = std::fma(U[5], F.Tm[5], std::fma(U[4], F.Tm[4], U[3] * F.Tm[3]));
    // invert_cov2d with dilation; degenerate if det < 1e-6
    const T det_pre = std::fma(a, c, -(b * b));
    T dil = T(cfg.dilation);
    a = a + dil;
    c = c + dil;
    T det = std::fma(a, c, -(b * b));
    if (!(det >= T(1e-6f))) return F;
    F.a = a;
    F.b = b;
    F.c = c;
    F.det = det;
    const T rdet = T(1) / det;
    F.A = c * rdet;
    F.B = (-b) * rdet;
    F.C = a * rdet;
    F.mx = std::fma(cam.fx, F.txz, cam.cx);
    F.my = std::fma(cam.fy, F.tyz, cam.cy);
    // activate_opacity; AA compensation (SPEC.md:646-654 mip: sqrt(det_pre / det_post), detached)
    T logit = P[off.op + g];
    F.o_raw = T(1) / (T(1) + M<T>::exp_(-logit));
    if (cfg.aa_mode == 3) F.ofac = det_pre > T(0) ? std::sqrt(det_pre / det) : T(0);
    F.o = (cfg.aa_mode == 1 || cfg.aa_mode == 3) ? F.o_raw * F.ofac : F.o_raw;
    T tau = T(cfg.tau_alpha);
    if (cfg.truncation == 1) {
        // fragment_alpha response mode: keep iff G >= exp(-sigma_cut^2 / 2), i.e. the
        // Mahalanobis distance Q <= sigma_cut^2, whatever the opacity
        F.has_bound = F.o > T(0);
        F.k2 = F.has_bound ? T(cfg.sigma_cut) * T(cfg.sigma_cut) : T(0);
    } else {
        F.has_bound = F.o > tau;
        F.k2 = F.has_bound ? T(-2) * M<T>::log_(tau / F.o) : T(0);
    }
    // eval_sh (view dir = mu - campos)
    T d0 = mu[0] - cam.pos[0], d1 = mu[1] - cam.pos[1], d2 = mu[2] - cam.pos[2];
    F.dlen = std::sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    F.dir[0] = d0 / F.dlen;
    F.dir[1] = d1 / F.dlen;
    F.dir[2] = d2 / F.dlen;
    int deg = cfg.sh_degree;
    T Y[16];
    sh_basis(F.dir[0], F.dir[1], F.dir[2], deg, Y);
    int nb = (deg + 1) * (deg + 1);
    const T* dc = P + off.dc + 3 * g;
    const T* rest = P + off.rest + 45 * g;
    for (int ch = 0; ch < 3; ++ch) {
        T acc = Y[0] * dc[ch];
        for (int k = 1; k < nb; ++k) acc = acc + Y[k] * rest[3 * (k - 1) + ch];
        F.raw[ch] = acc + T(0.5);
        F.rgb[ch] = F.raw[ch] < T(0) ? T(0) : F.raw[ch];
    }
    F.ok = true;
    return F;
}

// Conic quadratic form, fixed evaluation order shared with the kernels
// (ts_math.cuh tsx::conic_q; two correctly rounded products, two fused multiply-adds):
//   Q = fma(dy, fma(C, dy, (2B)*dx), (A*dx)*dx)
template <class T>
inline T conic_q(T A, T B2, T C, T dx, T dy) {
    return std::fma(dy, std::fma(C, dy, B2 * dx), (A * dx) * dx);
}

struct Rect {
    int tx0, ty0, tx1, ty1;  // inclusive; empty when tx0 > tx1
};

// bound_square / bound_rect -> inclusive tile rect.
// AABB->tile rule: pixel (i,j) samples at (i,j); the AABB
// covers the integer samples in [lo, hi] clipped to the image; tiles are the
// 16x16 blocks containing any of them.
template <class T>
Rect bound_tiles(const GFwd<T>& F, const Cam<T>& cam, const tso_render_config& cfg, T k2_plain) {
    Rect r{1, 1, 0, 0};
    if (!F.ok || !F.has_bound) return r;
    T rx, ry;
    if (cfg.bound_mode == 0) {
        T mid = T(0.5f) * (F.a + F.c);
        T disc = mid * mid - F.det;
        T lam = mid + std::sqrt(disc > T(0) ? disc : T(0));
        rx = ry = T(3) * std::sqrt(lam);
    } else {
        T k = std::sqrt(cfg.bound_mode == 1 ? k2_plain : F.k2);
        rx = k * std::sqrt(F.a);
        ry = k * std::sqrt(F.c);
    }
    T wm1 = T(cam.w - 1), hm1 = T(cam.h - 1);
    T lox = F.mx - rx, hix = F.mx + rx, loy = F.my - ry, hiy = F.my + ry;
    lox = lox < T(0) ? T(0) : lox;
    hix = hix > wm1 ? wm1 : hix;
    loy = loy < T(0) ? T(0) : loy;
    hiy = hiy > hm1 ? hm1 : hiy;
    if (!(lox <= hix) || !(loy <= hiy)) return r;
    int px0 = int(std::ceil(lox)), px1 = int(std::floor(hix));
    int py0 = int(std::ceil(loy)), py1 = int(std::floor(hiy));
    if (px0 > px1 || py0 > py1) return r;
    r.tx0 = px0 >> 4;
    r.tx1 = px1 >> 4;
    r.ty0 = py0 >> 4;
    r.ty1 = py1 >> 4;
    return r;
}

// tile_cull_exact: max of the Gaussian over the tile's
// sample rectangle; keep iff Q(p*) <= k2 (inclusive).  With the
// centre outside the rectangle the minimum of the convex Q lies on an edge
// facing the centre (at most one vertical + one horizontal edge); on an edge
// the 1D optimum t* = -(B/C) dx (resp. -(B/A) dy) is clamped to the edge.
template <class T>
bool tile_keep(T mx, T my, T A, T B, T C, T k2, int tx, int ty, const Cam<T>& cam) {
    T x0 = T(tx * TILE), y0 = T(ty * TILE);
    T x1 = T(std::min(tx * TILE + TILE - 1, cam.w - 1));
    T y1 = T(std::min(ty * TILE + TILE - 1, cam.h - 1));
    const bool inx = mx >= x0 && mx <= x1, iny = my >= y0 && my <= y1;
    if (inx && iny) return true;
    T nBA = (-B) / A, nBC = (-B) / C;
    T B2 = B + B;
    T best = T(INFINITY);
    if (!inx) {
        T dx = (mx < x0 ? x0 : x1) - mx;
        T lo = y0 - my, hi = y1 - my;
        T dy = nBC * dx;
        dy = dy < lo ? lo : (dy > hi ? hi : dy);
        T qv = conic_q(A, B2, C, dx, dy);
        best = qv < best ? qv : best;
    }
    if (!iny) {
        T dy = (my < y0 ? y0 : y1) - my;
        T lo = x0 - mx, hi = x1 - mx;
        T dx = nBA * dy;
        dx = dx < lo ? lo : (dx > hi ? hi : dx);
        T qv = conic_q(A, B2, C, dx, dy);
        best = qv < best ? qv : best;
    }
    return best <= k2;
}

template <class T>
T plain_k2(const tso_render_config& cfg) {
    if (cfg.truncation == 1) return T(cfg.sigma_cut) * T(cfg.sigma_cut);  // response mode: one cutoff for all
    return T(-2) * M<T>::log_(T(cfg.tau_alpha));
}

// ----------------------------------------------------------------------------
// Per-view pipeline state (render intermediates retained for backward)
// ----------------------------------------------------------------------------
template <class T>
struct View {
    int64_t N = 0;
    std::vector<GFwd<T>> F;
    std::vector<Rect> rect;
    std::vector<uint32_t> cnt, dkey;
    std::vector<uint64_t> keys;
    std::vector<uint32_t> vals;
    std::vector<uint32_t> ranges;  // 2*Tn
    int64_t I = 0;
};

template <class T>
uint32_t depth_key_of(T z) {
    float zf = float(z);
    return bits_of(zf) ^ 0x80000000u;
}

template <class T>
void preprocess_all(View<T>& V, const T* P, int64_t N, const Cam<T>& cam, const tso_render_config& cfg) {
    V.N = N;
    V.F.resize(N);
    V.rect.resize(N);
    V.cnt.assign(N, 0);
    V.dkey.assign(N, 0xFFFFFFFFu);
    T k2p = plain_k2<T>(cfg);
    pfor(N, [&](int64_t b, int64_t e) {
        for (int64_t g = b; g < e; ++g) {
            GFwd<T> F = gaussian_forward(P, N, g, cam, cfg);
            Rect r = bound_tiles(F, cam, cfg, k2p);
            uint32_t c = 0;
            for (int ty = r.ty0; ty <= r.ty1; ++ty)
                for (int tx = r.tx0; tx <= r.tx1; ++tx)
                    if (cfg.cull_mode == 0 || tile_keep(F.mx, F.my, F.A, F.B, F.C, F.k2, tx, ty, cam)) ++c;
            V.F[g] = F;
            V.rect[g] = r;
            V.cnt[g] = c;
            V.dkey[g] = c ? depth_key_of(F.zh) : 0xFFFFFFFFu;
        }
    });
}

// build_instances: Gaussian-major, row-major tiles within a Gaussian
template <class T>
void build_instances(View<T>& V, const Cam<T>& cam, const tso_render_config& cfg) {
    int64_t N = V.N;
    std::vector<int64_t> offs(N + 1, 0);
    for (int64_t g = 0; g < N; ++g) offs[g + 1] = offs[g] + V.cnt[g];
    V.I = offs[N];
    V.keys.resize(V.I);
    V.vals.resize(V.I);
    pfor(N, [&](int64_t b, int64_t e) {
        for (int64_t g = b; g < e; ++g) {
            if (!V.cnt[g]) continue;
            const GFwd<T>& F = V.F[g];
            const Rect& r = V.rect[g];
            int64_t o = offs[g];
            for (int ty = r.ty0; ty <= r.ty1; ++ty)
                for (int tx = r.tx0; tx <= r.tx1; ++tx)
                    if (cfg.cull_mode == 0 || tile_keep(F.mx, F.my, F.A, F.B, F.C, F.k2, tx, ty, cam)) {
                        uint64_t tile = uint64_t(ty) * cam.tiles_x + tx;
                        V.keys[o] = (tile << 32) | V.dkey[g];
                        V.vals[o] = uint32_t(g);
                        ++o;
                    }
        }
    });
}

// LSD radix, 8-bit digits, stable; sorts (key32, val) by key32
void lsd_radix_u32(std::vector<uint32_t>& k, std::vector<uint32_t>& v, int bits) {
    size_t n = k.size();
    std::vector<uint32_t> k2(n), v2(n);
    for (int sh = 0; sh < bits; sh += 8) {
        size_t cnt[257] = {0};
        for (size_t i = 0; i < n; ++i) cnt[((k[i] >> sh) & 255u) + 1]++;
        for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
        for (size_t i = 0; i < n; ++i) {
            size_t p = cnt[(k[i] >> sh) & 255u]++;
            k2[p] = k[i];
            v2[p] = v[i];
        }
        k.swap(k2);
        v.swap(v2);
    }
}

int64_t sort_two_stage(int64_t I, int tile_bits, uint64_t* keys, uint32_t* vals) {
    // stage 1: stable by depth (32-bit), carrying the instance position
    std::vector<uint32_t> dk(I), pos(I);
    for (int64_t i = 0; i < I; ++i) {
        dk[i] = uint32_t(keys[i] & 0xFFFFFFFFu);
        pos[i] = uint32_t(i);
    }
    lsd_radix_u32(dk, pos, 32);
    // stage 2: stable by tile
    std::vector<uint32_t> tk(I);
    for (int64_t i = 0; i < I; ++i) tk[i] = uint32_t(keys[pos[i]] >> 32);
    int tb = ((tile_bits + 7) / 8) * 8;
    lsd_radix_u32(tk, pos, tb);
    std::vector<uint64_t> nk(I);
    std::vector<uint32_t> nv(I);
    for (int64_t i = 0; i < I; ++i) {
        nk[i] = keys[pos[i]];
        nv[i] = vals[pos[i]];
    }
    std::memcpy(keys, nk.data(), I * 8);
    std::memcpy(vals, nv.data(), I * 4);
    // key bytes touched per SPEC.md:283 accounting: 4 B depth x 4 passes + tile bytes x passes
    // (16-bit tile keys up to 2^16 tiles, 32-bit keys above: SPEC.md:193)
    if (tb > 16) return I * 4 * 4 + I * 4 * (tb / 8);
    return I * 4 * 4 + I * (tb / 8) * (tb / 8);
}

void tile_ranges(int64_t I, const uint64_t* k, int32_t Tn, uint32_t* ranges) {
    // half-open; empty tiles get (lb, lb) where lb = #instances with tile < t (App. A.5)
    int64_t i = 0;
    for (int32_t t = 0; t < Tn; ++t) {
        int64_t b = i;
        while (i < I && int64_t(k[i] >> 32) == t) ++i;
        ranges[2 * t] = uint32_t(b);
        ranges[2 * t + 1] = uint32_t(i);
    }
}

// stable depth sort then stable tile sort (LSD, 8-bit digits);
// equal to the combined stable 64-bit sort (checked in tests against
// tso_sort_combined / std::stable_sort).
template <class T>
void sort_and_range(View<T>& V, const Cam<T>& cam) {
    int Tn = cam.tiles_x * cam.tiles_y;
    int tb = 1;
    while ((1 << tb) < Tn) ++tb;
    sort_two_stage(V.I, tb, V.keys.data(), V.vals.data());
    V.ranges.assign(2 * Tn, 0);
    tile_ranges(V.I, V.keys.data(), Tn, V.ranges.data());
}

// ----------------------------------------------------------------------------
// raster_forward: blend_tile, fragment_alpha (:316-324)
// ----------------------------------------------------------------------------
template <class T>
struct Frame {
    std::vector<T> rgb, Tf;
    std::vector<uint32_t> count;
};

template <class T>
void blend_all(const View<T>& V, const Cam<T>& cam, const tso_render_config& cfg, Frame<T>& fb,
               std::vector<double>* wsum = nullptr) {
    int Wd = cam.w, Hd = cam.h;
    fb.rgb.assign(size_t(Wd) * Hd * 3, T(0));
    fb.Tf.assign(size_t(Wd) * Hd, T(1));
    fb.count.assign(size_t(Wd) * Hd, 0);
    if (wsum) wsum->assign(size_t(Wd) * Hd, 0.0);
    int Tn = cam.tiles_x * cam.tiles_y;
    pfor_dyn(Tn, [&](int64_t t) {
        int tx = int(t % cam.tiles_x), ty = int(t / cam.tiles_x);
        uint32_t b = V.ranges[2 * t], e = V.ranges[2 * t + 1];
        for (int py = ty * TILE; py < std::min(Hd, ty * TILE + TILE); ++py)
            for (int px = tx * TILE; px < std::min(Wd, tx * TILE + TILE); ++px) {
                T Tt = T(1), C[3] = {T(0), T(0), T(0)};
                uint32_t last = 0;
                double ws = 0.0;
                for (uint32_t i = b; i < e; ++i) {
                    const GFwd<T>& F = V.F[V.vals[i]];
                    T dx = T(px) - F.mx, dy = T(py) - F.my;
                    T Q = conic_q(F.A, F.B + F.B, F.C, dx, dy);
                    if (!(Q <= F.k2)) continue;  // classic: o*G < tau; response: G < exp(-sigma_cut^2 / 2)
                    T G = M<T>::exp_blend(T(-0.5) * Q);
                    T al = F.o * G;
                    al = al > T(0.99) ? T(0.99) : al;
                    if (cfg.early_stop_compat) {
                        T test = Tt * (T(1) - al);
                        if (test < T(1e-4)) break;
                    }
                    T w = al * Tt;
                    for (int ch = 0; ch < 3; ++ch) C[ch] = C[ch] + w * F.rgb[ch];
                    ws += double(w);
                    Tt = Tt * (T(1) - al);
                    last = i - b + 1;
                    if (!cfg.early_stop_compat && Tt < T(1e-4)) break;  // blend, then stop
                }
                size_t p = size_t(py) * Wd + px;
                for (int ch = 0; ch < 3; ++ch) fb.rgb[3 * p + ch] = C[ch] + Tt * T(cfg.bg[ch]);
                fb.Tf[p] = Tt;
                fb.count[p] = last;
                if (wsum) (*wsum)[p] = ws + double(Tt);
            }
    });
}

template <class T>
bool valid_cam(const tso_camera* c) {
    if (!c || c->width <= 0 || c->height <= 0) return false;
    // TileGrid: 16-bit tile keys below 2^16 tiles, 32-bit keys above
    // (selected automatically: the combined key is tile << 32 | depth either way)
    int64_t tn = int64_t((c->width + 15) / 16) * ((c->height + 15) / 16);
    return tn < (int64_t(1) << 24);
}

template <class T>
int64_t render_impl(int64_t n, const T* P, const tso_camera* c, const tso_render_config* cfg, T* rgb, T* Tout,
                    uint32_t* cnt, std::vector<double>* wsum = nullptr) {
    if (!valid_cam<T>(c) || !cfg) return -1;
    Cam<T> cam(*c);
    View<T> V;
    preprocess_all(V, P, n, cam, *cfg);
    build_instances(V, cam, *cfg);
    sort_and_range(V, cam);
    Frame<T> fb;
    blend_all(V, cam, *cfg, fb, wsum);
    size_t np = size_t(cam.w) * cam.h;
    if (rgb) std::memcpy(rgb, fb.rgb.data(), np * 3 * sizeof(T));
    if (Tout) std::memcpy(Tout, fb.Tf.data(), np * sizeof(T));
    if (cnt) std::memcpy(cnt, fb.count.data(), np * 4);
    return V.I;
}

// ----------------------------------------------------------------------------
// loss_metrics: training_loss 0.8 L1 + 0.2 (1 - SSIM),
// 11x11 Gaussian window sigma 1.5, C1 = 0.01^2, C2 = 0.03^2, reflect padding.
// ----------------------------------------------------------------------------
inline int reflect_idx(int i, int n) {
    if (i < 0) return -i;
    if (i >= n) return 2 * (n - 1) - i;
    return i;
}

void gauss_window(double* g) {
    double s = 0;
    for (int i = 0; i < 11; ++i) {
        double d = i - 5;
        g[i] = std::exp(-(d * d) / (2.0 * 1.5 * 1.5));
        s += g[i];
    }
    for (int i = 0; i < 11; ++i) g[i] /= s;
}

// separable correlation with reflect padding over an H x W plane
void conv_plane(const double* in, double* out, int H, int W, const double* g) {
    std::vector<double> tmp(size_t(H) * W);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double s = 0;
            for (int o = -5; o <= 5; ++o) s += g[o + 5] * in[size_t(y) * W + reflect_idx(x + o, W)];
            tmp[size_t(y) * W + x] = s;
        }
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double s = 0;
            for (int o = -5; o <= 5; ++o) s += g[o + 5] * tmp[size_t(reflect_idx(y + o, H)) * W + x];
            out[size_t(y) * W + x] = s;
        }
}

// transpose of conv_plane (scatter form)
void conv_plane_T(const double* in, double* out, int H, int W, const double* g) {
    std::vector<double> tmp(size_t(H) * W, 0.0);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int o = -5; o <= 5; ++o)
                tmp[size_t(reflect_idx(y + o, H)) * W + x] += g[o + 5] * in[size_t(y) * W + x];
    std::fill(out, out + size_t(H) * W, 0.0);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int o = -5; o <= 5; ++o)
                out[size_t(y) * W + reflect_idx(x + o, W)] += g[o + 5] * tmp[size_t(y) * W + x];
}

template <class T>
double loss_impl(int H, int W, const T* X, const T* Yt, T* dX) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    size_t np = size_t(H) * W;
    double Mtot = double(np) * 3.0;
    double g[11];
    gauss_window(g);
    double l1 = 0.0, ssim_sum = 0.0;
    std::vector<std::vector<double>> grad(3, std::vector<double>(np));
    double ssim_ch[3] = {0.0, 0.0, 0.0};
    pfor_dyn(3, [&](int64_t ch) {
        std::vector<double> x(np), y(np), xx(np), yy(np), xy(np), mx(np), my(np), sxx(np), syy(np), sxy(np);
        for (size_t p = 0; p < np; ++p) {
            x[p] = double(X[3 * p + ch]);
            y[p] = double(Yt[3 * p + ch]);
            xx[p] = x[p] * x[p];
            yy[p] = y[p] * y[p];
            xy[p] = x[p] * y[p];
        }
        conv_plane(x.data(), mx.data(), H, W, g);
        conv_plane(y.data(), my.data(), H, W, g);
        conv_plane(xx.data(), sxx.data(), H, W, g);
        conv_plane(yy.data(), syy.data(), H, W, g);
        conv_plane(xy.data(), sxy.data(), H, W, g);
        std::vector<double> fa(np), fb(np), fc(np);
        for (size_t p = 0; p < np; ++p) {
            double ux = mx[p], uy = my[p];
            double vx = sxx[p] - ux * ux, vy = syy[p] - uy * uy, cxy = sxy[p] - ux * uy;
            double n1 = 2 * ux * uy + C1, n2 = 2 * cxy + C2;
            double d1 = ux * ux + uy * uy + C1, d2 = vx + vy + C2;
            double D = d1 * d2, S = n1 * n2 / D;
            ssim_ch[ch] += S;
            double dS_dux = (2 * uy * n2 - S * 2 * ux * d2) / D;
            double dS_dvx = -S / d2;
            double dS_dcxy = 2 * n1 / D;
            fa[p] = dS_dux - 2 * ux * dS_dvx - uy * dS_dcxy;
            fb[p] = 2 * dS_dvx;
            fc[p] = dS_dcxy;
        }
        std::vector<double> ta(np), tb(np), tc(np);
        conv_plane_T(fa.data(), ta.data(), H, W, g);
        conv_plane_T(fb.data(), tb.data(), H, W, g);
        conv_plane_T(fc.data(), tc.data(), H, W, g);
        for (size_t p = 0; p < np; ++p) {
            double dS = ta[p] + x[p] * tb[p] + y[p] * tc[p];
            double d = x[p] - y[p];
            double sgn = d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0);
            grad[ch][p] = (0.8 * sgn - 0.2 * dS) / Mtot;
        }
    });
    // deterministic reductions (fixed channel / pixel order)
    for (int ch = 0; ch < 3; ++ch) {
        for (size_t p = 0; p < np; ++p) l1 += std::fabs(double(X[3 * p + ch]) - double(Yt[3 * p + ch]));
        ssim_sum += ssim_ch[ch];
    }
    if (dX)
        for (size_t p = 0; p < np; ++p)
            for (int ch = 0; ch < 3; ++ch) dX[3 * p + ch] = T(grad[ch][p]);
    return 0.8 * (l1 / Mtot) + 0.2 * (1.0 - ssim_sum / Mtot);
}

// ----------------------------------------------------------------------------
// raster_backward.  Per pixel, a front-to-back pass over its
// list (up to the contributor count) evaluates each kept fragment's alpha and
// transmittance T_i; a reverse pass then maintains the normalised suffix colour
//   U_i = alpha_{i+1} c_{i+1} + (1 - alpha_{i+1}) U_{i+1},   U_last = c_bg
// (colour still to come behind fragment i, per unit of T_{i+1}/(1-alpha_i)), so
//   dL/dalpha_i = T_i * sum_ch g_ch (c_i,ch - U_i,ch)
// with no division by (1 - alpha) (SPEC.md:385, :430 design decision).
// backward_mode 0 runs this per pixel over the whole list; backward_mode 1
// (per-Gaussian buckets of 32) restores T at each bucket's
// start (forward checkpoints) and U at its end (checkpoints of
// the reverse pass), then replays the bucket's 32 instances for all pixels.  Both
// run the identical per-fragment op sequence and sum each instance's pixel
// contributions in pixel order, so they agree bitwise; the merge into per-Gaussian
// gradients is tile-major then instance order.
// Per-instance 2D grads: {dmx, dmy, dA, dB, dC, do, dr, dg, db}; B is the conic
// off-diagonal entering Q as 2B.
// ----------------------------------------------------------------------------
template <class T>
struct FragRec {
    T al, G, Tt, dx, dy;
    bool clamped;
    uint32_t i;  // instance position
};

// forward quantities of one fragment at transmittance Tt; false if not kept (Q > k2)
template <class T>
inline bool frag_eval(const GFwd<T>& F, T px, T py, T Tt, FragRec<T>& r) {
    T dx = px - F.mx, dy = py - F.my;
    T Q = conic_q(F.A, F.B + F.B, F.C, dx, dy);
    if (!(Q <= F.k2)) return false;
    T G = M<T>::exp_blend(T(-0.5) * Q);
    T og = F.o * G;
    r.clamped = og > T(0.99);
    r.al = r.clamped ? T(0.99) : og;
    r.G = G;
    r.Tt = Tt;
    r.dx = dx;
    r.dy = dy;
    return true;
}

// gradient of one fragment given the normalised suffix colour U behind it; then U <- U_{i-1}
template <class T>
inline void frag_grad(const GFwd<T>& F, const FragRec<T>& r, const T* gC, T* U, T* ig) {
    T w = r.al * r.Tt;
    T s = T(0);
    for (int ch = 0; ch < 3; ++ch) {
        ig[6 + ch] += w * gC[ch];
        s += gC[ch] * (F.rgb[ch] - U[ch]);
    }
    T dal = r.Tt * s;
    if (!r.clamped) {
        ig[5] += r.G * dal;
        T dQ = T(-0.5) * r.G * F.o * dal;
        ig[0] += dQ * (T(-2) * (F.A * r.dx + F.B * r.dy));
        ig[1] += dQ * (T(-2) * (F.B * r.dx + F.C * r.dy));
        ig[2] += dQ * r.dx * r.dx;
        ig[3] += dQ * T(2) * r.dx * r.dy;
        ig[4] += dQ * r.dy * r.dy;
    }
    for (int ch = 0; ch < 3; ++ch) U[ch] = r.al * F.rgb[ch] + (T(1) - r.al) * U[ch];
}

// list positions [j0, j1) of pixel (px, py) starting at transmittance T0, with the
// normalised suffix U_end behind position j1 (recs: scratch)
template <class T>
inline void pixel_range_backward(const View<T>& V, uint32_t b, uint32_t j0, uint32_t j1, T px, T py, const T* gC,
                                 T T0, const T* U_end, T* ig, std::vector<FragRec<T>>& recs) {
    recs.clear();
    T Tt = T0;
    for (uint32_t j = j0; j < j1; ++j) {
        FragRec<T> r;
        if (frag_eval(V.F[V.vals[b + j]], px, py, Tt, r)) {
            r.i = b + j;
            recs.push_back(r);
            Tt = Tt * (T(1) - r.al);
        }
    }
    T U[3] = {U_end[0], U_end[1], U_end[2]};
    for (size_t k = recs.size(); k-- > 0;)
        frag_grad(V.F[V.vals[recs[k].i]], recs[k], gC, U, ig + size_t(recs[k].i) * 9);
}

template <class T>
void raster_backward(const View<T>& V, const Cam<T>& cam, const tso_render_config& cfg, const Frame<T>& fb,
                     const T* dLdC, std::vector<T>& g2d /* N*9 */) {
    int Wd = cam.w, Hd = cam.h;
    std::vector<T> ig(size_t(V.I) * 9, T(0));
    int Tn = cam.tiles_x * cam.tiles_y;
    const int BK = 32;
    const T bg[3] = {T(cfg.bg[0]), T(cfg.bg[1]), T(cfg.bg[2])};
    pfor_dyn(Tn, [&](int64_t t) {
        int tx = int(t % cam.tiles_x), ty = int(t / cam.tiles_x);
        uint32_t b = V.ranges[2 * t], e = V.ranges[2 * t + 1];
        if (b == e) return;
        int x0 = tx * TILE, y0 = ty * TILE;
        int x1 = std::min(Wd, x0 + TILE), y1 = std::min(Hd, y0 + TILE);
        std::vector<FragRec<T>> recs;
        if (cfg.backward_mode == 0) {
            for (int py = y0; py < y1; ++py)
                for (int px = x0; px < x1; ++px) {
                    size_t p = size_t(py) * Wd + px;
                    pixel_range_backward(V, b, 0u, fb.count[p], T(px), T(py), dLdC + 3 * p, T(1), bg, ig.data(),
                                         recs);
                }
        } else {
            // checkpoints per pixel and bucket: T at the bucket's start (forward replay) and the
            // normalised suffix U behind its end (reverse replay)
            uint32_t maxc = 0;
            for (int py = y0; py < y1; ++py)
                for (int px = x0; px < x1; ++px) maxc = std::max(maxc, fb.count[size_t(py) * Wd + px]);
            uint32_t nb = (maxc + BK - 1) / BK;
            int npx = (x1 - x0) * (y1 - y0);
            std::vector<T> ckT(size_t(nb) * npx), ckU(size_t(nb) * npx * 3);
            for (int py = y0; py < y1; ++py)
                for (int px = x0; px < x1; ++px) {
                    size_t p = size_t(py) * Wd + px;
                    int lp = (py - y0) * (x1 - x0) + (px - x0);
                    const uint32_t cnt = fb.count[p];
                    recs.clear();
                    std::vector<uint32_t> first_rec(nb + 1, 0);  // first kept fragment of each bucket
                    T Tt = T(1);
                    for (uint32_t j = 0; j < nb * BK; ++j) {
                        if (j % BK == 0) {
                            ckT[size_t(j / BK) * npx + lp] = Tt;
                            first_rec[j / BK] = uint32_t(recs.size());
                        }
                        FragRec<T> r;
                        if (j < cnt && frag_eval(V.F[V.vals[b + j]], T(px), T(py), Tt, r)) {
                            r.i = b + j;
                            recs.push_back(r);
                            Tt = Tt * (T(1) - r.al);
                        }
                    }
                    first_rec[nb] = uint32_t(recs.size());
                    T U[3] = {bg[0], bg[1], bg[2]};
                    T scratch[9];
                    for (uint32_t k = nb; k-- > 0;) {
                        for (int ch = 0; ch < 3; ++ch) ckU[(size_t(k) * npx + lp) * 3 + ch] = U[ch];
                        for (uint32_t q = first_rec[k + 1]; q-- > first_rec[k];)
                            frag_grad(V.F[V.vals[recs[q].i]], recs[q], dLdC + 3 * p, U, scratch);
                    }
                }
            for (uint32_t k = 0; k < nb; ++k)          // buckets (32, 32, ..., rest)
                for (int py = y0; py < y1; ++py)
                    for (int px = x0; px < x1; ++px) {
                        size_t p = size_t(py) * Wd + px;
                        int lp = (py - y0) * (x1 - x0) + (px - x0);
                        const uint32_t j1 = std::min<uint32_t>((k + 1) * BK, fb.count[p]);
                        if (k * BK >= j1) continue;
                        pixel_range_backward(V, b, k * BK, j1, T(px), T(py), dLdC + 3 * p,
                                             ckT[size_t(k) * npx + lp], &ckU[(size_t(k) * npx + lp) * 3], ig.data(),
                                             recs);
                    }
        }
    });
    // deterministic merge, tile-major then instance order
    g2d.assign(size_t(V.N) * 9, T(0));
    for (int64_t i = 0; i < V.I; ++i) {
        T* d = g2d.data() + size_t(V.vals[i]) * 9;
        const T* s = ig.data() + size_t(i) * 9;
        for (int k = 0; k < 9; ++k) d[k] += s[k];
    }
}

// backward_project + SH/activation chain and
// accumulate_densify_stats.
template <class T>
void project_backward(const T* P, int64_t N, int64_t g, const GFwd<T>& F, const Cam<T>& cam,
                      const tso_render_config& cfg, const T* g2, T* G) {
    Off off(N);
    const T* W = cam.W;
    T dmx = g2[0], dmy = g2[1], dA = g2[2], dB = g2[3], dC = g2[4], dop = g2[5];
    // --- color / SH
    int deg = cfg.sh_degree, nb = (deg + 1) * (deg + 1);
    T drc[3];
    for (int ch = 0; ch < 3; ++ch) drc[ch] = F.raw[ch] < T(0) ? T(0) : g2[6 + ch];
    T Y[16], dY[16][3];
    sh_basis(F.dir[0], F.dir[1], F.dir[2], deg, Y);
    sh_basis_grad(F.dir[0], F.dir[1], F.dir[2], deg, dY);
    const T* dcp = P + off.dc + 3 * g;
    const T* rest = P + off.rest + 45 * g;
    T ddir[3] = {T(0), T(0), T(0)};
    for (int ch = 0; ch < 3; ++ch) {
        G[off.dc + 3 * g + ch] += Y[0] * drc[ch];
        for (int k = 1; k < nb; ++k) G[off.rest + 45 * g + 3 * (k - 1) + ch] += Y[k] * drc[ch];
        for (int k = 1; k < nb; ++k) {
            T c = rest[3 * (k - 1) + ch];
            for (int a = 0; a < 3; ++a) ddir[a] += drc[ch] * dY[k][a] * c;
        }
    }
    (void)dcp;
    T nd = F.dir[0] * ddir[0] + F.dir[1] * ddir[1] + F.dir[2] * ddir[2];
    T dmean[3];
    for (int a = 0; a < 3; ++a) dmean[a] = (ddir[a] - F.dir[a] * nd) / F.dlen;
    // --- opacity (through the AA factor; the Mip compensation is detached from Sigma2D)
    G[off.op + g] += ((dop * F.ofac) * F.o_raw) * (T(1) - F.o_raw);
    // --- conic -> dilated cov2d: dS' = -C' Gc C', Gc = [[dA, dB/2],[dB/2, dC]]
    T hb = T(0.5) * dB;
    T K00 = F.A * dA + F.B * hb, K01 = F.A * hb + F.B * dC;
    T K10 = F.B * dA + F.C * hb, K11 = F.B * hb + F.C * dC;
    T da = -(K00 * F.A + K01 * F.B);
    T db = T(-2) * (K00 * F.B + K01 * F.C);
    T dc = -(K10 * F.B + K11 * F.C);
    // --- cov2d = Tm S Tm^T : dS = Tm^T G2 Tm, dTm = 2 G2 Tm S
    T G2[4] = {da, T(0.5) * db, T(0.5) * db, dc};
    T Sf[9] = {F.S[0], F.S[1], F.S[2], F.S[1], F.S[3], F.S[4], F.S[2], F.S[4], F.S[5]};
    T dS[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            T s = T(0);
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) s += F.Tm[3 * r + i] * G2[2 * r + c] * F.Tm[3 * c + j];
            dS[3 * i + j] = s;
        }
    T TS[6];
    for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) {
            T s = T(0);
            for (int k = 0; k < 3; ++k) s += F.Tm[3 * r + k] * Sf[3 * k + j];
            TS[3 * r + j] = s;
        }
    T dTm[6];
    for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 3; ++j) dTm[3 * r + j] = T(2) * (G2[2 * r] * TS[j] + G2[2 * r + 1] * TS[3 + j]);
    // --- Tm = J W3 : dJ = dTm W3^T
    T dJ00 = dTm[0] * W[0] + dTm[1] * W[1] + dTm[2] * W[2];
    T dJ02 = dTm[0] * W[8] + dTm[1] * W[9] + dTm[2] * W[10];
    T dJ11 = dTm[3] * W[4] + dTm[4] * W[5] + dTm[5] * W[6];
    T dJ12 = dTm[3] * W[8] + dTm[4] * W[9] + dTm[5] * W[10];
    // --- camera point grads
    T z = F.zh, z2 = z * z, z3 = z2 * z;
    T dtx = dmx * cam.fx / z, dty = dmy * cam.fy / z;
    T dtz = -dmx * cam.fx * F.xh / z2 - dmy * cam.fy * F.yh / z2;
    dtz += -dJ00 * cam.fx / z2 - dJ11 * cam.fy / z2;
    if (!F.clx) {
        dtx += dJ02 * (-cam.fx / z2);
        dtz += dJ02 * (T(2) * cam.fx * F.xh / z3);
    } else {
        dtz += dJ02 * (cam.fx * F.ux / z2);
    }
    if (!F.cly) {
        dty += dJ12 * (-cam.fy / z2);
        dtz += dJ12 * (T(2) * cam.fy * F.yh / z3);
    } else {
        dtz += dJ12 * (cam.fy * F.uy / z2);
    }
    for (int j = 0; j < 3; ++j) dmean[j] += W[j] * dtx + W[4 + j] * dty + W[8 + j] * dtz;
    for (int j = 0; j < 3; ++j) G[off.means + 3 * g + j] += dmean[j];
    // --- Sigma = M M^T : dM = 2 dS M ; M = R diag(s)
    T dM[9];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
            T s = T(0);
            for (int j = 0; j < 3; ++j) s += dS[3 * i + j] * F.Mm[3 * j + k];
            dM[3 * i + k] = T(2) * s;
        }
    T dR[9];
    for (int k = 0; k < 3; ++k) {
        T ds = T(0);
        for (int i = 0; i < 3; ++i) {
            ds += F.R[3 * i + k] * dM[3 * i + k];
            dR[3 * i + k] = dM[3 * i + k] * F.s[k];
        }
        if (cfg.aa_mode == 1)  // through s_hat = sqrt(s^2 + f) and the opacity factor
            G[off.ls + 3 * g + k] += ds * ((F.s_raw[k] * F.s_raw[k]) / F.s[k]) + ((dop * F.o_raw) * F.ofac) * (F.aaf / F.s_h[k]);
        else
            G[off.ls + 3 * g + k] += ds * F.s[k];
    }
    T w = F.qw, x = F.qx, y = F.qy, zq = F.qz;
    T dqw = T(2) * (-zq * dR[1] + y * dR[2] + zq * dR[3] - x * dR[5] - y * dR[6] + x * dR[7]);
    T dqx = T(2) * (y * dR[1] + zq * dR[2] + y * dR[3] - T(2) * x * dR[4] - w * dR[5] + zq * dR[6] + w * dR[7] -
                    T(2) * x * dR[8]);
    T dqy = T(2) * (T(-2) * y * dR[0] + x * dR[1] + w * dR[2] + x * dR[3] + zq * dR[5] - w * dR[6] + zq * dR[7] -
                    T(2) * y * dR[8]);
    T dqz = T(2) * (T(-2) * zq * dR[0] - w * dR[1] + x * dR[2] + w * dR[3] - T(2) * zq * dR[4] + y * dR[5] +
                    x * dR[6] + y * dR[7]);
    T dot = w * dqw + x * dqx + y * dqy + zq * dqz;
    T qh[4] = {w, x, y, zq}, dq[4] = {dqw, dqx, dqy, dqz};
    for (int k = 0; k < 4; ++k) G[off.q + 4 * g + k] += (dq[k] - qh[k] * dot) / F.qn;
}

template <class T>
void backward_impl(int64_t n, const T* P, const tso_camera* c, const tso_render_config* cfg, const T* dLdC_hwc,
                   T* G, T* g2d_out, T* accum, T* vcount) {
    if (!valid_cam<T>(c)) return;
    Cam<T> cam(*c);
    View<T> V;
    preprocess_all(V, P, n, cam, *cfg);
    build_instances(V, cam, *cfg);
    sort_and_range(V, cam);
    Frame<T> fb;
    blend_all(V, cam, *cfg, fb);
    std::vector<T> g2d;
    raster_backward(V, cam, *cfg, fb, dLdC_hwc, g2d);
    if (g2d_out)
        for (size_t i = 0; i < g2d.size(); ++i) g2d_out[i] += g2d[i];
    pfor(n, [&](int64_t b, int64_t e) {
        for (int64_t g = b; g < e; ++g) {
            if (!V.cnt[g]) continue;  // invisible: zero gradient, stats untouched
            const T* g2 = g2d.data() + size_t(g) * 9;
            if (G) project_backward(P, n, g, V.F[g], cam, *cfg, g2, G);
            if (accum) accum[g] += std::sqrt(g2[0] * g2[0] + g2[1] * g2[1]);
            if (vcount) vcount[g] += T(1);
        }
    });
}

// ----------------------------------------------------------------------------
// optim: Adam; literal formula, fixed per-element op order.
// ----------------------------------------------------------------------------
inline int group_of(int64_t idx, int64_t N, int64_t* gi) {
    const int64_t b[7] = {0, 3 * N, 6 * N, 10 * N, 11 * N, 14 * N, 59 * N};
    const int64_t comp[6] = {3, 3, 4, 1, 3, 45};
    for (int k = 0; k < 6; ++k)
        if (idx < b[k + 1]) {
            *gi = (idx - b[k]) / comp[k];
            return k;
        }
    *gi = 0;
    return 5;
}

// adam_step_reference: the literal formula
template <class T>
inline void adam_elem(T& th, T g, T& m, T& v, T lr, T b1, T b2, T omb1, T omb2, T eps, T bc1, T bc2) {
    m = b1 * m + omb1 * g;
    v = b2 * v + omb2 * g * g;
    T mh = m / bc1;
    T vh = v / bc2;
    T den = std::sqrt(vh) + eps;
    th = th - (lr * mh) / den;
}

}  // namespace

// ============================================================================
// extern "C" surface
// ============================================================================
extern "C" {

void tso_set_workers(int n) { g_workers = n; }
int tso_get_workers(void) { return workers(); }
float tso_expf(float x) { return soft_expf(x); }
float tso_logf(float x) { return soft_logf(x); }

int tso_rotation_from_quaternion_f64(const double q[4], double R[9]) {
    double P[59] = {0};
    P[3] = P[4] = P[5] = 0;  // unit scales
    P[6] = q[0];
    P[7] = q[1];
    P[8] = q[2];
    P[9] = q[3];
    double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(qn >= 1e-4)) return 0;
    double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    R[0] = 1 - 2 * (y * y + z * z);
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = 1 - 2 * (x * x + z * z);
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = 1 - 2 * (x * x + y * y);
    return 1;
}

void tso_build_covariance3d_f64(const double R[9], const double s[3], double cov6[6]) {
    double Mm[9];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) Mm[3 * i + k] = R[3 * i + k] * s[k];
    auto d = [&](int i, int j) {
        return (Mm[3 * i] * Mm[3 * j] + Mm[3 * i + 1] * Mm[3 * j + 1]) + Mm[3 * i + 2] * Mm[3 * j + 2];
    };
    cov6[0] = d(0, 0);
    cov6[1] = d(0, 1);
    cov6[2] = d(0, 2);
    cov6[3] = d(1, 1);
    cov6[4] = d(1, 2);
    cov6[5] = d(2, 2);
}

void tso_eval_sh_f64(const double* coeffs48, const double dir[3], int deg, double rgb[3]) {
    double Y[16];
    sh_basis(dir[0], dir[1], dir[2], deg, Y);
    int nb = (deg + 1) * (deg + 1);
    for (int ch = 0; ch < 3; ++ch) {
        double acc = 0;
        for (int k = 0; k < nb; ++k) acc += Y[k] * coeffs48[3 * k + ch];
        acc += 0.5;
        rgb[ch] = acc < 0 ? 0 : acc;
    }
}

int tso_project_mean_f64(const tso_camera* c, const double mu[3], double m2[2], double t[3]) {
    Cam<double> cam(*c);
    const double* W = cam.W;
    t[0] = ((W[0] * mu[0] + W[1] * mu[1]) + W[2] * mu[2]) + W[3];
    t[1] = ((W[4] * mu[0] + W[5] * mu[1]) + W[6] * mu[2]) + W[7];
    t[2] = ((W[8] * mu[0] + W[9] * mu[1]) + W[10] * mu[2]) + W[11];
    if (!(t[2] > cam.nearp)) return 0;
    m2[0] = cam.fx * (t[0] / t[2]) + cam.cx;
    m2[1] = cam.fy * (t[1] / t[2]) + cam.cy;
    return 1;
}

void tso_project_covariance_f64(const tso_camera* c, const double t[3], const double S[6], double out[3]) {
    Cam<double> cam(*c);
    const double* W = cam.W;
    double ux = t[0] / t[2], uy = t[1] / t[2];
    ux = std::min(cam.limx, std::max(-cam.limx, ux));
    uy = std::min(cam.limy, std::max(-cam.limy, uy));
    double J00 = cam.fx / t[2], J02 = -(cam.fx * ux * t[2]) / (t[2] * t[2]);
    double J11 = cam.fy / t[2], J12 = -(cam.fy * uy * t[2]) / (t[2] * t[2]);
    double Tm[6];
    for (int j = 0; j < 3; ++j) {
        Tm[j] = J00 * W[j] + J02 * W[8 + j];
        Tm[3 + j] = J11 * W[4 + j] + J12 * W[8 + j];
    }
    double Sf[9] = {S[0], S[1], S[2], S[1], S[3], S[4], S[2], S[4], S[5]};
    double U[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) U[3 * i + j] = Tm[3 * i] * Sf[j] + Tm[3 * i + 1] * Sf[3 + j] + Tm[3 * i + 2] * Sf[6 + j];
    out[0] = U[0] * Tm[0] + U[1] * Tm[1] + U[2] * Tm[2];
    out[1] = U[0] * Tm[3] + U[1] * Tm[4] + U[2] * Tm[5];
    out[2] = U[3] * Tm[3] + U[4] * Tm[4] + U[5] * Tm[5];
}

int tso_invert_cov2d_f64(const double cov[3], double dil, double conic[3], double* det) {
    double a = cov[0] + dil, b = cov[1], c = cov[2] + dil;
    double d = a * c - b * b;
    *det = d;
    if (!(d >= 1e-6)) return 0;
    conic[0] = c / d;
    conic[1] = -b / d;
    conic[2] = a / d;
    return 1;
}

void tso_preprocess(int64_t n, const float* params, const tso_camera* c, const tso_render_config* cfg, float* splat,
                    int32_t* rect, uint32_t* tile_count, uint32_t* depth_key) {
    Cam<float> cam(*c);
    View<float> V;
    preprocess_all(V, params, n, cam, *cfg);
    for (int64_t g = 0; g < n; ++g) {
        const GFwd<float>& F = V.F[g];
        float* s = splat + 12 * g;
        if (F.ok) {
            float rec[12] = {F.mx, F.my, F.k2, F.o, F.A, F.B, F.C, F.zh, F.rgb[0], F.rgb[1], F.rgb[2], F.det};
            std::memcpy(s, rec, sizeof(rec));
        } else {
            std::memset(s, 0, 12 * sizeof(float));
        }
        rect[4 * g] = V.rect[g].tx0;
        rect[4 * g + 1] = V.rect[g].ty0;
        rect[4 * g + 2] = V.rect[g].tx1;
        rect[4 * g + 3] = V.rect[g].ty1;
        tile_count[g] = V.cnt[g];
        depth_key[g] = V.dkey[g];
    }
}

int64_t tso_build_instances(int64_t n, const float* splat, const int32_t* rect, const uint32_t* tile_count,
                            const uint32_t* depth_key, const tso_camera* c, const tso_render_config* cfg,
                            uint64_t* keys, uint32_t* vals) {
    Cam<float> cam(*c);
    int64_t o = 0;
    for (int64_t g = 0; g < n; ++g) {
        if (!tile_count[g]) continue;
        const float* s = splat + 12 * g;
        for (int ty = rect[4 * g + 1]; ty <= rect[4 * g + 3]; ++ty)
            for (int tx = rect[4 * g]; tx <= rect[4 * g + 2]; ++tx)
                if (cfg->cull_mode == 0 || tile_keep(s[0], s[1], s[4], s[5], s[6], s[2], tx, ty, cam)) {
                    uint64_t tile = uint64_t(ty) * cam.tiles_x + tx;
                    keys[o] = (tile << 32) | depth_key[g];
                    vals[o] = uint32_t(g);
                    ++o;
                }
    }
    return o;
}

void tso_sort_combined(int64_t I, uint64_t* keys, uint32_t* vals) {
    std::vector<size_t> perm(I);
    for (int64_t i = 0; i < I; ++i) perm[i] = size_t(i);
    std::stable_sort(perm.begin(), perm.end(), [&](size_t a, size_t b) { return keys[a] < keys[b]; });
    std::vector<uint64_t> nk(I);
    std::vector<uint32_t> nv(I);
    for (int64_t i = 0; i < I; ++i) {
        nk[i] = keys[perm[i]];
        nv[i] = vals[perm[i]];
    }
    std::memcpy(keys, nk.data(), I * 8);
    std::memcpy(vals, nv.data(), I * 4);
}

int64_t tso_sort_two_stage(int64_t I, int tile_bits, uint64_t* keys, uint32_t* vals) {
    return sort_two_stage(I, tile_bits, keys, vals);
}

void tso_tile_ranges(int64_t I, const uint64_t* k, int32_t Tn, uint32_t* ranges) { tile_ranges(I, k, Tn, ranges); }

int64_t tso_render(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg, float* rgb,
                   float* T, uint32_t* count) {
    return render_impl<float>(n, params, cam, cfg, rgb, T, count);
}

int64_t tso_render_f64(int64_t n, const double* params, const tso_camera* cam, const tso_render_config* cfg,
                       double* rgb, double* T, uint32_t* count) {
    return render_impl<double>(n, params, cam, cfg, rgb, T, count);
}

void tso_render_weight_sum(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg,
                           double* out) {
    std::vector<double> ws;
    render_impl<float>(n, params, cam, cfg, nullptr, nullptr, nullptr, &ws);
    std::memcpy(out, ws.data(), ws.size() * sizeof(double));
}

double tso_training_loss(int32_t H, int32_t W, const float* rgb, const float* target, float* dL) {
    return loss_impl<float>(H, W, rgb, target, dL);
}
double tso_training_loss_f64(int32_t H, int32_t W, const double* rgb, const double* target, double* dL) {
    return loss_impl<double>(H, W, rgb, target, dL);
}

void tso_backward(int64_t n, const float* params, const tso_camera* cam, const tso_render_config* cfg,
                  const float* dLdC, float* grads, float* grad2d, float* accum, float* vcount) {
    backward_impl<float>(n, params, cam, cfg, dLdC, grads, grad2d, accum, vcount);
}
void tso_backward_f64(int64_t n, const double* params, const tso_camera* cam, const tso_render_config* cfg,
                      const double* dLdC, double* grads, double* grad2d, double* accum, double* vcount) {
    backward_impl<double>(n, params, cam, cfg, dLdC, grads, grad2d, accum, vcount);
}

void tso_adam_step(int64_t n, float* th, const float* g, float* m, float* v, const float lr[6], float b1, float b2,
                   float eps, float bc1, float bc2, int32_t mode, const uint8_t* visible) {
    // Every mode applies the reference per-element op order, so
    // fused == reference bitwise.  mode 0 is restated as the
    // textbook multi-sweep form (moments sweep, then update sweep), modes 1/2 as the
    // single fused sweep; fused_backward modes (3, 4) have the end state of fused
    // (1) / skip-invisible (2).
    int64_t L = 59 * n;
    float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    if (mode == 3) mode = 1;
    if (mode == 4) mode = 2;
    if (mode == 0) {
        pfor(L, [&](int64_t b, int64_t e) {
            for (int64_t i = b; i < e; ++i) {
                m[i] = b1 * m[i] + omb1 * g[i];
                v[i] = b2 * v[i] + omb2 * g[i] * g[i];
            }
        });
        pfor(L, [&](int64_t b, int64_t e) {
            for (int64_t i = b; i < e; ++i) {
                int64_t gi;
                int grp = group_of(i, n, &gi);
                float mh = m[i] / bc1;
                float vh = v[i] / bc2;
                float den = std::sqrt(vh) + eps;
                th[i] = th[i] - (lr[grp] * mh) / den;
            }
        });
        return;
    }
    pfor(L, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            int64_t gi;
            int grp = group_of(i, n, &gi);
            if (mode == 2 && visible && !visible[gi]) continue;
            adam_elem<float>(th[i], g[i], m[i], v[i], lr[grp], b1, b2, omb1, omb2, eps, bc1, bc2);
        }
    });
}

void tso_adam_step_f64(int64_t n, double* th, const double* g, double* m, double* v, const double lr[6], double b1,
                       double b2, double eps, double bc1, double bc2) {
    int64_t L = 59 * n;
    for (int64_t i = 0; i < L; ++i) {
        int64_t gi;
        int grp = group_of(i, n, &gi);
        adam_elem<double>(th[i], g[i], m[i], v[i], lr[grp], b1, b2, 1.0 - b1, 1.0 - b2, eps, bc1, bc2);
    }
}

double tso_mean_lr(int64_t step, double extent) {
    // extent * 1.6e-4 * (1e-2)^(step/30000)
    double t = double(step) / 30000.0;
    return extent * 1.6e-4 * std::pow(1e-2, t);
}

// densify_and_prune (order App. A.10).  Thresholds are compared
// in log space against host-double constants.
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// cos(2 pi u), u in [0, 1): the device's cos2pi_det (ts_math.cuh) op for op
static inline float cos2pi_det(float u) {
    const float t = u * 4.0f;
    const int q = int(t);
    const float f = t - float(q);
    const float th = f * 1.57079632679489662f;
    const float x2 = th * th;
    float c = -1.1470745597729725e-11f;
    c = c * x2 + 2.08767569878681e-09f;
    c = c * x2 + -2.755731922398589e-07f;
    c = c * x2 + 2.48015873015873e-05f;
    c = c * x2 + -1.388888888888889e-03f;
    c = c * x2 + 4.1666666666666664e-02f;
    c = c * x2 + -0.5f;
    c = c * x2 + 1.0f;
    float sn = -7.647163731819816e-13f;
    sn = sn * x2 + 1.6059043836821613e-10f;
    sn = sn * x2 + -2.505210838544172e-08f;
    sn = sn * x2 + 2.755731922398589e-06f;
    sn = sn * x2 + -1.984126984126984e-04f;
    sn = sn * x2 + 8.333333333333333e-03f;
    sn = sn * x2 + -0.16666666666666666f;
    sn = sn * x2 + 1.0f;
    sn = sn * th;
    return q == 0 ? c : q == 1 ? -sn : q == 2 ? -c : sn;
}

extern "C" float tso_cos2pi(float u) { return cos2pi_det(u); }

static inline float u01(uint64_t seed, int64_t iter, int64_t parent, int code) {
    uint64_t h = mix64(mix64(mix64(seed ^ mix64(uint64_t(iter))) ^ uint64_t(parent)) ^ uint64_t(code));
    return (float(h >> 40) + 0.5f) * 0x1.0p-24f;
}

int64_t tso_densify_and_prune(int64_t n, const float* P, const float* m, const float* v, const float* accum,
                              const float* vcount, float grad_thresh, float extent, uint64_t seed, int64_t iter,
                              float* OP, float* OM, float* OV, int64_t* stats) {
    Off off(n);
    float log_small = float(std::log(0.01 * double(extent)));
    float log_big = float(std::log(0.1 * double(extent)));
    float logit_min = float(std::log(0.05 / 0.95));
    const float ln16 = 0x1.e148a2p-2f;
    std::vector<uint8_t> sel(n), small(n), prn(n);
    for (int64_t g = 0; g < n; ++g) {
        const float* ls = P + off.ls + 3 * g;
        const float* q = P + off.q + 4 * g;
        float mls = std::max(ls[0], std::max(ls[1], ls[2]));
        float qn = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        sel[g] = vcount[g] > 0.0f && (accum[g] / vcount[g]) > grad_thresh;
        small[g] = mls <= log_small;
        bool pr_common = (P[off.op + g] < logit_min) || !(qn >= 1e-4f);
        prn[g] = pr_common || (mls > log_big);
        // child prune evaluated on child scales
        (void)pr_common;
    }
    struct Row {
        int64_t src;
        int kind;  // 0 keep, 1 clone, 2 child0, 3 child1
    };
    std::vector<Row> rows;
    int64_t n_clone = 0, n_split = 0, n_pruned = 0;
    for (int64_t g = 0; g < n; ++g) {
        if (sel[g] && !small[g]) continue;  // split parent removed
        if (prn[g]) {
            ++n_pruned;
            continue;
        }
        rows.push_back({g, 0});
    }
    for (int64_t g = 0; g < n; ++g)
        if (sel[g] && small[g]) {
            ++n_clone;
            if (prn[g]) {
                ++n_pruned;
                continue;
            }
            rows.push_back({g, 1});
        }
    for (int64_t g = 0; g < n; ++g)
        if (sel[g] && !small[g]) {
            ++n_split;
            const float* ls = P + off.ls + 3 * g;
            const float* q = P + off.q + 4 * g;
            float mls = std::max(ls[0], std::max(ls[1], ls[2])) - ln16;
            float qn = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
            bool pc = (P[off.op + g] < logit_min) || !(qn >= 1e-4f) || (mls > log_big);
            for (int k = 0; k < 2; ++k) {
                if (pc) {
                    ++n_pruned;
                    continue;
                }
                rows.push_back({g, 2 + k});
            }
        }
    int64_t na = int64_t(rows.size());
    Off oo(na);
    for (int64_t r = 0; r < na; ++r) {
        int64_t g = rows[r].src;
        int kind = rows[r].kind;
        auto cp = [&](int64_t so, int64_t dof, int comp) {
            for (int k = 0; k < comp; ++k) {
                OP[dof + comp * r + k] = P[so + comp * g + k];
                OM[dof + comp * r + k] = kind == 0 ? m[so + comp * g + k] : 0.0f;
                OV[dof + comp * r + k] = kind == 0 ? v[so + comp * g + k] : 0.0f;
            }
        };
        cp(off.means, oo.means, 3);
        cp(off.ls, oo.ls, 3);
        cp(off.q, oo.q, 4);
        cp(off.op, oo.op, 1);
        cp(off.dc, oo.dc, 3);
        cp(off.rest, oo.rest, 45);
        if (kind >= 2) {
            int child = kind - 2;
            const float* ls = P + off.ls + 3 * g;
            const float* q = P + off.q + 4 * g;
            float qn = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
            float w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
            float R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                          2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                          2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
            float zs[3];
            for (int a = 0; a < 3; ++a) {
                float u1 = u01(seed, iter, g, child * 8 + a * 2);
                float u2 = u01(seed, iter, g, child * 8 + a * 2 + 1);
                // Box-Muller with the deterministic log / cos of the device (bitwise equal children)
                zs[a] = std::sqrt(-2.0f * soft_logf(u1)) * cos2pi_det(u2);
                zs[a] *= soft_expf(ls[a]);
            }
            for (int i = 0; i < 3; ++i)
                OP[oo.means + 3 * r + i] = P[off.means + 3 * g + i] + (R[3 * i] * zs[0] + R[3 * i + 1] * zs[1] + R[3 * i + 2] * zs[2]);
            for (int a = 0; a < 3; ++a) OP[oo.ls + 3 * r + a] = ls[a] - ln16;
        }
    }
    stats[0] = n_clone;
    stats[1] = n_split;
    stats[2] = n_pruned;
    return na;
}

void tso_opacity_reset(int64_t n, float* P) {
    // o <- min(o, 0.01) in logit space
    float lmax = float(std::log(0.01 / 0.99));
    Off off(n);
    for (int64_t g = 0; g < n; ++g) P[off.op + g] = P[off.op + g] < lmax ? P[off.op + g] : lmax;
}

// ---------------------------------------------------------------------------
// morton_reorder: quantise means to 21 bits per axis over the
// mean AABB inflated by 1e-6, interleave x-LSB-first into a 63-bit
// code, stable sort (code, index), permute every per-Gaussian array.
// Quantisation: q = min(2^21-1, uint(((p - lo) / ((hi - lo) + 1e-6)) * 2^21)),
// each op rounded to fp32 (the device computes the same expression).
// ---------------------------------------------------------------------------
uint64_t tso_morton_interleave(uint32_t qx, uint32_t qy, uint32_t qz, int bits) {
    uint64_t c = 0;
    const uint32_t q[3] = {qx, qy, qz};
    for (int b = 0; b < bits; ++b)
        for (int k = 0; k < 3; ++k) c |= uint64_t((q[k] >> b) & 1u) << (3 * b + k);
    return c;
}

void tso_morton_codes(int64_t n, const float* P, uint64_t* codes) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t g = 0; g < n; ++g)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], P[3 * g + k]);
            hi[k] = std::max(hi[k], P[3 * g + k]);
        }
    for (int64_t g = 0; g < n; ++g) {
        uint32_t q[3];
        for (int k = 0; k < 3; ++k) {
            const float span = (hi[k] - lo[k]) + 1e-6f;
            const float t = ((P[3 * g + k] - lo[k]) / span) * 2097152.0f;
            const uint32_t u = uint32_t(t);
            q[k] = u > 2097151u ? 2097151u : u;
        }
        codes[g] = tso_morton_interleave(q[0], q[1], q[2], 21);
    }
}

void tso_morton_reorder(int64_t n, float* P, float* M, float* V, float* accum, float* vcount, uint32_t* perm) {
    if (n <= 0) return;
    std::vector<uint64_t> code(n);
    tso_morton_codes(n, P, code.data());
    std::vector<uint32_t> idx(n);
    for (int64_t i = 0; i < n; ++i) idx[i] = uint32_t(i);
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return code[a] < code[b]; });
    const Off o(n);
    const int64_t starts[6] = {o.means, o.ls, o.q, o.op, o.dc, o.rest};
    const int width[6] = {3, 3, 4, 1, 3, 45};
    std::vector<float> tmp;
    for (float* B : {P, M, V}) {
        if (!B) continue;
        tmp.assign(B, B + 59 * n);
        for (int a = 0; a < 6; ++a)
            for (int64_t r = 0; r < n; ++r)
                for (int k = 0; k < width[a]; ++k)
                    B[starts[a] + r * width[a] + k] = tmp[starts[a] + int64_t(idx[r]) * width[a] + k];
    }
    for (float* B : {accum, vcount}) {
        if (!B) continue;
        tmp.assign(B, B + n);
        for (int64_t r = 0; r < n; ++r) B[r] = tmp[idx[r]];
    }
    if (perm) std::copy(idx.begin(), idx.end(), perm);
}

// One full training step on one view (SPEC.md:829-837 step body): render ->
// training_loss -> backward -> Adam, each stage timed (bench per-stage times,
// SPEC.md:839-847).  This is the timed CPU baseline unit.
double tso_train_step(int64_t n, float* params, float* m, float* v, const tso_camera* c,
                      const tso_render_config* cfg, const float* target, const float lr[6], float b1, float b2,
                      float eps, float bc1, float bc2, float* accum, float* vcount, double* st) {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    auto lap = [&](int k) {
        auto t1 = clk::now();
        if (st) st[k] = std::chrono::duration<double>(t1 - t0).count();
        t0 = t1;
    };
    Cam<float> cam(*c);
    View<float> V;
    preprocess_all(V, params, n, cam, *cfg);
    lap(0);
    build_instances(V, cam, *cfg);
    sort_and_range(V, cam);
    lap(1);
    Frame<float> fb;
    blend_all(V, cam, *cfg, fb);
    lap(2);
    std::vector<float> dL(fb.rgb.size());
    double loss = loss_impl<float>(cam.h, cam.w, fb.rgb.data(), target, dL.data());
    lap(3);
    std::vector<float> g2d;
    raster_backward(V, cam, *cfg, fb, dL.data(), g2d);
    lap(4);
    std::vector<float> G(size_t(59) * n, 0.0f);
    pfor(n, [&](int64_t b, int64_t e) {
        for (int64_t g = b; g < e; ++g) {
            if (!V.cnt[g]) continue;
            const float* g2 = g2d.data() + size_t(g) * 9;
            project_backward(params, n, g, V.F[g], cam, *cfg, g2, G.data());
            if (accum) accum[g] += std::sqrt(g2[0] * g2[0] + g2[1] * g2[1]);
            if (vcount) vcount[g] += 1.0f;
        }
    });
    lap(5);
    tso_adam_step(n, params, G.data(), m, v, lr, b1, b2, eps, bc1, bc2, 1, nullptr);
    lap(6);
    if (st) st[7] = double(V.I);
    return loss;
}

int32_t tso_sh_active_degree(int64_t iter) { return int32_t(std::min<int64_t>(3, iter / 1000)); }

void tso_set_sampling_rates(int64_t n, const float* nu) { g_nu.assign(nu, nu + n); }

// compute_sampling_rates; project_mean op order, J-clamp frustum
void tso_compute_sampling_rates(int64_t n, const float* params, const tso_camera* cams, int32_t ncams, float extent,
                                float* nu) {
    Off off(n);
    std::vector<Cam<float>> cs;
    for (int k = 0; k < ncams; ++k) cs.emplace_back(cams[k]);
    const float fallback = 1.0f / extent;
    pfor(n, [&](int64_t b, int64_t e) {
        for (int64_t g = b; g < e; ++g) {
            const float* mu = params + off.means + 3 * g;
            float best = 0.0f;
            bool any = false;
            for (const auto& cam : cs) {
                const float* W = cam.W;
                const float xh = ((W[0] * mu[0] + W[1] * mu[1]) + W[2] * mu[2]) + W[3];
                const float yh = ((W[4] * mu[0] + W[5] * mu[1]) + W[6] * mu[2]) + W[7];
                const float zh = ((W[8] * mu[0] + W[9] * mu[1]) + W[10] * mu[2]) + W[11];
                if (!(zh > cam.nearp)) continue;
                const float tx = xh / zh, ty = yh / zh;
                if (tx < -cam.limx || tx > cam.limx || ty < -cam.limy || ty > cam.limy) continue;
                const float f = cam.fx > cam.fy ? cam.fx : cam.fy;
                const float v = f / zh;
                best = any ? (v > best ? v : best) : v;
                any = true;
            }
            nu[g] = any ? best : fallback;
        }
    });
}

// apply_3d_filter_clip in log space
void tso_apply_3d_filter_clip(int64_t n, float* params, const float* nu, float kappa3d) {
    Off off(n);
    const float sk = std::sqrt(kappa3d);
    for (int64_t g = 0; g < n; ++g) {
        const float fl = soft_logf(sk / nu[g]);
        for (int k = 0; k < 3; ++k) {
            float& l = params[off.ls + 3 * g + k];
            l = l < fl ? fl : l;
        }
    }
}

double tso_scene_extent(int32_t nc, const double* c) {
    if (nc <= 1) return 1.0;
    double m[3] = {0, 0, 0};
    for (int i = 0; i < nc; ++i)
        for (int k = 0; k < 3; ++k) m[k] += c[3 * i + k] / nc;
    double r = 0;
    for (int i = 0; i < nc; ++i) {
        double d = 0;
        for (int k = 0; k < 3; ++k) d += (c[3 * i + k] - m[k]) * (c[3 * i + k] - m[k]);
        r = std::max(r, std::sqrt(d));
    }
    return 1.1 * r;
}

}  // extern "C"
