// K1 preprocess_fwd: one thread per Gaussian.
// activate_scales/opacity, rotation_from_quaternion (:59-67),
// build_covariance3d (:69-77), project_mean (:132-140), project_covariance
// (:142-150), invert_cov2d (:152-160), eval_sh (:79-87), bound_rect (:214-222)
// and the exact-cull COUNT pass (:224-232).  HBM-bound: reads 44 B + 12*D B of
// parameters, writes a 48 B splat row + 8 B rect + 4 B count + 4 B depth key.
#include "ts_internal.cuh"
#include "ts_math.cuh"
#include "ts_stage.cuh"

namespace ts {
namespace {

constexpr int kBlock = 128;

template <int DEG>
__global__ void __launch_bounds__(kBlock) preprocess_kernel(
    const float* __restrict__ P, int64_t N, DevCam cam, ts_render_config cfg, float4* __restrict__ splat,
    uint4* __restrict__ rect, float* __restrict__ ryv, uint32_t* __restrict__ tcount, uint32_t* __restrict__ dkey,
    uint32_t* __restrict__ dperm, uint32_t* __restrict__ vis_counter, const float* __restrict__ nu_hat,
    uint32_t* __restrict__ binH, int bin_chunk) {
    using namespace tsx;
    // staged inputs of the CTA's 128 Gaussians (one pass of independent 16-byte loads)
    constexpr int kMu = 0, kLs = kMu + 3 * kBlock + 4, kQ = kLs + 3 * kBlock + 4, kOp = kQ + 4 * kBlock + 4,
                  kDc = kOp + kBlock + 4, kRest = kDc + 3 * kBlock + 4;
    constexpr int deg = DEG;
    constexpr int nb = (deg + 1) * (deg + 1);
    constexpr int nrest = 3 * (nb - 1);
    __shared__ __align__(16) float sm[kRest + (nrest > 0 ? 45 * kBlock + 4 : 12 * kBlock + 4)];
    const Off off(N);
    const int64_t g0 = int64_t(blockIdx.x) * kBlock;
    const int64_t g = g0 + threadIdx.x;
    const int rows = int(tmin<int64_t>(kBlock, N - g0));
    int sh[6] = {0, 0, 0, 0, 0, 0};
    __shared__ unsigned long long bars[2];
    {
        const Span base[5] = {{sm + kMu, P + off.means + 3 * g0, 3 * rows},
                              {sm + kLs, P + off.ls + 3 * g0, 3 * rows},
                              {sm + kQ, P + off.q + 4 * g0, 4 * rows},
                              {sm + kOp, P + off.op + g0, rows},
                              {sm + kDc, P + off.dc + 3 * g0, 3 * rows}};
        // two barriers: the geometry rows gate the projection, the SH rows (the bulk of the
        // bytes) are awaited only before the colour evaluation
        mbar_init_all(bars, 2);
        int s5[5];
        tma_issue_spans(base, s5, &bars[0]);
        for (int k = 0; k < 5; ++k) sh[k] = s5[k];
        if constexpr (nrest > 0) {
            const Span sp[1] = {{sm + kRest, P + off.rest + g0 * 45, 45 * rows}};
            int s1[1];
            tma_issue_spans(sp, s1, &bars[1]);
            sh[5] = s1[0];
        }
        mbar_wait0(&bars[0]);
    }
    const bool live = g < N;  // dead lanes stay for the warp-cooperative cull below
    const int tid = threadIdx.x;
    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0, s2 = s0;
    uint32_t cnt = 0;
    uint4 rc = make_uint4(1u, 1u, 0u, 0u);  // empty: tx0=1 > tx1=0
    bool ok = false;
    float zh = 0.f;
    float ry_cull = 0.f;  // blend row-cull half-height (0: no tiles)
    // exact-cull inputs of the warp-cooperative pass (ntl = 0: nothing to test)
    uint32_t ntl_c = 0, rect0 = 0, magic_c = 0;
    int tw_c = 1;
    float mx_c = 0.f, my_c = 0.f, A_c = 0.f, B_c = 0.f, C_c = 0.f, k2_c = 0.f, nBA_c = 0.f, nBC_c = 0.f;
    bool big_c = false;
    do {
        if (!live) break;
        const float* W = cam.W;
        const float* mus = sm + kMu + sh[0] + 3 * tid;
        const float m0 = mus[0], m1 = mus[1], m2 = mus[2];
        // project_mean, fixed order (depth feeds the sort key)
        const float xh = add(fma_(W[2], m2, fma_(W[1], m1, mul(W[0], m0))), W[3]);
        const float yh = add(fma_(W[6], m2, fma_(W[5], m1, mul(W[4], m0))), W[7]);
        zh = add(fma_(W[10], m2, fma_(W[9], m1, mul(W[8], m0))), W[11]);
        if (!(zh > cam.nearp)) break;
        const float* qs = sm + kQ + sh[2] + 4 * tid;
        const float4 qv = make_float4(qs[0], qs[1], qs[2], qs[3]);
        const float qq = fma_(qv.w, qv.w, fma_(qv.z, qv.z, fma_(qv.y, qv.y, mul(qv.x, qv.x))));
        const float qn = sqrt_(qq);
        if (!(qn >= 1e-4f)) break;
        const float rq = div(1.f, qn);
        const float w = mul(qv.x, rq), x = mul(qv.y, rq), y = mul(qv.z, rq), z = mul(qv.w, rq);
        float R[9];
        {
            const float xx = mul(x, x), yy = mul(y, y), zz = mul(z, z), xy = mul(x, y), xz = mul(x, z),
                        yz = mul(y, z), wx = mul(w, x), wy = mul(w, y), wz = mul(w, z);
            R[0] = sub(1.f, mul(2.f, add(yy, zz)));
            R[1] = mul(2.f, sub(xy, wz));
            R[2] = mul(2.f, add(xz, wy));
            R[3] = mul(2.f, add(xy, wz));
            R[4] = sub(1.f, mul(2.f, add(xx, zz)));
            R[5] = mul(2.f, sub(yz, wx));
            R[6] = mul(2.f, sub(xz, wy));
            R[7] = mul(2.f, add(yz, wx));
            R[8] = sub(1.f, mul(2.f, add(xx, yy)));
        }
        float sc[3];
        const float* lss = sm + kLs + sh[1] + 3 * tid;
        sc[0] = expf_det(lss[0]);
        sc[1] = expf_det(lss[1]);
        sc[2] = expf_det(lss[2]);
        float ofac = 1.f;
        if (cfg.aa_mode == 1) {
            // apply_3d_filter_original, exact ops (feeds the tile rect)
            const float nu = nu_hat[g];
            const float f = div(cfg.kappa3d, mul(nu, nu));
            float q[3], hh[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                q[k] = mul(sc[k], sc[k]);
                hh[k] = add(q[k], f);
                sc[k] = sqrt_(hh[k]);
            }
            ofac = sqrt_(div(mul(mul(q[0], q[1]), q[2]), mul(mul(hh[0], hh[1]), hh[2])));
        }
        float Mm[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) Mm[3 * i + k] = mul(R[3 * i + k], sc[k]);
        auto sdot = [&](int i, int j) {
            return fma_(Mm[3 * i + 2], Mm[3 * j + 2], fma_(Mm[3 * i + 1], Mm[3 * j + 1], mul(Mm[3 * i], Mm[3 * j])));
        };
        const float S00 = sdot(0, 0), S01 = sdot(0, 1), S02 = sdot(0, 2), S11 = sdot(1, 1), S12 = sdot(1, 2),
                    S22 = sdot(2, 2);
        // project_covariance with clamped ratios
        const float limx = cam.limx, limy = cam.limy;
        const float rz = div(1.f, zh);
        const float txz = mul(xh, rz), tyz = mul(yh, rz);
        const float ux = txz < -limx ? -limx : (txz > limx ? limx : txz);
        const float uy = tyz < -limy ? -limy : (tyz > limy ? limy : tyz);
        // J = [[fx/z, 0, -fx u_x / z], [0, fy/z, -fy u_y / z]] (u = clamped x/z, y/z)
        const float J00 = mul(cam.fx, rz), J02 = mul(-mul(cam.fx, ux), rz);
        const float J11 = mul(cam.fy, rz), J12 = mul(-mul(cam.fy, uy), rz);
        float Tm[6];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            Tm[j] = fma_(J02, W[8 + j], mul(J00, W[j]));
            Tm[3 + j] = fma_(J12, W[8 + j], mul(J11, W[4 + j]));
        }
        const float Sf[9] = {S00, S01, S02, S01, S11, S12, S02, S12, S22};
        float U[6];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                U[3 * i + j] = fma_(Tm[3 * i + 2], Sf[6 + j], fma_(Tm[3 * i + 1], Sf[3 + j], mul(Tm[3 * i], Sf[j])));
        float a = fma_(U[2], Tm[2], fma_(U[1], Tm[1], mul(U[0], Tm[0])));
        const float b = fma_(U[2], Tm[5], fma_(U[1], Tm[4], mul(U[0], Tm[3])));
        float c = fma_(U[5], Tm[5], fma_(U[4], Tm[4], mul(U[3], Tm[3])));
        // invert_cov2d with dilation
        const float det_pre = fma_(a, c, -mul(b, b));
        a = add(a, cfg.dilation);
        c = add(c, cfg.dilation);
        const float det = fma_(a, c, -mul(b, b));
        if (!(det >= 1e-6f)) break;
        const float rdet = div(1.f, det);
        const float A = mul(c, rdet), B = mul(-b, rdet), C = mul(a, rdet);
        const float mx = fma_(cam.fx, txz, cam.cx), my = fma_(cam.fy, tyz, cam.cy);
        // activate_opacity; keep level set Q <= k2  (classic: o exp(-Q/2) >= tau)
        const float logit = sm[kOp + sh[3] + tid];
        const float o_raw = div(1.f, add(1.f, expf_det(-logit)));
        // Mip compensation: sqrt(det_pre / det_post), detached in the backward
        if (cfg.aa_mode == 3) ofac = det_pre > 0.f ? sqrt_(div(det_pre, det)) : 0.f;
        const float o = (cfg.aa_mode == 1 || cfg.aa_mode == 3) ? mul(o_raw, ofac) : o_raw;
        const float tau = cfg.tau_alpha;
        // classic truncation: o G >= tau; response truncation: G >= exp(-sigma_cut^2 / 2)
        const bool resp = cfg.truncation == 1;
        const bool has_bound = resp ? o > 0.f : o > tau;
        const float k2 = !has_bound ? 0.f : resp ? mul(cfg.sigma_cut, cfg.sigma_cut) : mul(-2.f, logf_det(div(tau, o)));
        ok = true;

        // ---- eval_sh (colour tolerance path: contraction allowed) ----
        const float cpx = -((W[0] * W[3] + W[4] * W[7]) + W[8] * W[11]);
        const float cpy = -((W[1] * W[3] + W[5] * W[7]) + W[9] * W[11]);
        const float cpz = -((W[2] * W[3] + W[6] * W[7]) + W[10] * W[11]);
        float d0 = m0 - cpx, d1 = m1 - cpy, d2 = m2 - cpz;
        const float il = rsqrtf(d0 * d0 + d1 * d1 + d2 * d2);
        d0 *= il;
        d1 *= il;
        d2 *= il;
        float Y[16];
        Y[0] = TS_SH_C0;
        if (deg >= 1) {
            Y[1] = -TS_SH_C1 * d1;
            Y[2] = TS_SH_C1 * d2;
            Y[3] = -TS_SH_C1 * d0;
        }
        if (deg >= 2) {
            const float xx = d0 * d0, yy = d1 * d1, zz = d2 * d2;
            Y[4] = TS_SH_C2_0 * d0 * d1;
            Y[5] = TS_SH_C2_1 * d1 * d2;
            Y[6] = TS_SH_C2_2 * (2.f * zz - xx - yy);
            Y[7] = TS_SH_C2_3 * d0 * d2;
            Y[8] = TS_SH_C2_4 * (xx - yy);
            if (deg >= 3) {
                Y[9] = TS_SH_C3_0 * d1 * (3.f * xx - yy);
                Y[10] = TS_SH_C3_1 * d0 * d1 * d2;
                Y[11] = TS_SH_C3_2 * d1 * (4.f * zz - xx - yy);
                Y[12] = TS_SH_C3_3 * d2 * (2.f * zz - 3.f * xx - 3.f * yy);
                Y[13] = TS_SH_C3_4 * d0 * (4.f * zz - xx - yy);
                Y[14] = TS_SH_C3_5 * d2 * (xx - yy);
                Y[15] = TS_SH_C3_6 * d0 * (xx - 3.f * yy);
            }
        }
        float rgb[3];
        if constexpr (nrest > 0) mbar_wait0(&bars[1]);
        const float* rs = sm + kRest + sh[5] + tid * 45;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            float acc = Y[0] * sm[kDc + sh[4] + 3 * tid + ch];
            _Pragma("unroll") for (int k = 1; k < nb; ++k) acc += Y[k] * rs[3 * (k - 1) + ch];
            acc += 0.5f;
            rgb[ch] = acc < 0.f ? 0.f : acc;
        }
        s0 = make_float4(mx, my, k2, o);
        s1 = make_float4(A, B, C, zh);
        s2 = make_float4(rgb[0], rgb[1], rgb[2], det);
        if (!has_bound) break;
        ry_cull = ellipse_ry(A, B, C, k2);

        // ---- bound (opacity-aware rect / rect / square) -> inclusive tile rect ----
        float rx, ry;
        if (cfg.bound_mode == 0) {
            const float mid = mul(0.5f, add(a, c));
            const float disc = sub(mul(mid, mid), det);
            const float lam = add(mid, sqrt_(disc > 0.f ? disc : 0.f));
            rx = ry = mul(3.f, sqrt_(lam));
        } else {
            const float kk = sqrt_(cfg.bound_mode == 1 && !resp ? mul(-2.f, logf_det(tau)) : k2);
            rx = mul(kk, sqrt_(a));
            ry = mul(kk, sqrt_(c));
        }
        const float wm1 = float(cam.w - 1), hm1 = float(cam.h - 1);
        float lox = sub(mx, rx), hix = add(mx, rx), loy = sub(my, ry), hiy = add(my, ry);
        lox = lox < 0.f ? 0.f : lox;
        hix = hix > wm1 ? wm1 : hix;
        loy = loy < 0.f ? 0.f : loy;
        hiy = hiy > hm1 ? hm1 : hiy;
        if (!(lox <= hix) || !(loy <= hiy)) break;
        const int px0 = int(ceilf(lox)), px1 = int(floorf(hix));
        const int py0 = int(ceilf(loy)), py1 = int(floorf(hiy));
        if (px0 > px1 || py0 > py1) break;
        const int tx0 = px0 >> 4, tx1 = px1 >> 4, ty0 = py0 >> 4, ty1 = py1 >> 4;
        const int ntl = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
        const bool big = ntl > 64;
        rc = make_uint4(uint32_t(tx0) | (uint32_t(tx1) << 16),
                        uint32_t(ty0) | (uint32_t(ty1) << 16) | (big ? 0x80000000u : 0u), 0u, 0u);
        uint64_t mask = 0;
        // per-chunk tile histogram of the bucketed binning (k_bin.cu), fire-and-forget REDs
        uint32_t* hrow = binH ? binH + size_t(g / bin_chunk) * size_t(cam.tiles_x * cam.tiles_y) : nullptr;
        if (cfg.cull_mode == 0) {
            cnt = uint32_t(ntl);
            if (!big) mask = ntl == 64 ? ~0ull : ((1ull << ntl) - 1ull);
            if (hrow)
                for (int tyy = ty0; tyy <= ty1; ++tyy)
                    for (int txx = tx0; txx <= tx1; ++txx) atomicAdd(hrow + tyy * cam.tiles_x + txx, 1u);
        } else {
            ntl_c = uint32_t(ntl);
            rect0 = uint32_t(tx0) | (uint32_t(ty0) << 16);
            tw_c = tx1 - tx0 + 1;
            magic_c = 0xFFFFFFFFu / uint32_t(tw_c);
            mx_c = mx, my_c = my, A_c = A, B_c = B, C_c = C, k2_c = k2;
            nBA_c = div(-B, A), nBC_c = div(-B, C);
            big_c = big;
        }
        rc.z = uint32_t(mask);
        rc.w = uint32_t(mask >> 32);
    } while (false);
    (void)ok;
    // every thread (also those that left the body early) sees the SH copy land before the
    // CTA can retire: shared memory must not be released under an in-flight bulk copy
    if constexpr (nrest > 0) mbar_wait0(&bars[1]);
    if (cfg.cull_mode != 0) {
        // tile_cull_exact, warp-cooperative: the warp's (Gaussian, rect tile) pairs are
        // enumerated as one list (exclusive scan of the rect sizes) and tested 32 at a
        // time, so lanes with small rects do not idle behind the warp's largest one.
        // The nonempty rects are ranked and their cull inputs tabled in shared memory (in
        // the warp's own, fully consumed SH staging rows); pair e belongs to the rect of
        // rank (owner of the window's first pair) + (segment starts in the window at or
        // before e), one OR-reduction per window.  Each Gaussian gathers its keep bits
        // (row-major rect order) from the window ballots.
        const unsigned kFull = 0xffffffffu;
        const int lane = threadIdx.x & 31;
        const int warp = threadIdx.x >> 5;
        uint32_t incl = ntl_c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - ntl_c;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const uint32_t ne = __ballot_sync(kFull, ntl_c != 0);
        const int rank = __popc(ne & ((1u << lane) - 1u));
        const int tb = nrest > 0 ? ((kRest + sh[5] + 45 * 32 * warp + 3) & ~3) : ((kRest + 3) & ~3) + 384 * warp;
        float4* tab = reinterpret_cast<float4*>(sm + tb);
        __syncwarp();  // the warp's lanes are done with their staged SH rows
        if (ntl_c) {
            tab[rank] = make_float4(mx_c, my_c, A_c, B_c);
            tab[32 + rank] = make_float4(C_c, k2_c, nBA_c, nBC_c);
            tab[64 + rank] = make_float4(__uint_as_float(rect0), __int_as_float(tw_c), __uint_as_float(magic_c),
                                         __uint_as_float(excl));
        }
        __syncwarp();
        uint32_t* hrow = binH ? binH + size_t(g0 / bin_chunk) * size_t(cam.tiles_x * cam.tiles_y) : nullptr;
        const bool hist = hrow != nullptr;
        uint64_t mask = 0;
        uint32_t bcnt = 0;
        int carry = -1;  // rank of the owner of pair base - 1
        for (uint32_t base = 0; base < total; base += 32) {
            const uint32_t e = base + uint32_t(lane);
            const uint32_t rel = excl - base;  // < 32 iff this lane's segment starts in the window
            const uint32_t sb = __reduce_or_sync(kFull, (ntl_c != 0 && rel < 32u) ? (1u << rel) : 0u);
            const int own = carry + __popc(sb & ((2u << lane) - 1u));
            carry += __popc(sb);
            bool keep = false;
            if (e < total) {
                const float4 p0 = tab[own], p1 = tab[32 + own], p2 = tab[64 + own];
                const uint32_t li = e - __float_as_uint(p2.w);
                const uint32_t otw = __float_as_uint(p2.y);
                // li / otw by a multiply-high (magic = floor((2^32-1)/otw) is at most one short)
                uint32_t q = __umulhi(li, __float_as_uint(p2.z));
                uint32_t r = li - q * otw;
                if (r >= otw) r -= otw, ++q;
                const uint32_t orect = __float_as_uint(p2.x);
                const int txx = int(orect & 0xffffu) + int(r), tyy = int(orect >> 16) + int(q);
                keep = tile_keep(p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, txx, tyy, cam.w, cam.h);
                if (keep & hist) atomicAdd(hrow + (uint32_t(tyy) * uint32_t(cam.tiles_x) + uint32_t(txx)), 1u);
            }
            const uint32_t K = __ballot_sync(kFull, keep);
            // this lane's pairs [excl, excl + ntl) -> mask bit (pair - excl); bits of other
            // lanes' pairs beyond the segment are cleared after the loop
            const int shf = int(base) - int(excl);
            if (shf > -32 && shf < 64) mask |= shf >= 0 ? (uint64_t(K) << shf) : uint64_t(K >> -shf);
            if (big_c) {  // rects of more than 64 tiles: count only
                const uint32_t lo = excl > base ? excl : base, hi = incl < base + 32 ? incl : base + 32;
                if (lo < hi) {
                    const uint32_t len = hi - lo;
                    bcnt += __popc((K >> (lo - base)) & (len == 32 ? kFull : ((1u << len) - 1u)));
                }
            }
        }
        if (big_c) {
            cnt = bcnt;
            mask = 0;
        } else {
            mask &= ntl_c >= 64 ? ~0ull : ((1ull << ntl_c) - 1ull);
            cnt = uint32_t(__popcll(mask));
        }
        rc.z = uint32_t(mask);
        rc.w = uint32_t(mask >> 32);
    }
    if (!live) return;
    splat[3 * g] = s0;
    splat[3 * g + 1] = s1;
    splat[3 * g + 2] = s2;
    rect[g] = rc;
    ryv[g] = ry_cull;
    tcount[g] = cnt;
    dkey[g] = cnt ? (__float_as_uint(zh) ^ 0x80000000u) : 0xFFFFFFFFu;
    dperm[g] = uint32_t(g);
    // warp-aggregated visible counter (bench V)
    const unsigned am = __activemask();
    const unsigned vis = __ballot_sync(am, cnt != 0);
    if ((threadIdx.x & 31) == __ffs(am) - 1 && vis) atomicAdd(vis_counter, __popc(vis));
}

}  // namespace

void launch_preprocess(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    if (c.N == 0) return;
    // the bucketed binning's chunk histograms are accumulated here (zeroed first)
    uint32_t* binH = nullptr;
    const int Tn = cam.tiles_x * cam.tiles_y;
    if (c.binning_mode == 0 && bin_supported(Tn)) {
        const int chunk = bin_chunk_for(c.N, c.sm_count);
        const size_t rows = size_t((c.N + chunk - 1) / chunk);
        if (ensure(c, c.binH, rows * Tn)) {
            binH = c.binH.p;
            cudaMemsetAsync(binH, 0, rows * Tn * 4, c.stream);
        }
    }
    const int64_t blocks = (c.N + kBlock - 1) / kBlock;
#define TS_PRE(D)                                                                                      \
    preprocess_kernel<D><<<unsigned(blocks), kBlock, 0, c.stream>>>(c.params.p, c.N, cam, cfg, c.splat.p, \
                                                                     c.rect.p, c.ryv.p, c.tcount.p, c.dkey[0].p,   \
                                                                     c.dperm[0].p, c.counters.p + 1, c.nu_hat.p,    \
                                                                     binH, bin_chunk_for(c.N, c.sm_count))
    switch (cfg.sh_degree) {
        case 0: TS_PRE(0); break;
        case 1: TS_PRE(1); break;
        case 2: TS_PRE(2); break;
        default: TS_PRE(3); break;
    }
#undef TS_PRE
    TS_LAUNCHED(c);
}

}  // namespace ts
