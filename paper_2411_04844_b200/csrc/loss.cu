// loss.cu -- fused projection-domain loss (L1 + valid-window SSIM with
// analytic gradient), iteration bookkeeping and the Adam step.
//
// Reference (/root/reference/pkg/src/splatct/):
//   l1_loss              loss.py:64-74     mean|pred-ref|, grad sign/count
//   _gaussian_window     loss.py:77-80     11 taps, sigma 1.5, normalised
//   _valid_corr(_adjoint) loss.py:83-101   separable, valid positions only
//   _ssim_slice          loss.py:112-141   SSIM map + d/dx via (d_mx, d_x2w, d_xyw)
//   ssim_loss            loss.py:159-180   L = max(ref) global; 1 - mean_z SSIM
//   total_loss_detailed  loss.py:210-239   zero-weight terms skipped (NaN parts)
//   OptimizerState.lr    optim.py:88-90 ; adam_step optim.py:109-144
//
// B200 design: the (m, n, p) sinogram has the slice index fastest, so one
// warp covers 32 consecutive slices of the same (view, detector) bin and
// every window statistic is computed for 32 independent slice images with
// fully coalesced loads.  Each thread owns one (slice, column) and walks the
// view axis keeping an 11-row ring of horizontally-correlated statistics in
// shared memory (f64, like the reference, because sigma_x^2 = E[x^2]-mu^2
// cancels).  Pass 1 writes the three SSIM derivative fields, pass 2 applies
// the transposed correlation and fuses the L1 term and the f32 store.
#include "common.cuh"

namespace splatct {

constexpr int KMAX = 11;
constexpr int LZ = 32;     // slices per CTA (lanes)
constexpr int LCOL = 4;    // columns per CTA
constexpr int LNT = LZ * LCOL;

struct Win {
    double gr[KMAX], gc[KMAX];
    int kr, kc;
};

static Win make_win(int m, int n) {
    Win W{};
    auto mk = [](int k, double* g) {
        double s = 0.0;
        for (int i = 0; i < k; ++i) {
            double x = i - (k - 1) / 2.0;
            g[i] = exp(-0.5 * (x / 1.5) * (x / 1.5));
            s += g[i];
        }
        for (int i = 0; i < k; ++i) g[i] /= s;
    };
    int kr = m < 11 ? m : 11, kc = n < 11 ? n : 11;
    kr -= 1 - kr % 2;
    kc -= 1 - kc % 2;
    W.kr = kr; W.kc = kc;
    mk(kr, W.gr);
    mk(kc, W.gc);
    return W;
}

struct LossLayout {
    int vr, vc, zc, nchunks;
    int64_t nb_v, nb_g;    // blocks per chunk of the SSIM-map and gradient passes
    size_t o_H, o_D, o_T, o_ps, o_pl, total;
};

static LossLayout loss_layout(int m, int n, int p) {
    LossLayout L{};
    Win W = make_win(m, n);
    L.vr = m - W.kr + 1;
    L.vc = n - W.kc + 1;
    L.zc = p < 64 ? p : 64;
    L.nchunks = (p + L.zc - 1) / L.zc;
    L.nb_v = ((int64_t)L.vr * L.vc * L.zc + 255) / 256;
    L.nb_g = ((int64_t)m * n * L.zc + 255) / 256;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align_up(b > 0 ? b : 1); return o; };
    L.o_H = take(sizeof(double) * 5 * (size_t)m * L.vc * L.zc);
    L.o_D = take(sizeof(double) * 3 * (size_t)L.vr * L.vc * L.zc);
    L.o_T = take(sizeof(double) * 3 * (size_t)L.vr * n * L.zc);
    L.o_ps = take(sizeof(double) * L.nb_v * L.nchunks);
    L.o_pl = take(sizeof(double) * L.nb_g * L.nchunks);
    L.total = off;
    return L;
}

// ---------------------------------------------------------------------------
// Four separable passes, one thread per output element, processed per chunk
// of ZC slices so the f64 intermediates (H, D, T) of a chunk stay L2-resident:
//   S1  H[5][m][vc][zc]  = row-direction window sums of x, y, x^2, y^2, xy
//   S2  D[3][vr][vc][zc] = column-direction sums -> SSIM map and its
//                          derivative fields (d_mx, d_x2w, d_xyw), sum of SSIM
//   G1  T[3][vr][n][zc]  = transposed row correlation of D
//   G2  grad[m][n][p]    = transposed column correlation of T, combined with
//                          x, y and the L1 sign term; sum |x - y|
// (loss.py:83-141: _valid_corr / _valid_corr_adjoint / _ssim_slice).  Every
// tap loop keeps two partial sums so the DFMA dependency chains are halved.
// ---------------------------------------------------------------------------
constexpr int ZC = 64;
constexpr int PT = 256;   // threads per block

template <int K>
__device__ __forceinline__ int ktaps(int k) { return K > 0 ? K : k; }

template <int KC_>
__global__ void __launch_bounds__(PT) k_ssim_h(const float* __restrict__ X, const float* __restrict__ Y,
                                              int m, int n, int p, int z0, int zc, Win W, int vc,
                                              double* __restrict__ H, const int* halt) {
    if (halted(halt)) return;
    const int64_t idx = blockIdx.x * (int64_t)PT + threadIdx.x;
    const int64_t tot = (int64_t)m * vc * zc;
    if (idx >= tot) return;
    const int zl = (int)(idx % zc);
    const int64_t vj = idx / zc;
    const int j = (int)(vj % vc), v = (int)(vj / vc);
    const int kc = ktaps<KC_>(W.kc);
    const float* xr = X + ((int64_t)v * n + j) * p + z0 + zl;
    const float* yr = Y + ((int64_t)v * n + j) * p + z0 + zl;
    double h[2][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
#pragma unroll
    for (int b = 0; b < (KC_ > 0 ? KC_ : KMAX); ++b) {
        if (KC_ == 0 && b >= kc) break;
        const double xv = (double)__ldg(xr + (int64_t)b * p);
        const double yv = (double)__ldg(yr + (int64_t)b * p);
        const double g = W.gc[b];
        double* hb = h[b & 1];
        hb[0] = fma(g, xv, hb[0]);
        hb[1] = fma(g, yv, hb[1]);
        hb[2] = fma(g, xv * xv, hb[2]);
        hb[3] = fma(g, yv * yv, hb[3]);
        hb[4] = fma(g, xv * yv, hb[4]);
    }
#pragma unroll
    for (int f = 0; f < 5; ++f) H[f * tot + idx] = h[0][f] + h[1][f];
}

template <int KR_>
__global__ void __launch_bounds__(PT) k_ssim_v(const double* __restrict__ H, int m, int zc, Win W,
                                              int vr, int vc, double c1, double c2,
                                              double* __restrict__ D, double* __restrict__ part,
                                              const int* halt) {
    if (halted(halt)) return;
    __shared__ double red[PT / 32];
    const int64_t idx = blockIdx.x * (int64_t)PT + threadIdx.x;
    const int64_t tot = (int64_t)vr * vc * zc;      // outputs
    const int64_t htot = (int64_t)m * vc * zc;      // H field stride
    const int64_t rstride = (int64_t)vc * zc;       // one row of H
    double s = 0.0;
    if (idx < tot) {
        const int kr = ktaps<KR_>(W.kr);
        const double* h0 = H + idx;   // row i of H has the same (j, zl) offset
        double a[2][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
#pragma unroll
        for (int t = 0; t < (KR_ > 0 ? KR_ : KMAX); ++t) {
            if (KR_ == 0 && t >= kr) break;
            const double g = W.gr[t];
            double* at = a[t & 1];
#pragma unroll
            for (int f = 0; f < 5; ++f) at[f] = fma(g, h0[f * htot + t * rstride], at[f]);
        }
        const double mx = a[0][0] + a[1][0], my = a[0][1] + a[1][1], x2w = a[0][2] + a[1][2],
                     y2w = a[0][3] + a[1][3], xyw = a[0][4] + a[1][4];
        const double sx2 = x2w - mx * mx, sy2 = y2w - my * my, sxy = xyw - mx * my;
        const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * sxy + c2;
        const double b1 = mx * mx + my * my + c1, b2 = sx2 + sy2 + c2;
        const double inv = 1.0 / (b1 * b2);   // 1/b1 = b2*inv, 1/b2 = b1*inv
        s = (a1 * a2) * inv;
        D[idx] = (2.0 * my * (a2 - a1)) * inv - 2.0 * mx * s * ((b2 - b1) * inv);
        D[tot + idx] = -s * (b1 * inv);
        D[2 * tot + idx] = 2.0 * a1 * inv;
    }
    const double r = block_sum<PT>(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}

template <int KC_>
__global__ void __launch_bounds__(PT) k_ssim_gh(const double* __restrict__ D, int n, int zc, Win W,
                                               int vr, int vc, double* __restrict__ T,
                                               const int* halt) {
    if (halted(halt)) return;
    const int64_t idx = blockIdx.x * (int64_t)PT + threadIdx.x;
    const int64_t tot = (int64_t)vr * n * zc;
    if (idx >= tot) return;
    const int zl = (int)(idx % zc);
    const int64_t is = idx / zc;
    const int s = (int)(is % n), i = (int)(is / n);
    const int kc = ktaps<KC_>(W.kc);
    const int64_t dtot = (int64_t)vr * vc * zc;
    const int blo = max(0, s - vc + 1), bhi = min(kc - 1, s);
    const double* d0 = D + ((int64_t)i * vc + s) * zc + zl;   // column jj = s - b
    double t[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int b = 0; b < (KC_ > 0 ? KC_ : KMAX); ++b) {
        if (KC_ == 0 && b >= kc) break;
        if (b < blo || b > bhi) continue;
        const double g = W.gc[b];
        const double* q = d0 - (int64_t)b * zc;
        double* tb = t[b & 1];
        tb[0] = fma(g, q[0], tb[0]);
        tb[1] = fma(g, q[dtot], tb[1]);
        tb[2] = fma(g, q[2 * dtot], tb[2]);
    }
    T[idx] = t[0][0] + t[1][0];
    T[tot + idx] = t[0][1] + t[1][1];
    T[2 * tot + idx] = t[0][2] + t[1][2];
}

template <int KR_>
__global__ void __launch_bounds__(PT) k_loss_gv(const float* __restrict__ X, const float* __restrict__ Y,
                                               const double* __restrict__ T, int m, int n, int p,
                                               int z0, int zc, Win W, int vr, int vc, double l1w,
                                               double l1_count, double ssw, double ssim_slices,
                                               float* __restrict__ G, double* __restrict__ part,
                                               const int* halt) {
    if (halted(halt)) return;
    __shared__ double red[PT / 32];
    const int64_t idx = blockIdx.x * (int64_t)PT + threadIdx.x;
    const int64_t tot = (int64_t)m * n * zc;
    double l1 = 0.0;
    if (idx < tot) {
        const int zl = (int)(idx % zc);
        const int64_t rs = idx / zc;
        const int s = (int)(rs % n), r = (int)(rs / n);
        const int64_t gi = rs * p + z0 + zl;
        const double xv = (double)__ldg(X + gi), yv = (double)__ldg(Y + gi);
        const double diff = xv - yv;
        l1 = fabs(diff);
        double g = 0.0;
        if (l1w > 0.0) g += l1w * ((double)((diff > 0) - (diff < 0)) / l1_count);
        if (ssw > 0.0) {
            const int kr = ktaps<KR_>(W.kr);
            const int64_t ttot = (int64_t)vr * n * zc;
            const int64_t rstride = (int64_t)n * zc;
            const int alo = max(0, r - vr + 1), ahi = min(kr - 1, r);
            const double* t0 = T + ((int64_t)r * n + s) * zc + zl;   // row i = r - a
            double A[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
            for (int a = 0; a < (KR_ > 0 ? KR_ : KMAX); ++a) {
                if (KR_ == 0 && a >= kr) break;
                if (a < alo || a > ahi) continue;
                const double gg = W.gr[a];
                const double* q = t0 - (int64_t)a * rstride;
                double* Aa = A[a & 1];
                Aa[0] = fma(gg, q[0], Aa[0]);
                Aa[1] = fma(gg, q[ttot], Aa[1]);
                Aa[2] = fma(gg, q[2 * ttot], Aa[2]);
            }
            double gs = A[0][0] + A[1][0];
            gs += 2.0 * xv * (A[0][1] + A[1][1]);
            gs += yv * (A[0][2] + A[1][2]);
            gs *= 1.0 / ((double)vr * (double)vc);
            g += ssw * (-gs / ssim_slices);
        }
        G[gi] = (float)g;
    }
    const double rr = block_sum<PT>(l1, red);
    if (threadIdx.x == 0) part[blockIdx.x] = rr;
}

__global__ void __launch_bounds__(1024) k_sino_max(const float* __restrict__ x, int64_t count,
                                                   double* __restrict__ out) {
    __shared__ float sh[32];
    float mv = -INFINITY;
    for (int64_t i = threadIdx.x; i < count; i += 1024) mv = fmaxf(mv, x[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mv;
    __syncthreads();
    if (threadIdx.x < 32) {
        mv = sh[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, o));
        if (threadIdx.x == 0) out[0] = (double)mv;
    }
}

__global__ void __launch_bounds__(256) k_sq_diff(const float* __restrict__ x,
                                                 const float* __restrict__ y, int64_t count,
                                                 double* __restrict__ part) {
    __shared__ double red[8];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < count; i += (int64_t)gridDim.x * 256) {
        const double d = (double)x[i] - (double)y[i];
        acc += d * d;
    }
    const double r = block_sum<256>(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void k_iter_finalize(const double* __restrict__ sums, double l1w, double ssw,
                                double tvw, double l1_count, double ssim_count, double tv_count,
                                double lr0, double lrf, int64_t max_iters, int64_t* step,
                                int64_t* iter, double* trace, int64_t trace_cap, double* adam,
                                int* halt) {
    if (*halt) return;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    const double l1 = l1w > 0 ? sums[0] / l1_count : nan;
    const double ss = ssw > 0 ? 1.0 - sums[1] / ssim_count : nan;
    const double tv = tvw > 0 ? sums[2] / tv_count : nan;
    double value = 0.0;
    if (l1w > 0) value += l1w * l1;
    if (ssw > 0) value += ssw * ss;
    if (tvw > 0) value += tvw * tv;
    const int64_t it = *iter;
    if (it < trace_cap) {
        trace[4 * it + 0] = value;
        trace[4 * it + 1] = l1;
        trace[4 * it + 2] = ss;
        trace[4 * it + 3] = tv;
    }
    if (!isfinite(value)) {
        *halt = 1;
        return;
    }
    const int64_t st = *step;
    const double T = (double)(max_iters > 1 ? max_iters : 1);
    const double frac = (double)(st < max_iters ? st : max_iters) / T;
    adam[0] = lr0 * pow(lrf / lr0, frac);
    adam[1] = 1.0 - pow(0.9, (double)(st + 1));
    adam[2] = 1.0 - pow(0.999, (double)(st + 1));
    *step = st + 1;
    *iter = it + 1;
}

__global__ void k_adam(double* __restrict__ P, const double* __restrict__ G,
                       double* __restrict__ M1, double* __restrict__ M2, int64_t n,
                       const double* __restrict__ adam, double sfloor, double sceil,
                       const int* halt) {
    if (halted(halt)) return;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= 5 * n) return;
    const double lr = adam[0], bc1 = adam[1], bc2 = adam[2];
    const double g = G[idx];
    const double m = 0.9 * M1[idx] + (1.0 - 0.9) * g;
    const double v = 0.999 * M2[idx] + (1.0 - 0.999) * g * g;
    double p = P[idx] - lr * (m / bc1) / (sqrt(v / bc2) + 1e-8);
    const int64_t row = idx / n;
    if (row == 3) p = fmin(fmax(p, sfloor), sceil);
    if (row == 4) p = fmax(p, 0.0);
    M1[idx] = m;
    M2[idx] = v;
    P[idx] = p;
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_loss_workspace_bytes(int m, int n, int p, size_t* bytes) {
    *bytes = loss_layout(m, n, p).total;
    return SPLATCT_OK;
}

int splatct_sino_max(const float* x, int64_t count, double* out, void* stream) {
    k_sino_max<<<1, 1024, 0, as_stream(stream)>>>(x, count, out);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_loss_fused(const float* pred, const float* ref, int m, int n, int p, double lmax,
                       double lambda1, double lambda2, double l1_count, double ssim_slices,
                       float* grad_pred, void* ws, size_t ws_bytes, double* sums,
                       const int* halt, void* stream) {
    SPLATCT_REQUIRE(m > 0 && n > 0 && p > 0, "invalid sinogram dims");
    LossLayout L = loss_layout(m, n, p);
    SPLATCT_REQUIRE(ws_bytes >= L.total, "loss workspace too small");
    cudaStream_t s = as_stream(stream);
    Win W = make_win(m, n);
    if (!(lmax > 0.0)) lmax = 1.0;
    const double c1 = (0.01 * lmax) * (0.01 * lmax), c2 = (0.03 * lmax) * (0.03 * lmax);
    char* base = reinterpret_cast<char*>(ws);
    double* H = reinterpret_cast<double*>(base + L.o_H);
    double* D = reinterpret_cast<double*>(base + L.o_D);
    double* T = reinterpret_cast<double*>(base + L.o_T);
    double* ps = reinterpret_cast<double*>(base + L.o_ps);
    double* pl = reinterpret_cast<double*>(base + L.o_pl);
    const bool k11 = W.kr == 11 && W.kc == 11;
    if (L.nchunks > 1 && p % L.zc != 0) {   // short last chunk leaves unused partial slots
        SPLATCT_CK(cudaMemsetAsync(ps, 0, sizeof(double) * L.nb_v * L.nchunks, s));
        SPLATCT_CK(cudaMemsetAsync(pl, 0, sizeof(double) * L.nb_g * L.nchunks, s));
    }
    for (int ci = 0; ci < L.nchunks; ++ci) {
        const int z0 = ci * L.zc, zc = min(L.zc, p - z0);
        if (lambda2 > 0.0) {
            const unsigned g1 = (unsigned)(((int64_t)m * L.vc * zc + 255) / 256);
            const unsigned g2 = (unsigned)(((int64_t)L.vr * L.vc * zc + 255) / 256);
            const unsigned g3 = (unsigned)(((int64_t)L.vr * n * zc + 255) / 256);
            if (k11) {
                k_ssim_h<11><<<g1, PT, 0, s>>>(pred, ref, m, n, p, z0, zc, W, L.vc, H, halt);
                SPLATCT_LAUNCH_CK();
                k_ssim_v<11><<<g2, PT, 0, s>>>(H, m, zc, W, L.vr, L.vc, c1, c2, D,
                                               ps + ci * L.nb_v, halt);
                SPLATCT_LAUNCH_CK();
                k_ssim_gh<11><<<g3, PT, 0, s>>>(D, n, zc, W, L.vr, L.vc, T, halt);
            } else {
                k_ssim_h<0><<<g1, PT, 0, s>>>(pred, ref, m, n, p, z0, zc, W, L.vc, H, halt);
                SPLATCT_LAUNCH_CK();
                k_ssim_v<0><<<g2, PT, 0, s>>>(H, m, zc, W, L.vr, L.vc, c1, c2, D,
                                              ps + ci * L.nb_v, halt);
                SPLATCT_LAUNCH_CK();
                k_ssim_gh<0><<<g3, PT, 0, s>>>(D, n, zc, W, L.vr, L.vc, T, halt);
            }
            SPLATCT_LAUNCH_CK();
        }
        const unsigned g4 = (unsigned)(((int64_t)m * n * zc + 255) / 256);
        if (k11)
            k_loss_gv<11><<<g4, PT, 0, s>>>(pred, ref, T, m, n, p, z0, zc, W, L.vr, L.vc, lambda1,
                                            l1_count, lambda2, ssim_slices, grad_pred,
                                            pl + ci * L.nb_g, halt);
        else
            k_loss_gv<0><<<g4, PT, 0, s>>>(pred, ref, T, m, n, p, z0, zc, W, L.vr, L.vc, lambda1,
                                           l1_count, lambda2, ssim_slices, grad_pred,
                                           pl + ci * L.nb_g, halt);
        SPLATCT_LAUNCH_CK();
    }
    if (lambda2 > 0.0) {
        if (int e = reduce_sum_f64(ps, L.nb_v * L.nchunks, sums + 1, s)) return e;
    } else {
        SPLATCT_CK(cudaMemsetAsync(sums + 1, 0, sizeof(double), s));
    }
    if (int e = reduce_sum_f64(pl, L.nb_g * L.nchunks, sums, s)) return e;
    return SPLATCT_OK;
}

int splatct_sum_sq_diff(const float* x, const float* y, int64_t count, double* ws, double* out,
                        void* stream) {
    cudaStream_t s = as_stream(stream);
    k_sq_diff<<<SPLATCT_SQDIFF_BLOCKS, 256, 0, s>>>(x, y, count, ws);
    SPLATCT_LAUNCH_CK();
    return reduce_sum_f64(ws, SPLATCT_SQDIFF_BLOCKS, out, s);
}

int splatct_iter_finalize(const double* sums, double lambda1, double lambda2, double lambda3,
                          double l1_count, double ssim_count, double tv_count, double lr0,
                          double lrf, int64_t max_iters, int64_t* step, int64_t* iter,
                          double* trace, int64_t trace_cap, double* adam, int* halt,
                          void* stream) {
    k_iter_finalize<<<1, 1, 0, as_stream(stream)>>>(sums, lambda1, lambda2, lambda3, l1_count,
                                                    ssim_count, tv_count, lr0, lrf, max_iters,
                                                    step, iter, trace, trace_cap, adam, halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_adam(double* params, const double* grads, double* m1, double* m2, int64_t n,
                 const double* adam, double sigma_floor, double sigma_ceiling, const int* halt,
                 void* stream) {
    if (n <= 0) return SPLATCT_OK;
    const int64_t tot = 5 * n;
    k_adam<<<(unsigned)((tot + 255) / 256), 256, 0, as_stream(stream)>>>(
        params, grads, m1, m2, n, adam, sigma_floor, sigma_ceiling, halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
