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
    int vr, vc;
    int64_t nblk_stats, nblk_grad;
    size_t o_D, o_ps, o_pl, total;
};

static LossLayout loss_layout(int m, int n, int p) {
    LossLayout L{};
    Win W = make_win(m, n);
    L.vr = m - W.kr + 1;
    L.vc = n - W.kc + 1;
    const int64_t zc = (p + LZ - 1) / LZ;
    L.nblk_stats = zc * ((L.vc + LCOL - 1) / LCOL);
    L.nblk_grad = zc * ((n + LCOL - 1) / LCOL);
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align_up(b > 0 ? b : 1); return o; };
    L.o_D = take(sizeof(double) * 3 * (size_t)L.vr * L.vc * p);
    L.o_ps = take(sizeof(double) * L.nblk_stats);
    L.o_pl = take(sizeof(double) * L.nblk_grad);
    L.total = off;
    return L;
}

// Pass 1: window statistics, SSIM map, derivative fields D (f64 [3][vr][vc][p]).
__global__ void __launch_bounds__(LNT) k_ssim_stats(const float* __restrict__ X,
                                                   const float* __restrict__ Y, int m, int n,
                                                   int p, Win W, double c1, double c2, int vr,
                                                   int vc, double* __restrict__ D,
                                                   double* __restrict__ part, const int* halt) {
    if (halted(halt)) return;
    extern __shared__ double ring[];   // [KMAX][5][LNT]
    __shared__ double red[LNT / 32];
    const int lane = threadIdx.x % LZ, cg = threadIdx.x / LZ;
    const int z = blockIdx.x * LZ + lane;
    const int j = blockIdx.y * LCOL + cg;
    const bool act = z < p && j < vc;
    double ssum = 0.0;
    const int kr = W.kr, kc = W.kc;
    for (int v = 0; v < m && act; ++v) {
        double h0 = 0, h1 = 0, h2 = 0, h3 = 0, h4 = 0;
        const int64_t rowb = ((int64_t)v * n + j) * p + z;
        for (int b = 0; b < kc; ++b) {
            const double xv = (double)__ldg(X + rowb + (int64_t)b * p);
            const double yv = (double)__ldg(Y + rowb + (int64_t)b * p);
            const double g = W.gc[b];
            h0 += g * xv;
            h1 += g * yv;
            h2 += g * (xv * xv);
            h3 += g * (yv * yv);
            h4 += g * (xv * yv);
        }
        const int slot = v % kr;
        double* rs = ring + (size_t)slot * 5 * LNT + threadIdx.x;
        rs[0 * LNT] = h0; rs[1 * LNT] = h1; rs[2 * LNT] = h2; rs[3 * LNT] = h3; rs[4 * LNT] = h4;
        if (v >= kr - 1) {
            const int i = v - kr + 1;
            double mx = 0, my = 0, x2w = 0, y2w = 0, xyw = 0;
            for (int a = 0; a < kr; ++a) {
                const double* q = ring + (size_t)((i + a) % kr) * 5 * LNT + threadIdx.x;
                const double g = W.gr[a];
                mx += g * q[0];
                my += g * q[LNT];
                x2w += g * q[2 * LNT];
                y2w += g * q[3 * LNT];
                xyw += g * q[4 * LNT];
            }
            const double sx2 = x2w - mx * mx, sy2 = y2w - my * my, sxy = xyw - mx * my;
            const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * sxy + c2;
            const double b1 = mx * mx + my * my + c1, b2 = sx2 + sy2 + c2;
            const double s = (a1 * a2) / (b1 * b2);
            ssum += s;
            const double dmx = (2.0 * my * (a2 - a1)) / (b1 * b2) - 2.0 * mx * s * (1.0 / b1 - 1.0 / b2);
            const double dx2 = -s / b2;
            const double dxy = 2.0 * a1 / (b1 * b2);
            const int64_t plane = (int64_t)vr * vc * p;
            const int64_t o = ((int64_t)i * vc + j) * p + z;
            D[o] = dmx;
            D[plane + o] = dx2;
            D[2 * plane + o] = dxy;
        }
    }
    const double r = block_sum<LNT>(ssum, red);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// Pass 2: transposed correlation of D, SSIM gradient, L1 term, f32 store.
__global__ void __launch_bounds__(LNT) k_loss_grad(const float* __restrict__ X,
                                                  const float* __restrict__ Y, int m, int n,
                                                  int p, Win W, int vr, int vc,
                                                  const double* __restrict__ D, double l1w,
                                                  double l1_count, double ssw, double ssim_slices,
                                                  float* __restrict__ G,
                                                  double* __restrict__ part, const int* halt) {
    if (halted(halt)) return;
    extern __shared__ double ring[];   // [KMAX][3][LNT]
    __shared__ double red[LNT / 32];
    const int lane = threadIdx.x % LZ, cg = threadIdx.x / LZ;
    const int z = blockIdx.x * LZ + lane;
    const int s = blockIdx.y * LCOL + cg;
    const bool act = z < p && s < n;
    const int kr = W.kr, kc = W.kc;
    const int64_t plane = (int64_t)vr * vc * p;
    const double inv_val = 1.0 / ((double)vr * (double)vc);
    double l1sum = 0.0;
    for (int r = 0; r < m && act; ++r) {
        if (ssw > 0.0 && r < vr) {
            double t0 = 0, t1 = 0, t2 = 0;
            for (int b = 0; b < kc; ++b) {
                const int jj = s - b;
                if (jj < 0 || jj >= vc) continue;
                const int64_t o = ((int64_t)r * vc + jj) * p + z;
                const double g = W.gc[b];
                t0 += g * D[o];
                t1 += g * D[plane + o];
                t2 += g * D[2 * plane + o];
            }
            double* rs = ring + (size_t)(r % kr) * 3 * LNT + threadIdx.x;
            rs[0] = t0; rs[LNT] = t1; rs[2 * LNT] = t2;
        }
        const int64_t idx = ((int64_t)r * n + s) * p + z;
        const double xv = (double)__ldg(X + idx), yv = (double)__ldg(Y + idx);
        const double diff = xv - yv;
        l1sum += fabs(diff);
        double g = 0.0;
        if (l1w > 0.0) g += l1w * ((double)((diff > 0) - (diff < 0)) / l1_count);
        if (ssw > 0.0) {
            double A1 = 0, A2 = 0, A3 = 0;
            for (int a = 0; a < kr; ++a) {
                const int i = r - a;
                if (i < 0 || i >= vr) continue;
                const double* q = ring + (size_t)(i % kr) * 3 * LNT + threadIdx.x;
                const double gg = W.gr[a];
                A1 += gg * q[0];
                A2 += gg * q[LNT];
                A3 += gg * q[2 * LNT];
            }
            double gs = A1;
            gs += 2.0 * xv * A2;
            gs += yv * A3;
            gs *= inv_val;
            g += ssw * (-gs / ssim_slices);
        }
        G[idx] = (float)g;
    }
    const double rr = block_sum<LNT>(l1sum, red);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = rr;
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
    double* D = reinterpret_cast<double*>(base + L.o_D);
    double* ps = reinterpret_cast<double*>(base + L.o_ps);
    double* pl = reinterpret_cast<double*>(base + L.o_pl);
    const unsigned zc = (unsigned)((p + LZ - 1) / LZ);
    if (lambda2 > 0.0) {
        const size_t sm = sizeof(double) * KMAX * 5 * LNT;
        static bool attr_set = false;
        if (!attr_set) {
            SPLATCT_CK(cudaFuncSetAttribute(k_ssim_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)sm));
            attr_set = true;
        }
        dim3 grid(zc, (unsigned)((L.vc + LCOL - 1) / LCOL));
        k_ssim_stats<<<grid, LNT, sm, s>>>(pred, ref, m, n, p, W, c1, c2, L.vr, L.vc, D, ps, halt);
        SPLATCT_LAUNCH_CK();
        if (int e = reduce_sum_f64(ps, L.nblk_stats, sums + 1, s)) return e;
    } else {
        SPLATCT_CK(cudaMemsetAsync(sums + 1, 0, sizeof(double), s));
    }
    {
        const size_t sm = sizeof(double) * KMAX * 3 * LNT;
        dim3 grid(zc, (unsigned)((n + LCOL - 1) / LCOL));
        k_loss_grad<<<grid, LNT, sm, s>>>(pred, ref, m, n, p, W, L.vr, L.vc, D, lambda1, l1_count,
                                          lambda2, ssim_slices, grad_pred, pl, halt);
        SPLATCT_LAUNCH_CK();
        if (int e = reduce_sum_f64(pl, L.nblk_grad, sums, s)) return e;
    }
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
