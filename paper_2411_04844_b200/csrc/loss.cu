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
#include "tc.cuh"
#include "tmap.cuh"

namespace splatct {

constexpr int KMAX = 11;
// 11x11 fast path: output columns per block.  7 (224 threads) makes the C2
// grids 576 / 592 blocks = ~2 full waves of 2 CTAs x 148 SMs (8 gave 1.7).
constexpr int R_COLS = 7;
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
    int64_t nb_s11, nb_g11;   // blocks of the 11x11 row-walking kernels
    bool k11;
    size_t o_H, o_D, o_T, o_ps, o_pl, o_D11, o_RS, total;
};

constexpr int ZC = 64;    // slices per chunk (one block = 4 columns x ZC slices)
constexpr int PT = 256;   // threads per block

static LossLayout loss_layout(int m, int n, int p) {
    LossLayout L{};
    Win W = make_win(m, n);
    L.vr = m - W.kr + 1;
    L.vc = n - W.kc + 1;
    L.zc = p < ZC ? p : ZC;
    L.nchunks = (p + ZC - 1) / ZC;
    L.nb_v = (int64_t)((L.vr + 3) / 4) * L.vc;
    L.nb_g = (int64_t)((m + 3) / 4) * n;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align_up(b > 0 ? b : 1); return o; };
    L.k11 = W.kr == 11 && W.kc == 11 && p % 4 == 0;
    L.nb_s11 = (int64_t)((p + 31) / 32) * ((L.vc + R_COLS - 1) / R_COLS);
    L.nb_g11 = (int64_t)((p + 31) / 32) * ((n + R_COLS - 1) / R_COLS);
    if (L.k11) {   // row-walking kernels: full-p D, no H/T
        L.o_H = L.o_T = 0;
        // the three derivative fields in f32: every statistic and the SSIM value
        // are f64 (the cancellation is in sigma^2 = E[x^2] - mu^2, done before
        // the store); the fields only feed the linear adjoint correlation
        L.o_D11 = take(sizeof(float) * 3 * (size_t)L.vr * L.vc * p);
        L.o_D = L.o_D11;
        L.o_RS = take(sizeof(double) * 2 * (size_t)L.vr * L.vc * p);   // ref window stats
        L.o_ps = take(sizeof(double) * L.nb_s11);
        L.o_pl = take(sizeof(double) * L.nb_g11);
    } else {
        L.o_H = take(sizeof(double) * 5 * (size_t)m * L.vc * ZC);
        L.o_D = take(sizeof(double) * 3 * (size_t)L.vr * L.vc * ZC);
        L.o_T = take(sizeof(double) * 3 * (size_t)L.vr * n * ZC);
        L.o_ps = take(sizeof(double) * L.nb_v * L.nchunks);
        L.o_pl = take(sizeof(double) * L.nb_g * L.nchunks);
    }
    L.total = off;
    return L;
}

// ---------------------------------------------------------------------------
// Four separable passes, processed per chunk of ZC = 64 slices so the f64
// intermediates (H, D, T) of a chunk stay L2-resident:
//   S1  H[5][m][vc][ZC]  = row-direction window sums of x, y, x^2, y^2, xy
//   S2  D[3][vr][vc][ZC] = column-direction sums -> SSIM map and its
//                          derivative fields (d_mx, d_x2w, d_xyw), sum of SSIM
//   G1  T[3][vr][n][ZC]  = transposed row correlation of D
//   G2  grad[m][n][p]    = transposed column correlation of T, combined with
//                          x, y and the L1 sign term; sum |x - y|
// (loss.py:83-141: _valid_corr / _valid_corr_adjoint / _ssim_slice).
// A block computes 4 consecutive outputs along the filtered axis for 64
// slices; it first stages the 4 + 10 input positions it needs in shared
// memory (coalesced 256 B rows), so every tap is an immediate-offset LDS and
// each input value is read from L2 once per block instead of 11 times.
// Tap loops keep two partial sums (even / odd taps) to halve DFMA chains.
// ---------------------------------------------------------------------------
constexpr int OB = 4;            // outputs per block along the filtered axis
constexpr int SPAN = OB + KMAX - 1;

template <int K>
__device__ __forceinline__ int ktaps(int k) { return K > 0 ? K : k; }

// S1: block (row v, columns j0..j0+3); stage x, y columns j0..j0+13.
template <int KC_>
__global__ void __launch_bounds__(PT) k_ssim_h(const float* __restrict__ X, const float* __restrict__ Y,
                                              int m, int n, int p, int z0, int zc, Win W, int vc,
                                              double* __restrict__ H, const int* halt) {
    if (halted(halt)) return;
    __shared__ float sx[SPAN][ZC], sy[SPAN][ZC];
    const int zl = threadIdx.x & (ZC - 1), o = threadIdx.x / ZC;
    const int j0 = blockIdx.x * OB, v = blockIdx.y;
    const int kc = ktaps<KC_>(W.kc);
    const int ncol = min(OB + kc - 1, n - j0);
    for (int e = threadIdx.x; e < SPAN * ZC; e += PT) {
        const int cidx = e / ZC, z = e & (ZC - 1);
        float xv = 0.f, yv = 0.f;
        if (cidx < ncol && z < zc) {
            const int64_t gi = ((int64_t)v * n + j0 + cidx) * p + z0 + z;
            xv = __ldg(X + gi);
            yv = __ldg(Y + gi);
        }
        sx[cidx][z] = xv;
        sy[cidx][z] = yv;
    }
    __syncthreads();
    const int j = j0 + o;
    if (zl >= zc || j >= vc) return;
    double h[2][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
#pragma unroll
    for (int b = 0; b < (KC_ > 0 ? KC_ : KMAX); ++b) {
        if (KC_ == 0 && b >= kc) break;
        const double xv = (double)sx[o + b][zl];
        const double yv = (double)sy[o + b][zl];
        const double g = W.gc[b];
        double* hb = h[b & 1];
        hb[0] = fma(g, xv, hb[0]);
        hb[1] = fma(g, yv, hb[1]);
        hb[2] = fma(g, xv * xv, hb[2]);
        hb[3] = fma(g, yv * yv, hb[3]);
        hb[4] = fma(g, xv * yv, hb[4]);
    }
    const int64_t tot = (int64_t)m * vc * ZC;
    const int64_t idx = ((int64_t)v * vc + j) * ZC + zl;
#pragma unroll
    for (int f = 0; f < 5; ++f) H[f * tot + idx] = h[0][f] + h[1][f];
}

// S2: block (rows i0..i0+3, column j); stage H rows i0..i0+13 of column j.
template <int KR_>
__global__ void __launch_bounds__(PT) k_ssim_v(const double* __restrict__ H, int m, int zc, Win W,
                                              int vr, int vc, double c1, double c2,
                                              double* __restrict__ D, double* __restrict__ part,
                                              const int* halt) {
    if (halted(halt)) return;
    __shared__ double sh[5][SPAN][ZC];
    __shared__ double red[PT / 32];
    const int zl = threadIdx.x & (ZC - 1), o = threadIdx.x / ZC;
    const int i0 = blockIdx.x * OB, j = blockIdx.y;
    const int kr = ktaps<KR_>(W.kr);
    const int nrow = min(OB + kr - 1, m - i0);
    const int64_t htot = (int64_t)m * vc * ZC;
    for (int e = threadIdx.x; e < SPAN * ZC; e += PT) {
        const int r = e / ZC, z = e & (ZC - 1);
        const int64_t hi = ((int64_t)(i0 + r) * vc + j) * ZC + z;
#pragma unroll
        for (int f = 0; f < 5; ++f) sh[f][r][z] = (r < nrow && z < zc) ? H[f * htot + hi] : 0.0;
    }
    __syncthreads();
    const int i = i0 + o;
    double s = 0.0;
    if (zl < zc && i < vr) {
        double a[2][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
#pragma unroll
        for (int t = 0; t < (KR_ > 0 ? KR_ : KMAX); ++t) {
            if (KR_ == 0 && t >= kr) break;
            const double g = W.gr[t];
            double* at = a[t & 1];
#pragma unroll
            for (int f = 0; f < 5; ++f) at[f] = fma(g, sh[f][o + t][zl], at[f]);
        }
        const double mx = a[0][0] + a[1][0], my = a[0][1] + a[1][1], x2w = a[0][2] + a[1][2],
                     y2w = a[0][3] + a[1][3], xyw = a[0][4] + a[1][4];
        const double sx2 = x2w - mx * mx, sy2 = y2w - my * my, sxy = xyw - mx * my;
        const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * sxy + c2;
        const double b1 = mx * mx + my * my + c1, b2 = sx2 + sy2 + c2;
        const double inv = 1.0 / (b1 * b2);   // 1/b1 = b2*inv, 1/b2 = b1*inv
        s = (a1 * a2) * inv;
        const int64_t tot = (int64_t)vr * vc * ZC;
        const int64_t idx = ((int64_t)i * vc + j) * ZC + zl;
        D[idx] = (2.0 * my * (a2 - a1)) * inv - 2.0 * mx * s * ((b2 - b1) * inv);
        D[tot + idx] = -s * (b1 * inv);
        D[2 * tot + idx] = 2.0 * a1 * inv;
    }
    const double r = block_sum<PT>(s, red);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// G1: block (row i, columns s0..s0+3); stage D columns s0-10..s0+3 of row i
// (zero outside [0, vc)).  T[i][s] = sum_b gc[b] D[i][s-b].
template <int KC_>
__global__ void __launch_bounds__(PT) k_ssim_gh(const double* __restrict__ D, int n, int zc, Win W,
                                               int vr, int vc, double* __restrict__ T,
                                               const int* halt) {
    if (halted(halt)) return;
    __shared__ double sd[3][SPAN][ZC];
    const int zl = threadIdx.x & (ZC - 1), o = threadIdx.x / ZC;
    const int s0 = blockIdx.x * OB, i = blockIdx.y;
    const int kc = ktaps<KC_>(W.kc);
    const int base = s0 - (kc - 1);   // staged column q holds D column base + q
    const int64_t dtot = (int64_t)vr * vc * ZC;
    for (int e = threadIdx.x; e < SPAN * ZC; e += PT) {
        const int q = e / ZC, z = e & (ZC - 1);
        const int jj = base + q;
        const bool ok = q < OB + kc - 1 && jj >= 0 && jj < vc && z < zc;
        const int64_t di = ((int64_t)i * vc + jj) * ZC + z;
#pragma unroll
        for (int f = 0; f < 3; ++f) sd[f][q][z] = ok ? D[f * dtot + di] : 0.0;
    }
    __syncthreads();
    const int s = s0 + o;
    if (zl >= zc || s >= n) return;
    double t[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int b = 0; b < (KC_ > 0 ? KC_ : KMAX); ++b) {
        if (KC_ == 0 && b >= kc) break;
        const double g = W.gc[b];
        const int q = o + (kc - 1) - b;   // column s - b
        double* tb = t[b & 1];
#pragma unroll
        for (int f = 0; f < 3; ++f) tb[f] = fma(g, sd[f][q][zl], tb[f]);
    }
    const int64_t tot = (int64_t)vr * n * ZC;
    const int64_t idx = ((int64_t)i * n + s) * ZC + zl;
    T[idx] = t[0][0] + t[1][0];
    T[tot + idx] = t[0][1] + t[1][1];
    T[2 * tot + idx] = t[0][2] + t[1][2];
}

// G2: block (rows r0..r0+3, column s); stage T rows r0-10..r0+3 of column s
// (zero outside [0, vr)).  A_f[r] = sum_a gr[a] T_f[r-a].
template <int KR_>
__global__ void __launch_bounds__(PT) k_loss_gv(const float* __restrict__ X, const float* __restrict__ Y,
                                               const double* __restrict__ T, int m, int n, int p,
                                               int z0, int zc, Win W, int vr, int vc, double l1w,
                                               double l1_count, double ssw, double ssim_slices,
                                               float* __restrict__ G, double* __restrict__ part,
                                               const int* halt) {
    if (halted(halt)) return;
    __shared__ double st[3][SPAN][ZC];
    __shared__ double red[PT / 32];
    const int zl = threadIdx.x & (ZC - 1), o = threadIdx.x / ZC;
    const int r0 = blockIdx.x * OB, s = blockIdx.y;
    const int kr = ktaps<KR_>(W.kr);
    if (ssw > 0.0) {
        const int base = r0 - (kr - 1);
        const int64_t ttot = (int64_t)vr * n * ZC;
        for (int e = threadIdx.x; e < SPAN * ZC; e += PT) {
            const int q = e / ZC, z = e & (ZC - 1);
            const int ii = base + q;
            const bool ok = q < OB + kr - 1 && ii >= 0 && ii < vr && z < zc;
            const int64_t ti = ((int64_t)ii * n + s) * ZC + z;
#pragma unroll
            for (int f = 0; f < 3; ++f) st[f][q][z] = ok ? T[f * ttot + ti] : 0.0;
        }
        __syncthreads();
    }
    const int r = r0 + o;
    double l1 = 0.0;
    if (zl < zc && r < m) {
        const int64_t gi = ((int64_t)r * n + s) * p + z0 + zl;
        const double xv = (double)__ldg(X + gi), yv = (double)__ldg(Y + gi);
        const double diff = xv - yv;
        l1 = fabs(diff);
        double g = 0.0;
        if (l1w > 0.0) g += l1w * ((double)((diff > 0) - (diff < 0)) / l1_count);
        if (ssw > 0.0) {
            double A[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
            for (int a = 0; a < (KR_ > 0 ? KR_ : KMAX); ++a) {
                if (KR_ == 0 && a >= kr) break;
                const double gg = W.gr[a];
                const int q = o + (kr - 1) - a;   // row r - a
                double* Aa = A[a & 1];
#pragma unroll
                for (int f = 0; f < 3; ++f) Aa[f] = fma(gg, st[f][q][zl], Aa[f]);
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
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = rr;
}

// ---------------------------------------------------------------------------
// 11 x 11 window fast path (the default: every image with >= 11 views and
// detectors, p % 4 == 0).  A block owns 32 slices x R_COLS output columns and
// walks the view axis.  Input rows (R_COLS + 10 columns x 32 slices) are gathered with
// cp.async into a 3-deep shared-memory ring two rows ahead of the compute, and
// the last 11 rows of horizontal window sums live in REGISTERS: the row loop
// is unrolled by 11 so every ring slot is a compile-time index.  f64
// throughout like loss.py:112-141.
// ---------------------------------------------------------------------------
constexpr int R_SPAN = R_COLS + 10;       // staged input columns
constexpr int R_NT = 32 * R_COLS;
constexpr int R_AHEAD = 2;                // rows staged ahead of the compute (3 measured no faster)
constexpr int R_BUF = R_AHEAD + 1;        // staging ring depth
constexpr int G_AHEAD = 2;                // gradient kernel (48 KB static smem bound)
constexpr int G_BUF = G_AHEAD + 1;

__device__ __forceinline__ void cp16_zfill(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit_group() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Each thread issues (and later converts) the same 16-byte chunks of every
// staged row, so the f32 landing buffer is private per chunk: only the
// converted f64 row (read by 11 neighbouring columns) needs a barrier.
constexpr int S_CHUNKS = 2 * R_SPAN * 8;                  // x, y: R_SPAN columns x 8 chunks
constexpr int S_SLOTS = (S_CHUNKS + R_NT - 1) / R_NT;      // chunks per thread

// MODE 0: all five window moments from X and Y (loss.py:112-141).
// MODE 1: the reference-only moments (mean_y, E[y^2]) are read from RS, the
//         per-window statistics of the measured sinogram computed once per
//         run (MODE 2), so the per-iteration pass carries three fields.
// MODE 2: writes RS = {mean_y, E[y^2]} per valid window (X unused).
// Tensor maps of the stats kernel's row loads (use = 0: cp.async path).
struct StatMaps {
    CUtensorMap x, y, rs;   // X, Y [m][n][p] box {32, R_SPAN, 1}; RS [2][vr][vc][p] f64 box {32, R_COLS, 1, 2}
    int use;
};
constexpr unsigned S_ROWBYTES = R_SPAN * 32 * 4;       // one x or y box
constexpr unsigned S_RSBYTES = 2 * R_COLS * 32 * 8;    // one RS box

template <int MODE>
__global__ void __launch_bounds__(R_NT, MODE == 1 ? 2 : 1) k_ssim_stats11(const float* __restrict__ X,
                                                          const float* __restrict__ Y, int m, int n,
                                                          int p, Win W, double c1, double c2,
                                                          int vr, int vc, float* __restrict__ D,
                                                          double* __restrict__ part,
                                                          double* __restrict__ RS,
                                                          const __grid_constant__ StatMaps tm,
                                                          const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    constexpr int NF = MODE == 0 ? 5 : (MODE == 1 ? 3 : 2);   // ring fields
    // landing ring (f32), read in place: one slot more than the staging depth,
    // so a row is rewritten only after every warp has passed the barrier that
    // follows its last read
    constexpr int S_BUF = R_BUF + 1;
    __shared__ __align__(128) float sf[S_BUF][2][R_SPAN][32];
    // MODE 1: the reference window moments of an output row, staged with the
    // input rows (4 slots: a slot is rewritten two barriers after its read)
    constexpr int RS_BUF = R_AHEAD + 2;
    static_assert(RS_BUF == S_BUF, "one mbarrier per slot covers both rings");
    __shared__ __align__(128) double srs[MODE == 1 ? RS_BUF : 1][2][MODE == 1 ? R_COLS : 1][32];
    __shared__ double red[R_NT / 32];
    // TMA path: thread 0 loads a row's boxes (x, y, and in MODE 1 the reference
    // moments of output row v - 10) behind the slot's mbarrier; the tensor
    // maps zero-fill columns and slices outside the sinogram
    // ("full", count 1 + bytes) and released by every warp ("empty", count
    // R_COLS) once it has read the slot, so warps never meet at a block
    // barrier: thread 0 re-issues a slot only after all warps released it
    __shared__ __align__(8) uint64_t sbar[S_BUF], ebar[S_BUF];
    if (tm.use) {
        if (threadIdx.x == 0) {
            for (int b = 0; b < S_BUF; ++b) {
                tc::mbar_init(&sbar[b], 1);
                tc::mbar_init(&ebar[b], R_COLS);
            }
            tc::mbar_init_fence();
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, cl = threadIdx.x >> 5;
    const int zb = blockIdx.x * 32, j0 = blockIdx.y * R_COLS;
    const int z = zb + lane, j = j0 + cl;
    const bool act = z < p && j < vc;
    const int64_t plane = (int64_t)vr * vc * p;
    const int64_t rowstride = (int64_t)n * p;
    // per-thread chunk table (fixed for every row)
    int64_t goff[S_SLOTS];
    int soff[S_SLOTS];
    bool gok[S_SLOTS], mine[S_SLOTS];
#pragma unroll
    for (int k = 0; k < S_SLOTS; ++k) {
        const int e = threadIdx.x + k * R_NT;
        mine[k] = e < S_CHUNKS;
        const int arr = e / (R_SPAN * 8), rem = e % (R_SPAN * 8);
        const int col = rem >> 3, q = rem & 7;
        gok[k] = mine[k] && j0 + col < n && zb + 4 * q < p;
        goff[k] = gok[k] ? (int64_t)(j0 + col) * p + zb + 4 * q : 0;
        soff[k] = (arr * R_SPAN + col) * 32 + 4 * q;     // within one [2][R_SPAN][32] row
        if (arr) goff[k] = -goff[k] - 1;                  // sign selects Y
        if (MODE == 2 && !arr) mine[k] = false;           // ref-only: no X rows
    }
    // MODE 1 staging of RS: thread t copies 16 bytes (two slices) of one
    // (field, column) row segment: 2 fields x R_COLS columns x 16 chunks
    const int rs_f = threadIdx.x / (R_COLS * 16), rs_c = (threadIdx.x / 16) % R_COLS,
              rs_q = threadIdx.x % 16;
    const bool rs_ok = MODE == 1 && rs_f < 2 && j0 + rs_c < vc && zb + 2 * rs_q < p;
    auto issue_tma = [&](int v) {   // thread 0
        if (v >= m) return;
        const int slot = v % S_BUF, u = v - 10;
        const bool rs = MODE == 1 && u >= 0 && u < vr;
        const unsigned bar = tc::smem_u32(&sbar[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                     "r"((MODE == 2 ? 1u : 2u) * S_ROWBYTES + (rs ? S_RSBYTES : 0u))
                     : "memory");
        if (MODE != 2)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tc::smem_u32(&sf[slot][0][0][0])),
                "l"(&tm.x), "r"(zb), "r"(j0), "r"(v), "r"(bar)
                : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tc::smem_u32(&sf[slot][1][0][0])),
            "l"(&tm.y), "r"(zb), "r"(j0), "r"(v), "r"(bar)
            : "memory");
        if (rs)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(tc::smem_u32(&srs[slot][0][0][0])),
                "l"(&tm.rs), "r"(zb), "r"(j0), "r"(u), "r"(0), "r"(bar)
                : "memory");
    };
    auto issue = [&](int v) {
        if (tm.use) {
            if (threadIdx.x == 0) issue_tma(v);
            return;
        }
        if (MODE == 1) {   // reference moments of output row v - 10 (needed at iteration v)
            const int u = v - 10;
            if (u >= 0 && u < vr && rs_f < 2) {
                const double* src =
                    rs_ok ? RS + rs_f * plane + ((int64_t)u * vc + j0 + rs_c) * p + zb + 2 * rs_q
                          : RS;
                cp16_zfill(&srs[v % RS_BUF][rs_f][rs_c][2 * rs_q], src, rs_ok);
            }
        }
        if (v < m) {
            float* buf = &sf[v % S_BUF][0][0][0];
#pragma unroll
            for (int k = 0; k < S_SLOTS; ++k) {
                if (!mine[k]) continue;
                const bool isy = goff[k] < 0;
                const int64_t o = isy ? -goff[k] - 1 : goff[k];
                const float* src = (isy ? Y : X) + (gok[k] ? v * rowstride + o : 0);
                cp16_zfill(buf + soff[k], src, gok[k]);
            }
        }
        cp_commit_group();
    };
#pragma unroll
    for (int q = 0; q < R_AHEAD; ++q) issue(q);
    double ring[11][NF];
    double ssum = 0.0;
    for (int v0 = 0; v0 < m; v0 += 11) {
#pragma unroll
        for (int ph = 0; ph < 11; ++ph) {
            const int v = v0 + ph;
            if (v >= m) break;
            if (tm.use) {
                tc::mbar_wait(&sbar[v % S_BUF], (uint32_t)(v / S_BUF) & 1u);   // row v landed
                const int w = v + R_AHEAD;   // next row to stage: its slot held row w - 4
                if (threadIdx.x == 0 && w < m) {
                    if (w >= S_BUF)
                        tc::mbar_wait(&ebar[w % S_BUF], (uint32_t)(w / S_BUF - 1) & 1u);
                    issue_tma(w);
                }
            } else {
                cp_wait_group<R_AHEAD - 1>();   // my chunks of row v landed (later rows in flight)
                issue(v + R_AHEAD);   // slot (v+2) % 4: last read at row v-2, before the previous barrier
                __syncthreads();      // row v complete in shared memory
            }
            // MODE 1: the reference window moments of output row v-10, loaded
            // before the row's arithmetic so their latency overlaps it
            double rs_my = 0.0, rs_y2 = 0.0;
            if (MODE == 1 && v >= 10 && act) {   // staged with row v (cp.async, barrier above)
                rs_my = srs[v % RS_BUF][0][cl][lane];
                rs_y2 = srs[v % RS_BUF][1][cl][lane];
            }
            const float* xr = &sf[v % S_BUF][0][cl][lane];
            const float* yr = &sf[v % S_BUF][1][cl][lane];
            double h[2][NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) h[0][f] = h[1][f] = 0.0;
#pragma unroll
            for (int b = 0; b < 11; ++b) {
                double* hb = h[b & 1];
                const double yv = (double)yr[32 * b];
                if (MODE == 2) {          // {y, y^2}
                    const double gy = W.gc[b] * yv;
                    hb[0] += gy;
                    hb[1] = fma(gy, yv, hb[1]);
                } else {
                    const double xv = (double)xr[32 * b];
                    const double gx = W.gc[b] * xv;
                    hb[0] += gx;                       // x
                    hb[1] = fma(gx, xv, hb[1]);        // x^2
                    hb[2] = fma(gx, yv, hb[2]);        // xy
                    if (MODE == 0) {
                        const double gy = W.gc[b] * yv;
                        hb[3] += gy;                   // y
                        hb[4] = fma(gy, yv, hb[4]);    // y^2
                    }
                }
            }
#pragma unroll
            for (int f = 0; f < NF; ++f) ring[ph][f] = h[0][f] + h[1][f];
            if (tm.use) {   // this warp is done with slot v % 4 (rows and moments)
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&ebar[v % S_BUF]);
            }
            if (v >= 10 && act) {
                double a[2][NF];
#pragma unroll
                for (int f = 0; f < NF; ++f) a[0][f] = a[1][f] = 0.0;
#pragma unroll
                for (int t = 0; t < 11; ++t) {   // row v-10+t lives in slot (ph+1+t) % 11
                    const double g = W.gr[t];
                    double* at = a[t & 1];
#pragma unroll
                    for (int f = 0; f < NF; ++f) at[f] = fma(g, ring[(ph + 1 + t) % 11][f], at[f]);
                }
                const int64_t o = ((int64_t)(v - 10) * vc + j) * p + z;
                if (MODE == 2) {
                    RS[o] = a[0][0] + a[1][0];
                    RS[plane + o] = a[0][1] + a[1][1];
                } else {
                    const double mx = a[0][0] + a[1][0], x2w = a[0][1] + a[1][1],
                                 xyw = a[0][2] + a[1][2];
                    const double my = MODE == 0 ? a[0][3] + a[1][3] : rs_my;
                    const double y2w = MODE == 0 ? a[0][4] + a[1][4] : rs_y2;
                    const double sx2 = x2w - mx * mx, sy2 = y2w - my * my, sxy = xyw - mx * my;
                    const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * sxy + c2;
                    const double b1 = mx * mx + my * my + c1, b2 = sx2 + sy2 + c2;
                    const double inv = 1.0 / (b1 * b2);   // 1/b1 = b2*inv, 1/b2 = b1*inv
                    const double s = (a1 * a2) * inv;
                    ssum += s;
                    D[o] = (float)((2.0 * my * (a2 - a1)) * inv - 2.0 * mx * s * ((b2 - b1) * inv));
                    D[plane + o] = (float)(-s * (b1 * inv));
                    D[2 * plane + o] = (float)(2.0 * a1 * inv);
                }
            }
        }
    }
    if (!tm.use) cp_wait_group<0>();
    if (MODE != 2) {
        const double r = block_sum<R_NT>(ssum, red);
        if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = r;
    }
}

constexpr int G_DCHUNKS = 3 * R_SPAN * 8;                    // D (f32): 3 fields x 17 cols x 8
constexpr int G_DSLOTS = (G_DCHUNKS + R_NT - 1) / R_NT;
constexpr int G_XCHUNKS = 2 * R_COLS * 8;                    // x, y: R_COLS cols x 8 chunks

// The staged rows of the gradient kernel (bytes): D fields 3 x R_SPAN x 32 f32,
// x and y R_COLS x 32 f32 each -- also the TMA boxes' sizes.
constexpr unsigned G_DBYTES = 3 * R_SPAN * 32 * 4;
constexpr unsigned G_XBYTES = R_COLS * 32 * 4;

// Tensor maps of the gradient kernel's row loads (use = 0: cp.async path).
struct GradMaps {
    CUtensorMap d, x, y;   // D [3][vr][vc][p] box {32, R_SPAN, 1, 3}; X, Y [m][n][p] box {32, R_COLS, 1}
    int use;
};

__global__ void __launch_bounds__(R_NT, 2) k_loss_grad11(const float* __restrict__ X,
                                                         const float* __restrict__ Y, int m, int n,
                                                         int p, Win W, int vr, int vc,
                                                         const float* __restrict__ D, double l1w,
                                                         double l1_count, double ssw,
                                                         double ssim_slices, float* __restrict__ G,
                                                         double* __restrict__ part,
                                                         const __grid_constant__ GradMaps tm,
                                                         const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    float gcf[11];   // the column window in f32 for the horizontal adjoint pass
#pragma unroll
    for (int b = 0; b < 11; ++b) gcf[b] = (float)W.gc[b];
    // per staged row: D columns s0-10 .. s0+7 (3 fields) and x, y columns s0 .. s0+7
    __shared__ __align__(128) float sd[G_BUF][3][R_SPAN][32];
    __shared__ __align__(128) float sxy[G_BUF][2][R_COLS][32];
    __shared__ double red[R_NT / 32];
    // TMA path: one thread loads a row's three boxes (D fields, x, y) behind a
    // per-buffer mbarrier instead of 224 threads issuing 16-byte cp.async chunks;
    // the tensor maps zero-fill columns and slices outside the sinogram
    __shared__ __align__(8) uint64_t gbar[G_BUF];
    if (tm.use) {
        if (threadIdx.x == 0) {
            for (int b = 0; b < G_BUF; ++b) tc::mbar_init(&gbar[b], 1);
            tc::mbar_init_fence();
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, cl = threadIdx.x >> 5;
    const int zb = blockIdx.x * 32, s0 = blockIdx.y * R_COLS;
    const int z = zb + lane, s = s0 + cl;
    const bool act = z < p && s < n;
    const int64_t plane = (int64_t)vr * vc * p;
    const bool ss = ssw > 0.0;
    // constant factors of loss.py:64-74 (sign / count) and the SSIM chain rule
    const double l1f = l1w > 0.0 ? l1w / l1_count : 0.0;
    const double ssf = ss ? -ssw / (ssim_slices * (double)vr * (double)vc) : 0.0;
    int64_t dgo[G_DSLOTS];
    int dso[G_DSLOTS];
    bool dok[G_DSLOTS], dmine[G_DSLOTS];
#pragma unroll
    for (int k = 0; k < G_DSLOTS; ++k) {
        const int e = threadIdx.x + k * R_NT;
        dmine[k] = e < G_DCHUNKS;
        const int f = e / (R_SPAN * 8), rem = e % (R_SPAN * 8);
        const int col = rem >> 3, q = rem & 7;
        const int jj = s0 - 10 + col;
        dok[k] = dmine[k] && jj >= 0 && jj < vc && zb + 4 * q < p;
        dgo[k] = dok[k] ? f * plane + (int64_t)jj * p + zb + 4 * q : 0;
        dso[k] = (f * R_SPAN + col) * 32 + 4 * q;
    }
    const bool xmine = threadIdx.x < G_XCHUNKS;
    const int xarr = threadIdx.x / (R_COLS * 8), xrem = threadIdx.x % (R_COLS * 8);
    const int xcol = xrem >> 3, xq = xrem & 7;
    const bool xok = xmine && s0 + xcol < n && zb + 4 * xq < p;
    const int64_t xgo = xok ? (int64_t)(s0 + xcol) * p + zb + 4 * xq : 0;
    const float* xsrc = xarr ? Y : X;
    const int64_t drow = (int64_t)vc * p, xrowstride = (int64_t)n * p;
    auto issue_tma = [&](int r) {   // thread 0
        if (r >= m) return;
        const int buf = r % G_BUF;
        const bool dr = ss && r < vr;
        const unsigned bar = tc::smem_u32(&gbar[buf]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                     "r"((dr ? G_DBYTES : 0u) + 2u * G_XBYTES)
                     : "memory");
        if (dr)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(tc::smem_u32(&sd[buf][0][0][0])),
                "l"(&tm.d), "r"(zb), "r"(s0 - 10), "r"(r), "r"(0), "r"(bar)
                : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tc::smem_u32(&sxy[buf][0][0][0])),
            "l"(&tm.x), "r"(zb), "r"(s0), "r"(r), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(tc::smem_u32(&sxy[buf][1][0][0])),
            "l"(&tm.y), "r"(zb), "r"(s0), "r"(r), "r"(bar)
            : "memory");
    };
    auto issue = [&](int r) {
        if (tm.use) {
            if (threadIdx.x == 0) issue_tma(r);
            return;
        }
        if (r < m) {
            const int buf = r % G_BUF;
            if (ss && r < vr) {
                float* db = &sd[buf][0][0][0];
#pragma unroll
                for (int k = 0; k < G_DSLOTS; ++k)
                    if (dmine[k]) cp16_zfill(db + dso[k], D + (dok[k] ? r * drow + dgo[k] : 0), dok[k]);
            }
            if (xmine)
                cp16_zfill(&sxy[buf][xarr][xcol][4 * xq], xsrc + (xok ? r * xrowstride + xgo : 0), xok);
        }
        cp_commit_group();
    };
#pragma unroll
    for (int q = 0; q < G_AHEAD; ++q) issue(q);
    double ring[11][3];
#pragma unroll
    for (int q = 0; q < 11; ++q) ring[q][0] = ring[q][1] = ring[q][2] = 0.0;
    double l1sum = 0.0;
    for (int r0 = 0; r0 < m; r0 += 11) {
#pragma unroll
        for (int ph = 0; ph < 11; ++ph) {
            const int r = r0 + ph;
            if (r >= m) break;
            if (tm.use)
                tc::mbar_wait(&gbar[r % G_BUF], (uint32_t)(r / G_BUF) & 1u);   // row r landed
            else
                cp_wait_group<G_AHEAD - 1>();
            __syncthreads();   // and every warp is past row r - 1: its buffer is free
            issue(r + G_AHEAD);
            const int buf = r % G_BUF;
            if (ss && r < vr) {
                // the derivative fields are f32 already: their 11-tap horizontal
                // correlation runs on the FP32 pipe (two interleaved partial sums,
                // ~1e-7 relative), widened once per field for the f64 vertical pass
                float t[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
#pragma unroll
                for (int b = 0; b < 11; ++b) {    // column s - b = staged column cl + 10 - b
                    const float g = gcf[b];
                    float* tb = t[b & 1];
#pragma unroll
                    for (int f = 0; f < 3; ++f)
                        tb[f] = fmaf(g, sd[buf][f][cl + 10 - b][lane], tb[f]);
                }
#pragma unroll
                for (int f = 0; f < 3; ++f) ring[ph][f] = (double)t[0][f] + (double)t[1][f];
            } else {
#pragma unroll
                for (int f = 0; f < 3; ++f) ring[ph][f] = 0.0;   // rows >= vr contribute 0
            }
            if (act) {
                const double xv = (double)sxy[buf][0][cl][lane];
                const double yv = (double)sxy[buf][1][cl][lane];
                const double diff = xv - yv;
                l1sum += fabs(diff);
                double g = l1f * (double)((diff > 0) - (diff < 0));
                if (ss) {
                    // row r - a lives in slot (ph - a) mod 11; rows < 0 are the zeroed slots
                    double A[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
                    for (int a = 0; a < 11; ++a) {
                        const double gg = W.gr[a];
                        double* Aa = A[a & 1];
#pragma unroll
                        for (int f = 0; f < 3; ++f) Aa[f] = fma(gg, ring[(ph - a + 11) % 11][f], Aa[f]);
                    }
                    double gs = A[0][0] + A[1][0];
                    gs += 2.0 * xv * (A[0][1] + A[1][1]);
                    gs += yv * (A[0][2] + A[1][2]);
                    g += ssf * gs;
                }
                G[((int64_t)r * n + s) * p + z] = (float)g;
            }
        }
    }
    if (!tm.use) cp_wait_group<0>();   // TMA: rows >= m are never issued, all issued were waited
    const double rr = block_sum<R_NT>(l1sum, red);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = rr;
}

// Tensor maps for k_ssim_stats11 (X may be null in MODE 2; RS only in MODE 1).
static StatMaps stat_maps(const float* X, const float* Y, const double* RS, int m, int n, int p,
                          int vr, int vc) {
    StatMaps g;
    memset(&g, 0, sizeof(g));
    const cuuint64_t fp = (cuuint64_t)p * 4;
    const cuuint64_t xdim[3] = {(cuuint64_t)p, (cuuint64_t)n, (cuuint64_t)m};
    const cuuint64_t xstr[2] = {fp, fp * n};
    const cuuint32_t xbox[3] = {32, R_SPAN, 1};
    const cuuint64_t rdim[4] = {(cuuint64_t)p, (cuuint64_t)vc, (cuuint64_t)vr, 2};
    const cuuint64_t rstr[3] = {2 * fp, 2 * fp * vc, 2 * fp * vc * vr};
    const cuuint32_t rbox[4] = {32, R_COLS, 1, 2};
    bool ok = encode_tiled(&g.y, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, xdim, xstr, xbox,
                           CU_TENSOR_MAP_SWIZZLE_NONE);
    if (ok && X)
        ok = encode_tiled(&g.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, xdim, xstr, xbox,
                          CU_TENSOR_MAP_SWIZZLE_NONE);
    if (ok && RS)
        ok = encode_tiled(&g.rs, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, RS, rdim, rstr, rbox,
                          CU_TENSOR_MAP_SWIZZLE_NONE);
    g.use = ok;
    return g;
}

// Tensor maps for k_loss_grad11 (p % 4 == 0 and 16-byte aligned bases: the
// k11 path's requirements); use = 0 when TMA is unavailable.
static GradMaps grad_maps(const float* X, const float* Y, const float* D, int m, int n, int p,
                          int vr, int vc) {
    GradMaps g;
    const cuuint64_t fp = (cuuint64_t)p * 4;
    const cuuint64_t ddim[4] = {(cuuint64_t)p, (cuuint64_t)vc, (cuuint64_t)vr, 3};
    const cuuint64_t dstr[3] = {fp, fp * vc, fp * vc * vr};
    const cuuint32_t dbox[4] = {32, R_SPAN, 1, 3};
    const cuuint64_t xdim[3] = {(cuuint64_t)p, (cuuint64_t)n, (cuuint64_t)m};
    const cuuint64_t xstr[2] = {fp, fp * n};
    const cuuint32_t xbox[3] = {32, R_COLS, 1};
    g.use = encode_tiled(&g.d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, D, ddim, dstr, dbox,
                         CU_TENSOR_MAP_SWIZZLE_NONE) &&
            encode_tiled(&g.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, xdim, xstr, xbox,
                         CU_TENSOR_MAP_SWIZZLE_NONE) &&
            encode_tiled(&g.y, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, xdim, xstr, xbox,
                         CU_TENSOR_MAP_SWIZZLE_NONE);
    return g;
}

// max(x) over count floats: per-block maxima (grid-stride, 16 B loads), then
// a single-block max.  NaN-free input (the sinogram is validated finite).
__global__ void __launch_bounds__(256) k_sino_max_part(const float* __restrict__ x, int64_t count,
                                                       float* __restrict__ part) {
    __shared__ float sh[8];
    float mv = -INFINITY;
    const int64_t n4 = ((uintptr_t)x % 16 == 0) ? count / 4 : 0;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n4; i += (int64_t)gridDim.x * 256) {
        const float4 v = x4[i];
        mv = fmaxf(mv, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (int64_t i = 4 * n4 + blockIdx.x * 256 + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * 256)
        mv = fmaxf(mv, x[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mv;
    __syncthreads();
    if (threadIdx.x < 32) {
        mv = threadIdx.x < 8 ? sh[threadIdx.x] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, o));
        if (threadIdx.x == 0) part[blockIdx.x] = mv;
    }
}

__global__ void k_sino_max_final(const float* __restrict__ part, int n, double* __restrict__ out) {
    float mv = -INFINITY;
    for (int i = threadIdx.x; i < n; i += 32) mv = fmaxf(mv, part[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, o));
    if (threadIdx.x == 0) out[0] = (double)mv;
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

// Optional first stage (one 1024-thread block, Part.n[f] > 0): sums[f] is
// reduced here from the block partials the loss and the adjoint left, in the
// fixed order of k_reduce_sum (bitwise its result), saving three launches.
struct FinParts {
    const double* p[3];   // l1, ssim, tv partials (or null: sums[f] is final)
    int64_t n[3];
    double* scratch;      // FIN_BLOCKS x 3 block sums, then a ticket word (zero between calls)
    const double* sched;  // optional {lr, 1-b1^t, 1-b2^t} per pre-increment step (host-computed)
    int64_t sched_len;
};
#ifndef FIN_BLOCKS_N
#define FIN_BLOCKS_N 32
#endif
constexpr int FIN_BLOCKS = FIN_BLOCKS_N, FIN_NT = 256;

__global__ void k_iter_finalize(double* __restrict__ sums, FinParts parts, double l1w,
                                double ssw, double tvw, double l1_count, double ssim_count,
                                double tv_count, double lr0, double lrf, int64_t max_iters,
                                int64_t* step, int64_t* iter, double* trace, int64_t trace_cap,
                                double* adam, int* halt) {
    griddep_wait();
    if (*halt) return;
    if (parts.scratch != nullptr) {
        // FIN_BLOCKS blocks each sum a fixed slice of every partial array, the
        // last block to finish combines the block sums in block order
        // (deterministic whichever block is last) and does the bookkeeping
        __shared__ double sh[FIN_NT / 32];
        __shared__ bool last;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            if (parts.p[f] == nullptr) continue;   // uniform
            const int64_t per = (parts.n[f] + FIN_BLOCKS - 1) / FIN_BLOCKS;
            const int64_t lo = blockIdx.x * per, hi = min(parts.n[f], lo + per);
            double a0 = 0.0, a1 = 0.0;
            int64_t i = lo + threadIdx.x;
            for (; i + FIN_NT < hi; i += 2 * FIN_NT) {
                a0 += parts.p[f][i];
                a1 += parts.p[f][i + FIN_NT];
            }
            if (i < hi) a0 += parts.p[f][i];
            const double r = block_sum<FIN_NT>(a0 + a1, sh);
            if (threadIdx.x == 0) parts.scratch[f * FIN_BLOCKS + blockIdx.x] = r;
        }
        if (threadIdx.x == 0) {
            __threadfence();
            unsigned* ticket = reinterpret_cast<unsigned*>(parts.scratch + 3 * FIN_BLOCKS);
            last = atomicAdd(ticket, 1u) == FIN_BLOCKS - 1;
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        __shared__ double bs[3 * FIN_BLOCKS];   // the block sums, loaded in parallel
        if (threadIdx.x < 3 * FIN_BLOCKS)
            bs[threadIdx.x] = reinterpret_cast<volatile double*>(parts.scratch)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x != 0) return;
        for (int f = 0; f < 3; ++f) {
            if (parts.p[f] == nullptr) continue;
            double t = 0.0;
            for (int b = 0; b < FIN_BLOCKS; ++b) t += bs[f * FIN_BLOCKS + b];
            sums[f] = t;
        }
        *reinterpret_cast<unsigned*>(parts.scratch + 3 * FIN_BLOCKS) = 0u;   // next call
    } else if (threadIdx.x != 0) {
        return;
    }
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
    if (parts.sched != nullptr && st >= 0 && st < parts.sched_len) {
        // the schedule as the reference computes it on the host (Python float
        // powers, optim.py:88-90, 123-126), tabulated once per run
        adam[0] = parts.sched[3 * st];
        adam[1] = parts.sched[3 * st + 1];
        adam[2] = parts.sched[3 * st + 2];
    } else {
        const double T = (double)(max_iters > 1 ? max_iters : 1);
        const double frac = (double)(st < max_iters ? st : max_iters) / T;
        adam[0] = lr0 * pow(lrf / lr0, frac);
        adam[1] = 1.0 - pow(0.9, (double)(st + 1));
        adam[2] = 1.0 - pow(0.999, (double)(st + 1));
    }
    *step = st + 1;
    *iter = it + 1;
}

__global__ void k_adam(double* __restrict__ P, const double* __restrict__ G,
                       double* __restrict__ M1, double* __restrict__ M2, int64_t n,
                       const double* __restrict__ adam, double sfloor, double sceil,
                       const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= 5 * n) return;
    adam_elem(P, G, M1, M2, idx, (int)(idx / n), adam[0], adam[1], adam[2], sfloor, sceil);
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_loss_workspace_bytes(int m, int n, int p, size_t* bytes) {
    *bytes = loss_layout(m, n, p).total;
    return SPLATCT_OK;
}

int splatct_sino_max(const float* x, int64_t count, double* out, void* stream) {
    // out[1 ..] is scratch for the per-block maxima (caller passes
    // double[1 + SPLATCT_SQDIFF_BLOCKS])
    cudaStream_t s = as_stream(stream);
    float* part = reinterpret_cast<float*>(out + 1);
    k_sino_max_part<<<SPLATCT_SQDIFF_BLOCKS, 256, 0, s>>>(x, count, part);
    SPLATCT_LAUNCH_CK();
    k_sino_max_final<<<1, 32, 0, s>>>(part, SPLATCT_SQDIFF_BLOCKS, out);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"

static int loss_fused_impl(const float* pred, const float* ref, int m, int n, int p, double lmax,
                           double lambda1, double lambda2, double l1_count, double ssim_slices,
                           float* grad_pred, void* ws, size_t ws_bytes, double* sums,
                           const int* halt, void* stream, bool prepared, bool defer = false) {
    // defer: leave the block partials in ws (splatct_loss_partials) for
    // splatct_iter_finalize_partials to reduce, instead of two reduce launches
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
    const bool k11 = L.k11;
    if (k11) {
        float* D11 = reinterpret_cast<float*>(base + L.o_D11);
        const dim3 gs((p + 31) / 32, (L.vc + R_COLS - 1) / R_COLS),
            gg((p + 31) / 32, (n + R_COLS - 1) / R_COLS);
        if (lambda2 > 0.0) {
            double* RS = reinterpret_cast<double*>(base + L.o_RS);
            if (prepared)
                SPLATCT_CK(launch_pdl(k_ssim_stats11<1>, gs, dim3(R_NT), 0, s, pred, ref, m, n, p,
                                      W, c1, c2, L.vr, L.vc, D11, ps, RS,
                                      stat_maps(pred, ref, RS, m, n, p, L.vr, L.vc), halt));
            else
                k_ssim_stats11<0><<<gs, R_NT, 0, s>>>(pred, ref, m, n, p, W, c1, c2, L.vr, L.vc,
                                                      D11, ps, RS,
                                                      stat_maps(pred, ref, nullptr, m, n, p,
                                                                L.vr, L.vc),
                                                      halt);
            SPLATCT_LAUNCH_CK();
            if (!defer)
                if (int e = reduce_sum_f64(ps, L.nb_s11, sums + 1, s)) return e;
        } else {
            SPLATCT_CK(cudaMemsetAsync(sums + 1, 0, sizeof(double), s));
        }
        const GradMaps gm = grad_maps(pred, ref, D11, m, n, p, L.vr, L.vc);
        SPLATCT_CK(launch_pdl(k_loss_grad11, gg, dim3(R_NT), 0, s, pred, ref, m, n, p, W, L.vr,
                              L.vc, D11, lambda1, l1_count, lambda2, ssim_slices, grad_pred, pl,
                              gm, halt));
        SPLATCT_LAUNCH_CK();
        return defer ? SPLATCT_OK : reduce_sum_f64(pl, L.nb_g11, sums, s);
    }
    for (int ci = 0; ci < L.nchunks; ++ci) {
        const int z0 = ci * ZC, zc = min(ZC, p - z0);
        if (lambda2 > 0.0) {
            const dim3 g1((L.vc + 3) / 4, m), g2((L.vr + 3) / 4, L.vc), g3((n + 3) / 4, L.vr);
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
        const dim3 g4((m + 3) / 4, n);
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
        if (!defer)
            if (int e = reduce_sum_f64(ps, L.nb_v * L.nchunks, sums + 1, s)) return e;
    } else {
        SPLATCT_CK(cudaMemsetAsync(sums + 1, 0, sizeof(double), s));
    }
    if (!defer)
        if (int e = reduce_sum_f64(pl, L.nb_g * L.nchunks, sums, s)) return e;
    return SPLATCT_OK;
}

// TV terms across a z-slab boundary, added after the fact (the slab's adjoint
// ran without halo planes, so the halo exchange overlaps it; loss.py:183-207):
// the forward difference into the upper neighbour's first plane is owned by
// this slab -- value |hi - v[c-1]| and subgradient -sign(hi - v[c-1]) at
// plane c-1 -- and the lower neighbour's difference into plane 0 contributes
// +sign(v[0] - lo) there.  One block, fixed order: deterministic; the value
// is added to *tv_sum.
__global__ void __launch_bounds__(1024) k_tv_halo_fixup(const float* __restrict__ vol,
                                                        float* __restrict__ dl,
                                                        const float* __restrict__ lo,
                                                        const float* __restrict__ hi, int64_t npix,
                                                        int c, double coef,
                                                        double* __restrict__ tv_sum,
                                                        const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t p = threadIdx.x; p < npix; p += blockDim.x) {
        const int64_t col = p * c;
        if (hi) {
            const float v = vol[col + c - 1];
            const float d = hi[p] - v;
            acc += fabs((double)d);
            const float sg = (float)((d > 0.f) - (d < 0.f));
            dl[col + c - 1] = (float)fma(-(double)sg, coef, (double)dl[col + c - 1]);
        }
        if (lo) {
            const float d = vol[col] - lo[p];
            const float sg = (float)((d > 0.f) - (d < 0.f));
            dl[col] = (float)fma((double)sg, coef, (double)dl[col]);
        }
    }
    const double r = block_sum<1024>(acc, red);
    if (threadIdx.x == 0 && hi) *tv_sum += r;
}

extern "C" {

int splatct_loss_fused(const float* pred, const float* ref, int m, int n, int p, double lmax,
                       double lambda1, double lambda2, double l1_count, double ssim_slices,
                       float* grad_pred, void* ws, size_t ws_bytes, double* sums,
                       const int* halt, void* stream) {
    return loss_fused_impl(pred, ref, m, n, p, lmax, lambda1, lambda2, l1_count, ssim_slices,
                           grad_pred, ws, ws_bytes, sums, halt, stream, false);
}

int splatct_loss_prepare_ref(const float* ref, int m, int n, int p, void* ws, size_t ws_bytes,
                             void* stream) {
    SPLATCT_REQUIRE(m > 0 && n > 0 && p > 0, "invalid sinogram dims");
    LossLayout L = loss_layout(m, n, p);
    SPLATCT_REQUIRE(ws_bytes >= L.total, "loss workspace too small");
    if (!L.k11) return SPLATCT_OK;   // the generic path recomputes everything
    Win W = make_win(m, n);
    char* base = reinterpret_cast<char*>(ws);
    const dim3 gs((p + 31) / 32, (L.vc + R_COLS - 1) / R_COLS);
    k_ssim_stats11<2><<<gs, R_NT, 0, as_stream(stream)>>>(
        nullptr, ref, m, n, p, W, 0.0, 0.0, L.vr, L.vc, nullptr, nullptr,
        reinterpret_cast<double*>(base + L.o_RS),
        stat_maps(nullptr, ref, nullptr, m, n, p, L.vr, L.vc), nullptr);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_loss_fused_prepared(const float* pred, const float* ref, int m, int n, int p,
                                double lmax, double lambda1, double lambda2, double l1_count,
                                double ssim_slices, float* grad_pred, void* ws, size_t ws_bytes,
                                double* sums, const int* halt, void* stream) {
    return loss_fused_impl(pred, ref, m, n, p, lmax, lambda1, lambda2, l1_count, ssim_slices,
                           grad_pred, ws, ws_bytes, sums, halt, stream, true);
}

int splatct_sum_sq_diff(const float* x, const float* y, int64_t count, double* ws, double* out,
                        void* stream) {
    cudaStream_t s = as_stream(stream);
    k_sq_diff<<<SPLATCT_SQDIFF_BLOCKS, 256, 0, s>>>(x, y, count, ws);
    SPLATCT_LAUNCH_CK();
    return reduce_sum_f64(ws, SPLATCT_SQDIFF_BLOCKS, out, s);
}

int splatct_tv_halo_fixup(const float* vol_yxz, float* dl_yxz, const float* halo_lo,
                          const float* halo_hi, int w, int h, int c, double lambda_tv,
                          double tv_count, double* tv_sum, const int* halt, void* stream) {
    if (!halo_lo && !halo_hi) return SPLATCT_OK;
    SPLATCT_CK(launch_pdl(k_tv_halo_fixup, dim3(1), dim3(1024), 0, as_stream(stream), vol_yxz,
                          dl_yxz, halo_lo, halo_hi, (int64_t)w * h, c,
                          tv_count > 0.0 ? lambda_tv / tv_count : 0.0, tv_sum, halt));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_iter_finalize(const double* sums, double lambda1, double lambda2, double lambda3,
                          double l1_count, double ssim_count, double tv_count, double lr0,
                          double lrf, int64_t max_iters, int64_t* step, int64_t* iter,
                          double* trace, int64_t trace_cap, double* adam, int* halt,
                          void* stream) {
    const FinParts none{{nullptr, nullptr, nullptr}, {0, 0, 0}, nullptr, nullptr, 0};
    SPLATCT_CK(launch_pdl(k_iter_finalize, dim3(1), dim3(1), 0, as_stream(stream),
                          const_cast<double*>(sums), none, lambda1, lambda2, lambda3, l1_count,
                          ssim_count, tv_count, lr0, lrf, max_iters, step, iter, trace, trace_cap,
                          adam, halt));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_iter_finalize_partials(double* sums, const double* l1_part, int64_t n_l1,
                                   const double* ssim_part, int64_t n_ssim,
                                   const double* tv_part, int64_t n_tv, double* scratch,
                                   const double* sched, int64_t sched_len, double lambda1,
                                   double lambda2, double lambda3, double l1_count,
                                   double ssim_count, double tv_count, double lr0, double lrf,
                                   int64_t max_iters, int64_t* step, int64_t* iter,
                                   double* trace, int64_t trace_cap, double* adam, int* halt,
                                   void* stream) {
    SPLATCT_REQUIRE(scratch != nullptr, "finalize scratch required");
    const FinParts parts{{n_l1 > 0 ? l1_part : nullptr, n_ssim > 0 ? ssim_part : nullptr,
                          n_tv > 0 ? tv_part : nullptr},
                         {n_l1, n_ssim, n_tv},
                         scratch,
                         sched_len > 0 ? sched : nullptr,
                         sched_len};
    SPLATCT_CK(launch_pdl(k_iter_finalize, dim3(FIN_BLOCKS), dim3(FIN_NT), 0, as_stream(stream), sums,
                          parts, lambda1, lambda2, lambda3, l1_count, ssim_count, tv_count, lr0,
                          lrf, max_iters, step, iter, trace, trace_cap, adam, halt));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_loss_partials(int m, int n, int p, double lambda2, void* ws, size_t ws_bytes,
                          const double** l1_part, int64_t* n_l1, const double** ssim_part,
                          int64_t* n_ssim) {
    SPLATCT_REQUIRE(m > 0 && n > 0 && p > 0, "invalid sinogram dims");
    LossLayout L = loss_layout(m, n, p);
    SPLATCT_REQUIRE(ws_bytes >= L.total, "loss workspace too small");
    char* base = reinterpret_cast<char*>(ws);
    *l1_part = reinterpret_cast<const double*>(base + L.o_pl);
    *n_l1 = L.k11 ? L.nb_g11 : L.nb_g * L.nchunks;
    *ssim_part = reinterpret_cast<const double*>(base + L.o_ps);
    *n_ssim = lambda2 > 0.0 ? (L.k11 ? L.nb_s11 : L.nb_v * L.nchunks) : 0;
    return SPLATCT_OK;
}

int splatct_loss_fused_prepared_deferred(const float* pred, const float* ref, int m, int n, int p,
                                         double lmax, double lambda1, double lambda2,
                                         double l1_count, double ssim_slices, float* grad_pred,
                                         void* ws, size_t ws_bytes, double* sums,
                                         const int* halt, void* stream) {
    return loss_fused_impl(pred, ref, m, n, p, lmax, lambda1, lambda2, l1_count, ssim_slices,
                           grad_pred, ws, ws_bytes, sums, halt, stream, true, true);
}

int splatct_adam(double* params, const double* grads, double* m1, double* m2, int64_t n,
                 const double* adam, double sigma_floor, double sigma_ceiling, const int* halt,
                 void* stream) {
    if (n <= 0) return SPLATCT_OK;
    const int64_t tot = 5 * n;
    SPLATCT_CK(launch_pdl(k_adam, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0,
                          as_stream(stream), params, grads, m1, m2, n, adam, sigma_floor,
                          sigma_ceiling, halt));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
