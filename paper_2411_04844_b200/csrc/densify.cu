// densify.cu -- adaptive density control (clone / split / prune) on the device.
//
// Restates densify.densify_and_prune (reference densify.py:86-147) and the
// Adam-moment remap (optim.py:92-106) so a densification event never moves
// the cloud through host memory:
//
//   classify   per Gaussian: avg = accum / iters; prune = sigma > 3 box
//              (| avg <= tau); hot = avg >= tau & !prune; clone / split
//              candidates by sigma <= theta (densify.py:97-110)
//   select     the k highest-avg candidates of a class (_limit,
//              densify.py:73-83) by an exact 4 x 16-bit radix select on the
//              f64 bits (avg > 0, so the bits order like the values)
//   apply      new cloud = [kept originals | clones | split children]
//              (densify.py:112-147) from three exclusive scans; clone
//              intensity x 0.5, children mu + noise * sigma (the host draws
//              the reference's numpy PCG64 normals, optim.py:394) and
//              sigma / cbrt 2; moments carried for survivors, zero otherwise.
//
// Arithmetic is the reference's f64 expression by expression (no FMA
// contraction), so the new cloud is bit-identical to the host restatement.
// Ties in avg exactly at the selection cut are broken by lower index (numpy's
// argsort there is an unstable introsort with unspecified tie order).
#include "common.cuh"

namespace splatct {

namespace {

enum : uint8_t { D_KEEP = 0, D_PRUNE = 1, D_CLONE_C = 2, D_SPLIT_C = 3, D_CLONE = 4, D_SPLIT = 5 };

constexpr int HBINS = 1 << 16;

struct SelState {
    unsigned long long prefix, mask;
    long long remaining;
};

struct DensifyLayout {
    size_t o_state, o_hist, o_flag, o_pos, o_scan, total;
};

DensifyLayout dlayout(int64_t n) {
    DensifyLayout L{};
    size_t off = 0;
    auto take = [&](size_t b) {
        const size_t o = off;
        off = align_up(off + b);
        return o;
    };
    L.o_state = take(sizeof(SelState));
    L.o_hist = take(sizeof(uint32_t) * HBINS);
    L.o_flag = take(sizeof(uint32_t) * 3 * (size_t)(n + 1));
    L.o_pos = take(sizeof(uint32_t) * 3 * (size_t)(n + 1));
    L.o_scan = take(scan_temp_bytes(n + 1));
    L.total = off;
    return L;
}

template <typename T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

__global__ void k_classify(const double* __restrict__ P, const double* __restrict__ accum,
                           int64_t n, double iters, double tau, double theta, double sigma_prune,
                           int grad_prune, uint8_t* __restrict__ cls,
                           unsigned long long* __restrict__ keys,
                           unsigned long long* __restrict__ counts) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    uint8_t c = D_KEEP;
    if (i < n) {
        const double avg = accum[i] / iters;
        const double sigma = P[3 * n + i];
        bool prune = sigma > sigma_prune;
        if (grad_prune) prune = prune || avg <= tau;
        const bool hot = avg >= tau && !prune;
        c = prune ? D_PRUNE : (hot ? (sigma <= theta ? D_CLONE_C : D_SPLIT_C) : D_KEEP);
        cls[i] = c;
        keys[i] = (unsigned long long)__double_as_longlong(avg);
    }
    // warp-aggregated integer counts (order-independent)
    const int lane = threadIdx.x & 31;
    const unsigned bp = __ballot_sync(0xffffffffu, c == D_PRUNE);
    const unsigned bc = __ballot_sync(0xffffffffu, c == D_CLONE_C);
    const unsigned bs = __ballot_sync(0xffffffffu, c == D_SPLIT_C);
    if (lane == 0) {
        if (bp) atomicAdd(&counts[0], (unsigned long long)__popc(bp));
        if (bc) atomicAdd(&counts[1], (unsigned long long)__popc(bc));
        if (bs) atomicAdd(&counts[2], (unsigned long long)__popc(bs));
    }
}

__global__ void k_sel_init(SelState* st, long long k) {
    st->prefix = 0ull;
    st->mask = 0ull;
    st->remaining = k;
}

// histogram of the next 16-bit digit of the still-matching candidates
__global__ void k_sel_hist(const uint8_t* __restrict__ cls,
                           const unsigned long long* __restrict__ keys, int64_t n, int which,
                           const SelState* __restrict__ st, int shift,
                           uint32_t* __restrict__ hist) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const unsigned long long pre = st->prefix, msk = st->mask;
    bool act = false;
    unsigned d = 0;
    if (i < n && cls[i] == which) {
        const unsigned long long k = keys[i];
        act = (k & msk) == pre;
        d = (unsigned)(k >> shift) & 0xffffu;
    }
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (!act) return;
    const unsigned peers = __match_any_sync(am, d);          // lanes sharing the digit
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[d], (uint32_t)__popc(peers));
}

// one block: find the digit holding the remaining-th largest key, narrow the
// prefix, and clear the histogram for the next pass
__global__ void __launch_bounds__(1024) k_sel_pick(SelState* __restrict__ st,
                                                   uint32_t* __restrict__ hist, int shift) {
    constexpr int PER = HBINS / 1024;
    __shared__ long long incl[1024];
    const int t = threadIdx.x;
    uint32_t mine[PER];
    long long s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        mine[j] = hist[t * PER + j];
        s += mine[j];
    }
    incl[t] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const long long v = t >= o ? incl[t - o] : 0;
        __syncthreads();
        incl[t] += v;
        __syncthreads();
    }
    const long long total = incl[1023];
    const long long above = total - incl[t];   // keys in higher bins than this thread's
    const long long rem = st->remaining;
    __syncthreads();
    if (above < rem && rem <= above + s) {     // exactly one thread
        long long acc = above;
        for (int j = PER - 1; j >= 0; --j) {
            if (rem <= acc + (long long)mine[j]) {
                st->remaining = rem - acc;
                st->prefix |= (unsigned long long)(t * PER + j) << shift;
                st->mask |= 0xffffull << shift;
                break;
            }
            acc += mine[j];
        }
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) hist[t * PER + j] = 0u;
}

__global__ void k_sel_ties(const uint8_t* __restrict__ cls,
                           const unsigned long long* __restrict__ keys, int64_t n, int which,
                           const SelState* __restrict__ st, uint32_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    flag[i] = (i < n && cls[i] == which && keys[i] == st->prefix) ? 1u : 0u;
}

__global__ void k_sel_mark(uint8_t* __restrict__ cls, const unsigned long long* __restrict__ keys,
                           int64_t n, int which, const SelState* __restrict__ st,
                           const uint32_t* __restrict__ tie_rank) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || cls[i] != which) return;
    const unsigned long long k = keys[i], thr = st->prefix;
    if (k > thr || (k == thr && (long long)tie_rank[i] < st->remaining))
        cls[i] = (uint8_t)(which + 2);
}

__global__ void k_mark_all(uint8_t* __restrict__ cls, int64_t n, int which) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && cls[i] == which) cls[i] = (uint8_t)(which + 2);
}

__global__ void k_apply_flags(const uint8_t* __restrict__ cls, int64_t n,
                              uint32_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const uint8_t c = i < n ? cls[i] : D_PRUNE;
    const int64_t s = n + 1;
    flag[i] = (i < n && c != D_PRUNE && c != D_SPLIT) ? 1u : 0u;
    flag[s + i] = c == D_CLONE ? 1u : 0u;
    flag[2 * s + i] = (i < n && c == D_SPLIT) ? 1u : 0u;
}

__global__ void k_apply(const double* __restrict__ P, const double* __restrict__ M1,
                        const double* __restrict__ M2, const uint8_t* __restrict__ cls,
                        const uint32_t* __restrict__ pos, const double* __restrict__ noise,
                        int64_t n, int64_t nn, double cbrt2, double* __restrict__ Q,
                        double* __restrict__ Q1, double* __restrict__ Q2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = n + 1;
    const uint8_t c = cls[i];
    if (c == D_PRUNE) return;
    const int64_t nkept = pos[n], nclone = pos[s + n];
    double p[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) p[r] = P[r * n + i];
    if (c == D_SPLIT) {
        const int64_t row = nkept + nclone + 2 * (int64_t)pos[2 * s + i];
        const double sg = __ddiv_rn(p[3], cbrt2);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const double* z = noise + (2 * (int64_t)pos[2 * s + i] + t) * 3;
#pragma unroll
            for (int a = 0; a < 3; ++a)
                Q[a * nn + row + t] = __dadd_rn(p[a], __dmul_rn(z[a], p[3]));
            Q[3 * nn + row + t] = sg;
            Q[4 * nn + row + t] = p[4];
#pragma unroll
            for (int r = 0; r < 5; ++r) {
                Q1[r * nn + row + t] = 0.0;
                Q2[r * nn + row + t] = 0.0;
            }
        }
        return;
    }
    if (c == D_CLONE) p[4] = __dmul_rn(p[4], 0.5);
    const int64_t row = pos[i];                               // kept original
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        Q[r * nn + row] = p[r];
        Q1[r * nn + row] = M1[r * n + i];
        Q2[r * nn + row] = M2[r * n + i];
    }
    if (c == D_CLONE) {
        const int64_t crow = nkept + pos[s + i];
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            Q[r * nn + crow] = p[r];
            Q1[r * nn + crow] = 0.0;
            Q2[r * nn + crow] = 0.0;
        }
    }
}

inline unsigned blocks(int64_t n, int nt = 256) { return (unsigned)((n + nt - 1) / nt); }

}  // namespace
}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_densify_workspace_bytes(int64_t n, size_t* bytes) {
    SPLATCT_REQUIRE(n >= 0 && bytes != nullptr, "densify_workspace_bytes: bad arguments");
    *bytes = dlayout(n).total;
    return SPLATCT_OK;
}

int splatct_densify_classify(const double* params, const double* accum, int64_t n, double iters,
                             double tau, double theta, double sigma_prune, int grad_prune,
                             uint8_t* cls, uint64_t* keys, uint64_t* counts, void* stream) {
    SPLATCT_REQUIRE(n >= 0 && iters > 0, "densify_classify: bad n / iters");
    cudaStream_t s = as_stream(stream);
    SPLATCT_CK(cudaMemsetAsync(counts, 0, 3 * sizeof(uint64_t), s));
    if (n == 0) return SPLATCT_OK;
    k_classify<<<blocks(n), 256, 0, s>>>(params, accum, n, iters, tau, theta, sigma_prune,
                                         grad_prune, cls,
                                         reinterpret_cast<unsigned long long*>(keys),
                                         reinterpret_cast<unsigned long long*>(counts));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_densify_select(uint8_t* cls, const uint64_t* keys, int64_t n, int which, int64_t k,
                           int64_t count, void* ws, size_t ws_bytes, void* stream) {
    SPLATCT_REQUIRE(which == D_CLONE_C || which == D_SPLIT_C,
                    "densify_select: class must be 2 (clone) or 3 (split)");
    const DensifyLayout L = dlayout(n);
    SPLATCT_REQUIRE(ws_bytes >= L.total, "densify_select: workspace too small");
    cudaStream_t s = as_stream(stream);
    if (k <= 0 || count <= 0 || n == 0) return SPLATCT_OK;
    if (k >= count) {
        k_mark_all<<<blocks(n), 256, 0, s>>>(cls, n, which);
        SPLATCT_LAUNCH_CK();
        return SPLATCT_OK;
    }
    const auto* kk = reinterpret_cast<const unsigned long long*>(keys);
    SelState* st = at<SelState>(ws, L.o_state);
    uint32_t* hist = at<uint32_t>(ws, L.o_hist);
    SPLATCT_CK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * HBINS, s));
    k_sel_init<<<1, 1, 0, s>>>(st, (long long)k);
    SPLATCT_LAUNCH_CK();
    for (int shift = 48; shift >= 0; shift -= 16) {
        k_sel_hist<<<blocks(n), 256, 0, s>>>(cls, kk, n, which, st, shift, hist);
        SPLATCT_LAUNCH_CK();
        k_sel_pick<<<1, 1024, 0, s>>>(st, hist, shift);
        SPLATCT_LAUNCH_CK();
    }
    uint32_t* flag = at<uint32_t>(ws, L.o_flag);
    uint32_t* rank = at<uint32_t>(ws, L.o_pos);
    k_sel_ties<<<blocks(n + 1), 256, 0, s>>>(cls, kk, n, which, st, flag);
    SPLATCT_LAUNCH_CK();
    if (int e = exclusive_scan_u32(flag, rank, n + 1, at<void>(ws, L.o_scan), s)) return e;
    k_sel_mark<<<blocks(n), 256, 0, s>>>(cls, kk, n, which, st, rank);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_densify_apply(const double* params, const double* m1, const double* m2,
                          const uint8_t* cls, const double* noise, int64_t n, int64_t n_new,
                          double cbrt2, double* new_params, double* new_m1, double* new_m2,
                          void* ws, size_t ws_bytes, void* stream) {
    const DensifyLayout L = dlayout(n);
    SPLATCT_REQUIRE(ws_bytes >= L.total, "densify_apply: workspace too small");
    SPLATCT_REQUIRE(n >= 0 && n_new >= 0, "densify_apply: bad sizes");
    if (n == 0 || n_new == 0) return SPLATCT_OK;
    cudaStream_t s = as_stream(stream);
    uint32_t* flag = at<uint32_t>(ws, L.o_flag);
    uint32_t* pos = at<uint32_t>(ws, L.o_pos);
    const int64_t st = n + 1;
    k_apply_flags<<<blocks(n + 1), 256, 0, s>>>(cls, n, flag);
    SPLATCT_LAUNCH_CK();
    for (int q = 0; q < 3; ++q)
        if (int e = exclusive_scan_u32(flag + q * st, pos + q * st, n + 1, at<void>(ws, L.o_scan), s))
            return e;
    k_apply<<<blocks(n), 256, 0, s>>>(params, m1, m2, cls, pos, noise, n, n_new, cbrt2,
                                      new_params, new_m1, new_m2);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
