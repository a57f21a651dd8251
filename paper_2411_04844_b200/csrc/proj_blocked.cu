// proj_blocked.cu -- 4-row blocked form of the projector operator and its
// application.
//
// The CSR operators of proj.cu spend one 1 KB z-column load (L1 -> registers)
// per (row, column) weight, i.e. 256 FMAs per 1 KB: the kernels are
// L1-throughput bound.  Adjacent rays of a view cross mostly the same pixels,
// and adjacent pixels are crossed by mostly the same rays, so rows are grouped
// four at a time:
//   kind 0 (forward, A):  rays 4g .. 4g+3 (consecutive detectors of a view);
//   kind 1 (adjoint, A^T): the 2x2 pixel quad (2qx..2qx+1, 2qy..2qy+1).
// A group entry is (column, w[4]) with the four member rows' weights (zero
// where a row does not touch the column).  One column load now feeds up to
// four rows: ~2.5x fewer L1 bytes and load instructions per useful FMA.
// The weights are exactly the CSR weights (same f32 values), summed per row
// in the same ascending-column order for the adjoint (rows of A^T are sorted
// by ray), so the blocked and unblocked operators agree to f32 rounding of
// the accumulation order only.
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace splatct {

constexpr int BLK_NT = 256;
constexpr int BLK_CAP = 8192;   // max gathered entries per group (4 rows)

// kind 0: 4 rays, kind 2: 8 rays, kind 1: 2x2 pixel quads; kinds 3 / 4: bands
// of 8 / 16 consecutive rays whose entries are sliding 4-ray windows (below).
struct GroupMap {
    int kind, nrows, w, h;
    __host__ __device__ bool band() const { return kind == 3 || kind == 4; }
    __host__ __device__ bool rays() const { return kind != 1; }
    __host__ __device__ int rows() const {
        return kind == 2 || kind == 3 ? 8 : (kind == 4 ? 16 : 4);
    }
    __host__ __device__ int64_t ngroups() const {
        if (rays()) return (nrows + rows() - 1) / rows();
        return (int64_t)((w + 1) / 2) * ((h + 1) / 2);
    }
    // member row k (0..rows()-1) of group g, or -1
    __host__ __device__ int64_t row(int64_t g, int k) const {
        if (rays()) {
            const int64_t r = (int64_t)rows() * g + k;
            return r < nrows ? r : -1;
        }
        const int qw = (w + 1) / 2;
        const int qx = (int)(g % qw), qy = (int)(g / qw);
        const int x = 2 * qx + (k & 1), y = 2 * qy + (k >> 1);
        return (x < w && y < h) ? (int64_t)y * w + x : -1;
    }
};

// One CTA per group: gather the member rows' entries, bitonic-sort by column,
// merge equal columns into one (column, w[4]) entry.  mode 0 counts, mode 1
// writes at gptr[g] (mode 2: writes, always through the sort).
//
// Band kinds (3, 4): a pixel of a band of B rays is crossed by a few
// consecutive rays (its bilinear support spans ~2-3 detector bins).  Each
// pixel's (ray, weight) run is cut into windows of 4 consecutive rays from its
// first ray k0 on, and one entry (k0 << 27 | pixel, w[4]) is written per
// window, ray k's weight in slot k mod 4, entries sorted by (k0, pixel).  A warp then walks
// the band with a sliding 4-row accumulator window (k_bspmm_band): a pixel's
// z-column is gathered once per band instead of once per aligned 4-ray group
// it touches (C2: ~1.55 -> ~1.15 gathers per pixel and view).
__global__ void __launch_bounds__(BLK_NT) k_block_build(GroupMap gm, const int64_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ idx,
                                                        const float* __restrict__ val,
                                                        const float2* __restrict__ order_dir,
                                                        int mode,
                                                        int64_t* __restrict__ gcount,
                                                        const int64_t* __restrict__ gptr,
                                                        int32_t* __restrict__ gidx,
                                                        float4* __restrict__ gval,
                                                        int* __restrict__ overflow, int cap,
                                                        int* __restrict__ maxlen) {
    // cap (a power of two <= BLK_CAP): the largest group of this operator, from
    // its count pass; it sizes the shared arrays, so small groups run more CTAs per SM
    extern __shared__ unsigned char smem[];
    uint32_t* key = reinterpret_cast<uint32_t*>(smem);            // [cap]
    uint32_t* pay = key + cap;                                    // [cap] (k << 28 | src)
    float* wv = reinterpret_cast<float*>(pay + cap);              // [cap]
    __shared__ int64_t beg[16], len[16];
    __shared__ int total, nuniq;
    const int64_t g = blockIdx.x;
    const int NR = gm.rows();
    if (threadIdx.x < 16) {
        const int64_t r = (int)threadIdx.x < NR ? gm.row(g, threadIdx.x) : -1;
        beg[threadIdx.x] = r >= 0 ? ptr[r] : 0;
        len[threadIdx.x] = r >= 0 ? ptr[r + 1] - ptr[r] : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int k = 0; k < NR; ++k) t += len[k];
        if (t > cap) {
            atomicExch(overflow, 1);
            t = 0;
        }
        if (maxlen) atomicMax(maxlen, (int)t);
        total = (int)t;
    }
    __syncthreads();
    const int L = total;
    int P = 1;
    while (P < L) P <<= 1;
    // march order: sort by the pixel's position along the group's ray
    // direction (13-bit quantised, then pixel id), so the warps of a CTA sweep
    // the slice together and share L1 lines; pixel order otherwise.
    const bool march = !gm.band() && order_dir != nullptr && (int64_t)gm.w * gm.h <= (1 << 19);
    float2 dir = make_float2(0.f, 0.f);
    if (march) dir = order_dir[g];
    const float cx = 0.5f * (gm.w - 1), cy = 0.5f * (gm.h - 1);
    const float R = 0.5f * sqrtf((float)gm.w * gm.w + (float)gm.h * gm.h) + 1.f;
    for (int i = threadIdx.x; i < P; i += BLK_NT) {
        if (i < L) {
            int k = 0;
            int64_t off = i;
            while (off >= len[k]) { off -= len[k]; ++k; }
            const int64_t j = beg[k] + off;
            const uint32_t pix = (uint32_t)idx[j];
            if (march) {
                const float px = (float)(pix % gm.w) - cx, py = (float)(pix / gm.w) - cy;
                int tq = (int)((px * dir.x + py * dir.y + R) * 4.f);
                tq = min(max(tq, 0), 8191);
                key[i] = ((uint32_t)tq << 19) | pix;
            } else {
                key[i] = pix;
            }
            pay[i] = ((uint32_t)k << 28) | (uint32_t)i;
            wv[i] = mode != 0 ? val[j] : 0.f;
        } else {
            key[i] = 0xffffffffu;
            pay[i] = 0xffffffffu;
        }
    }
    __syncthreads();
    // Rows already sorted by column (the pixel quads' rows of A^T, sorted by
    // ray): the (key, row) order the sort below builds is a merge of the rows,
    // so each distinct key is placed by binary searches instead.  Its first
    // occurrence (lowest row) is its head; the head's rank is the number of
    // heads with a smaller key, summed over the rows from a prefix count.
    if (!march && !gm.band() && mode == 1) {
        int st[9];
        st[0] = 0;
        for (int k = 0; k < NR; ++k) st[k + 1] = st[k] + (int)len[k];
        bool unsorted = false;
        for (int i = threadIdx.x; i + 1 < L; i += BLK_NT)
            if ((pay[i] >> 28) == (pay[i + 1] >> 28) && key[i] >= key[i + 1]) unsorted = true;
        if (!__syncthreads_or(unsorted)) {
            // entries of row kk with a key < x
            auto lower = [&](int kk, uint32_t x) {
                int lo = st[kk], hi = st[kk + 1];
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (key[mid] < x) lo = mid + 1; else hi = mid;
                }
                return lo - st[kk];
            };
            // heads, counted per contiguous chunk, then an exclusive block scan
            const int chunk = (L + BLK_NT - 1) / BLK_NT;
            const int c0 = min(L, (int)threadIdx.x * chunk), c1 = min(L, c0 + chunk);
            int nh = 0;
            for (int i = c0; i < c1; ++i) {
                const int k = (int)(pay[i] >> 28);
                const uint32_t x = key[i];
                bool head = true;
                for (int kk = 0; kk < k && head; ++kk) {
                    const int lb = lower(kk, x);
                    head = !(lb < st[kk + 1] - st[kk] && key[st[kk] + lb] == x);
                }
                nh += head;
                pay[i] = ((uint32_t)k << 28) | (head ? 1u : 0u);
            }
            __shared__ int wsum[BLK_NT / 32];
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            int inc = nh;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (lane == 31) wsum[wid] = inc;
            __syncthreads();
            int base = 0;
            for (int q = 0; q < wid; ++q) base += wsum[q];
            if (threadIdx.x == BLK_NT - 1) nuniq = base + inc;
            int run = base + inc - nh;
            for (int i = c0; i < c1; ++i) {
                const uint32_t h = pay[i] & 1u;
                pay[i] = (uint32_t)run;   // heads before entry i
                run += (int)h;
            }
            __syncthreads();
            const int nu = nuniq;
            auto pre = [&](int j) { return j < L ? (int)pay[j] : nu; };
            // every entry re-derives its row and head flag; heads write
            for (int i = threadIdx.x; i < L; i += BLK_NT) {
                int k = 0;
                while (i >= st[k + 1]) ++k;
                const uint32_t x = key[i];
                if (pre(i + 1) == pre(i)) continue;   // not a head
                float wr[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                int pos = 0;
                for (int kk = 0; kk < NR; ++kk) {
                    const int lb = kk == k ? i - st[k] : lower(kk, x);
                    pos += pre(st[kk] + lb) - pre(st[kk]);
                    if (kk == k) wr[kk] = wv[i];
                    else if (kk > k && lb < st[kk + 1] - st[kk] && key[st[kk] + lb] == x)
                        wr[kk] = wv[st[kk] + lb];
                }
                const int64_t o = gptr[g] + pos;
                gidx[o] = (int32_t)x;
                gval[o * (NR / 4)] = make_float4(wr[0], wr[1], wr[2], wr[3]);
                if (NR == 8) gval[o * 2 + 1] = make_float4(wr[4], wr[5], wr[6], wr[7]);
            }
            return;
        }
    }
    // bitonic sort of (key, pay) pairs, ascending by key then payload
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < P / 2; t += BLK_NT) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = ((uint64_t)key[lo] << 32) | pay[lo];
                const uint64_t b = ((uint64_t)key[hi] << 32) | pay[hi];
                if ((a > b) == up) {
                    key[lo] = (uint32_t)(b >> 32); pay[lo] = (uint32_t)b;
                    key[hi] = (uint32_t)(a >> 32); pay[hi] = (uint32_t)a;
                }
            }
            __syncthreads();
        }
    }
    if (gm.band()) {   // sorted by (pixel, ray): cut each pixel's run into 4-ray windows
        uint32_t* wkey = reinterpret_cast<uint32_t*>(wv + cap);   // [cap] k0 << 27 | pixel
        uint32_t* wpos = wkey + cap;                              // [cap] first entry
        if (threadIdx.x == 0) nuniq = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < L; i += BLK_NT) {
            if (i > 0 && key[i] == key[i - 1]) continue;   // not a run head
            for (int j = i; j < L && key[j] == key[i];) {
                const uint32_t k0 = pay[j] >> 28;
                const int slot = atomicAdd(&nuniq, 1);
                wkey[slot] = (k0 << 27) | key[i];
                wpos[slot] = (uint32_t)j;
                while (j < L && key[j] == key[i] && (pay[j] >> 28) <= k0 + 3) ++j;
            }
        }
        __syncthreads();
        const int nw = nuniq;
        if (mode == 0) {
            if (threadIdx.x == 0) gcount[g] = nw;
            return;
        }
        int P2 = 1;
        while (P2 < nw) P2 <<= 1;
        for (int i = nw + threadIdx.x; i < P2; i += BLK_NT) wkey[i] = wpos[i] = 0xffffffffu;
        __syncthreads();
        // (k0, pixel) keys are unique: the order is deterministic
        for (int size = 2; size <= P2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < P2 / 2; t += BLK_NT) {
                    const int lo = 2 * t - (t & (stride - 1));
                    const int hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    if ((wkey[lo] > wkey[hi]) == up) {
                        const uint32_t a = wkey[lo], b = wpos[lo];
                        wkey[lo] = wkey[hi]; wpos[lo] = wpos[hi];
                        wkey[hi] = a; wpos[hi] = b;
                    }
                }
                __syncthreads();
            }
        }
        for (int t = threadIdx.x; t < nw; t += BLK_NT) {
            const uint32_t k0 = wkey[t] >> 27;
            const uint32_t pix = key[wpos[t]];
            float wr[4] = {0.f, 0.f, 0.f, 0.f};
            // ray k of the window goes to slot k mod 4 (the apply kernel's ring)
            for (int e = (int)wpos[t]; e < L && key[e] == pix && (pay[e] >> 28) <= k0 + 3; ++e)
                wr[(pay[e] >> 28) & 3] = wv[pay[e] & 0x0fffffffu];
            const int64_t o = gptr[g] + t;
            gidx[o] = (int32_t)wkey[t];
            gval[o] = make_float4(wr[0], wr[1], wr[2], wr[3]);
        }
        return;
    }
    // run heads -> unique columns (serial scan by one warp is enough here)
    if (threadIdx.x == 0) nuniq = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
        int base = 0;
        for (int i0 = 0; i0 < L; i0 += 32) {
            const int i = i0 + threadIdx.x;
            const bool head = i < L && (i == 0 || key[i] != key[i - 1]);
            const unsigned m = __ballot_sync(0xffffffffu, head);
            const int pos = base + __popc(m & ((1u << threadIdx.x) - 1u));
            if (head && mode != 0) {
                float wr[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                for (int e = i; e < L && key[e] == key[i]; ++e) {
                    const uint32_t pl = pay[e];
                    wr[pl >> 28] = wv[pl & 0x0fffffffu];
                }
                const int64_t o = gptr[g] + pos;
                gidx[o] = (int32_t)(march ? (key[i] & 0x7ffffu) : key[i]);
                gval[o * (NR / 4)] = make_float4(wr[0], wr[1], wr[2], wr[3]);
                if (NR == 8) gval[o * 2 + 1] = make_float4(wr[4], wr[5], wr[6], wr[7]);
            }
            base += __popc(m);
        }
        if (threadIdx.x == 0) nuniq = base;
    }
    __syncthreads();
    if (threadIdx.x == 0 && mode == 0) gcount[g] = nuniq;
}

// Count pass for the column-keyed kinds (0, 1, 2): the number of distinct
// pixels among a group's member rows, which is the fill's unique-key count
// (the march key is a function of the pixel).  An open-addressing set in
// shared memory (load factor <= 1/2) replaces the fill's sort: one CAS per
// entry instead of a bitonic network.
constexpr int HC_BITS = 14;
constexpr int HC_SLOTS = 1 << HC_BITS;   // 2 x BLK_CAP
static_assert(HC_SLOTS >= 2 * BLK_CAP, "hash set load factor");

__global__ void __launch_bounds__(BLK_NT) k_block_count_hash(GroupMap gm,
                                                             const int64_t* __restrict__ ptr,
                                                             const int32_t* __restrict__ idx,
                                                             int64_t* __restrict__ gcount,
                                                             int* __restrict__ overflow,
                                                             int* __restrict__ maxlen) {
    extern __shared__ unsigned char smem[];
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem);   // [HC_SLOTS]
    __shared__ int64_t beg[8], len[8];
    __shared__ int nuniq, ok;
    const int64_t g = blockIdx.x;
    const int NR = gm.rows();
    if (threadIdx.x < 8) {
        const int64_t r = (int)threadIdx.x < NR ? gm.row(g, threadIdx.x) : -1;
        beg[threadIdx.x] = r >= 0 ? ptr[r] : 0;
        len[threadIdx.x] = r >= 0 ? ptr[r + 1] - ptr[r] : 0;
    }
    for (int i = threadIdx.x; i < HC_SLOTS; i += BLK_NT) tab[i] = 0xffffffffu;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int k = 0; k < NR; ++k) t += len[k];
        ok = t <= BLK_CAP;
        if (!ok) atomicExch(overflow, 1);
        else atomicMax(maxlen, (int)t);
        nuniq = 0;
    }
    __syncthreads();
    if (!ok) return;   // the fill rejects the operator
    int mine = 0;
    for (int k = 0; k < NR; ++k) {
        for (int64_t i = threadIdx.x; i < len[k]; i += BLK_NT) {
            const uint32_t pix = (uint32_t)idx[beg[k] + i];
            uint32_t s = (pix * 2654435761u) >> (32 - HC_BITS);
            for (;;) {
                const uint32_t old = atomicCAS(&tab[s], 0xffffffffu, pix);
                if (old == 0xffffffffu) { ++mine; break; }
                if (old == pix) break;
                s = (s + 1) & (HC_SLOTS - 1);
            }
        }
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&nuniq, mine);
    __syncthreads();
    if (threadIdx.x == 0) gcount[g] = nuniq;
}

// ---------------------------------------------------------------------------
// Blocked application: warp per group, lanes over slices.
// ---------------------------------------------------------------------------
template <int V>
__device__ __forceinline__ void ldvb(const float* p, float (&o)[V]) {
    if constexpr (V == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
    } else if constexpr (V == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __ldg(p);
    }
}
template <int V>
__device__ __forceinline__ void stvb(float* p, const float (&o)[V]) {
    if constexpr (V == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
    } else {
        p[0] = o[0];
    }
}

struct TvB {
    const float* vol;
    const float* halo_lo;
    const float* halo_hi;
    double coef;   // lambda_tv / tv_count (one DFMA per voxel instead of a DDIV)
    double* partial;
    int w, h;
};

__device__ __forceinline__ int sgnf(float d) { return (d > 0.f) - (d < 0.f); }

// Empty-space skipping (null occ: off); one uint64 per pixel column.
// Forward (mode 1): bit tz = the column's 16-slice segment in z tile tz has a
// non-zero voxel (recorded by the voxelizer as it stores the volume); other
// segments are exactly zero.  Adjoint (mode 2): bit tz = a Gaussian footprint
// covers the column in z tile tz (what the voxelizer backward reads).
// Adjoint (mode 2): a 2x2-pixel quad x z-chunk whose one-voxel neighbourhood
// no footprint covers is skipped entirely: the volume is zero there, so its
// TV value and subgradient are zero, and its output is left unwritten -- the
// caller (the training step's voxelizer backward) reads the adjoint only
// inside Gaussian footprints.
struct Occ {
    const unsigned long long* occ;
    int w, ntx, mode;   // mode 1: forward entry skipping, 2: adjoint quad skipping
    const int32_t* order = nullptr;   // CTA visit order (group-major launches only)
};

constexpr int BS_WARPS = 4;
#ifndef BS_MINB
#define BS_MINB 6   // CTAs per SM (80 registers); swept 4..8, tools/jobs/bs_minb.sh
#endif
constexpr int UNR = 8;    // z-vector gathers in flight per warp (16 measured no faster)

// Per-lane accumulators of the R group rows over the lane's V slices, held
// as packed pairs so every (row, slice pair) update is one FFMA2.
template <int R, int V>
struct AccR {
    static constexpr int P = (V + 1) / 2;
    float2 a[R][P];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
            for (int q = 0; q < P; ++q) a[k][q] = make_float2(0.f, 0.f);
    }
    // w: the entry's R row weights as R/4 float4
    __device__ __forceinline__ void add(const float4* w, const float (&x)[V]) {
#pragma unroll
        for (int k4 = 0; k4 < R / 4; ++k4) {
            const float4 w4 = w[k4];
            const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * k4 + j;
                if constexpr (V == 1) {
                    a[k][0].x = fmaf(wk[j], x[0], a[k][0].x);
                } else {
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        a[k][q] = ffma2(make_float2(wk[j], wk[j]),
                                        make_float2(x[2 * q], x[2 * q + 1]), a[k][q]);
                }
            }
        }
    }
    // store row K (if st) and restart it at zero
    template <int K>
    __device__ __forceinline__ void flush(bool st, float* p) {
        if (st) {
            float o[V];
            row(K, o);
            stvb<V>(p, o);
        }
#pragma unroll
        for (int q = 0; q < P; ++q) a[K][q] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ void row(int k, float (&o)[V]) const {
        if constexpr (V == 1) {
            o[0] = a[k][0].x;
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                o[2 * q] = a[k][q].x;
                o[2 * q + 1] = a[k][q].y;
            }
        }
    }
};

// TV epilogue for a whole 2x2 pixel quad (the adjoint's group): the four
// own z-vectors are loaded once and serve as each other's x / y neighbours,
// so a lane loads 4 own + at most 8 outside neighbour vectors instead of 20;
// the quad's TV value is one warp reduction.  Same arithmetic per voxel as
// the per-row forward-difference subgradient of loss.tv_loss (loss.py:195-206),
// z neighbours from adjacent lanes (shuffles) or, at warp / slab edges, from
// memory / halos.
template <int V>
__device__ __forceinline__ void tv_epilogue_quad(const TvB& a, const GroupMap& gm, int64_t g,
                                                 int zb, int c, bool zok,
                                                 const AccR<4, V>& acc, float* __restrict__ Y,
                                                 double& tvsum) {
    const int lane = threadIdx.x & 31;
    const int qw = (gm.w + 1) / 2;
    const int x0 = 2 * (int)(g % qw), y0 = 2 * (int)(g / qw);
    bool has[4];
    const float* col[4];
    float v[4][V];
    float up_prev[4], dn_next[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int x = x0 + (k & 1), y = y0 + (k >> 1);
        has[k] = x < gm.w && y < gm.h;
        col[k] = a.vol + ((int64_t)y * gm.w + x) * c;
        if (has[k] && zok) ldvb<V>(col[k] + zb, v[k]);
        else
#pragma unroll
            for (int t = 0; t < V; ++t) v[k][t] = 0.f;
        up_prev[k] = __shfl_up_sync(0xffffffffu, v[k][V - 1], 1);
        dn_next[k] = __shfl_down_sync(0xffffffffu, v[k][0], 1);
    }
    if (!zok) return;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!has[k]) continue;   // warp-uniform
        const int dx = k & 1, dy = k >> 1;
        const int x = x0 + dx, y = y0 + dy;
        int gs[V];
        float s1[V];
#pragma unroll
        for (int t = 0; t < V; ++t) { gs[t] = 0; s1[t] = 0.f; }
        // one axis: forward difference to the next neighbour, subgradient from
        // the previous one; in-quad neighbours come from registers
        auto axis = [&](bool has_next, int kn, const float* ncol, bool has_prev, int kp,
                        const float* pcol) {
            if (has_next) {
                float n[V];
                if (kn >= 0) {
#pragma unroll
                    for (int t = 0; t < V; ++t) n[t] = v[kn][t];
                } else {
                    ldvb<V>(ncol + zb, n);
                }
#pragma unroll
                for (int t = 0; t < V; ++t) {
                    const float d = n[t] - v[k][t];
                    s1[t] += fabsf(d);
                    gs[t] -= sgnf(d);
                }
            }
            if (has_prev) {
                float pv[V];
                if (kp >= 0) {
#pragma unroll
                    for (int t = 0; t < V; ++t) pv[t] = v[kp][t];
                } else {
                    ldvb<V>(pcol + zb, pv);
                }
#pragma unroll
                for (int t = 0; t < V; ++t) gs[t] += sgnf(v[k][t] - pv[t]);
            }
        };
        axis(x + 1 < gm.w, dx == 0 ? k + 1 : -1, col[k] + c, x > 0, dx == 1 ? k - 1 : -1,
             col[k] - c);
        axis(y + 1 < gm.h, dy == 0 ? k + 2 : -1, col[k] + (int64_t)gm.w * c, y > 0,
             dy == 1 ? k - 2 : -1, col[k] - (int64_t)gm.w * c);
        const int64_t row = (int64_t)y * gm.w + x;
        float ak[V], o[V];
        acc.row(k, ak);
#pragma unroll
        for (int t = 0; t < V; ++t) {
            const int z = zb + t;
            float zn = 0.f;
            bool hn = true;
            if (t + 1 < V) {
                zn = v[k][t + 1];
            } else if (z + 1 < c) {
                zn = lane < 31 ? dn_next[k] : __ldg(col[k] + z + 1);
            } else if (a.halo_hi) {
                zn = __ldg(a.halo_hi + row);
            } else {
                hn = false;
            }
            if (hn) {
                const float d = zn - v[k][t];
                s1[t] += fabsf(d);
                gs[t] -= sgnf(d);
            }
            float zp = 0.f;
            bool hp = true;
            if (t > 0) {
                zp = v[k][t - 1];
            } else if (z > 0) {
                zp = lane > 0 ? up_prev[k] : __ldg(col[k] + z - 1);
            } else if (a.halo_lo) {
                zp = __ldg(a.halo_lo + row);
            } else {
                hp = false;
            }
            if (hp) gs[t] += sgnf(v[k][t] - zp);
            o[t] = (float)fma((double)gs[t], a.coef, (double)ak[t]);
            tvsum += (double)s1[t];
        }
        stvb<V>(Y + row * c + zb, o);
    }
}

// Warp per (group, z-chunk of 32*V slices); the R rows of a group share every
// column load.  Entries are staged per warp in shared memory and consumed
// UNR at a time (UNR independent vector loads in flight).
template <int V, bool TV, int R>
__global__ void __launch_bounds__(32 * BS_WARPS, R == 8 ? 4 : BS_MINB) k_bspmm(GroupMap gm, const int64_t* __restrict__ gptr,
                                                        const int32_t* __restrict__ gidx,
                                                        const float4* __restrict__ gval,
                                                        const float* __restrict__ X,
                                                        float* __restrict__ Y, int c, int zsplit,
                                                        int zmajor, TvB tv, Occ oc,
                                                        const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    constexpr int RW = R / 4;   // float4 weight words per entry
    __shared__ int s_col[BS_WARPS][32];
    __shared__ float4 s_w[BS_WARPS][32 * RW];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // CTA b runs the work of CTA order[b]: the host lists the longest first
    const int64_t bid = oc.order ? (int64_t)oc.order[blockIdx.x] : (int64_t)blockIdx.x;
    const int64_t gw = bid * BS_WARPS + wid;
    // zmajor (gathered operand larger than L2): z-chunk-major order, so the
    // warps in flight share one z-chunk and the L2 working set is 1/zsplit of
    // the operand (C4: 512 MB volume); otherwise a group's chunks run together
    // and share its entry list
    const int64_t ngr = gm.ngroups();
    const int64_t g = zmajor ? gw % ngr : gw / zsplit;
    const int zch = zmajor ? (int)(gw / ngr) : (int)(gw % zsplit);
    if (g >= ngr || zch >= zsplit) return;
    const int zb = zch * 32 * V + lane * V;
    const bool zok = zb < c;
    // empty-space skipping (forward only): the z tiles this warp's chunk covers;
    // an entry whose pixel column has no Gaussian in them reads only zeros
    unsigned long long zmask = ~0ull;
    if (oc.mode == 1) {
        const int zlo = zch * 32 * V, zhi = min(zlo + 32 * V, c) - 1;
        const int tlo = zlo / 16, thi = zhi / 16;
        zmask = (thi >= 63 ? ~0ull : ((1ull << (thi + 1)) - 1ull)) & ~((1ull << tlo) - 1ull);
    }
    const int zl = zok ? zb : 0;   // keep loads in bounds for idle lanes
    if (oc.mode == 2) {   // adjoint quads (kind 1): skip all-empty neighbourhoods
        const int qw = (gm.w + 1) / 2;
        const int x0 = 2 * (int)(g % qw), y0 = 2 * (int)(g / qw);
        const int zlo = zch * 32 * V, zhi = min(zlo + 32 * V, c) - 1;
        const bool halo = (zlo == 0 && tv.halo_lo) || (zhi == c - 1 && tv.halo_hi);
        const int tlo = max(zlo - 1, 0) / 16, thi = min(zhi + 1, c - 1) / 16;
        const unsigned long long zm =
            (thi >= 63 ? ~0ull : ((1ull << (thi + 1)) - 1ull)) & ~((1ull << tlo) - 1ull);
        // footprint coverage of the quad's pixels and their one-pixel ring: the
        // 4 x 4 neighbourhood's words are loaded one per lane, then a vote
        const int xx = x0 - 1 + (lane & 3), yy = y0 - 1 + ((lane >> 2) & 3);
        const bool in = lane < 16 && xx >= 0 && xx < gm.w && yy >= 0 && yy < gm.h;
        const bool cov = in && (oc.occ[(int64_t)yy * gm.w + xx] & zm) != 0ull;
        if (!halo && !__any_sync(0xffffffffu, cov)) {   // warp-uniform
            if (TV && tv.partial && lane == 0) tv.partial[zch * ngr + g] = 0.0;
            return;
        }
    }
    AccR<R, V> acc;
    acc.zero();
    const int64_t b = gptr[g], e = gptr[g + 1];
    // entries of the next batch are prefetched into registers while the
    // current batch is consumed from shared memory
    int nc = 0;
    float4 nw[RW];
#pragma unroll
    for (int q = 0; q < RW; ++q) nw[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b + lane < e) {
        nc = __ldcs(gidx + b + lane);
#pragma unroll
        for (int q = 0; q < RW; ++q) nw[q] = __ldcs(gval + (b + lane) * RW + q);
    }
    for (int64_t j0 = b; j0 < e; j0 += 32) {
        __syncwarp();
        int cnt = (int)min((int64_t)32, e - j0);
        if (oc.mode == 1) {   // keep the entries whose column is occupied, in order
            bool keep = lane < cnt;
            if (keep) keep = (oc.occ[nc] & zmask) != 0ull;   // the pixel column's segments
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int slot = __popc(km & ((1u << lane) - 1u));
                s_col[wid][slot] = nc;
#pragma unroll
                for (int q = 0; q < RW; ++q) s_w[wid][slot * RW + q] = nw[q];
            }
            cnt = __popc(km);
        } else {
            s_col[wid][lane] = nc;
#pragma unroll
            for (int q = 0; q < RW; ++q) s_w[wid][lane * RW + q] = nw[q];
        }
        __syncwarp();
        if (j0 + 32 + lane < e) {
            nc = __ldcs(gidx + j0 + 32 + lane);
#pragma unroll
            for (int q = 0; q < RW; ++q) nw[q] = __ldcs(gval + (j0 + 32 + lane) * RW + q);
        }
        int jj = 0;
        for (; jj + UNR <= cnt; jj += UNR) {   // UNR z-vector gathers in flight
            float xv[UNR][V];
#pragma unroll
            for (int u = 0; u < UNR; ++u) ldvb<V>(X + (int64_t)s_col[wid][jj + u] * c + zl, xv[u]);
#pragma unroll
            for (int u = 0; u < UNR; ++u) acc.add(&s_w[wid][(jj + u) * RW], xv[u]);
        }
        for (; jj + 4 <= cnt; jj += 4) {
            float xv[4][V];
#pragma unroll
            for (int u = 0; u < 4; ++u) ldvb<V>(X + (int64_t)s_col[wid][jj + u] * c + zl, xv[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc.add(&s_w[wid][(jj + u) * RW], xv[u]);
        }
        for (; jj < cnt; ++jj) {
            float xv[V];
            ldvb<V>(X + (int64_t)s_col[wid][jj] * c + zl, xv);
            acc.add(&s_w[wid][jj * RW], xv);
        }
    }
    if constexpr (TV) {   // TV groups are the adjoint's 2x2 pixel quads (R == 4)
        double tvsum = 0.0;
        tv_epilogue_quad<V>(tv, gm, g, zb, c, zok, acc, Y, tvsum);
        if (tv.partial) {   // slot (z-chunk, quad): written once, reduced in fixed order
            tvsum = warp_sum(tvsum);
            if (lane == 0) tv.partial[zch * ngr + g] = tvsum;
        }
    } else {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int64_t row = gm.row(g, k);
            if (row < 0) continue;   // uniform across the warp
            float ak[V];
            acc.row(k, ak);
            if (zok) stvb<V>(Y + row * c + zb, ak);
        }
    }
}

// Band form of the forward (kinds 3 / 4): warp per (band of B rays, z-chunk),
// entries in (k0, pixel) order, each feeding rays k0..k0+3 of the band.  The
// accumulators are a ring of 4 rays, ray k in slot k mod 4 (the build stored
// the weights in that order): before an entry with a later k0, the window's
// first ray is complete (no later entry touches it), so it is stored and its
// slot restarts at zero for ray base + 4.  Every ray of the band is stored once.
#ifndef BAND_MINB
#define BAND_MINB 5
#endif
template <int V, int B>
__global__ void __launch_bounds__(32 * BS_WARPS, BAND_MINB) k_bspmm_band(GroupMap gm,
                                                                const int64_t* __restrict__ gptr,
                                                                const int32_t* __restrict__ gidx,
                                                                const float4* __restrict__ gval,
                                                                const float* __restrict__ X,
                                                                float* __restrict__ Y, int c,
                                                                int zsplit, int zmajor, Occ oc,
                                                                const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ int s_col[BS_WARPS][32];
    __shared__ float4 s_w[BS_WARPS][32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)BS_WARPS + wid;
    const int64_t ngr = gm.ngroups();
    const int64_t g = zmajor ? gw % ngr : gw / zsplit;
    const int zch = zmajor ? (int)(gw / ngr) : (int)(gw % zsplit);
    if (g >= ngr || zch >= zsplit) return;
    const int zb = zch * 32 * V + lane * V;
    const bool zok = zb < c;
    unsigned long long zmask = ~0ull;
    if (oc.mode == 1) {
        const int zlo = zch * 32 * V, zhi = min(zlo + 32 * V, c) - 1;
        const int tlo = zlo / 16, thi = zhi / 16;
        zmask = (thi >= 63 ? ~0ull : ((1ull << (thi + 1)) - 1ull)) & ~((1ull << tlo) - 1ull);
    }
    const int zl = zok ? zb : 0;
    AccR<4, V> acc;
    acc.zero();
    const int64_t row0 = g * (int64_t)B;
    int base = 0;   // band ray held in window slot 0
    auto advance = [&]() {   // store ray `base` (slot base mod 4) and restart its slot
        const int64_t row = row0 + base;
        const bool st = row < gm.nrows && zok;
        switch (base & 3) {   // warp-uniform
            case 0: acc.flush<0>(st, Y + row * c + zb); break;
            case 1: acc.flush<1>(st, Y + row * c + zb); break;
            case 2: acc.flush<2>(st, Y + row * c + zb); break;
            default: acc.flush<3>(st, Y + row * c + zb); break;
        }
        ++base;
    };
    const int64_t b = gptr[g], e = gptr[g + 1];
    int nc = 0;
    float4 nw = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b + lane < e) {
        nc = __ldcs(gidx + b + lane);
        nw = __ldcs(gval + b + lane);
    }
    auto consume = [&](int j, const float (&xv)[V]) {
        const int k0 = (int)((unsigned)s_col[wid][j] >> 27);   // warp-uniform
        while (base < k0) advance();
        acc.add(&s_w[wid][j], xv);
    };
    for (int64_t j0 = b; j0 < e; j0 += 32) {
        __syncwarp();
        int cnt = (int)min((int64_t)32, e - j0);
        if (oc.mode == 1) {   // keep the entries whose column is occupied, in order
            bool keep = lane < cnt;
            if (keep) keep = (oc.occ[nc & 0x07ffffff] & zmask) != 0ull;
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int slot = __popc(km & ((1u << lane) - 1u));
                s_col[wid][slot] = nc;
                s_w[wid][slot] = nw;
            }
            cnt = __popc(km);
        } else {
            s_col[wid][lane] = nc;
            s_w[wid][lane] = nw;
        }
        __syncwarp();
        if (j0 + 32 + lane < e) {
            nc = __ldcs(gidx + j0 + 32 + lane);
            nw = __ldcs(gval + j0 + 32 + lane);
        }
        int jj = 0;
        for (; jj + UNR <= cnt; jj += UNR) {   // UNR z-vector gathers in flight
            float xv[UNR][V];
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                ldvb<V>(X + (int64_t)(s_col[wid][jj + u] & 0x07ffffff) * c + zl, xv[u]);
#pragma unroll
            for (int u = 0; u < UNR; ++u) consume(jj + u, xv[u]);
        }
        for (; jj < cnt; ++jj) {
            float xv[V];
            ldvb<V>(X + (int64_t)(s_col[wid][jj] & 0x07ffffff) * c + zl, xv);
            consume(jj, xv);
        }
    }
    while (base < B) advance();
}

template <int V, bool TV>
static int launch_bspmm_v(const GroupMap& gm, const int64_t* gptr, const int32_t* gidx,
                          const float* gval, const float* X, float* Y, int c, const TvB& tv,
                          const Occ& oc, int64_t vol_bytes, const int* halt, cudaStream_t s) {
    const int zsplit = (c + 32 * V - 1) / (32 * V);
    const int64_t warps = gm.ngroups() * zsplit;
    // z-chunk-major order once the volume (the forward's gathered operand; a
    // proxy for the adjoint's sinogram) outgrows ~3/4 of L2
    const int zmajor = zsplit > 1 && vol_bytes > ((int64_t)96 << 20);
    const unsigned grid = (unsigned)((warps + BS_WARPS - 1) / BS_WARPS);
    Occ oc_ = oc;
    if (gm.band()) oc_.order = nullptr;
    const float4* gv = reinterpret_cast<const float4*>(gval);
    if (!TV && gm.band()) {
        if (gm.kind == 4)
            SPLATCT_CK(launch_pdl(k_bspmm_band<V, 16>, dim3(grid), dim3(32 * BS_WARPS), 0, s, gm,
                                  gptr, gidx, gv, X, Y, c, zsplit, zmajor, oc_, halt));
        else
            SPLATCT_CK(launch_pdl(k_bspmm_band<V, 8>, dim3(grid), dim3(32 * BS_WARPS), 0, s, gm,
                                  gptr, gidx, gv, X, Y, c, zsplit, zmajor, oc_, halt));
    } else if (!TV && gm.rows() == 8)
        SPLATCT_CK(launch_pdl(k_bspmm<V, false, 8>, dim3(grid), dim3(32 * BS_WARPS), 0, s, gm,
                              gptr, gidx, gv, X, Y, c, zsplit, zmajor, tv, oc_, halt));
    else
        SPLATCT_CK(launch_pdl(k_bspmm<V, TV, 4>, dim3(grid), dim3(32 * BS_WARPS), 0, s, gm, gptr,
                              gidx, gv, X, Y, c, zsplit, zmajor, tv, oc_, halt));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

static int vec_width(int c) {
    if (c % 4 == 0 && c >= 128) return 4;
    if (c % 2 == 0 && c >= 64) return 2;
    return 1;
}

template <bool TV>
static int launch_bspmm(const GroupMap& gm, const int64_t* gptr, const int32_t* gidx,
                        const float* gval, const float* X, float* Y, int c, const TvB& tv,
                        const int* halt, cudaStream_t s, const Occ& oc = Occ{nullptr, 0, 0, 0},
                        int64_t vol_bytes = 0) {
    const int V = vec_width(c);
    SPLATCT_REQUIRE((uintptr_t)X % (4 * V) == 0 && (uintptr_t)Y % (4 * V) == 0 &&
                        (!TV || (uintptr_t)tv.vol % (4 * V) == 0),
                    "projector operands must be %d-byte aligned", 4 * V);
    if (V == 4)
        return launch_bspmm_v<4, TV>(gm, gptr, gidx, gval, X, Y, c, tv, oc, vol_bytes, halt, s);
    if (V == 2)
        return launch_bspmm_v<2, TV>(gm, gptr, gidx, gval, X, Y, c, tv, oc, vol_bytes, halt, s);
    return launch_bspmm_v<1, TV>(gm, gptr, gidx, gval, X, Y, c, tv, oc, vol_bytes, halt, s);
}

// key, payload, weight per gathered entry; band kinds add the window key and position
static size_t block_smem(int kind, int cap) {
    return (size_t)cap * (kind == 3 || kind == 4 ? 20 : 12);
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_proj_tv_partial_len(int w, int h, int c, int64_t* len) {
    const int V = vec_width(c);   // one slot per (z-chunk, 2 x 2 quad)
    *len = (int64_t)((w + 1) / 2) * ((h + 1) / 2) * ((c + 32 * V - 1) / (32 * V));
    return SPLATCT_OK;
}

int splatct_proj_block_scratch_bytes(int nrows, int kind, int w, int h, size_t* bytes) {
    GroupMap gm{kind, nrows, w, h};
    const int64_t ng = gm.ngroups();
    *bytes = align_up(sizeof(int64_t) * (ng + 1)) + scan_temp_bytes(ng + 1) + 256;
    return SPLATCT_OK;
}

int splatct_proj_block_count(const int64_t* ptr, const int32_t* idx, int nrows, int kind, int w,
                             int h, const float* order_dir, int64_t* gptr, void* scratch,
                             size_t scratch_bytes, int64_t* nb, void* stream) {
    SPLATCT_REQUIRE(kind >= 0 && kind <= 4,
                    "kind must be 0 (4-ray groups), 1 (pixel quads), 2 (8-ray groups) or 3 / 4 "
                    "(8 / 16-ray bands)");
    SPLATCT_REQUIRE(kind == 1 || (int64_t)w * h <= (1 << 27), "band entries pack pixel < 2^27");
    GroupMap gm{kind, nrows, w, h};
    const int64_t ng = gm.ngroups();
    size_t need = 0;
    splatct_proj_block_scratch_bytes(nrows, kind, w, h, &need);
    SPLATCT_REQUIRE(scratch_bytes >= need, "block scratch too small");
    cudaStream_t s = as_stream(stream);
    int64_t* cnt = reinterpret_cast<int64_t*>(scratch);
    char* scan_tmp = reinterpret_cast<char*>(scratch) + align_up(sizeof(int64_t) * (ng + 1));
    int* overflow = reinterpret_cast<int*>(scan_tmp + scan_temp_bytes(ng + 1));
    int* maxlen = overflow + 1;   // the largest group's entry count, for the fill
    SPLATCT_CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ng + 1), s));
    SPLATCT_CK(cudaMemsetAsync(overflow, 0, 2 * sizeof(int), s));
    static bool attr = false;
    if (!attr) {
        SPLATCT_CK(cudaFuncSetAttribute(k_block_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)block_smem(3, BLK_CAP)));
        SPLATCT_CK(cudaFuncSetAttribute(k_block_count_hash,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        HC_SLOTS * (int)sizeof(uint32_t)));
        attr = true;
    }
    // SPLATCT_BLOCK_COUNT=sort counts with the fill's sort (test knob)
    const char* how = getenv("SPLATCT_BLOCK_COUNT");
    if (!gm.band() && !(how && !strcmp(how, "sort"))) {
        k_block_count_hash<<<(unsigned)ng, BLK_NT, HC_SLOTS * sizeof(uint32_t), s>>>(
            gm, ptr, idx, cnt, overflow, maxlen);
    } else {
        k_block_build<<<(unsigned)ng, BLK_NT, block_smem(kind, BLK_CAP), s>>>(
            gm, ptr, idx, nullptr, reinterpret_cast<const float2*>(order_dir), 0, cnt, nullptr,
            nullptr, nullptr, overflow, BLK_CAP, maxlen);
    }
    SPLATCT_LAUNCH_CK();
    if (int e = exclusive_scan_i64(cnt, gptr, ng + 1, scan_tmp, s)) return e;
    int ovf = 0;
    SPLATCT_CK(cudaMemcpyAsync(nb, gptr + ng, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaMemcpyAsync(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    SPLATCT_REQUIRE(!ovf, "a row group has more than %d entries", BLK_CAP);
    return SPLATCT_OK;
}

int splatct_proj_block_fill(const int64_t* ptr, const int32_t* idx, const float* val, int nrows,
                            int kind, int w, int h, const float* order_dir, const int64_t* gptr,
                            int32_t* gidx, float* gval, void* scratch, size_t scratch_bytes,
                            void* stream) {
    GroupMap gm{kind, nrows, w, h};
    const int64_t ng = gm.ngroups();
    size_t need = 0;
    splatct_proj_block_scratch_bytes(nrows, kind, w, h, &need);
    SPLATCT_REQUIRE(scratch_bytes >= need, "block scratch too small");
    SPLATCT_REQUIRE((uintptr_t)gval % 16 == 0, "gval must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    int* overflow = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) +
                                           align_up(sizeof(int64_t) * (ng + 1)) +
                                           scan_temp_bytes(ng + 1));
    // SPLATCT_BLOCK_FILL=sort: rows sorted by column are merged through the sort too (test knob)
    const char* how = getenv("SPLATCT_BLOCK_FILL");
    const int mode = how && !strcmp(how, "sort") ? 2 : 1;
    // the shared arrays are sized for the largest group the count pass saw
    int maxlen = 0;
    SPLATCT_CK(cudaMemcpyAsync(&maxlen, overflow + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    int cap = 256;
    while (cap < maxlen && cap < BLK_CAP) cap <<= 1;
    k_block_build<<<(unsigned)ng, BLK_NT, block_smem(kind, cap), s>>>(
        gm, ptr, idx, val, reinterpret_cast<const float2*>(order_dir), mode, nullptr, gptr, gidx,
        reinterpret_cast<float4*>(gval), overflow, cap, nullptr);
    SPLATCT_LAUNCH_CK();
    int ovf = 0;
    SPLATCT_CK(cudaMemcpyAsync(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    SPLATCT_REQUIRE(!ovf, "a row group has more entries than its count pass saw "
                          "(splatct_proj_block_fill needs the scratch of splatct_proj_block_count)");
    return SPLATCT_OK;
}

int splatct_proj_forward_ctas(int n_rays, int kind, int w, int h, int c, int64_t* ctas,
                              int* zsplit, int* ordered) {
    SPLATCT_REQUIRE(n_rays >= 0 && c > 0 && w > 0 && h > 0, "invalid sizes");
    GroupMap gm{kind, n_rays, 0, 0};
    const int V = vec_width(c);
    const int zs = (c + 32 * V - 1) / (32 * V);
    *zsplit = zs;
    *ctas = (gm.ngroups() * zs + BS_WARPS - 1) / BS_WARPS;
    const bool zmajor = zs > 1 && (int64_t)w * h * c * 4 > ((int64_t)96 << 20);
    *ordered = gm.band() ? 0 : (zmajor ? 2 : 1);
    return SPLATCT_OK;
}

int splatct_proj_forward_blocked(const int64_t* gptr, const int32_t* gidx, const float* gval,
                                 int n_rays, int kind, const float* vol_yxz, float* sino, int c,
                                 const uint64_t* col_occ, int w, int h, const int* halt,
                                 void* stream) {
    return splatct_proj_forward_blocked_ordered(gptr, gidx, gval, n_rays, kind, vol_yxz, sino, c,
                                                col_occ, w, h, nullptr, halt, stream);
}

int splatct_proj_forward_blocked_ordered(const int64_t* gptr, const int32_t* gidx,
                                         const float* gval, int n_rays, int kind,
                                         const float* vol_yxz, float* sino, int c,
                                         const uint64_t* col_occ, int w, int h,
                                         const int32_t* cta_order, const int* halt,
                                         void* stream) {
    SPLATCT_REQUIRE(n_rays >= 0 && c > 0 && w > 0 && h > 0, "invalid sizes");
    SPLATCT_REQUIRE(kind == 0 || kind == 2 || kind == 3 || kind == 4,
                    "forward groups are kind 0, 2, 3 or 4");
    SPLATCT_REQUIRE(col_occ == nullptr || c <= 64 * 16, "occupancy needs <= 64 z tiles");
    GroupMap gm{kind, n_rays, 0, 0};
    TvB tv{};
    Occ oc{reinterpret_cast<const unsigned long long*>(col_occ), w, (w + 15) / 16,
           col_occ ? 1 : 0};
    oc.order = cta_order;
    return launch_bspmm<false>(gm, gptr, gidx, gval, vol_yxz, sino, c, tv, halt,
                               as_stream(stream), oc, (int64_t)w * h * c * 4);
}

int splatct_proj_adjoint_blocked(const int64_t* gptr, const int32_t* gidx, const float* gval,
                                 int w, int h, int c, const float* gsino, const float* vol_yxz,
                                 const float* halo_lo, const float* halo_hi, double lambda_tv,
                                 double tv_count, float* out_yxz, double* tv_partial,
                                 const uint64_t* col_occ, const int* halt, void* stream) {
    SPLATCT_REQUIRE(w > 0 && h > 0 && c > 0, "invalid sizes");
    SPLATCT_REQUIRE(col_occ == nullptr || c <= 64 * 16, "occupancy needs <= 64 z tiles");
    GroupMap gm{1, w * h, w, h};
    TvB tv{vol_yxz, halo_lo, halo_hi, tv_count > 0.0 ? lambda_tv / tv_count : 0.0, tv_partial,
           w, h};
    const Occ oc{reinterpret_cast<const unsigned long long*>(col_occ), w, (w + 15) / 16,
                 col_occ ? 2 : 0};
    cudaStream_t s = as_stream(stream);
    if (vol_yxz != nullptr && lambda_tv > 0.0) {
        SPLATCT_REQUIRE(tv_count > 0.0, "tv_count must be positive");
        return launch_bspmm<true>(gm, gptr, gidx, gval, gsino, out_yxz, c, tv, halt, s, oc,
                                  (int64_t)w * h * c * 4);
    }
    return launch_bspmm<false>(gm, gptr, gidx, gval, gsino, out_yxz, c, tv, halt, s, oc,
                               (int64_t)w * h * c * 4);
}

}  // extern "C"
