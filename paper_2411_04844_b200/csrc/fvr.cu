// fvr.cu -- Fast Volume Reconstruction on B200: footprints, radix-sorted
// tile bins, tile-owned forward splat, Gaussian-owned backward.
//
// Reference semantics (paths under /root/reference/pkg/src/splatct/):
//   footprint  [floor(mu_a)-h_a, floor(mu_a)+h_a] intersect [0, dim_a)
//              _kernels.py:45-47,61-78 (true floor, out-of-volume dropped)
//   forward    V[z,y,x] += I * ez[oz] * ey[oy] * ex[ox]           _kernels.py:51-78
//              e[k] = exp(-(b - d)^2 / (2 sigma^2)), b = k - h, d = mu - floor(mu)
//   backward   dI += u g ; dmu += u g I r / sigma^2 ; dsigma += u g I |r|^2 / sigma^3
//              _kernels.py:132-205 ; accum += |dmu| fvr.py:266-273
//
// B200 design:
//   * volume stored yxz (slice fastest) so a tile's (y,x) column is a
//     contiguous 64 B segment;
//   * per-Gaussian tile counts, an exclusive scan, then (tile, Gaussian) pairs
//     emitted densely in Gaussian / slot order and stably LSD-radix-sorted by
//     tile id (pair count read on the device) -> per-tile lists in ascending
//     Gaussian id (bit-exact against the CPU restatement, deterministic sums);
//   * forward: one CTA per 16^3 tile, each thread owns a (y,x) column of 16
//     voxels in registers; per-Gaussian separable tables staged in shared
//     memory; every voxel stored exactly once (no memset, no atomics);
//   * backward: one warp per Gaussian (lanes over z) reading the upstream
//     straight from L2, separable moment contraction (x inner, y outer, z
//     per lane), warp-shuffle reduction, f64 chain rule; no atomics, no
//     partial buffers, deterministic.
#include <cuda.h>
#include <cudaTypedefs.h>
#include "tmap.cuh"

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "tc.cuh"

namespace splatct {

constexpr int TT = SPLATCT_TILE;   // tile edge (16)
constexpr int SORT_NT = 256;
#ifndef SORT_IPT_N
#define SORT_IPT_N 16
#endif
constexpr int SORT_IPT = SORT_IPT_N;   // keys per thread of a radix pass
constexpr int SORT_CHUNK = SORT_NT * SORT_IPT;
constexpr int RADIX = 256;
constexpr int MAX_PASSES = 4;     // 8-bit digits of a 32-bit tile id
constexpr int BIN_NT = 256;       // Gaussians per block in the emit pass

// Per-Gaussian record written by the footprint pass: integer floor (global
// voxel coordinates), fractional offsets, 0.5/sigma^2 and intensity in f32,
// so the tile kernels never touch f64.
struct __align__(16) GRec {
    int fx, fy, fz;
    float inv2;       // log2(e) / (2 sigma^2)
    float dx, dy, dz, I;
};

struct FvrLayout {
    int64_t n;
    int w, h, c, hx, hy, hz;
    int ntx, nty, ntz;
    int64_t nt;
    int S;            // slots per Gaussian (power of two >= max tiles per Gaussian)
    int Sl;           // log2(S)
    int64_t np;       // worst-case number of (tile, Gaussian) pairs
    int passes;
    int64_t sort_blocks;
    int64_t emit_blocks;
    size_t o_fp, o_k0, o_v0, o_k1, o_v1, o_tcount, o_tstart, o_ctl, o_tickets, o_ghist, o_stat_e,
        o_stat_s, o_pocc, o_fcov, ctl_bytes, o_rec, o_flag, o_pos, o_order, o_scan2,
        total;
    int final_buf;    // which (k,v) buffer holds the sorted result
};

static int axis_span(int half, int dim) {
    int s = (2 * half + TT - 1) / TT + 1;
    int nta = (dim + TT - 1) / TT;
    return s < nta ? s : nta;
}

static FvrLayout make_layout(int64_t n, int w, int h, int c, int hx, int hy, int hz) {
    FvrLayout L{};
    L.n = n;
    L.w = w; L.h = h; L.c = c; L.hx = hx; L.hy = hy; L.hz = hz;
    L.ntx = (w + TT - 1) / TT;
    L.nty = (h + TT - 1) / TT;
    L.ntz = (c + TT - 1) / TT;
    L.nt = (int64_t)L.ntx * L.nty * L.ntz;
    {   // slot field of a pair's value: a power of two >= the maximum tiles per
        // Gaussian (value = Gaussian << Sl | slot); worst-case pair count
        const int s_raw = axis_span(hx, w) * axis_span(hy, h) * axis_span(hz, c);
        L.Sl = 0;
        while ((1 << L.Sl) < s_raw) ++L.Sl;
        L.S = 1 << L.Sl;
        L.np = n * s_raw;
    }
    int bits = 0;
    while (((int64_t)1 << bits) < L.nt) ++bits;   // keys in [0, nt)
    L.passes = (bits + 7) / 8;
    if (L.passes < 1) L.passes = 1;
    L.sort_blocks = (L.np + SORT_CHUNK - 1) / SORT_CHUNK;
    L.emit_blocks = (n + BIN_NT - 1) / BIN_NT;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += align_up(bytes > 0 ? bytes : 1); return o; };
    L.o_fp = take(sizeof(int32_t) * 6 * (size_t)n);
    L.o_k0 = take(sizeof(uint32_t) * (size_t)L.np);
    L.o_v0 = take(sizeof(uint32_t) * (size_t)L.np);
    L.o_k1 = take(sizeof(uint32_t) * (size_t)L.np);
    L.o_v1 = take(sizeof(uint32_t) * (size_t)L.np);
    L.o_tcount = take(sizeof(uint32_t) * 4);   // forward's dynamic tile counter
    L.o_tstart = take(sizeof(uint32_t) * (size_t)(L.nt + 1));
    // per-call control block, zeroed by one memset: block tickets, the pair
    // count, per-pass global digit counts, the emit pass's look-back words,
    // then every sort pass's per-(block, digit) look-back words
    L.o_ctl = off;
    L.o_tickets = take(sizeof(uint32_t) * 8);
    L.o_ghist = take(sizeof(uint32_t) * RADIX * MAX_PASSES);
    L.o_stat_e = take(sizeof(unsigned long long) * (size_t)(L.emit_blocks > 0 ? L.emit_blocks : 1));
    L.o_stat_s = take(sizeof(unsigned long long) * RADIX * (size_t)L.passes *
                      (size_t)(L.sort_blocks > 0 ? L.sort_blocks : 1));
    L.ctl_bytes = off - L.o_ctl;
    // empty-space masks (zeroed and written by the masked forward)
    // per pixel column (y * w + x): bit tz set when its 16-slice segment in z
    // tile tz holds a non-zero voxel (the projector forward's skip test)
    L.o_pocc = take(sizeof(unsigned long long) * (size_t)w * h);
    // per pixel column: bit tz set when a Gaussian footprint covers the column
    // inside z tile tz (what the backward reads; the adjoints' skip test)
    L.o_fcov = take(sizeof(unsigned long long) * (size_t)w * h);
    L.o_rec = take(sizeof(GRec) * (size_t)n);
    // backward visiting order for volumes that exceed L2 (Gaussians sorted by
    // their first tile): first-slot flags, their exclusive scan, the list
    L.o_flag = take(sizeof(uint32_t) * (size_t)(L.np + 1));
    L.o_pos = take(sizeof(uint32_t) * (size_t)(L.np + 1));
    L.o_order = take(sizeof(uint32_t) * (size_t)(n + 1));
    L.o_scan2 = take(scan_temp_bytes(L.np + 1));
    L.total = off;
    L.final_buf = L.passes % 2;   // pass p reads buf p%2, writes (p+1)%2
    return L;
}

template <typename T>
static inline T* at(void* base, size_t off) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + off);
}
template <typename T>
static inline const T* at(const void* base, size_t off) {
    return reinterpret_cast<const T*>(reinterpret_cast<const char*>(base) + off);
}

// --------------------------------------------------------------------------
// footprints + pair emission
// --------------------------------------------------------------------------
// Look-back status words: 2-bit flag (1 = aggregate, 2 = inclusive prefix) |
// 62-bit value; the words are zeroed once per bin call.
constexpr unsigned long long LB_A = 1ull << 62, LB_P = 2ull << 62, LB_V = LB_A - 1;

// Walk back from block b over predecessors' status words (stride apart)
// until an inclusive prefix is found; returns the exclusive prefix of b.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* st, int64_t b,
                                                       int64_t stride) {
    unsigned long long excl = 0;
    for (int64_t pred = b - 1; pred >= 0; --pred) {
        unsigned long long w;
        do {
            w = *reinterpret_cast<volatile unsigned long long*>(&st[pred * stride]);
        } while ((w >> 62) == 0);
        excl += w & LB_V;
        if ((w >> 62) == 2) break;
    }
    return excl;
}

// The same walk for a whole warp, 32 predecessors per step (blocks that start
// together all publish aggregates first, so a serial walk would be long):
// the nearest inclusive word ends the sum.  Returns the exclusive prefix.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* st, int64_t b) {
    const int lane = threadIdx.x & 31;
    unsigned long long excl = 0;
    for (int64_t top = b - 1; top >= 0; top -= 32) {
        const int64_t pred = top - lane;
        unsigned long long w = 0;
        if (pred >= 0) {
            do {
                w = *reinterpret_cast<volatile unsigned long long*>(&st[pred]);
            } while ((w >> 62) == 0);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, pred >= 0 && (w >> 62) == 2);
        // lanes up to (and including) the nearest inclusive word contribute
        const int stop = incl ? __ffs(incl) - 1 : 31;
        unsigned long long v = (pred >= 0 && lane <= stop) ? (w & LB_V) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (incl) break;
    }
    return excl;
}

// Footprints + dense (tile, Gaussian) pairs in one pass.  Each block takes
// BIN_NT Gaussians in index order (block ids from a ticket, so look-back
// predecessors are always resident): footprint, GRec and tile count per
// Gaussian, a block scan of the counts, a decoupled look-back for the block's
// offset, then the block's pairs are written cooperatively (coalesced) in
// Gaussian order and (tz, ty, tx) slot order -- the value encodes
// Gaussian << Sl | slot.  The kernel also counts every sort pass's digits
// (global histograms), so each sort pass is a single kernel.
// Optional Adam step fused ahead of the binning (G null: none): each thread
// first updates its own Gaussian's five parameters and moments (adam_elem,
// bitwise k_adam's), then bins the updated Gaussian -- one pass and one
// launch fewer per training step.
struct AdamFuse {
    const double* G;
    double *M1, *M2;
    const double* s;   // {lr, 1 - b1^t, 1 - b2^t} from the iteration finalize
    double sfloor, sceil;
};

__global__ void __launch_bounds__(BIN_NT) k_bin_emit(
    const double* __restrict__ P, int64_t n, int w, int h, int c, int zoff, int hx, int hy,
    int hz, int ntx, int nty, int Sl, int passes, int ybits, int32_t* __restrict__ fp,
    GRec* __restrict__ rec, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
    uint32_t* __restrict__ ghist, unsigned long long* __restrict__ status,
    uint32_t* __restrict__ tickets, AdamFuse af, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ unsigned s_blk;
    __shared__ uint32_t s_off[BIN_NT + 1];
    __shared__ int4 s_tile[BIN_NT];        // tx0, ty0, tz0, nx | ny << 16
    __shared__ int s_ylo[BIN_NT];          // footprint's first row (row-ordered keys)
    __shared__ uint32_t s_warp[BIN_NT / 32];
    __shared__ uint32_t s_hist[MAX_PASSES][RADIX];
    __shared__ unsigned long long s_base;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t == 0) s_blk = atomicAdd(&tickets[0], 1u);
    if (t < RADIX)
        for (int p = 0; p < MAX_PASSES; ++p) s_hist[p][t] = 0u;
    __syncthreads();
    const int64_t blk = s_blk;
    const int64_t i = blk * BIN_NT + t;
    if (af.G != nullptr && i < n) {   // P is read back below by this thread only
        const double lr = af.s[0], bc1 = af.s[1], bc2 = af.s[2];
#pragma unroll
        for (int f = 0; f < 5; ++f)
            adam_elem(const_cast<double*>(P), af.G, af.M1, af.M2, f * n + i, f, lr, bc1, bc2,
                      af.sfloor, af.sceil);
    }
    uint32_t cnt = 0;
    int4 ti = make_int4(0, 0, 0, 1 | (1 << 16));
    int ylo0 = 0;
    if (i < n) {
        const int half[3] = {hx, hy, hz};
        const int dim[3] = {w, h, c};
        const int org[3] = {0, 0, zoff};
        int lo[3], hi[3];
        bool empty = false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            // local coordinates: global footprint minus the slab origin
            double f = floor(P[a * n + i]) - org[a];
            double l = f - half[a], u = f + half[a];
            if (l < 0.0) l = 0.0;
            if (u > dim[a] - 1) u = dim[a] - 1;
            if (!(l <= u)) {   // also catches NaN
                empty = true;
                lo[a] = 1; hi[a] = 0;
            } else {
                lo[a] = (int)l; hi[a] = (int)u;
            }
            fp[6 * i + 2 * a] = lo[a];
            fp[6 * i + 2 * a + 1] = hi[a];
        }
        if (!empty) {   // binned Gaussians have |floor(mu)| <= dim + half: int32 is exact
            GRec r;
            const double mx = P[i], my = P[n + i], mz = P[2 * n + i], sg = P[3 * n + i];
            const double fx = floor(mx), fy = floor(my), fz = floor(mz);
            r.fx = (int)fx; r.fy = (int)fy; r.fz = (int)fz;
            r.dx = (float)(mx - fx); r.dy = (float)(my - fy); r.dz = (float)(mz - fz);
            r.inv2 = (float)(0.5 / (sg * sg) * 1.4426950408889634);   // exp(-a) = exp2(-a log2 e)
            r.I = (float)P[4 * n + i];
            rec[i] = r;
            const int nx = hi[0] / TT - lo[0] / TT + 1, ny = hi[1] / TT - lo[1] / TT + 1;
            const int nz = hi[2] / TT - lo[2] / TT + 1;
            cnt = (uint32_t)(nx * ny * nz);
            ti = make_int4(lo[0] / TT, lo[1] / TT, lo[2] / TT, nx | (ny << 16));
            ylo0 = lo[1];
        }
    }
    s_tile[t] = ti;
    s_ylo[t] = ylo0;
    // block exclusive scan of the counts
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < BIN_NT / 32 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane < BIN_NT / 32) s_warp[lane] = v;
    }
    __syncthreads();
    const uint32_t excl = (wid > 0 ? s_warp[wid - 1] : 0u) + inc - cnt;
    const uint32_t total = s_warp[BIN_NT / 32 - 1];
    s_off[t] = excl;
    if (t == BIN_NT - 1) s_off[BIN_NT] = excl + cnt;
    if (wid == 0) {   // decoupled look-back over the preceding blocks' totals, 32 at a time
        unsigned long long base = 0;
        if (blk == 0) {
            if (lane == 0) atomicExch(&status[0], LB_P | (unsigned long long)total);
        } else {
            if (lane == 0) atomicExch(&status[blk], LB_A | (unsigned long long)total);
            base = lookback_warp(status, blk);
            if (lane == 0) atomicExch(&status[blk], LB_P | (base + total));
        }
        if (lane == 0) {
            s_base = base;
            if (blk == (int64_t)gridDim.x - 1) tickets[1] = (uint32_t)(base + total);   // pairs
        }
    }
    __syncthreads();
    const uint64_t base = s_base;
    for (uint32_t q = t; q < total; q += BIN_NT) {
        // owner: the last Gaussian whose offset is <= q (empty Gaussians share offsets)
        int lo = 0, hi = BIN_NT;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_off[mid] <= q) lo = mid; else hi = mid;
        }
        const uint32_t slot = q - s_off[lo];
        const int4 g = s_tile[lo];
        const int nx = g.w & 0xffff, ny = g.w >> 16;
        // small exact quotients through f32 (slot < S, a few thousand at most:
        // the half-unit margin dwarfs the approximate division's error)
        const int sy = (int)__fdividef((float)slot + 0.5f, (float)nx);
        const int sz = (int)__fdividef((float)sy + 0.5f, (float)ny);
        const int tx = g.x + (int)slot - sy * nx, ty = g.y + sy - sz * ny, tz = g.z + sz;
        // row-ordered bins (ybits > 0): inside a tile, the pairs are ordered by the
        // footprint's first row relative to the tile (in [-16, 15] for boxes up
        // to 17 rows; quantised to ybits), then by Gaussian -- so a k8 step of the
        // forward sees Gaussians covering similar rows and whole warps skip it
        uint32_t key = (uint32_t)((tz * nty + ty) * ntx + tx);
        if (ybits) {
            const int rel = min(max(s_ylo[lo] - TT * ty + 16, 0), 31);
            key = (key << ybits) | ((uint32_t)rel >> (5 - ybits));
        }
        keys[base + q] = key;
        vals[base + q] = ((uint32_t)(blk * BIN_NT + lo) << Sl) | slot;
        for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    if (t < RADIX)
        for (int p = 0; p < passes; ++p)
            if (s_hist[p][t]) atomicAdd(&ghist[p * RADIX + t], s_hist[p][t]);
}

// --------------------------------------------------------------------------
// stable LSD radix sort, 8-bit digits
// --------------------------------------------------------------------------
// One stable LSD pass ("onesweep"): a block takes SORT_CHUNK keys, each warp
// a contiguous run of 32 * SORT_IPT kept in registers.  Warps rank their own
// keys (match_any per 32-key round, per-warp digit counters in shared
// memory, warp-synchronous); the block's per-digit totals are published and
// each digit's offset among preceding blocks comes from a decoupled
// look-back (one thread per digit); the global digit offsets come from the
// histograms counted by k_bin_emit.  Three block barriers per pass, one
// kernel per pass, no separate histogram or scan.
__global__ void __launch_bounds__(SORT_NT) k_onesweep(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, const uint32_t* __restrict__ npairs,
    int shift, const uint32_t* __restrict__ ghist, unsigned long long* __restrict__ status,
    uint32_t* __restrict__ ticket, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    constexpr int NW = SORT_NT / 32;
    __shared__ unsigned s_blk;
    __shared__ uint32_t wh[NW][RADIX];    // per-warp digit counts, then local warp offsets
    __shared__ uint32_t s_warp[NW], s_lwarp[NW];
    __shared__ uint32_t s_lstart[RADIX], s_gstart[RADIX];   // digit starts: block-local, global
    __shared__ uint32_t sk[SORT_CHUNK], sv[SORT_CHUNK];      // the block's keys, locally sorted
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t == 0) s_blk = atomicAdd(ticket, 1u);
#pragma unroll
    for (int q = 0; q < NW; ++q) wh[q][t] = 0u;
    __syncthreads();
    const int64_t b = s_blk;
    const int64_t np = *npairs;
    const int64_t base = b * (int64_t)SORT_CHUNK;
    if (base >= np) return;   // block-uniform: later tickets are past the end too
    const int64_t wbase = base + (int64_t)wid * 32 * SORT_IPT + lane;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t k[SORT_IPT], v[SORT_IPT], rk[SORT_IPT];
#pragma unroll
    for (int r = 0; r < SORT_IPT; ++r) {
        const int64_t g = wbase + r * 32;
        const bool valid = g < np;
        k[r] = valid ? kin[g] : 0u;
        v[r] = valid ? vin[g] : 0u;
        const uint32_t d = valid ? (k[r] >> shift) & 255u : (uint32_t)RADIX;   // invalid: own group
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = valid ? wh[wid][d] : 0u;
        rk[r] = before + __popc(peers & lt_mask);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wh[wid][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // digit t: block total, offset among preceding blocks, global digit offset
        uint32_t mine = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) mine += wh[q][t];
        unsigned long long* st = status + t;   // word (block, digit) at block * RADIX + digit
        unsigned long long prev = 0;
        if (b == 0) {
            atomicExch(&st[0], LB_P | (unsigned long long)mine);
        } else {
            atomicExch(&st[b * RADIX], LB_A | (unsigned long long)mine);
            prev = lookback(st, b, RADIX);
            atomicExch(&st[b * RADIX], LB_P | (prev + mine));
        }
        // exclusive scans over digits: global digit counts and this block's totals
        const uint32_t gd = ghist[t];
        uint32_t inc = gd, linc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            const uint32_t lu = __shfl_up_sync(0xffffffffu, linc, o);
            if (lane >= o) {
                inc += u;
                linc += lu;
            }
        }
        if (lane == 31) {
            s_warp[wid] = inc;
            s_lwarp[wid] = linc;
        }
        __syncthreads();
        uint32_t gpre = inc - gd, lpre = linc - mine;
        for (int q = 0; q < wid; ++q) {
            gpre += s_warp[q];
            lpre += s_lwarp[q];
        }
        s_gstart[t] = (uint32_t)prev + gpre;   // global position of the block's first key t
        s_lstart[t] = lpre;                    // its position in the block's sorted order
        uint32_t acc = lpre;
#pragma unroll
        for (int q = 0; q < NW; ++q) {   // local warp offsets for digit t, in warp order
            const uint32_t c2 = wh[q][t];
            wh[q][t] = acc;
            acc += c2;
        }
    }
    __syncthreads();
    // sort the block's keys in shared memory, then write each digit's run with
    // consecutive threads at consecutive global positions (coalesced)
    int nvalid = 0;
#pragma unroll
    for (int r = 0; r < SORT_IPT; ++r) {
        const int64_t g = wbase + r * 32;
        if (g < np) {
            const uint32_t lp = wh[wid][(k[r] >> shift) & 255u] + rk[r];
            sk[lp] = k[r];
            sv[lp] = v[r];
        }
    }
    nvalid = (int)min((int64_t)SORT_CHUNK, np - base);
    __syncthreads();
    for (int i = t; i < nvalid; i += SORT_NT) {
        const uint32_t kk = sk[i];
        const uint32_t d = (kk >> shift) & 255u;
        const uint32_t pos = s_gstart[d] + ((uint32_t)i - s_lstart[d]);
        kout[pos] = kk;
        vout[pos] = sv[i];
    }
}

// --------------------------------------------------------------------------
// forward: one CTA per 16^3 tile on the tensor cores.
//
// Inside a tile the splat is a rank-K sum of separable factors,
//   V[y][x][z] = sum_k ex_k[x] * (I_k ey_k[y] ez_k[z]),
// i.e. a GEMM D[x][(y,z)] = A[x][k] B[k][(y,z)] with A = ex (16 x K) and B the
// per-Gaussian outer product I ey (x) ez (K x 256).  Each warp owns two y rows
// (N = 32 = 4 n8 tiles) and all 16 x (M = 16) and runs mma.sync m16n8k8 TF32
// with the 3xTF32 split (a_hi b_hi + a_hi b_lo + a_lo b_hi, fp32 accumulate),
// which keeps fp32-level accuracy (the volume target is 1e-5 relative L2).
// The separable tables (I ey, ex, ez; zero outside box, tile and volume) are
// built 64 Gaussians at a time (FWD_BATCH) in shared memory exactly as before; padding
// rows are zero so partial k8 steps contribute nothing.  Accumulators go
// through an XOR-swizzled shared-memory tile for coalesced stores.
// --------------------------------------------------------------------------
#ifndef FWD_TPG
// table-builder threads per Gaussian: 4 = 64-Gaussian batches, half the block
// barriers per Gaussian of 32-Gaussian batches (C2 0.100 -> 0.092 ms; 2 would
// need 53 KB of static shared memory)
#define FWD_TPG 4
#endif
constexpr int FWD_BATCH = 256 / FWD_TPG;   // Gaussians staged per round
#ifndef FWD_MINB
#define FWD_MINB 4   // CTAs per SM (64 registers)
#endif
// per Gaussian row: ex_hi[16] | ex_lo[16] (TF32 split, A operand) | I ey[16] | ez[16] | pad
constexpr int TAB_STRIDE = 72;  // 72 mod 32 = 8: the four k rows of a fragment hit distinct banks

// Separable weight of tile-local coordinate l on one axis (zero outside the
// box or the local volume): exp(-(b - d)^2 inv2), b = coord - floor(mu).
__device__ __forceinline__ float tab_weight(int coord_local, int origin, int dim, int f, int half,
                                            float d, float inv2) {
    const int b = coord_local + origin - f;
    if (coord_local >= dim || b > half || b < -half) return 0.f;
    const float r = (float)b - d;
    return exp2f(-inv2 * r * r);   // inv2 carries log2(e)
}

// x = hi + lo with hi a TF32 value (round-half-away on the 13 dropped bits;
// inputs are finite and >= 0) and lo exact in fp32 (the MMA reads its top 19
// bits, |lo| <= 2^-11 |x|, so the split keeps ~2^-22 relative accuracy).
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
    hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(256, FWD_MINB) k_fvr_fwd(const GRec* __restrict__ rec, int w, int h, int c,
                                                 int zoff, int hx, int hy, int hz, int ntx,
                                                 int nty, int64_t nt, int S,
                                                 const uint32_t* __restrict__ tstart,
                                                 const uint32_t* __restrict__ svals,
                                                 float* __restrict__ vol,
                                                 unsigned int* __restrict__ counter, int fetch,
                                                 unsigned long long* __restrict__ pocc,
                                                 unsigned long long* __restrict__ fcov,
                                                 const __grid_constant__ CUtensorMap tmap,
                                                 int use_tma, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ __align__(16) float tab[FWD_BATCH * TAB_STRIDE];
    // [y*16+x][z/4] with the 16-byte chunk XOR-swizzled by (row >> 1) & 3: exactly
    // TMA's 64-byte swizzle, so the tile leaves through one bulk tensor store
    __shared__ __align__(1024) float4 sacc[TT * TT][TT / 4];
    __shared__ int64_t s_next;
    __shared__ unsigned s_rows[TT];   // footprint coverage: x bits per tile row
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;        // mma fragment coordinates
    const int r0 = 2 * wid;                        // this warp's two tile rows (y)
    const int ntz = (int)(nt / ((int64_t)ntx * nty));
    // persistent CTAs fetch tiles dynamically (uneven per-tile cost); tiles are
    // visited z-fastest so consecutive fetches write adjacent 64 B column
    // segments (HBM-friendly for the all-zero tiles of sparse volumes)
    // `fetch` consecutive tiles are claimed per counter bump (1 for dense
    // volumes, up to 32 for sparse ones where most tiles are empty zero-stores)
    for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_next = (int64_t)atomicAdd(counter, (unsigned)fetch);
    __syncthreads();
    const int64_t kc = s_next;
    if (kc >= nt) break;
    const int kend = (int)min(kc + fetch, nt);
    for (int k32 = (int)kc; k32 < kend; ++k32) {   // nt < 2^31 (check_args)
    const int tzi = k32 % ntz;
    const int rest = k32 / ntz;
    const int txi = rest % ntx, tyi = rest / ntx;
    const int64_t t = ((int64_t)tzi * nty + tyi) * ntx + txi;
    const int x0 = txi * TT, y0 = tyi * TT, z0 = tzi * TT;
    const uint32_t beg = tstart[t], end = tstart[t + 1];
    const bool empty = beg == end;
    if (use_tma && threadIdx.x == 0)   // sacc is rewritten after this tile's barriers
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    // (the previous tile's readers passed the barrier after their read)
    if (threadIdx.x < TT) s_rows[threadIdx.x] = 0u;
    float acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    const int tg = threadIdx.x / FWD_TPG, tj = threadIdx.x % FWD_TPG;   // table builder: Gaussian, part

    // the next batch's Gaussian records are loaded while this batch's MMAs run,
    // from pair values loaded one batch earlier still (the value -> record
    // chain would otherwise stall the warp in order at the record load)
    GRec rn;
    if (beg + tg < end) rn = rec[svals[beg + tg] >> S];   // S = log2(slots per Gaussian)
    uint32_t vn = beg + FWD_BATCH + tg < end ? svals[beg + FWD_BATCH + tg] : 0u;
    for (uint32_t b0 = beg; b0 < end; b0 += FWD_BATCH) {
        const int nb = (int)min((uint32_t)FWD_BATCH, end - b0);
        const int nk = (nb + 7) & ~7;
        const GRec r = rn;
        if (b0 + FWD_BATCH + tg < end) rn = rec[vn >> S];
        if (b0 + 2 * FWD_BATCH + tg < end) vn = svals[b0 + 2 * FWD_BATCH + tg];
        __syncthreads();
        if (tg < nk) {
            float* row = tab + tg * TAB_STRIDE;
            uint32_t* urow = reinterpret_cast<uint32_t*>(row);
            if (tg < nb) {
                if (fcov) {   // footprint coverage of this tile's columns: rows tj, tj + 8
                    const int bx0 = max(r.fx - hx, x0), bx1 = min(min(r.fx + hx, w - 1), x0 + TT - 1);
                    const int by0 = max(r.fy - hy, y0), by1 = min(min(r.fy + hy, h - 1), y0 + TT - 1);
                    if (bx0 <= bx1) {
                        const unsigned xb = ((2u << (bx1 - x0)) - 1u) & ~((1u << (bx0 - x0)) - 1u);
#pragma unroll
                        for (int rr = 0; rr < TT / FWD_TPG; ++rr) {
                            const int yy = y0 + tj + FWD_TPG * rr;
                            if (yy >= by0 && yy <= by1) atomicOr(&s_rows[tj + FWD_TPG * rr], xb);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < 3 * TT / FWD_TPG; ++q) {
                    const int e = tj + FWD_TPG * q, a = e / TT, l = e % TT;   // compile-time a per q
                    if (a == 0) {
                        uint32_t hi, lo;
                        tf32_split(tab_weight(x0 + l, 0, w, r.fx, hx, r.dx, r.inv2), hi, lo);
                        urow[l] = hi;
                        urow[TT + l] = lo;
                    } else if (a == 1) {
                        row[2 * TT + l] = tab_weight(y0 + l, 0, h, r.fy, hy, r.dy, r.inv2) * r.I;
                    } else {
                        row[3 * TT + l] = tab_weight(z0 + l, zoff, c, r.fz, hz, r.dz, r.inv2);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4 * TT / FWD_TPG; ++q) row[tj + FWD_TPG * q] = 0.f;   // k8 padding
            }
        }
        __syncthreads();
        for (int k0 = 0; k0 < nk; k0 += 8) {
            const float* ra = tab + (k0 + t4) * TAB_STRIDE;       // Gaussian k0 + t
            const float* rb = tab + (k0 + t4 + 4) * TAB_STRIDE;   // Gaussian k0 + t + 4
            const float ya0 = ra[2 * TT + r0], ya1 = ra[2 * TT + r0 + 1];
            const float yb0 = rb[2 * TT + r0], yb1 = rb[2 * TT + r0 + 1];
            // none of the step's 8 Gaussians reaches this warp's two rows: its B
            // operand is all zero and the step would add exact zeros (skipping it
            // is bitwise neutral); row-ordered bins make this common
            if (!__any_sync(0xffffffffu, ya0 != 0.f || ya1 != 0.f || yb0 != 0.f || yb1 != 0.f))
                continue;
            const uint32_t* ua = reinterpret_cast<const uint32_t*>(ra);
            const uint32_t* ub = reinterpret_cast<const uint32_t*>(rb);
            // A[x][k] = ex_k[x], pre-split by the table builder
            const uint32_t ah[4] = {ua[g], ua[g + 8], ub[g], ub[g + 8]};
            const uint32_t al[4] = {ua[TT + g], ua[TT + g + 8], ub[TT + g], ub[TT + g + 8]};
            const float za0 = ra[3 * TT + g], za1 = ra[3 * TT + g + 8];
            const float zb0 = rb[3 * TT + g], zb1 = rb[3 * TT + g + 8];
            // n-tile j: row r0 + (j >> 1), z = (j & 1) * 8 + n
            uint32_t bh[4][2], bl[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float ya = (j >> 1) ? ya1 : ya0, yb = (j >> 1) ? yb1 : yb0;
                const float za = (j & 1) ? za1 : za0, zb = (j & 1) ? zb1 : zb0;
                tf32_split(ya * za, bh[j][0], bl[j][0]);   // B[k=t][n=g]
                tf32_split(yb * zb, bh[j][1], bl[j][1]);   // B[k=t+4][n=g]
            }
            // each k8 step accumulates from zero (small terms first) and is
            // added to the fp32 accumulators with round-to-nearest: the tensor
            // core's truncating accumulation then only biases one step's
            // partial sum, not the tile's running total.  The four n-tiles'
            // chains are interleaved so consecutive HMMAs are independent.
            float d[4][4];
#pragma unroll
            for (int j = 0; j < 4; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_tf32(d[j], al, bh[j][0], bh[j][1]);
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_tf32(d[j], ah, bl[j][0], bl[j][1]);
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_tf32(d[j], ah, bh[j][0], bh[j][1]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[j][q] += d[j][q];
        }
    }
    if (!empty) {   // accumulators -> swizzled [column][z] tile
        float* sf = reinterpret_cast<float*>(sacc);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int y = r0 + (j >> 1);
            const int z = (j & 1) * 8 + 2 * t4;
            const int q = z >> 2, hf = z & 3;   // float4 chunk, offset 0 or 2
#pragma unroll
            for (int hx8 = 0; hx8 < 2; ++hx8) {
                const int col = y * TT + g + 8 * hx8;
                float2* dst = reinterpret_cast<float2*>(
                    sf + (col * 4 + (q ^ ((col >> 1) & 3))) * 4 + hf);
                *dst = make_float2(acc[j][2 * hx8], acc[j][2 * hx8 + 1]);
            }
        }
        if (use_tma) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
    }
    if (fcov && !empty && ntz <= 64) {   // after the last batch's barrier: rows complete
        const int x = x0 + (threadIdx.x & (TT - 1)), y = y0 + (threadIdx.x >> 4);
        if (x < w && y < h && ((s_rows[threadIdx.x >> 4] >> (threadIdx.x & (TT - 1))) & 1u))
            atomicOr(&fcov[(int64_t)y * w + x], 1ull << tzi);
        __syncthreads();   // before the next tile zeroes the rows
    }
    // store: non-empty tiles leave through one TMA bulk tensor store (the
    // tensor map clips tiles at the volume edges); otherwise the tile's 256
    // columns x 64 B are written 8 columns per warp instruction (4 lanes x
    // 16 B per column); empty tiles store zeros directly
    if (use_tma && !empty) {
        if (threadIdx.x == 0) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&sacc[0][0]);
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                "cp.async.bulk.commit_group;\n" ::"l"(&tmap), "r"(z0), "r"(x0), "r"(y0), "r"(sa)
                : "memory");
        }
        if (pocc && ntz <= 64) {   // column segment occupancy from the staged tile
            const int x = x0 + (threadIdx.x & (TT - 1)), y = y0 + (threadIdx.x >> 4);
            bool nz = false;
#pragma unroll
            for (int q = 0; q < TT / 4; ++q) {
                const float4 v = sacc[threadIdx.x][q];
                nz |= v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f;
            }
            if (nz && x < w && y < h) atomicOr(&pocc[(int64_t)y * w + x], 1ull << tzi);
        }
    } else if ((c & 3) == 0 && z0 + TT <= c) {
        const int ch = lane & 3;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int cid = wid * 32 + i * 8 + (lane >> 2);
            const int x = x0 + (cid & (TT - 1)), y = y0 + cid / TT;
            const float4 v = empty ? make_float4(0.f, 0.f, 0.f, 0.f)
                                   : sacc[cid][ch ^ ((cid >> 1) & 3)];
            if (x < w && y < h)
                *reinterpret_cast<float4*>(vol + ((int64_t)y * w + x) * c + z0 + 4 * ch) = v;
            if (pocc && !empty && ntz <= 64) {   // column segment occupancy (4 lanes per column)
                const bool nz = v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f;
                const unsigned b = __ballot_sync(0xffffffffu, nz);
                if (ch == 0 && ((b >> (lane & ~3)) & 0xfu) && x < w && y < h)
                    atomicOr(&pocc[(int64_t)y * w + x], 1ull << tzi);
            }
        }
    } else {   // ragged z tile: one column per thread, scalar stores
        const int cid = threadIdx.x;
        const int x = x0 + (cid & (TT - 1)), y = y0 + cid / TT;
        if (x < w && y < h) {
            float* col = vol + ((int64_t)y * w + x) * c;
            bool nz = false;
#pragma unroll
            for (int q = 0; q < TT / 4; ++q) {
                const float4 v = empty ? make_float4(0.f, 0.f, 0.f, 0.f)
                                       : sacc[cid][q ^ ((cid >> 1) & 3)];
                if (z0 + 4 * q + 0 < c) { col[z0 + 4 * q + 0] = v.x; nz |= v.x != 0.f; }
                if (z0 + 4 * q + 1 < c) { col[z0 + 4 * q + 1] = v.y; nz |= v.y != 0.f; }
                if (z0 + 4 * q + 2 < c) { col[z0 + 4 * q + 2] = v.z; nz |= v.z != 0.f; }
                if (z0 + 4 * q + 3 < c) { col[z0 + 4 * q + 3] = v.w; nz |= v.w != 0.f; }
            }
            if (pocc && nz && ntz <= 64) atomicOr(&pocc[(int64_t)y * w + x], 1ull << tzi);
        }
    }
    }   // tile
    }   // fetch
    if (use_tma && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    // every CTA has made its last claim once it gets here: the last one to
    // exit resets the claim counter (and the exit ticket) for the next forward
    if (threadIdx.x == 0 && atomicAdd(&counter[2], 1u) == gridDim.x - 1) {
        counter[0] = 0u;
        counter[2] = 0u;
    }
}

// --------------------------------------------------------------------------
// forward on the FP32 pipe: register-blocked FFMA2 with the work cut to the
// footprints at warp granularity.
//
// One 64-thread CTA per 16^3 tile (persistent, tiles claimed from a counter).
// A thread owns two adjacent columns (x, x+1) of two adjacent rows (y, y+1),
// 16 slices each: 32 float2 accumulators {V[y][x][z], V[y][x+1][z]}.  A warp
// owns 8 rows x 16 columns x 16 slices.  Per 32-Gaussian batch of the tile
// list (ascending id: deterministic sums) the table builders write, per
// Gaussian, ex (column pairs), I ey, ez (zero outside box, tile and volume)
// and the integer footprint inside the tile (rows, columns, z halves); each
// warp then ballots the Gaussians whose rows meet its 8 rows and walks only
// those.  The z overlap of a box with a 16-slice tile is a prefix, a suffix or
// both halves, so only covered half-tiles are summed (uniform branch).  Per
// Gaussian and lane: w = (I ey[y], I ey[y+1]) x {ex[x], ex[x+1]} (two FMUL2),
// then acc[r][z] += w[r] * ez[z] (one FFMA2 per row and slice).  Columns leave
// as 64-byte float4 runs straight from registers.
// --------------------------------------------------------------------------
constexpr int FF_THREADS = 64;
constexpr int FF_BATCH = 32;

struct __align__(16) FTab {
    float ez[16];     // z weights (zero outside box, tile, volume)
    float2 ex[8];     // x weights, column pairs
    float2 ey[8];     // I * y weights, row pairs
    int ym;           // rows covered (bits 0..15) | z halves (bit 16: low, bit 17: high)
    int xm;           // columns covered by the footprint (coverage mask)
    int pad[2];
};

template <bool MASKS>
__global__ void __launch_bounds__(FF_THREADS, 8)
    k_fvr_fwd_ff(const GRec* __restrict__ rec, int w, int h, int c, int zoff, int hx, int hy,
                 int hz, int ntx, int nty, int64_t nt, int S,
                 const uint32_t* __restrict__ tstart, const uint32_t* __restrict__ svals,
                 float* __restrict__ vol, unsigned int* __restrict__ counter, int fetch,
                 unsigned long long* __restrict__ pocc, unsigned long long* __restrict__ fcov,
                 const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ FTab tab[FF_BATCH];
    __shared__ int64_t s_next;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int xp = lane & 7;                   // column pair
    const int rp = wid * 4 + (lane >> 3);      // row pair: rows 2 rp, 2 rp + 1
    const int ntz = (int)(nt / ((int64_t)ntx * nty));
    const int tg = threadIdx.x >> 1, th = threadIdx.x & 1;   // table builder: Gaussian, half
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_next = (int64_t)atomicAdd(counter, (unsigned)fetch);
        __syncthreads();
        const int64_t kc = s_next;
        if (kc >= nt) break;
        const int kend = (int)min(kc + fetch, nt);
        for (int k32 = (int)kc; k32 < kend; ++k32) {
            const int tzi = k32 % ntz;
            const int rest = k32 / ntz;
            const int txi = rest % ntx, tyi = rest / ntx;
            const int64_t t = ((int64_t)tzi * nty + tyi) * ntx + txi;
            const int x0 = txi * TT, y0 = tyi * TT, z0 = tzi * TT;
            const uint32_t beg = tstart[t], end = tstart[t + 1];
            float2 acc0[16], acc1[16];
#pragma unroll
            for (int z = 0; z < 16; ++z) acc0[z] = acc1[z] = make_float2(0.f, 0.f);
            unsigned cov0 = 0u, cov1 = 0u;
            GRec rn;
            if (beg + tg < end) rn = rec[svals[beg + tg] >> S];
            for (uint32_t b0 = beg; b0 < end; b0 += FF_BATCH) {
                const int nb = (int)min((uint32_t)FF_BATCH, end - b0);
                const GRec r = rn;
                if (b0 + FF_BATCH + tg < end) rn = rec[svals[b0 + FF_BATCH + tg] >> S];
                __syncthreads();   // the previous batch's table reads are done
                if (tg < nb) {     // half th: entries 8 th .. 8 th + 7 of ex, ey, ez
                    FTab& T = tab[tg];
                    float vx[8], vy[8], vz[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int l = 8 * th + q;
                        vx[q] = tab_weight(x0 + l, 0, w, r.fx, hx, r.dx, r.inv2);
                        vy[q] = tab_weight(y0 + l, 0, h, r.fy, hy, r.dy, r.inv2) * r.I;
                        vz[q] = tab_weight(z0 + l, zoff, c, r.fz, hz, r.dz, r.inv2);
                    }
                    float4* ex4 = reinterpret_cast<float4*>(T.ex) + 2 * th;
                    float4* ey4 = reinterpret_cast<float4*>(T.ey) + 2 * th;
                    float4* ez4 = reinterpret_cast<float4*>(T.ez) + 2 * th;
                    ex4[0] = make_float4(vx[0], vx[1], vx[2], vx[3]);
                    ex4[1] = make_float4(vx[4], vx[5], vx[6], vx[7]);
                    ey4[0] = make_float4(vy[0], vy[1], vy[2], vy[3]);
                    ey4[1] = make_float4(vy[4], vy[5], vy[6], vy[7]);
                    ez4[0] = make_float4(vz[0], vz[1], vz[2], vz[3]);
                    ez4[1] = make_float4(vz[4], vz[5], vz[6], vz[7]);
                    if (th == 0) {   // integer footprint inside the tile (a3): rows, columns, z halves
                        const int by0 = max(r.fy - hy, y0), by1 = min(min(r.fy + hy, h - 1), y0 + TT - 1);
                        const int bx0 = max(r.fx - hx, x0), bx1 = min(min(r.fx + hx, w - 1), x0 + TT - 1);
                        const int bz0 = max(r.fz - zoff - hz, z0);
                        const int bz1 = min(min(r.fz - zoff + hz, c - 1), z0 + TT - 1);
                        int ym = 0, xm = 0;
                        if (by0 <= by1 && bx0 <= bx1 && bz0 <= bz1) {
                            ym = (int)(((2u << (by1 - y0)) - 1u) & ~((1u << (by0 - y0)) - 1u));
                            xm = (int)(((2u << (bx1 - x0)) - 1u) & ~((1u << (bx0 - x0)) - 1u));
                            if (bz0 - z0 < 8) ym |= 1 << 16;
                            if (bz1 - z0 >= 8) ym |= 1 << 17;
                        }
                        T.ym = ym;
                        T.xm = xm;
                    }
                }
                __syncthreads();
                // the Gaussians whose rows meet this warp's 8 rows
                unsigned todo = __ballot_sync(
                    0xffffffffu, lane < nb && ((tab[lane].ym >> (8 * wid)) & 0xFF) != 0);
                while (todo) {
                    const int kb = __ffs(todo) - 1;
                    todo &= todo - 1u;
                    const FTab& T = tab[kb];
                    const int2 m = *reinterpret_cast<const int2*>(&T.ym);
                    const float2 e = T.ex[xp];
                    const float2 wy = T.ey[rp];
                    const float4* ez4 = reinterpret_cast<const float4*>(T.ez);
                    const float4 za = ez4[0], zb = ez4[1], zc = ez4[2], zd = ez4[3];
                    const float2 wa = make_float2(e.x * wy.x, e.y * wy.x);
                    const float2 wb = make_float2(e.x * wy.y, e.y * wy.y);
                    if (MASKS) {
                        if ((m.x >> (2 * rp)) & 1) cov0 |= (unsigned)m.y;
                        if ((m.x >> (2 * rp + 1)) & 1) cov1 |= (unsigned)m.y;
                    }
#define FF_Q(Z, V, K)                                                        \
    acc0[K] = ffma2(make_float2(V, V), wa, acc0[K]);                         \
    acc1[K] = ffma2(make_float2(V, V), wb, acc1[K]);
                    if (m.x & (1 << 16)) {
                        FF_Q(0, za.x, 0) FF_Q(0, za.y, 1) FF_Q(0, za.z, 2) FF_Q(0, za.w, 3)
                        FF_Q(0, zb.x, 4) FF_Q(0, zb.y, 5) FF_Q(0, zb.z, 6) FF_Q(0, zb.w, 7)
                    }
                    if (m.x & (1 << 17)) {
                        FF_Q(0, zc.x, 8) FF_Q(0, zc.y, 9) FF_Q(0, zc.z, 10) FF_Q(0, zc.w, 11)
                        FF_Q(0, zd.x, 12) FF_Q(0, zd.y, 13) FF_Q(0, zd.z, 14) FF_Q(0, zd.w, 15)
                    }
#undef FF_Q
                }
            }
            // store: each column's 16 slices are one 64-byte run
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int y = y0 + 2 * rp + rr;
#pragma unroll
                for (int hc = 0; hc < 2; ++hc) {
                    const int x = x0 + 2 * xp + hc;
                    if (x >= w || y >= h) continue;
                    float v[16];
#pragma unroll
                    for (int z = 0; z < 16; ++z)
                        v[z] = rr ? (hc ? acc1[z].y : acc1[z].x) : (hc ? acc0[z].y : acc0[z].x);
                    float* col = vol + ((int64_t)y * w + x) * c + z0;
                    if ((c & 3) == 0 && z0 + TT <= c) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            reinterpret_cast<float4*>(col)[q] =
                                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int z = 0; z < 16; ++z)
                            if (z0 + z < c) col[z] = v[z];
                    }
                    if (MASKS && ntz <= 64) {
                        bool nz = false;
#pragma unroll
                        for (int z = 0; z < 16; ++z) nz |= v[z] != 0.f;
                        if (nz) atomicOr(&pocc[(int64_t)y * w + x], 1ull << tzi);
                        if ((((rr ? cov1 : cov0) >> (2 * xp + hc)) & 1u))
                            atomicOr(&fcov[(int64_t)y * w + x], 1ull << tzi);
                    }
                }
            }
        }
    }
}

// --------------------------------------------------------------------------
// forward on the 5th-generation tensor cores (tcgen05, the default).
//
// Per 16^3 tile the splat is the rank-K GEMM D[(y,x)][z] = sum_k A[(y,x)][k] B[k][z]
// with A = (I ey) (x) ex (the 256-row outer product of Gaussian k) and B = ez.
// D is two M = 128 accumulators (rows y 0..7 / 8..15) of N = 16 slices in
// TMEM; K runs over the tile's Gaussian list (ascending id) in stages of 32.
// fp32-level accuracy from the 3xTF32 split (hi = x & ~0x1fff, lo = x - hi):
// D += Alo Bhi + Ahi Blo + Ahi Bhi per k8 chunk (validated bitwise by
// splatct_tc_selftest).  Warp roles, one persistent 416-thread CTA per SM
// over a contiguous, cost-balanced range of tiles:
//   * 8 producer warps: per stage, the separable tables (ex, I ey, ez; zero
//     outside box, tile and volume) into shared memory, then each thread forms
//     its row's 32 outer-product values, splits them and writes A straight into
//     TMEM (tcgen05.st; A never touches shared memory), and B (16 x 32, K-major)
//     into a shared-memory stage; the footprint coverage rows for the masks;
//   * 1 MMA warp: one elected thread issues 24 kind::tf32 MMAs per stage
//     (M 128, N 16, K 8; A from TMEM) and commits to mbarriers;
//   * 4 epilogue warps: tcgen05.ld of the two accumulators (a thread gets one
//     pixel column's 16 slices per half), 64-byte column stores, empty-space
//     masks; empty tiles store zeros without touching the tensor core.
// Stages (A in TMEM, B in shared memory) and accumulators are double-buffered.
// --------------------------------------------------------------------------
constexpr int TC_KS = 32;          // Gaussians per stage
constexpr int TC_P_WARPS = 16;   // 4 lane quadrants x 2 row halves x 2 k halves
constexpr int TC_THREADS = 32 * (TC_P_WARPS + 1 + 4);
constexpr int TC_TS = TC_KS + 4;   // table row stride (floats): conflict-free LDS.128 rows
constexpr int TC_ALPHA = 4;        // cost of an empty tile, in (tile, Gaussian) pairs

struct TcSmem {
    float ex[2][16][TC_TS], ey[2][16][TC_TS], ez[2][16][TC_TS];   // [buf][coordinate][k]
    uint32_t bop[2][2][TC_KS * 16];                               // [slot][hi, lo] B, K-major
    uint32_t covw[4][TC_P_WARPS][16];                              // per tile: rows' covered columns
    uint64_t a_full[2], a_empty[2], d_full[2], d_empty[2], cov_full[4];
    uint32_t tbase;
    int t_begin, t_end;
};

// first tile t with cost(t) = tstart[t] + ALPHA t >= target (cost is increasing)
__device__ __forceinline__ int64_t tc_lower(const uint32_t* tstart, int64_t nt, int64_t target) {
    int64_t lo = 0, hi = nt;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)tstart[mid] + TC_ALPHA * mid < target) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void p_bar() {   // the 256 producer threads
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * TC_P_WARPS) : "memory");
}

constexpr int TC_LIST_CAP = 7680;   // non-empty tiles per CTA (the 120 KB dynamic list)

// Walks the stages (32-Gaussian slices) of the CTA's non-empty tile list.
struct TcStage {
    int i;          // list index
    uint32_t k0;    // first Gaussian of the stage within the tile
    __device__ __forceinline__ void next(const int4* list) {
        k0 += TC_KS;
        if (k0 >= (uint32_t)list[i].z) {
            k0 = 0;
            ++i;
        }
    }
};

template <bool MASKS>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_fvr_fwd_tc(const GRec* __restrict__ rec, int w, int h, int c, int zoff, int hx, int hy,
                 int hz, int ntx, int nty, int64_t nt, int S,
                 const uint32_t* __restrict__ tstart, const uint32_t* __restrict__ svals,
                 float* __restrict__ vol, unsigned long long* __restrict__ pocc,
                 unsigned long long* __restrict__ fcov, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ __align__(128) TcSmem sm;
    __shared__ int s_wcount[TC_THREADS / 32 + 1];
    extern __shared__ int4 tlist[];   // {tile, begin, count, 0} of the CTA's non-empty tiles
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntz = (int)(nt / ((int64_t)ntx * nty));
    const int64_t nxy = (int64_t)ntx * nty;
    if (warp == TC_P_WARPS) tc::tmem_alloc(&sm.tbase, 512);
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&sm.a_full[i], TC_P_WARPS);
            tc::mbar_init(&sm.a_empty[i], 1);
            tc::mbar_init(&sm.d_full[i], 1);
            tc::mbar_init(&sm.d_empty[i], 4);
        }
        for (int i = 0; i < 4; ++i) tc::mbar_init(&sm.cov_full[i], TC_P_WARPS);
        tc::mbar_init_fence();
        const int64_t F = (int64_t)tstart[nt] + TC_ALPHA * nt;
        const int64_t G = gridDim.x;
        sm.t_begin = (int)tc_lower(tstart, nt, (F * blockIdx.x + G - 1) / G);
        sm.t_end = blockIdx.x + 1 == gridDim.x
                       ? (int)nt
                       : (int)tc_lower(tstart, nt, (F * (blockIdx.x + 1) + G - 1) / G);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t t0 = sm.tbase;
    const int tb = sm.t_begin, te = sm.t_end;
    // the non-empty tiles of [tb, te), in order, into shared memory (block-wide
    // compaction): the roles then walk stages without global loads on their
    // critical paths
    int nlist = 0;
    for (int base = tb; base < te; base += TC_THREADS) {
        const int t = base + tid;
        uint32_t b = 0, e = 0;
        if (t < te) {
            b = tstart[t];
            e = tstart[t + 1];
        }
        const bool ne = e > b;
        const unsigned bal = __ballot_sync(0xffffffffu, ne);
        if (lane == 0) s_wcount[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int k = 0; k < TC_THREADS / 32; ++k) {
                const int v = s_wcount[k];
                s_wcount[k] = acc;
                acc += v;
            }
            s_wcount[TC_THREADS / 32] = acc;
        }
        __syncthreads();
        if (ne) {
            const int pos = nlist + s_wcount[warp] + __popc(bal & ((1u << lane) - 1u));
            const int tz = (int)(t / nxy), rr = (int)(t % nxy);
            tlist[pos] = make_int4(t, (int)b, (int)(e - b), (tz << 20) | ((rr / ntx) << 10) | (rr % ntx));
        }
        nlist += s_wcount[TC_THREADS / 32];
        __syncthreads();
    }

    if (warp < TC_P_WARPS) {
        // ------------------------------------------------------------ producers
        // warp w: TMEM lane quadrant q = w % 4, accumulator half hf (rows y 0-7 /
        // 8-15), stage k half ks (Gaussians 16 ks .. 16 ks + 15)
        const int q = warp & 3, hf = (warp >> 2) & 1, ks = warp >> 3;
        const int m = 32 * q + lane;                 // accumulator row (TMEM lane)
        const int ty = 8 * hf + (m >> 4), tx = m & 15;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        const int gi = tid >> 4, part = tid & 15;    // table builder: Gaussian, coordinate
        // stage cursor (cur) and the two prefetch cursors: the Gaussian id of
        // stage +2 and the record of stage +1 are loaded ahead of their use
        TcStage cur{0, 0u}, n1, n2;
        n1 = cur;
        if (nlist > 0) n1.next(tlist);
        n2 = n1;
        if (n2.i < nlist) n2.next(tlist);
        // raw sorted pair value of Gaussian gi of a stage (0xffffffff: none); the
        // shift to the Gaussian id happens a stage later, off the load's latency
        auto sval = [&](const TcStage& st) -> uint32_t {
            if (st.i >= nlist) return 0xffffffffu;
            const int4 d = tlist[st.i];
            return st.k0 + gi < (uint32_t)d.z ? svals[d.y + st.k0 + gi] : 0xffffffffu;
        };
        GRec rcur, rnext;
        uint32_t v2 = sval(n2);
        {
            const uint32_t v0 = sval(cur), v1 = sval(n1);
            if (v0 != 0xffffffffu) rcur = rec[v0 >> S];
            if (v1 != 0xffffffffu) rnext = rec[v1 >> S];
        }
        unsigned cov = 0u;   // lanes 0..15 of each warp: row `part`'s covered columns
        uint32_t gs = 0, dt = 0;
        // tables of stage gs live in buffer gs & 1; stage gs's are built at the end of stage gs - 1
        auto build = [&](const TcStage& st, const GRec& r, int buf) {
            const int4 d = tlist[st.i];
            const int nb = (int)min((uint32_t)TC_KS, (uint32_t)d.z - st.k0);
            const int x0 = (d.w & 1023) * TT, y0 = ((d.w >> 10) & 1023) * TT, z0 = (d.w >> 20) * TT;
            float vx = 0.f, vy = 0.f, vz = 0.f;
            unsigned rows = 0u;
            if (gi < nb) {
                vx = tab_weight(x0 + part, 0, w, r.fx, hx, r.dx, r.inv2);
                vy = tab_weight(y0 + part, 0, h, r.fy, hy, r.dy, r.inv2) * r.I;
                vz = tab_weight(z0 + part, zoff, c, r.fz, hz, r.dz, r.inv2);
                if (MASKS) {   // integer footprint inside the tile (a3): row `part`
                    const int yy = y0 + part;
                    const int bx0 = max(r.fx - hx, x0), bx1 = min(min(r.fx + hx, w - 1), x0 + TT - 1);
                    if (yy >= r.fy - hy && yy <= r.fy + hy && yy < h && bx0 <= bx1)
                        rows = ((2u << (bx1 - x0)) - 1u) & ~((1u << (bx0 - x0)) - 1u);
                }
            }
            sm.ex[buf][part][gi] = vx;
            sm.ey[buf][part][gi] = vy;
            sm.ez[buf][part][gi] = vz;
            if (MASKS) {   // OR over the warp's two Gaussians (lanes part, part + 16)
                rows |= __shfl_xor_sync(0xffffffffu, rows, 16);
                cov |= rows;
            }
        };
        if (cur.i < nlist) build(cur, rcur, 0);
        p_bar();
        while (cur.i < nlist) {
            const uint32_t cnt = (uint32_t)tlist[cur.i].z;
            const int nb = (int)min((uint32_t)TC_KS, cnt - cur.k0);
            const int nk8 = (nb + 7) >> 3;
            const int slot = gs & 1, buf = gs & 1;
            // prefetch: record of stage +2 (its id was loaded a stage ago), id of stage +3
            GRec rn2;
            if (v2 != 0xffffffffu) rn2 = rec[v2 >> S];
            TcStage n3 = n2;
            if (n3.i < nlist) n3.next(tlist);
            const uint32_t v3 = sval(n3);
            // the MMAs of the stage that last used this slot are complete
            tc::mbar_wait(&sm.a_empty[slot], ((gs >> 1) & 1) ^ 1);
            tc::fence_after();
            // A: this row's outer-product values of k chunks 2 ks, 2 ks + 1, split,
            // straight into TMEM
            const float* ey = sm.ey[buf][ty];
            const float* ex = sm.ex[buf][tx];
            const uint32_t acol = t0 + lane_addr + 128 + slot * 128 + hf * 64;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = 2 * ks + jj;
                if (j < nk8) {
                    const float4 ya = *reinterpret_cast<const float4*>(ey + 8 * j);
                    const float4 yb = *reinterpret_cast<const float4*>(ey + 8 * j + 4);
                    const float4 xa = *reinterpret_cast<const float4*>(ex + 8 * j);
                    const float4 xb = *reinterpret_cast<const float4*>(ex + 8 * j + 4);
                    const float v[8] = {ya.x * xa.x, ya.y * xa.y, ya.z * xa.z, ya.w * xa.w,
                                        yb.x * xb.x, yb.y * xb.y, yb.z * xb.z, yb.w * xb.w};
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        hi[e] = __float_as_uint(v[e]) & 0xffffe000u;
                        lo[e] = __float_as_uint(v[e] - __uint_as_float(hi[e]));
                    }
                    tc::st_x8(acol + 8 * j, hi);
                    tc::st_x8(acol + 32 + 8 * j, lo);
                }
            }
            {   // B: ez (16 slices x 32 Gaussians), canonical K-major, one per thread
                const int n = tid >> 5, kk = tid & 31;
                const float v = sm.ez[buf][n][kk];
                const uint32_t vh = __float_as_uint(v) & 0xffffe000u;
                const int off = (128 * (kk >> 3) + 64 * ((kk & 7) >> 2) + 32 * (n >> 3) +
                                 4 * (n & 7) + (kk & 3));
                sm.bop[slot][0][off] = vh;
                sm.bop[slot][1][off] = __float_as_uint(v - __uint_as_float(vh));
            }
            tc::wait_st();
            tc::fence_proxy_async();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sm.a_full[slot]);
            const bool last = cur.k0 + TC_KS >= cnt;   // the tile's last stage
            if (MASKS && last) {   // the tile's footprint coverage rows, for the epilogue
                const int cb = dt & 3;
                if (lane < 16) sm.covw[cb][warp][lane] = cov;
                cov = 0u;
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sm.cov_full[cb]);
            }
            if (last) ++dt;
            // the next stage's tables (the other buffer), from the prefetched record
            if (n1.i < nlist) build(n1, rnext, buf ^ 1);
            p_bar();
            cur = n1;
            n1 = n2;
            n2 = n3;
            rnext = rn2;
            v2 = v3;
            ++gs;
        }
    } else if (warp == TC_P_WARPS) {
        // ---------------------------------------------------------------- MMA
        if (lane == 0) {
            const uint32_t id = tc::idesc_tf32(128, 16);
            uint32_t gs = 0;
            for (int li = 0; li < nlist; ++li) {
                const uint32_t cnt = (uint32_t)tlist[li].z;
                for (uint32_t k0 = 0; k0 < cnt; k0 += TC_KS, ++gs) {
                    const int nb = (int)min((uint32_t)TC_KS, cnt - k0);
                    const int nk8 = (nb + 7) >> 3;
                    const int slot = gs & 1;
                    tc::mbar_wait(&sm.d_empty[slot], ((gs >> 1) & 1) ^ 1);
                    tc::mbar_wait(&sm.a_full[slot], (gs >> 1) & 1);
                    tc::fence_after();
                    const uint32_t bh = tc::smem_u32(sm.bop[slot][0]);
                    const uint32_t bl = tc::smem_u32(sm.bop[slot][1]);
                    // each stage sums into a fresh accumulator (the epilogue adds the
                    // stages in fp32, round to nearest): the small cross terms first
                    for (int hf = 0; hf < 2; ++hf) {
                        const uint32_t d = t0 + slot * 32 + hf * 16;
                        const uint32_t a = t0 + 128 + slot * 128 + hf * 64;
                        for (int j = 0; j < nk8; ++j) {
                            const uint64_t dh = tc::smem_desc(bh + 512 * j, 256, 128);
                            const uint64_t dl = tc::smem_desc(bl + 512 * j, 256, 128);
                            tc::mma_tf32_ts(d, a + 32 + 8 * j, dh, id, j ? 1u : 0u);
                            tc::mma_tf32_ts(d, a + 8 * j, dl, id, 1u);
                        }
                        for (int j = 0; j < nk8; ++j) {
                            const uint64_t dh = tc::smem_desc(bh + 512 * j, 256, 128);
                            tc::mma_tf32_ts(d, a + 8 * j, dh, id, 1u);
                        }
                    }
                    tc::commit(&sm.a_empty[slot]);   // this slot's A and B are free again
                    tc::commit(&sm.d_full[slot]);    // the stage's partial sums are final
                }
            }
        }
        __syncwarp();
    } else {
        // ----------------------------------------------------------- epilogue
        const int q = warp & 3;
        const int m = 32 * q + lane;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        uint32_t gs = 0, dt = 0;
        int li = 0;
        for (int t = tb; t < te; ++t) {
            uint32_t cnt = 0;
            if (li < nlist && tlist[li].x == t) cnt = (uint32_t)tlist[li++].z;
            const int tzi = (int)(t / nxy), rest = (int)(t % nxy);
            const int x0 = (rest % ntx) * TT, y0 = (rest / ntx) * TT, z0 = tzi * TT;
            float acc[2][16];
#pragma unroll
            for (int z = 0; z < 16; ++z) acc[0][z] = acc[1][z] = 0.f;
            for (uint32_t k0 = 0; k0 < cnt; k0 += TC_KS, ++gs) {
                const int slot = gs & 1;
                tc::mbar_wait(&sm.d_full[slot], (gs >> 1) & 1);
                tc::fence_after();
                uint32_t v0[16], v1[16];
                tc::ld_x16(t0 + lane_addr + slot * 32, v0);
                tc::ld_x16(t0 + lane_addr + slot * 32 + 16, v1);
                tc::wait_ld();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sm.d_empty[slot]);
#pragma unroll
                for (int z = 0; z < 16; ++z) {
                    acc[0][z] += __uint_as_float(v0[z]);
                    acc[1][z] += __uint_as_float(v1[z]);
                }
            }
            unsigned cov[2] = {0u, 0u};
            if (MASKS && cnt > 0) {
                const int cb = dt & 3;
                tc::mbar_wait(&sm.cov_full[cb], (dt >> 2) & 1);
#pragma unroll
                for (int wv = 0; wv < TC_P_WARPS; ++wv) {
                    cov[0] |= sm.covw[cb][wv][m >> 4];
                    cov[1] |= sm.covw[cb][wv][8 + (m >> 4)];
                }   // row r's columns: warps hold rows part = lane of Gaussians 2 w, 2 w + 1
            }
            if (cnt > 0) ++dt;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int y = y0 + 8 * hf + (m >> 4), x = x0 + (m & 15);
                if (x >= w || y >= h) continue;
                float* col = vol + ((int64_t)y * w + x) * c + z0;
                if ((c & 3) == 0 && z0 + TT <= c) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq)
                        reinterpret_cast<float4*>(col)[qq] =
                            make_float4(acc[hf][4 * qq], acc[hf][4 * qq + 1], acc[hf][4 * qq + 2],
                                        acc[hf][4 * qq + 3]);
                } else {
#pragma unroll
                    for (int z = 0; z < 16; ++z)
                        if (z0 + z < c) col[z] = acc[hf][z];
                }
                if (MASKS && ntz <= 64 && cnt > 0) {
                    bool nz = false;
#pragma unroll
                    for (int z = 0; z < 16; ++z) nz |= acc[hf][z] != 0.f;
                    if (nz) atomicOr(&pocc[(int64_t)y * w + x], 1ull << tzi);
                    if ((cov[hf] >> (m & 15)) & 1u) atomicOr(&fcov[(int64_t)y * w + x], 1ull << tzi);
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == TC_P_WARPS) tc::tmem_free(t0, 512);
}

// --------------------------------------------------------------------------
// the non-decomposed splat (fvr.reconstruct_nodecomp -> splat_plain,
// _kernels.py:81-129): the reference keeps it to validate and benchmark the
// decomposition -- every box voxel pays its own squared distance and its own
// exponential.  Same tile bins and tile-owned accumulation as the forward
// (one 256-thread CTA per 16^3 tile, a thread per (y, x) column of 16 slices,
// the tile list in ascending Gaussian id: deterministic), so the two paths
// differ only in the arithmetic per contribution: one exp2 + 3 FMA here
// against one FMA on separable tables in the decomposed kernels.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fvr_fwd_plain(const GRec* __restrict__ rec, int w, int h,
                                                    int c, int zoff, int hx, int hy, int hz,
                                                    int ntx, int nty, int S,
                                                    const uint32_t* __restrict__ tstart,
                                                    const uint32_t* __restrict__ svals,
                                                    float* __restrict__ vol) {
    const int64_t t = blockIdx.x;
    const int txi = (int)(t % ntx), tyi = (int)((t / ntx) % nty), tzi = (int)(t / ((int64_t)ntx * nty));
    const int x = txi * TT + (threadIdx.x & 15), y = tyi * TT + (threadIdx.x >> 4), z0 = tzi * TT;
    __shared__ GRec sr[64];
    float acc[16];
#pragma unroll
    for (int z = 0; z < 16; ++z) acc[z] = 0.f;
    const uint32_t beg = tstart[t], end = tstart[t + 1];
    for (uint32_t b0 = beg; b0 < end; b0 += 64) {
        const int nb = (int)min(64u, end - b0);
        __syncthreads();
        if ((int)threadIdx.x < nb) sr[threadIdx.x] = rec[svals[b0 + threadIdx.x] >> S];
        __syncthreads();
        for (int k = 0; k < nb; ++k) {
            const GRec r = sr[k];
            const int bx = x - r.fx, by = y - r.fy;
            if (bx < -hx || bx > hx || by < -hy || by > hy) continue;   // footprint (a3)
            const float rx = (float)bx - r.dx, ry = (float)by - r.dy;
            const float dxy = fmaf(rx, rx, ry * ry);
#pragma unroll
            for (int z = 0; z < 16; ++z) {
                const int bz = z0 + z + zoff - r.fz;
                const float rz = (float)bz - r.dz;
                const float e = r.I * exp2f(-r.inv2 * fmaf(rz, rz, dxy));
                acc[z] += (bz >= -hz && bz <= hz) ? e : 0.f;
            }
        }
    }
    if (x < w && y < h) {
        float* col = vol + ((int64_t)y * w + x) * c + z0;
#pragma unroll
        for (int z = 0; z < 16; ++z)
            if (z0 + z < c) col[z] = acc[z];
    }
}

// tstart[t] = lower_bound(sorted keys, t) for t in [0, nt] from the key
// boundaries: sorted position j starts every tile in (key[j-1], key[j]], and
// tstart[nt] = number of pairs (read on the device: the bins are dense).
// One coalesced pass; each tile start is written exactly once.
// It also readies the forward that follows the bins: the tile-claim counter
// and its exit ticket (fcounter[0], [2]) are zeroed, and so are the two
// empty-space masks (mask_words u64; the masked forward ORs into them), which
// would otherwise each take a memset node between the bins and the forward.
__global__ void k_tile_starts(const uint32_t* __restrict__ skeys,
                              const uint32_t* __restrict__ npairs, int64_t nt, int ybits,
                              uint32_t* __restrict__ tstart, unsigned int* __restrict__ fcounter,
                              unsigned long long* __restrict__ masks, int64_t mask_words,
                              const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    const int64_t np = npairs ? (int64_t)*npairs : 0;
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j == 0) {
        fcounter[0] = 0u;
        fcounter[2] = 0u;
    }
    for (int64_t k = j; k < mask_words; k += (int64_t)gridDim.x * blockDim.x) masks[k] = 0ull;
    if (j > np) return;
    const int64_t prev = j == 0 ? -1 : (int64_t)(skeys[j - 1] >> ybits);
    const int64_t cur = j == np ? nt : (int64_t)(skeys[j] >> ybits);
    for (int64_t t = prev + 1; t <= cur; ++t) tstart[t] = (uint32_t)j;
}

// --------------------------------------------------------------------------
// backward: one warp per Gaussian, lanes over z, upstream read straight from
// global memory (the C2 upstream, 64 MB, stays L2-resident between the loss
// and this kernel).  The box's columns are walked (y outer, x inner) with the
// separable factors in per-warp shared tables, so per column a lane does one
// coalesced load and three FMAs:
//   C_k(y) = sum_x ex rx^k u(y,x,z)           (k = 0, 1, 2)
//   A0 += ey C0, Ax += ey C1, Ay += ey ry C0, Ar += ey (C2 + ry^2 C0)
// and the lane-private z factors ez, rz are applied once at the end.  One
// warp sums a Gaussian's moments in a fixed order: deterministic, with no
// partial buffer and no combine pass.  Gradient formulas: _kernels.py:132-205.
// --------------------------------------------------------------------------
constexpr int BG_WARPS = 4;
constexpr int BG_XC = 17;   // box columns per register row (default box 17^3)

// Fast path for boxes up to 17 columns x 17 slices (the default 17^3 box):
// the 32 lanes take two columns at a time (lane = column parity x 16 slices),
// so a row costs 9 column-pair loads instead of 17 half-empty ones; the 17th
// slice of the box is one lanes-over-columns load per row.  Lane-private x
// tables (9 pairs x {e, e r, e r^2}) stay in registers, the two halves are
// combined once per Gaussian.  Same moments as the general path below.
template <bool PF>   // PF: prefetch the next row (register-hungry; more ILP)
__device__ __forceinline__ void bwd_moments17(const GRec& r, int xlo, int nx, int ylo, int ny,
                                              int zlo, int nz, int w, int c, int zoff,
                                              const float* __restrict__ up, float& S0, float& Sx,
                                              float& Sy, float& Sz, float& S2) {
    const int lane = threadIdx.x & 31, hf = lane >> 4, zl = lane & 15;
    // slice of this lane (first 16 of the box) and the optional 17th slice
    const bool zok = zl < nz;
    const float rz = (float)(zlo + zl + zoff - r.fz) - r.dz;
    const float ez = zok ? exp2f(-r.inv2 * rz * rz) : 0.f;
    const bool has16 = nz > 16;
    const float rz16 = (float)(zlo + 16 + zoff - r.fz) - r.dz;
    const float ez16 = has16 ? exp2f(-r.inv2 * rz16 * rz16) : 0.f;
    // x weights: column pair k -> column 2k + hf (main), column lane (17th slice)
    float2 wx01[9];   // {e, e r}: one FFMA2 per column
    float wx2[9];
    uint32_t coff[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int col = 2 * k + hf;
        const float rx = (float)(xlo + col - r.fx) - r.dx;
        const float ex = col < nx ? exp2f(-r.inv2 * rx * rx) : 0.f;
        wx01[k] = make_float2(ex, ex * rx);
        wx2[k] = ex * rx * rx;
        coff[k] = (uint32_t)min(col, nx - 1) * (uint32_t)c;
    }
    const float rxp = (float)(xlo + lane - r.fx) - r.dx;
    const float exp_ = (has16 && lane < nx) ? exp2f(-r.inv2 * rxp * rxp) : 0.f;
    const float wp0 = exp_, wp1 = exp_ * rxp, wp2 = exp_ * rxp * rxp;
    const uint32_t poff = (uint32_t)min(lane, nx - 1) * (uint32_t)c + 16u;
    const int64_t rstride = (int64_t)w * c;
    const float* row = up + ((int64_t)ylo * w + xlo) * c + zlo + (zok ? zl : 0);
    const float* prow = up + ((int64_t)ylo * w + xlo) * c + zlo;
    float A0 = 0.f, Ax = 0.f, Ay = 0.f, Ar = 0.f;   // main slices, per lane
    float Q0 = 0.f, Qx = 0.f, Qy = 0.f, Qr = 0.f;   // 17th slice, per column lane
    float u[9], un[9], pu = 0.f, pn = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) u[k] = zok ? __ldg(row + coff[k]) : 0.f;
    if (has16) pu = __ldg(prow + poff);
    for (int yi = 0; yi < ny; ++yi) {
        const bool more = yi + 1 < ny;
        if (!PF && yi > 0) {   // load this row now
            row += rstride;
            prow += rstride;
#pragma unroll
            for (int k = 0; k < 9; ++k) u[k] = zok ? __ldg(row + coff[k]) : 0.f;
            if (has16) pu = __ldg(prow + poff);
        }
        if (PF && more) {   // prefetch the next row
            row += rstride;
            prow += rstride;
#pragma unroll
            for (int k = 0; k < 9; ++k) un[k] = zok ? __ldg(row + coff[k]) : 0.f;
            if (has16) pn = __ldg(prow + poff);
        }
        const float ry = (float)(ylo + yi - r.fy) - r.dy;
        const float ey = exp2f(-r.inv2 * ry * ry);
        float2 C01 = make_float2(0.f, 0.f);
        float C2 = 0.f;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            C01 = ffma2(make_float2(u[k], u[k]), wx01[k], C01);
            C2 = fmaf(wx2[k], u[k], C2);
        }
        const float C0 = C01.x, C1 = C01.y;
        const float eyry = ey * ry, eyry2 = eyry * ry;
        A0 = fmaf(ey, C0, A0);
        Ax = fmaf(ey, C1, Ax);
        Ay = fmaf(eyry, C0, Ay);
        Ar = fmaf(ey, C2, fmaf(eyry2, C0, Ar));
        Q0 = fmaf(ey * wp0, pu, Q0);
        Qx = fmaf(ey * wp1, pu, Qx);
        Qy = fmaf(eyry * wp0, pu, Qy);
        Qr = fmaf(fmaf(ey, wp2, eyry2 * wp0), pu, Qr);
        if (PF && more) {
#pragma unroll
            for (int k = 0; k < 9; ++k) u[k] = un[k];
            pu = pn;
        }
    }
    // the two column-parity halves hold the same slices: fold them, then apply
    // the lane-private z factors (lanes 16..31 duplicate lanes 0..15: weight 0)
    A0 += __shfl_xor_sync(0xffffffffu, A0, 16);
    Ax += __shfl_xor_sync(0xffffffffu, Ax, 16);
    Ay += __shfl_xor_sync(0xffffffffu, Ay, 16);
    Ar += __shfl_xor_sync(0xffffffffu, Ar, 16);
    const float eh = hf ? 0.f : ez;
    S0 = eh * A0;
    Sx = eh * Ax;
    Sy = eh * Ay;
    Sz = eh * rz * A0;
    S2 = eh * fmaf(rz * rz, A0, Ar);
    // 17th slice: per-column-lane partials, all with the same z factor
    S0 = fmaf(ez16, Q0, S0);
    Sx = fmaf(ez16, Qx, Sx);
    Sy = fmaf(ez16, Qy, Sy);
    Sz = fmaf(ez16 * rz16, Q0, Sz);
    S2 = fmaf(ez16, fmaf(rz16 * rz16, Q0, Qr), S2);
}

// FAST-path moments with the upstream rows brought in by TMA: one lane
// issues a {20 z, 17 x, 1 y} box load per row into a 4-slot per-warp ring
// (completion on per-slot mbarriers, out-of-volume taps zero-filled), so three
// rows are in flight ahead of the arithmetic at the cost of one instruction
// per row.  Lanes then read their column-pair words from shared memory.
constexpr int BT_RING = 4;
constexpr int BT_ZB = 20;   // box z extent: 17 taps from a 16 B-aligned start (z0 & ~3)
constexpr int BT_SLOT = 1408;                      // 17 x 20 x 4 B = 1360, rounded to 128 B
constexpr unsigned BT_BYTES = 17u * BT_ZB * 4u;

// Column of step k for half-warp hf: {0-3, 8-11, 16} and {4-7, 12-15}.  The
// half-warps then sit 4 columns = 80 words apart (= 16 banks), so a step's 32
// shared-memory reads hit 32 distinct banks (adjacent columns, 20 words apart,
// would overlap by 4 banks).
__device__ __forceinline__ int tcol(int k, int hf) { return 8 * (k >> 2) + (k & 3) + 4 * hf; }

__device__ __forceinline__ void bwd_moments17_tma(const GRec& r, int xlo, int nx, int ylo, int ny,
                                                  int zlo, int nz, int zoff,
                                                  const CUtensorMap* tmap, float* ring,
                                                  unsigned long long* bars, float& S0, float& Sx,
                                                  float& Sy, float& Sz, float& S2) {
    const int lane = threadIdx.x & 31, hf = lane >> 4, zl = lane & 15;
    const bool zok = zl < nz;
    const float rz = (float)(zlo + zl + zoff - r.fz) - r.dz;
    const float ez = zok ? exp2f(-r.inv2 * rz * rz) : 0.f;
    const bool has16 = nz > 16;
    const float rz16 = (float)(zlo + 16 + zoff - r.fz) - r.dz;
    const float ez16 = has16 ? exp2f(-r.inv2 * rz16 * rz16) : 0.f;
    float2 wx01[9];
    float wx2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int col = tcol(k, hf);
        const float rx = (float)(xlo + col - r.fx) - r.dx;
        const float ex = col < nx ? exp2f(-r.inv2 * rx * rx) : 0.f;
        wx01[k] = make_float2(ex, ex * rx);
        wx2[k] = ex * rx * rx;
    }
    const float rxp = (float)(xlo + lane - r.fx) - r.dx;
    const float exp_ = (has16 && lane < nx) ? exp2f(-r.inv2 * rxp * rxp) : 0.f;
    const float wp0 = exp_, wp1 = exp_ * rxp, wp2 = exp_ * rxp * rxp;
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
    const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bars);
    auto issue = [&](int yi) {   // lane 0
        const int q = yi % BT_RING;
        const unsigned b = bar_s + 8 * q, dst = ring_s + BT_SLOT * q;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b),
                     "r"(BT_BYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
            "l"(tmap), "r"(zlo & ~3), "r"(xlo), "r"(ylo + yi), "r"(b)
            : "memory");
    };
    if (lane == 0)
        for (int q = 0; q < BT_RING - 1 && q < ny; ++q) issue(q);
    float A0 = 0.f, Ax = 0.f, Ay = 0.f, Ar = 0.f;
    float Q0 = 0.f, Qx = 0.f, Qy = 0.f, Qr = 0.f;
    for (int yi = 0; yi < ny; ++yi) {
        __syncwarp();   // every lane is done with the slot refilled next (row yi - 1)
        if (lane == 0 && yi + BT_RING - 1 < ny) issue(yi + BT_RING - 1);
        const int q = yi % BT_RING;
        const unsigned parity = (unsigned)(yi / BT_RING) & 1u;
        {   // wait for row yi
            unsigned done = 0;
            do {
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                    " selp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(done)
                    : "r"(bar_s + 8 * q), "r"(parity)
                    : "memory");
            } while (!done);
        }
        const float* src = ring + (BT_SLOT / 4) * q + (zlo & 3);
        const float ry = (float)(ylo + yi - r.fy) - r.dy;
        const float ey = exp2f(-r.inv2 * ry * ry);
        float2 C01 = make_float2(0.f, 0.f);
        float C2 = 0.f;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            // column 20 (k = 8, upper half-warp) lies past the box: never read it
            // columns past the footprint (nx < 17) are never read either: the masked
            // adjoint leaves upstream outside every footprint unwritten (0 x NaN = NaN)
            const float u = (zok && (k < 8 || !hf) && tcol(k, hf) < nx)
                                ? src[tcol(k, hf) * BT_ZB + zl] : 0.f;
            C01 = ffma2(make_float2(u, u), wx01[k], C01);
            C2 = fmaf(wx2[k], u, C2);
        }
        const float pu = (has16 && lane < nx) ? src[lane * BT_ZB + 16] : 0.f;
        const float C0 = C01.x, C1 = C01.y;
        const float eyry = ey * ry, eyry2 = eyry * ry;
        A0 = fmaf(ey, C0, A0);
        Ax = fmaf(ey, C1, Ax);
        Ay = fmaf(eyry, C0, Ay);
        Ar = fmaf(ey, C2, fmaf(eyry2, C0, Ar));
        Q0 = fmaf(ey * wp0, pu, Q0);
        Qx = fmaf(ey * wp1, pu, Qx);
        Qy = fmaf(eyry * wp0, pu, Qy);
        Qr = fmaf(fmaf(ey, wp2, eyry2 * wp0), pu, Qr);
    }
    A0 += __shfl_xor_sync(0xffffffffu, A0, 16);
    Ax += __shfl_xor_sync(0xffffffffu, Ax, 16);
    Ay += __shfl_xor_sync(0xffffffffu, Ay, 16);
    Ar += __shfl_xor_sync(0xffffffffu, Ar, 16);
    const float eh = hf ? 0.f : ez;
    S0 = eh * A0;
    Sx = eh * Ax;
    Sy = eh * Ay;
    Sz = eh * rz * A0;
    S2 = eh * fmaf(rz * rz, A0, Ar);
    S0 = fmaf(ez16, Q0, S0);
    Sx = fmaf(ez16, Qx, Sx);
    Sy = fmaf(ez16, Qy, Sy);
    Sz = fmaf(ez16 * rz16, Q0, Sz);
    S2 = fmaf(ez16, fmaf(rz16 * rz16, Q0, Qr), S2);
}

// The same moments for a full 17 x 17 x 17 box (every interior Gaussian), with
// the row loop unrolled: two box rows per TMA load ({20 z, 17 x, 2 y}, 3-slot
// ring: up to 6 rows in flight, half the issues and barrier waits), the row
// weights {ey, ey ry, ey ry^2} from a per-warp table, and no per-element
// selects -- the 18th column (k = 8 of the odd half) and the lanes past the
// 17th column re-read column 16 (inside the footprint, finite) against a zero
// weight.  Row 17 of the last load is never read.
#ifndef SPLATCT_BT2_ROWS
#define SPLATCT_BT2_ROWS 2
#endif
#ifndef SPLATCT_BT2_RING
#define SPLATCT_BT2_RING 3
#endif
constexpr int BT2_ROWS = SPLATCT_BT2_ROWS;          // box rows per TMA load
constexpr int BT2_RING = SPLATCT_BT2_RING;
constexpr int BT2_NB = (17 + BT2_ROWS - 1) / BT2_ROWS;   // loads per box
constexpr int BT2_SLOT = (BT2_ROWS * 17 * BT_ZB * 4 + 127) / 128 * 128;
constexpr unsigned BT2_BYTES = (unsigned)BT2_ROWS * 17u * BT_ZB * 4u;

__device__ __forceinline__ void bwd_moments17_tma_full(const GRec& r, int xlo, int ylo, int zlo,
                                                       int zoff, const CUtensorMap* tmap2,
                                                       float* ring, unsigned long long* bars,
                                                       float4* ytab, float& S0, float& Sx,
                                                       float& Sy, float& Sz, float& S2) {
    const int lane = threadIdx.x & 31, hf = lane >> 4, zl = lane & 15;
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
    const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bars);
    auto issue = [&](int bi) {   // lane 0: rows 2 bi, 2 bi + 1
        const int q = bi % BT2_RING;
        const unsigned b = bar_s + 8 * q, dst = ring_s + BT2_SLOT * q;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b),
                     "r"(BT2_BYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
            "l"(tmap2), "r"(zlo & ~3), "r"(xlo), "r"(ylo + BT2_ROWS * bi), "r"(b)
            : "memory");
    };
    if (lane == 0)
        for (int q = 0; q < BT2_RING && q < BT2_NB; ++q) issue(q);
    const float rz = (float)(zlo + zl + zoff - r.fz) - r.dz;
    const float ez = exp2f(-r.inv2 * rz * rz);
    const float rz16 = (float)(zlo + 16 + zoff - r.fz) - r.dz;
    const float ez16 = exp2f(-r.inv2 * rz16 * rz16);
    float2 wx01[9];
    float wx2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int col = tcol(k, k < 8 ? hf : 0);
        const float rx = (float)(xlo + col - r.fx) - r.dx;
        const float ex = (k < 8 || !hf) ? exp2f(-r.inv2 * rx * rx) : 0.f;
        wx01[k] = make_float2(ex, ex * rx);
        wx2[k] = ex * rx * rx;
    }
    const int pl = lane < 17 ? lane : 16;
    const float rxp = (float)(xlo + lane - r.fx) - r.dx;
    const float exq = lane < 17 ? exp2f(-r.inv2 * rxp * rxp) : 0.f;
    if (lane < 17) {
        const float ry = (float)(ylo + lane - r.fy) - r.dy;
        const float ey = exp2f(-r.inv2 * ry * ry);
        ytab[lane] = make_float4(ey, ey * ry, ey * ry * ry, 0.f);
    }
    int off[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) off[k] = tcol(k, k < 8 ? hf : 0) * BT_ZB + zl + (zlo & 3);
    const int offp = pl * BT_ZB + 16 + (zlo & 3);
    float A0 = 0.f, Ax = 0.f, Ay = 0.f, Ar = 0.f, P0 = 0.f, P1 = 0.f, P2 = 0.f;
#pragma unroll
    for (int bi = 0; bi < BT2_NB; ++bi) {
        __syncwarp();   // every lane is done with box bi - 1's slot (refilled next); ytab visible
        if (lane == 0 && bi >= 1 && bi + BT2_RING - 1 < BT2_NB) issue(bi + BT2_RING - 1);
        const int q = bi % BT2_RING;
        {
            const unsigned parity = (unsigned)(bi / BT2_RING) & 1u;
            unsigned done = 0;
            do {
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                    " selp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(done)
                    : "r"(bar_s + 8 * q), "r"(parity)
                    : "memory");
            } while (!done);
        }
        const float* src = ring + (BT2_SLOT / 4) * q;
#pragma unroll
        for (int rr = 0; rr < BT2_ROWS; ++rr) {
            const int yi = BT2_ROWS * bi + rr;
            if (yi > 16) break;
            const float* rs = src + rr * (17 * BT_ZB);
            float2 C01 = make_float2(0.f, 0.f);
            float C2 = 0.f;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const float u = rs[off[k]];
                C01 = ffma2(make_float2(u, u), wx01[k], C01);
                C2 = fmaf(wx2[k], u, C2);
            }
            const float pu = rs[offp];
            const float4 t = ytab[yi];
            A0 = fmaf(t.x, C01.x, A0);
            Ax = fmaf(t.x, C01.y, Ax);
            Ay = fmaf(t.y, C01.x, Ay);
            Ar = fmaf(t.x, C2, fmaf(t.z, C01.x, Ar));
            P0 = fmaf(t.x, pu, P0);
            P1 = fmaf(t.y, pu, P1);
            P2 = fmaf(t.z, pu, P2);
        }
    }
    A0 += __shfl_xor_sync(0xffffffffu, A0, 16);
    Ax += __shfl_xor_sync(0xffffffffu, Ax, 16);
    Ay += __shfl_xor_sync(0xffffffffu, Ay, 16);
    Ar += __shfl_xor_sync(0xffffffffu, Ar, 16);
    const float eh = hf ? 0.f : ez;
    S0 = eh * A0;
    Sx = eh * Ax;
    Sy = eh * Ay;
    Sz = eh * rz * A0;
    S2 = eh * fmaf(rz * rz, A0, Ar);
    const float Q0 = exq * P0, Qx = exq * rxp * P0, Qy = exq * P1;
    const float Qr = fmaf(exq * rxp * rxp, P0, exq * P2);
    S0 = fmaf(ez16, Q0, S0);
    Sx = fmaf(ez16, Qx, Sx);
    Sy = fmaf(ez16, Qy, Sy);
    Sz = fmaf(ez16 * rz16, Q0, Sz);
    S2 = fmaf(ez16, fmaf(rz16 * rz16, Q0, Qr), S2);
}

// flags[j] = 1 for the sorted pair that is its Gaussian's first tile (slot 0)
__global__ void k_first_flags(const uint32_t* __restrict__ svals, const uint32_t* __restrict__ tstart,
                              int64_t nt, int64_t np, int S, uint32_t* __restrict__ flags) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j > np) return;
    const uint32_t npairs = tstart[nt];
    flags[j] = (j < (int64_t)npairs && (svals[j] & ((1u << S) - 1u)) == 0u) ? 1u : 0u;
}

__global__ void k_order_scatter(const uint32_t* __restrict__ svals,
                                const uint32_t* __restrict__ flags,
                                const uint32_t* __restrict__ pos, int64_t np, int S,
                                uint32_t* __restrict__ order) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j > np) return;
    if (j == np) order[0] = pos[np];                      // count of listed Gaussians
    else if (flags[j]) order[1 + pos[j]] = svals[j] >> S;
}

// FAST: every box is at most 17 columns x 17 slices (box halves hx, hz <= 8),
// so only the column-pair path is compiled (its own register budget).
// ORD: visit Gaussians in first-tile order (order[0] = count, order[1..])
template <bool FAST, bool ORD>
__global__ void __launch_bounds__(32 * BG_WARPS, FAST ? 6 : 4) k_fvr_bwd(const double* __restrict__ P, int64_t n,
                                                          const uint32_t* __restrict__ order,
                                                          const int32_t* __restrict__ fp,
                                                          const GRec* __restrict__ rec, int w,
                                                          int h, int c, int zoff,
                                                          const float* __restrict__ up,
                                                          double* __restrict__ G,
                                                          double* __restrict__ accum,
                                                          const __grid_constant__ CUtensorMap utmap,
                                                          const __grid_constant__ CUtensorMap utmap2,
                                                          int use_tma, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    // per warp: the 1-row ring (general boxes) or the 2-row ring (full boxes)
    constexpr int RING_FL = (BT_RING * BT_SLOT > BT2_RING * BT2_SLOT ? BT_RING * BT_SLOT
                                                                      : BT2_RING * BT2_SLOT) / 4;
    __shared__ __align__(128) float bring[FAST ? BG_WARPS : 1][FAST ? RING_FL : 1];
    __shared__ float4 ytab[FAST ? BG_WARPS : 1][17];
    __shared__ __align__(8) unsigned long long bbar[BG_WARPS][BT_RING];
    __shared__ float xt[3][BG_WARPS][32];   // ex, ex rx, ex rx^2
    __shared__ float2 yt[BG_WARPS][32];   // {ey, ry}
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (FAST && use_tma) {   // every ring barrier initialised once, before any copy in the CTA
        if (threadIdx.x < BG_WARPS * BT_RING) {
            const unsigned b = (unsigned)__cvta_generic_to_shared(&bbar[0][0]) + 8 * threadIdx.x;
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        __syncthreads();
    }
    const int64_t gw = blockIdx.x * (int64_t)BG_WARPS + wid;
    if (gw >= (ORD ? (int64_t)order[0] : n)) return;   // warp-uniform: warp-level syncs only
    const int64_t i = ORD ? (int64_t)order[1 + gw] : gw;
    const int xlo = fp[6 * i], xhi = fp[6 * i + 1], ylo = fp[6 * i + 2], yhi = fp[6 * i + 3];
    const int zlo = fp[6 * i + 4], zhi = fp[6 * i + 5];
    float S0 = 0.f, Sx = 0.f, Sy = 0.f, Sz = 0.f, S2 = 0.f;
    if (FAST || (xlo <= xhi && ylo <= yhi && zlo <= zhi && xhi - xlo < 17 && zhi - zlo < 17)) {
        if (xlo <= xhi && ylo <= yhi && zlo <= zhi) {
            const GRec r = rec[i];
            if (FAST && use_tma && xhi - xlo == 16 && yhi - ylo == 16 && zhi - zlo == 16)
                bwd_moments17_tma_full(r, xlo, ylo, zlo, zoff, &utmap2, bring[FAST ? wid : 0],
                                       bbar[wid], ytab[FAST ? wid : 0], S0, Sx, Sy, Sz, S2);
            else if (FAST && use_tma)
                bwd_moments17_tma(r, xlo, xhi - xlo + 1, ylo, yhi - ylo + 1, zlo, zhi - zlo + 1,
                                  zoff, &utmap, bring[FAST ? wid : 0], bbar[wid], S0, Sx, Sy, Sz,
                                  S2);
            else
                bwd_moments17<!FAST>(r, xlo, xhi - xlo + 1, ylo, yhi - ylo + 1, zlo,
                                     zhi - zlo + 1, w, c, zoff, up, S0, Sx, Sy, Sz, S2);
        }
    } else if (xlo <= xhi && ylo <= yhi && zlo <= zhi) {
        const GRec r = rec[i];
        for (int zc = zlo; zc <= zhi; zc += 32) {
            const int z = zc + lane;
            const bool zok = z <= zhi;
            const float rz = (float)(z + zoff - r.fz) - r.dz;
            const float ez = zok ? exp2f(-r.inv2 * rz * rz) : 0.f;
            const float* ubase = up + (zok ? z : zlo);
            float A0 = 0.f, Ax = 0.f, Ay = 0.f, Ar = 0.f;
            for (int yc = ylo; yc <= yhi; yc += 32) {
                const int ny = min(32, yhi - yc + 1);
                for (int xc = xlo; xc <= xhi; xc += BG_XC) {
                    const int nx = min(BG_XC, xhi - xc + 1);
                    __syncwarp();   // previous chunk's table reads are done
                    {
                        const float ry = (float)(yc + lane - r.fy) - r.dy;
                        yt[wid][lane] = make_float2(lane < ny ? exp2f(-r.inv2 * ry * ry) : 0.f, ry);
                        const float rx = (float)(xc + lane - r.fx) - r.dx;
                        const float ex = lane < nx ? exp2f(-r.inv2 * rx * rx) : 0.f;
                        xt[0][wid][lane] = ex;
                        xt[1][wid][lane] = ex * rx;
                        xt[2][wid][lane] = ex * rx * rx;
                    }
                    __syncwarp();
                    // a whole row (<= BG_XC columns) of loads is issued at once and
                    // the next row is prefetched while this one is consumed.
                    // Columns beyond nx re-read column nx-1 (valid memory, L1 hit)
                    // and meet a zero weight, so the loads need no k-predicate.
                    float wx0[BG_XC], wx1[BG_XC], wx2[BG_XC];
                    uint32_t coff[BG_XC];
#pragma unroll
                    for (int k = 0; k < BG_XC; ++k) {
                        wx0[k] = xt[0][wid][k];
                        wx1[k] = xt[1][wid][k];
                        wx2[k] = xt[2][wid][k];
                        coff[k] = (uint32_t)min(k, nx - 1) * (uint32_t)c;
                    }
                    const float* row = ubase + ((int64_t)yc * w + xc) * c;
                    const int64_t rstride = (int64_t)w * c;
                    float ua[BG_XC], ub[BG_XC];
#define BG_LOAD(U)                                                        \
    _Pragma("unroll") for (int k = 0; k < BG_XC; ++k) U[k] = zok ? __ldg(row + coff[k]) : 0.f;
#define BG_CONSUME(U, YI)                                                 \
    {                                                                     \
        float C0 = 0.f, C1 = 0.f, C2 = 0.f;                               \
        _Pragma("unroll") for (int k = 0; k < BG_XC; ++k) {               \
            C0 = fmaf(wx0[k], U[k], C0);                                  \
            C1 = fmaf(wx1[k], U[k], C1);                                  \
            C2 = fmaf(wx2[k], U[k], C2);                                  \
        }                                                                 \
        const float2 ey = yt[wid][YI];                                    \
        A0 = fmaf(ey.x, C0, A0);                                          \
        Ax = fmaf(ey.x, C1, Ax);                                          \
        Ay = fmaf(ey.x * ey.y, C0, Ay);                                   \
        Ar = fmaf(ey.x, fmaf(ey.y * ey.y, C0, C2), Ar);                   \
    }
                    BG_LOAD(ua);
                    for (int yi = 0; yi < ny; yi += 2) {
                        const bool more = yi + 1 < ny;
                        if (more) { row += rstride; BG_LOAD(ub); }
                        BG_CONSUME(ua, yi);
                        if (!more) break;
                        if (yi + 2 < ny) { row += rstride; BG_LOAD(ua); }
                        BG_CONSUME(ub, yi + 1);
                    }
#undef BG_LOAD
#undef BG_CONSUME
                }
            }
            S0 = fmaf(ez, A0, S0);
            Sx = fmaf(ez, Ax, Sx);
            Sy = fmaf(ez, Ay, Sy);
            Sz = fmaf(ez * rz, A0, Sz);
            S2 = fmaf(ez, fmaf(rz * rz, A0, Ar), S2);
        }
    }
    S0 = warp_sum(S0);
    Sx = warp_sum(Sx);
    Sy = warp_sum(Sy);
    Sz = warp_sum(Sz);
    S2 = warp_sum(S2);
    if (lane == 0) {   // chain rule in f64 (fvr.py:227-273)
        const double amp = P[4 * n + i], sg = P[3 * n + i];
        const double inv_s2 = 1.0 / (sg * sg), inv_s3 = inv_s2 / sg;
        const double k2 = amp * inv_s2;
        const double gx = k2 * Sx, gy = k2 * Sy, gz = k2 * Sz;
        G[i] = gx;
        G[n + i] = gy;
        G[2 * n + i] = gz;
        G[3 * n + i] = amp * inv_s3 * S2;
        G[4 * n + i] = S0;
        if (accum) accum[i] += sqrt(gx * gx + gy * gy + gz * gz);
    }
}

// --------------------------------------------------------------------------
// backward, spatially ordered (the default for boxes <= 17^3): persistent
// CTAs walk the tile-sorted (tile, Gaussian) pairs and take each Gaussian at
// its first tile (slot 0), so every CTA sweeps one contiguous run of tiles and
// the Gaussians resident on an SM at any moment are neighbours -- their boxes
// overlap, and the upstream rows they read are L1 hits instead of one private
// L2 stream per Gaussian (the TMA row ring read 1.2 GB from L2 per C2 launch).
// A full 17^3 box (every interior Gaussian) runs a branch-free row loop with
// compile-time column offsets: 9 column-pair loads + 1 seventeenth-slice load,
// 9 FFMA2 + 9 FFMA and 7 row FMAs per row, the row weights {ey, ey ry, ey ry^2}
// from a per-warp table.  Footprints clipped by the volume take the clamped
// general path (bwd_moments17).  Moments, reduction and f64 chain rule as in
// k_fvr_bwd; each Gaussian is summed by one warp in a fixed order
// (deterministic, independent of which warp takes it).
// --------------------------------------------------------------------------
constexpr int BS_WARPS = 16;

template <int C>   // compile-time volume depth (0: runtime c)
__device__ __forceinline__ void bwd_moments17_full(const GRec& r, int xlo, int ylo, int zlo,
                                                   int w, int c_rt, int zoff,
                                                   const float* __restrict__ up,
                                                   const float4* ytab, float& S0, float& Sx,
                                                   float& Sy, float& Sz, float& S2) {
    const int cc = C ? C : c_rt;
    const int lane = threadIdx.x & 31, hf = lane >> 4, zl = lane & 15;
    const float rz = (float)(zlo + zl + zoff - r.fz) - r.dz;
    const float ez = exp2f(-r.inv2 * rz * rz);
    const float rz16 = (float)(zlo + 16 + zoff - r.fz) - r.dz;
    const float ez16 = exp2f(-r.inv2 * rz16 * rz16);
    float2 wx01[9];
    float wx2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {   // column 2k + hf; column 17 (k = 8, hf = 1) is not in the box
        const float rx = (float)(xlo + 2 * k + hf - r.fx) - r.dx;
        const float ex = (k < 8 || !hf) ? exp2f(-r.inv2 * rx * rx) : 0.f;
        wx01[k] = make_float2(ex, ex * rx);
        wx2[k] = ex * rx * rx;
    }
    const int pl = lane < 17 ? lane : 16;   // 17th slice: lanes over columns
    const float rxp = (float)(xlo + lane - r.fx) - r.dx;
    const float exp_ = lane < 17 ? exp2f(-r.inv2 * rxp * rxp) : 0.f;
    const int64_t rstride = (int64_t)w * cc;
    const float* pb = up + ((int64_t)ylo * w + xlo + hf) * cc + zlo + zl;
    const float* pp = up + ((int64_t)ylo * w + xlo + pl) * cc + zlo + 16;
    float A0 = 0.f, Ax = 0.f, Ay = 0.f, Ar = 0.f, P0 = 0.f, P1 = 0.f, P2 = 0.f;
    float ua[9], ub[9], pa, pbv;
#define BS_LOAD(U, PU)                                                              \
    {                                                                               \
        _Pragma("unroll") for (int k = 0; k < 8; ++k) U[k] = __ldg(pb + 2 * k * cc); \
        U[8] = hf ? 0.f : __ldg(pb + 16 * cc);                                      \
        PU = __ldg(pp);                                                             \
        pb += rstride;                                                              \
        pp += rstride;                                                              \
    }
#define BS_ROW(U, PU, YI)                                                           \
    {                                                                               \
        float2 C01 = make_float2(0.f, 0.f);                                         \
        float C2 = 0.f;                                                             \
        _Pragma("unroll") for (int k = 0; k < 9; ++k) {                             \
            C01 = ffma2(make_float2(U[k], U[k]), wx01[k], C01);                     \
            C2 = fmaf(wx2[k], U[k], C2);                                            \
        }                                                                           \
        const float4 t = ytab[YI];                                                  \
        A0 = fmaf(t.x, C01.x, A0);                                                  \
        Ax = fmaf(t.x, C01.y, Ax);                                                  \
        Ay = fmaf(t.y, C01.x, Ay);                                                  \
        Ar = fmaf(t.x, C2, fmaf(t.z, C01.x, Ar));                                   \
        P0 = fmaf(t.x, PU, P0);                                                     \
        P1 = fmaf(t.y, PU, P1);                                                     \
        P2 = fmaf(t.z, PU, P2);                                                     \
    }
    BS_LOAD(ua, pa);
#pragma unroll
    for (int yi = 0; yi < 16; yi += 2) {   // rows 0..15 in pairs, next row in flight
        BS_LOAD(ub, pbv);
        BS_ROW(ua, pa, yi);
        if (yi + 2 < 17) BS_LOAD(ua, pa);
        BS_ROW(ub, pbv, yi + 1);
    }
    BS_ROW(ua, pa, 16);
#undef BS_LOAD
#undef BS_ROW
    A0 += __shfl_xor_sync(0xffffffffu, A0, 16);
    Ax += __shfl_xor_sync(0xffffffffu, Ax, 16);
    Ay += __shfl_xor_sync(0xffffffffu, Ay, 16);
    Ar += __shfl_xor_sync(0xffffffffu, Ar, 16);
    const float eh = hf ? 0.f : ez;
    S0 = eh * A0;
    Sx = eh * Ax;
    Sy = eh * Ay;
    Sz = eh * rz * A0;
    S2 = eh * fmaf(rz * rz, A0, Ar);
    // 17th slice: per-column sums over rows, column weights applied once
    const float Q0 = exp_ * P0, Qx = exp_ * rxp * P0, Qy = exp_ * P1;
    const float Qr = fmaf(exp_ * rxp * rxp, P0, exp_ * P2);
    S0 = fmaf(ez16, Q0, S0);
    Sx = fmaf(ez16, Qx, Sx);
    Sy = fmaf(ez16, Qy, Sy);
    Sz = fmaf(ez16 * rz16, Q0, Sz);
    S2 = fmaf(ez16, fmaf(rz16 * rz16, Q0, Qr), S2);
}

template <int C>
__global__ void __launch_bounds__(32 * BS_WARPS, 1)
    k_fvr_bwd_sp(const double* __restrict__ P, int64_t n, const uint32_t* __restrict__ svals,
                 const uint32_t* __restrict__ tstart, int64_t nt, int Sl,
                 const int32_t* __restrict__ fp, const GRec* __restrict__ rec, int w, int h,
                 int c, int zoff, const float* __restrict__ up, double* __restrict__ G,
                 double* __restrict__ accum, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    __shared__ float4 ytab[BS_WARPS][17];   // per warp: {ey, ey ry, ey ry^2} per box row
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t np = tstart[nt];
    // contiguous pair range of this CTA (tile order): one run of neighbouring tiles
    const uint32_t per = (np + gridDim.x - 1) / gridDim.x;
    const uint32_t j0 = min(np, blockIdx.x * per), j1 = min(np, j0 + per);
    const uint32_t smask = (1u << Sl) - 1u;
    for (uint32_t jb = j0 + 32u * wid; jb < j1; jb += 32u * BS_WARPS) {
        const uint32_t j = jb + lane;
        const uint32_t v = j < j1 ? svals[j] : 1u;
        unsigned first = __ballot_sync(0xffffffffu, j < j1 && (v & smask) == 0u);
        while (first) {
            const int src = __ffs(first) - 1;
            first &= first - 1u;
            const int64_t i = (int64_t)(__shfl_sync(0xffffffffu, v, src) >> Sl);
            const int xlo = fp[6 * i], xhi = fp[6 * i + 1], ylo = fp[6 * i + 2];
            const int yhi = fp[6 * i + 3], zlo = fp[6 * i + 4], zhi = fp[6 * i + 5];
            const GRec r = rec[i];
            float S0, Sx, Sy, Sz, S2;
            if (xhi - xlo == 16 && yhi - ylo == 16 && zhi - zlo == 16) {
                __syncwarp();   // the previous Gaussian's table reads are done
                if (lane < 17) {
                    const float ry = (float)(ylo + lane - r.fy) - r.dy;
                    const float ey = exp2f(-r.inv2 * ry * ry);
                    ytab[wid][lane] = make_float4(ey, ey * ry, ey * ry * ry, 0.f);
                }
                __syncwarp();
                bwd_moments17_full<C>(r, xlo, ylo, zlo, w, c, zoff, up, ytab[wid], S0, Sx, Sy,
                                      Sz, S2);
            } else {
                bwd_moments17<false>(r, xlo, xhi - xlo + 1, ylo, yhi - ylo + 1, zlo,
                                     zhi - zlo + 1, w, c, zoff, up, S0, Sx, Sy, Sz, S2);
            }
            S0 = warp_sum(S0);
            Sx = warp_sum(Sx);
            Sy = warp_sum(Sy);
            Sz = warp_sum(Sz);
            S2 = warp_sum(S2);
            if (lane == 0) {   // chain rule in f64 (fvr.py:227-273)
                const double amp = P[4 * n + i], sg = P[3 * n + i];
                const double inv_s2 = 1.0 / (sg * sg), inv_s3 = inv_s2 / sg;
                const double k2 = amp * inv_s2;
                const double gx = k2 * Sx, gy = k2 * Sy, gz = k2 * Sz;
                G[i] = gx;
                G[n + i] = gy;
                G[2 * n + i] = gz;
                G[3 * n + i] = amp * inv_s3 * S2;
                G[4 * n + i] = S0;
                if (accum) accum[i] += sqrt(gx * gx + gy * gy + gz * gz);
            }
        }
    }
}

// --------------------------------------------------------------------------
// backward, tile-staged (the default for boxes <= 17^3 with c % 4 == 0).
//
// A Gaussian's clipped box starts in its first tile (slot 0 of its pairs)
// and spans at most 2 x 2 x 2 tiles from there.  A persistent CTA (one per
// SM, 16 warps) claims work units = (tile column tx, ty) x (a run of BT_ZCH z
// tiles) and sweeps z: the upstream "slabs" -- tiles (tx..tx+1, ty..ty+1) of
// one z tile, 32 x 32 x 16 floats = 64 KB -- arrive by one TMA box load each
// into a 3-slab shared-memory ring (slab tz + 2 loads while tile tz is
// processed).  Warps then take the Gaussians whose first tile is (tx, ty, tz)
// (ballot over the tile's sorted pairs) and read their 17^3 boxes from shared
// memory: the upstream is read from L2 once per unit (about 4x its size in
// total, from the 2 x 2 tile halo) instead of once per Gaussian (the TMA row
// kernel's 1.2 GB per C2 launch).
// Per Gaussian, lanes take the box's 17 x 17 (column, slice) pairs as 10 slots
// (s = lane + 32 i: column s / 17, slice s % 17) and, per row, accumulate the
// y moments T0 += ey u, T1 += ey ry u, T2 += ey ry^2 u (conflict-free LDS:
// slot i of lane l reads bank (16 x + z) mod 32); x and z weights are applied
// once per slot at the end, then one warp reduction and the f64 chain rule
// (fvr.py:227-273).  Footprints clipped by the volume take the clamped
// global-memory path (bwd_moments17).  Deterministic: each Gaussian is summed
// by one warp in a fixed order.
// --------------------------------------------------------------------------
constexpr int BT_WARPS = 16;
constexpr int BT_ZCH = 16;                 // z tiles per work unit
constexpr int BT_SLAB = 32 * 32 * 16;      // floats per slab
constexpr unsigned BT_SLAB_BYTES = BT_SLAB * 4u;

struct __align__(16) BtWarp {
    float4 ey[17];      // {ey, ey ry, ey ry^2, 0} per box row
};

// Moments of one full-box (17^3) Gaussian from a staged tile column: slab
// buffers bA (z tile tz) and bB (tz + 1), each [y 32][x 32][z 16] floats in
// the 64 B swizzle, (xr, yr) the box origin inside the 32 x 32 window.  Lanes:
// column parity hf x slice zl (slices 0..15 of the box, columns 2k + hf); the
// 17th slice with lanes over columns.  ey holds {ey, ey ry, ey ry^2} per row.
// Used by k_fvr_bwd_ts and k_fvr_bwd_ts2 (identical arithmetic, bitwise equal).
__device__ __forceinline__ void bt_full_moments(const float* __restrict__ slab, int bA, int bB,
                                                int tz, int xr, int yr, const GRec& r, int xlo,
                                                int zlo, int zoff, const float4* ey, int lane,
                                                float& S0, float& Sx, float& Sy, float& Sz,
                                                float& S2) {
    const int hf = lane >> 4, zl = lane & 15;
    auto soff = [&](int colr, int za) {
        const int rr = yr * 32 + xr + colr, zz = za & 15;
        return ((za >> 4) == tz ? bA : bB) * BT_SLAB + rr * 16 +
               (((zz >> 2) ^ ((rr >> 1) & 3)) << 2) + (zz & 3);
    };
    int off[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) off[k] = soff(min(2 * k + hf, 16), zlo + zl);
    const int pl = lane < 17 ? lane : 16;
    const int offp = soff(pl, zlo + 16);
    const float rz = (float)(zlo + zl + zoff - r.fz) - r.dz;
    const float ez = exp2f(-r.inv2 * rz * rz);
    const float rz16 = (float)(zlo + 16 + zoff - r.fz) - r.dz;
    const float ez16 = exp2f(-r.inv2 * rz16 * rz16);
    float2 wx01[9];
    float wx2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const float rx = (float)(xlo + 2 * k + hf - r.fx) - r.dx;
        const float ex = (k < 8 || !hf) ? exp2f(-r.inv2 * rx * rx) : 0.f;
        wx01[k] = make_float2(ex, ex * rx);
        wx2[k] = ex * rx * rx;
    }
    const float rxp = (float)(xlo + lane - r.fx) - r.dx;
    const float exq = lane < 17 ? exp2f(-r.inv2 * rxp * rxp) : 0.f;
    float A0 = 0.f, Ax = 0.f, Ay = 0.f, Ar = 0.f, P0 = 0.f, P1 = 0.f, P2 = 0.f;
#pragma unroll
    for (int yi = 0; yi < 17; ++yi) {
        float2 C01 = make_float2(0.f, 0.f);
        float C2 = 0.f;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const float uu = slab[off[k] + 512 * yi];
            C01 = ffma2(make_float2(uu, uu), wx01[k], C01);
            C2 = fmaf(wx2[k], uu, C2);
        }
        const float pu = slab[offp + 512 * yi];
        const float4 t = ey[yi];
        A0 = fmaf(t.x, C01.x, A0);
        Ax = fmaf(t.x, C01.y, Ax);
        Ay = fmaf(t.y, C01.x, Ay);
        Ar = fmaf(t.x, C2, fmaf(t.z, C01.x, Ar));
        P0 = fmaf(t.x, pu, P0);
        P1 = fmaf(t.y, pu, P1);
        P2 = fmaf(t.z, pu, P2);
    }
    A0 += __shfl_xor_sync(0xffffffffu, A0, 16);
    Ax += __shfl_xor_sync(0xffffffffu, Ax, 16);
    Ay += __shfl_xor_sync(0xffffffffu, Ay, 16);
    Ar += __shfl_xor_sync(0xffffffffu, Ar, 16);
    const float eh = hf ? 0.f : ez;
    S0 = eh * A0;
    Sx = eh * Ax;
    Sy = eh * Ay;
    Sz = eh * rz * A0;
    S2 = eh * fmaf(rz * rz, A0, Ar);
    const float Q0 = exq * P0, Qx = exq * rxp * P0, Qy = exq * P1;
    const float Qr = fmaf(exq * rxp * rxp, P0, exq * P2);
    S0 = fmaf(ez16, Q0, S0);
    Sx = fmaf(ez16, Qx, Sx);
    Sy = fmaf(ez16, Qy, Sy);
    Sz = fmaf(ez16 * rz16, Q0, Sz);
    S2 = fmaf(ez16, fmaf(rz16 * rz16, Q0, Qr), S2);
}

// the warp's per-row table {ey, ey ry, ey ry^2} for a full box starting at row ylo
__device__ __forceinline__ void bt_row_table(float4* ey, const GRec& r, int ylo, int lane) {
    __syncwarp();
    if (lane < 17) {
        const float ry = (float)(ylo + lane - r.fy) - r.dy;
        const float e = exp2f(-r.inv2 * ry * ry);
        ey[lane] = make_float4(e, e * ry, e * ry * ry, 0.f);
    }
    __syncwarp();
}

// f64 chain rule of one Gaussian's moments (fvr.py:227-273), lane 0
__device__ __forceinline__ void bt_chain(const double* __restrict__ P, int64_t n, int64_t gi,
                                         float S0, float Sx, float Sy, float Sz, float S2,
                                         double* __restrict__ G, double* __restrict__ accum) {
    const double amp = P[4 * n + gi], sg = P[3 * n + gi];
    const double inv_s2 = 1.0 / (sg * sg), inv_s3 = inv_s2 / sg;
    const double k2 = amp * inv_s2;
    const double gx = k2 * Sx, gy = k2 * Sy, gz = k2 * Sz;
    G[gi] = gx;
    G[n + gi] = gy;
    G[2 * n + gi] = gz;
    G[3 * n + gi] = amp * inv_s3 * S2;
    G[4 * n + gi] = S0;
    if (accum) accum[gi] += sqrt(gx * gx + gy * gy + gz * gz);
}

__global__ void __launch_bounds__(32 * BT_WARPS, 1)
    k_fvr_bwd_ts(const double* __restrict__ P, int64_t n, const uint32_t* __restrict__ svals,
                 const uint32_t* __restrict__ tstart, int ntx, int nty, int ntz, int Sl,
                 const int32_t* __restrict__ fp, const GRec* __restrict__ rec, int w, int h,
                 int c, int zoff, const float* __restrict__ up,
                 const __grid_constant__ CUtensorMap utmap, unsigned int* __restrict__ counter,
                 double* __restrict__ G, double* __restrict__ accum, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    extern __shared__ __align__(1024) float slab[];      // [3][y 32][x 32][z 16]
    __shared__ BtWarp wt[BT_WARPS];
    __shared__ __align__(8) unsigned long long sbar[3];
    __shared__ int s_unit;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int b = 0; b < 3; ++b) tc::mbar_init(reinterpret_cast<uint64_t*>(&sbar[b]), 1);
        tc::mbar_init_fence();
    }
    __syncthreads();
    const uint32_t smask = (1u << Sl) - 1u;
    const int nzch = (ntz + BT_ZCH - 1) / BT_ZCH;
    const int units = ntx * nty * nzch;
    // slab (z tile) held by each ring buffer, and loads issued per buffer (the
    // mbarrier phase); plain scalars (no local-memory array)
    int held0 = -1, held1 = -1, held2 = -1;
    uint32_t ld0 = 0u, ld1 = 0u, ld2 = 0u;
    const int64_t nxy = (int64_t)ntx * nty;
    for (;;) {
        __syncthreads();
        if (tid == 0) s_unit = (int)atomicAdd(counter, 1u);
        __syncthreads();
        const int u = s_unit;
        if (u >= units) break;
        const int col = u / nzch, ch = u % nzch;
        const int tx = col % ntx, ty = col / ntx;
        const int tz0 = ch * BT_ZCH, tz1 = min(ntz, tz0 + BT_ZCH);
        // issue the load of slab sz into its ring buffer (thread 0; caller syncs first)
        auto load = [&](int sz_) {
            const int b = sz_ % 3;
            int& held = b == 0 ? held0 : (b == 1 ? held1 : held2);
            uint32_t& lds = b == 0 ? ld0 : (b == 1 ? ld1 : ld2);
            if (held == sz_ || sz_ >= ntz) return;
            held = sz_;
            ++lds;
            if (tid == 0) {
                const unsigned bar = tc::smem_u32(&sbar[b]);
                const unsigned dst = tc::smem_u32(slab + b * BT_SLAB);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                             "r"(BT_SLAB_BYTES)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
                    "l"(&utmap), "r"(16 * sz_), "r"(16 * tx), "r"(16 * ty), "r"(bar)
                    : "memory");
            }
        };
        auto wait_slab = [&](int sz_) {
            if (sz_ >= ntz) return;
            const int b = sz_ % 3;
            const uint32_t lds = b == 0 ? ld0 : (b == 1 ? ld1 : ld2);
            tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[b]), (lds - 1u) & 1u);
        };
        // a new unit is another tile column: land every outstanding slab load of
        // the previous unit (a prefetch may never have been waited for), then
        // forget what the buffers hold
        if (ld0) tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[0]), (ld0 - 1u) & 1u);
        if (ld1) tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[1]), (ld1 - 1u) & 1u);
        if (ld2) tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[2]), (ld2 - 1u) & 1u);
        held0 = held1 = held2 = -1;
        for (int tz = tz0; tz < tz1; ++tz) {
            const int64_t t = (int64_t)tz * nxy + (int64_t)ty * ntx + tx;
            const uint32_t pb = tstart[t], pe = tstart[t + 1];
            if (pb == pe) continue;   // no pairs: no Gaussian starts here
            __syncthreads();          // every warp is done with the slab tz - 1 buffer
            load(tz);
            load(tz + 1);
            if (tz + 1 < tz1) {       // prefetch for the next tile of the unit
                const int64_t t2 = t + nxy;
                if (tstart[t2 + 1] > tstart[t2]) load(tz + 2);
            }
            wait_slab(tz);
            wait_slab(tz + 1);
            // the Gaussians whose first tile is t
            for (uint32_t jb = pb + 32u * warp; jb < pe; jb += 32u * BT_WARPS) {
                const uint32_t j = jb + lane;
                const uint32_t v = j < pe ? svals[j] : 1u;
                unsigned first = __ballot_sync(0xffffffffu, j < pe && (v & smask) == 0u);
                while (first) {
                    const int src = __ffs(first) - 1;
                    first &= first - 1u;
                    const int64_t i = (int64_t)(__shfl_sync(0xffffffffu, v, src) >> Sl);
                    const int xlo = fp[6 * i], xhi = fp[6 * i + 1], ylo = fp[6 * i + 2];
                    const int yhi = fp[6 * i + 3], zlo = fp[6 * i + 4], zhi = fp[6 * i + 5];
                    const GRec r = rec[i];
                    float S0 = 0.f, Sx = 0.f, Sy = 0.f, Sz = 0.f, S2 = 0.f;
                    if (xhi - xlo == 16 && yhi - ylo == 16 && zhi - zlo == 16) {
                        BtWarp& W = wt[warp];
                        bt_row_table(W.ey, r, ylo, lane);
                        bt_full_moments(slab, tz % 3, (tz + 1) % 3, tz, xlo - 16 * tx, ylo - 16 * ty,
                                        r, xlo, zlo, zoff, W.ey, lane, S0, Sx, Sy, Sz, S2);
                    } else {
                        bwd_moments17<false>(r, xlo, xhi - xlo + 1, ylo, yhi - ylo + 1, zlo,
                                             zhi - zlo + 1, w, c, zoff, up, S0, Sx, Sy, Sz, S2);
                    }
                    S0 = warp_sum(S0);
                    Sx = warp_sum(Sx);
                    Sy = warp_sum(Sy);
                    Sz = warp_sum(Sz);
                    S2 = warp_sum(S2);
                    if (lane == 0) {   // chain rule in f64 (fvr.py:227-273)
                        const double amp = P[4 * n + i], sg = P[3 * n + i];
                        const double inv_s2 = 1.0 / (sg * sg), inv_s3 = inv_s2 / sg;
                        const double k2 = amp * inv_s2;
                        const double gx = k2 * Sx, gy = k2 * Sy, gz = k2 * Sz;
                        G[i] = gx;
                        G[n + i] = gy;
                        G[2 * n + i] = gz;
                        G[3 * n + i] = amp * inv_s3 * S2;
                        G[4 * n + i] = S0;
                        if (accum) accum[i] += sqrt(gx * gx + gy * gy + gz * gz);
                    }
                }
            }
        }
    }
    __syncthreads();
    // drain: a prefetched slab nobody waited for must land before the CTA exits
    if (ld0) tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[0]), (ld0 - 1u) & 1u);
    if (ld1) tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[1]), (ld1 - 1u) & 1u);
    if (ld2) tc::mbar_wait(reinterpret_cast<uint64_t*>(&sbar[2]), (ld2 - 1u) & 1u);
}

// --------------------------------------------------------------------------
// backward, tile-staged and asynchronous (SPLATCT_BWD_KERNEL=ts2).
//
// Same staging as k_fvr_bwd_ts (a tile column's upstream slabs, 32 x 32 x 16
// floats with the 64 B swizzle, one TMA box each, a 3-slab ring), but no
// block-wide barrier per tile.  A producer warp claims work units (a tile
// column x BT2Z_CH z tiles), scans the unit's tile bins for the Gaussians
// whose first tile each tile is (slot 0), publishes that list through a
// 2-entry queue (an entry is cut early when the list is full, so any density
// fits), and streams only the slabs those Gaussians read into the ring, each
// behind a "full" mbarrier and released through an "empty" mbarrier that
// every consumer warp arrives on once it has moved past the slab.  Consumer
// warps claim single Gaussians from the entry in tile order, so a tile's
// Gaussians run concurrently while later slabs land.  Per Gaussian the
// arithmetic is k_fvr_bwd_ts's (bit-identical moments).
// --------------------------------------------------------------------------
#ifndef BT2Z_CONS_N
#define BT2Z_CONS_N 16
#endif
constexpr int BT2Z_CONS = BT2Z_CONS_N;            // consumer warps
#ifndef BT2Z_CH_N
#define BT2Z_CH_N 4
#endif
constexpr int BT2Z_CH = BT2Z_CH_N;                // z tiles per claimed unit
constexpr int BT2Z_CAP = 1024;                    // Gaussians per queue entry
constexpr int BT2Z_THREADS = 32 * (BT2Z_CONS + 2);   // + scanner + loader warps

struct BtEntry {
    int tx, ty, tz0, ntiles, end;
    int gofs[BT2Z_CH + 1];   // list prefix per tile
    int sseq[BT2Z_CH + 1];   // ring sequence number of slab tz0 + i, or -1 (not needed)
    uint32_t gl[BT2Z_CAP];   // Gaussian ids, tile order, ascending pair order per tile
};

__global__ void __launch_bounds__(BT2Z_THREADS, 1)
    k_fvr_bwd_ts2(const double* __restrict__ P, int64_t n, const uint32_t* __restrict__ svals,
                  const uint32_t* __restrict__ tstart, int ntx, int nty, int ntz, int Sl,
                  const int32_t* __restrict__ fp, const GRec* __restrict__ rec, int w, int h,
                  int c, int zoff, const float* __restrict__ up,
                  const __grid_constant__ CUtensorMap utmap, unsigned int* __restrict__ counter,
                  double* __restrict__ G, double* __restrict__ accum, const int* halt) {
    griddep_wait();
    if (halted(halt)) return;
    extern __shared__ __align__(1024) float slab[];      // [3][y 32][x 32][z 16]
    __shared__ BtWarp wt[BT2Z_CONS];
    __shared__ BtEntry uq[2];
    __shared__ unsigned int uclaim[2];
    __shared__ __align__(8) uint64_t full[3], empty[3], ufull[2], uempty[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int b = 0; b < 3; ++b) {
            tc::mbar_init(&full[b], 1);
            tc::mbar_init(&empty[b], BT2Z_CONS);
        }
        for (int e = 0; e < 2; ++e) {
            tc::mbar_init(&ufull[e], 1);
            tc::mbar_init(&uempty[e], BT2Z_CONS + 1);   // consumers + the loader
        }
        tc::mbar_init_fence();
    }
    __syncthreads();
    const int64_t nxy = (int64_t)ntx * nty;
    const uint32_t smask = (1u << Sl) - 1u;
    if (warp == BT2Z_CONS + 1) {
        // -------------------------------------------------------------- loader
        // streams each entry's needed slabs into the ring, in sequence order
        if (lane == 0) {
            for (uint32_t k = 0;; ++k) {
                const int e = k & 1;
                tc::mbar_wait(&ufull[e], (k >> 1) & 1);
                const BtEntry& U = uq[e];
                if (U.end) break;
                const int tx = U.tx, ty = U.ty, t0 = U.tz0, nt = U.ntiles;
                int sq[BT2Z_CH + 1];
#pragma unroll
                for (int i = 0; i <= BT2Z_CH; ++i) sq[i] = i <= nt ? U.sseq[i] : -1;
                tc::mbar_arrive(&uempty[e]);   // done reading the entry
#pragma unroll
                for (int i = 0; i <= BT2Z_CH; ++i) {
                    const int q = sq[i];
                    if (q < 0) continue;
                    const int b = q % 3;
                    tc::mbar_wait(&empty[b], ((q / 3) & 1) ^ 1);   // its last reader is done
                    const unsigned bar = tc::smem_u32(&full[b]);
                    const unsigned dst = tc::smem_u32(slab + b * BT_SLAB);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                                 "r"(BT_SLAB_BYTES)
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
                        "l"(&utmap), "r"(16 * (t0 + i)), "r"(16 * tx), "r"(16 * ty), "r"(bar)
                        : "memory");
                }
            }
        }
        return;
    }
    if (warp == BT2Z_CONS) {
        // ------------------------------------------------------------- scanner
        const int nzch = (ntz + BT2Z_CH - 1) / BT2Z_CH;
        const int units = ntx * nty * nzch;
        uint32_t k = 0, seq = 0;
        for (;;) {
            int u = 0;
            if (lane == 0) u = (int)atomicAdd(counter, 1u);
            u = __shfl_sync(0xffffffffu, u, 0);
            const bool last = u >= units;
            const int col = last ? 0 : u / nzch, ch = last ? 0 : u % nzch;
            const int tx = col % ntx, ty = col / ntx;
            const int tzA = ch * BT2Z_CH, tzE = last ? 0 : min(ntz, tzA + BT2Z_CH);
            // a claimed unit becomes one or more queue entries (cut when full)
            // the unit's tile bounds, one load per lane: lane 2i / 2i + 1 hold the
            // pair range of tile tzA + i
            uint32_t tb = 0u;
            if (lane < 2 * (tzE - tzA))
                tb = tstart[(int64_t)(tzA + (lane >> 1)) * nxy + (int64_t)ty * ntx + tx + (lane & 1)];
            int tz = tzA;
            uint32_t jn = __shfl_sync(0xffffffffu, tb, 0);
            do {
                const int e = k & 1;
                if (lane == 0) tc::mbar_wait(&uempty[e], ((k >> 1) & 1) ^ 1);   // entry free
                __syncwarp();
                BtEntry& U = uq[e];
                if (last) {
                    if (lane == 0) {
                        U.end = 1;
                        tc::mbar_arrive(&ufull[e]);
                    }
                    return;
                }
                const int t0 = tz;
                int cnt = 0, nt = 0;
                if (lane == 0) U.gofs[0] = 0;
                // scan tiles t0.. while the list has room; a tile may be split
                while (tz < tzE) {
                    const uint32_t pe = __shfl_sync(0xffffffffu, tb, 2 * (tz - tzA) + 1);
                    // 4 batches of 32 pairs per round (independent loads in flight)
                    while (jn < pe && cnt + 32 <= BT2Z_CAP) {
                        const int nb = cnt + 128 <= BT2Z_CAP ? 4 : 1;
                        uint32_t v[4];
                        bool ok[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t j = jn + 32 * q + lane;
                            ok[q] = q < nb && j < pe;
                            v[q] = ok[q] ? svals[j] : 0u;
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const bool f = ok[q] && (v[q] & smask) == 0u;
                            const unsigned m = __ballot_sync(0xffffffffu, f);
                            if (f) U.gl[cnt + __popc(m & ((1u << lane) - 1u))] = v[q] >> Sl;
                            cnt += __popc(m);
                        }
                        jn = min(jn + 32u * nb, pe);
                    }
                    if (lane == 0) U.gofs[nt + 1] = cnt;
                    ++nt;
                    if (jn < pe) break;          // list full inside tile tz: continue it next entry
                    ++tz;
                    if (tz < tzE) jn = __shfl_sync(0xffffffffu, tb, 2 * (tz - tzA));
                    if (nt == BT2Z_CH) break;
                }
                // slabs t0 .. t0 + nt (the last only inside the volume) are read by
                // the tiles that have Gaussians: tile i reads slabs i and i + 1
                __syncwarp();   // every lane's list writes precede lane 0's release
                if (lane == 0) {
                    U.tx = tx;
                    U.ty = ty;
                    U.tz0 = t0;
                    U.ntiles = nt;
                    U.end = 0;
                    for (int i = 0; i <= nt; ++i) {
                        const bool need = (i < nt && U.gofs[i + 1] > U.gofs[i]) ||
                                          (i > 0 && U.gofs[i] > U.gofs[i - 1]);
                        U.sseq[i] = need && t0 + i < ntz ? (int)seq++ : -1;
                    }
                    uclaim[e] = 0u;
                    tc::mbar_arrive(&ufull[e]);   // release: the entry is written
                }
                __syncwarp();
                ++k;
            } while (tz < tzE);
        }
    }
    // -------------------------------------------------------------- consumers
    BtWarp& W = wt[warp];
    for (uint32_t k = 0;; ++k) {
        const int e = k & 1;
        tc::mbar_wait(&ufull[e], (k >> 1) & 1);
        const BtEntry& U = uq[e];
        if (U.end) break;
        const int total = U.gofs[U.ntiles];
        int rel = 0;            // slabs of the entry this warp has released
        int waited = -1;        // highest slab of the entry this warp has waited for
        int cur = -1;
        // a slab is released only after it landed: the arrival then belongs to
        // this use of the buffer, and no load is in flight when the CTA exits
        auto wait_upto = [&](int lim) {
            for (int sl = waited + 1; sl <= lim && sl <= U.ntiles; ++sl) {
                const int q = U.sseq[sl];
                if (q >= 0) tc::mbar_wait(&full[q % 3], (q / 3) & 1);
                waited = sl;
            }
        };
        // in slab order, each slab waited for and then released: a later slab's
        // load may depend on this warp's release of an earlier one
        auto release_below = [&](int lim) {
            for (; rel < lim && rel <= U.ntiles; ++rel) {
                wait_upto(rel);
                __syncwarp();
                const int q = U.sseq[rel];
                if (q >= 0 && lane == 0) tc::mbar_arrive(&empty[q % 3]);
            }
        };
        for (;;) {
            int idx = 0;
            if (lane == 0) idx = (int)atomicAdd(&uclaim[e], 1u);
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx >= total) break;
            int i = cur < 0 ? 0 : cur;
            while (U.gofs[i + 1] <= idx) ++i;
            if (i != cur) {   // moved on: slabs before tile i have no more readers here
                cur = i;
                release_below(i);
                wait_upto(i + 1);
            }
            const int tz = U.tz0 + i;
            const int64_t gi = U.gl[idx];
            const int xlo = fp[6 * gi], xhi = fp[6 * gi + 1], ylo = fp[6 * gi + 2];
            const int yhi = fp[6 * gi + 3], zlo = fp[6 * gi + 4], zhi = fp[6 * gi + 5];
            const GRec r = rec[gi];
            float S0 = 0.f, Sx = 0.f, Sy = 0.f, Sz = 0.f, S2 = 0.f;
            if (xhi - xlo == 16 && yhi - ylo == 16 && zhi - zlo == 16) {
                const int qa = U.sseq[i], qb = U.sseq[i + 1];
                bt_row_table(W.ey, r, ylo, lane);
                bt_full_moments(slab, qa % 3, qb < 0 ? 0 : qb % 3, tz, xlo - 16 * U.tx,
                                ylo - 16 * U.ty, r, xlo, zlo, zoff, W.ey, lane, S0, Sx, Sy, Sz,
                                S2);
            } else {
                bwd_moments17<false>(r, xlo, xhi - xlo + 1, ylo, yhi - ylo + 1, zlo, zhi - zlo + 1,
                                     w, c, zoff, up, S0, Sx, Sy, Sz, S2);
            }
            S0 = warp_sum(S0);
            Sx = warp_sum(Sx);
            Sy = warp_sum(Sy);
            Sz = warp_sum(Sz);
            S2 = warp_sum(S2);
            if (lane == 0) bt_chain(P, n, gi, S0, Sx, Sy, Sz, S2, G, accum);
        }
        release_below(U.ntiles + 1);   // the entry's remaining slabs
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&uempty[e]);
    }
}

__global__ void k_grad_norm_accum(const double* __restrict__ G, int64_t n,
                                  double* __restrict__ accum, const int* halt) {
    if (halted(halt)) return;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double gx = G[i], gy = G[n + i], gz = G[2 * n + i];
    accum[i] += sqrt(gx * gx + gy * gy + gz * gz);
}

__global__ void k_export_items(const uint32_t* __restrict__ svals, int64_t np, int S,
                               int32_t* __restrict__ items) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < np) items[j] = (int32_t)(svals[j] >> S);   // S = log2(slots)
}

static int check_args(int64_t n, int w, int h, int c, int hx, int hy, int hz, size_t ws_bytes,
                      const FvrLayout& L) {
    SPLATCT_REQUIRE(n >= 0 && w > 0 && h > 0 && c > 0, "invalid sizes n=%lld dims=(%d,%d,%d)",
                    (long long)n, w, h, c);
    SPLATCT_REQUIRE(hx >= 0 && hy >= 0 && hz >= 0, "negative box half");
    SPLATCT_REQUIRE(L.np < ((int64_t)1 << 32) - 1 && (n << L.Sl) < ((int64_t)1 << 32),
                    "too many (tile, Gaussian) pairs: %lld", (long long)L.np);
    SPLATCT_REQUIRE(L.nt < ((int64_t)1 << 31), "too many tiles");
    SPLATCT_REQUIRE(ws_bytes >= L.total, "workspace too small: %zu < %zu", ws_bytes, L.total);
    return SPLATCT_OK;
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_fvr_workspace_bytes(int64_t n, int w, int h, int c, int hx, int hy, int hz,
                                size_t* bytes) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    *bytes = L.total;
    return SPLATCT_OK;
}

static int fvr_bin_impl(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                        int hy, int hz, void* ws, size_t ws_bytes, const int* halt, void* stream,
                        bool row_order, AdamFuse af = AdamFuse{nullptr, nullptr, nullptr, nullptr, 0.0, 0.0}) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    if (int e = check_args(n, w, h, c, hx, hy, hz, ws_bytes, L)) return e;
    // row order uses the key bits the radix passes sort anyway (no extra pass),
    // at most 4, and only for boxes up to 17 rows (relative first row in [-16, 15])
    int tile_bits = 0;
    while (((int64_t)1 << tile_bits) < L.nt) ++tile_bits;
    const int ybits = row_order && hy <= 8 ? min(4, 8 * L.passes - tile_bits) : 0;
    cudaStream_t s = as_stream(stream);
    uint32_t* tickets = at<uint32_t>(ws, L.o_tickets);   // [0] emit, [1] pair count, [2..] passes
    const uint32_t* npairs = tickets + 1;
    if (n > 0) {
        SPLATCT_CK(cudaMemsetAsync(at<char>(ws, L.o_ctl), 0, L.ctl_bytes, s));
        SPLATCT_CK(launch_pdl(k_bin_emit, dim3((unsigned)L.emit_blocks), dim3(BIN_NT), 0, s,
                              params, n, w, h, c, z0, hx, hy, hz, L.ntx, L.nty, L.Sl, L.passes,
                              ybits, at<int32_t>(ws, L.o_fp), at<GRec>(ws, L.o_rec),
                              at<uint32_t>(ws, L.o_k0), at<uint32_t>(ws, L.o_v0),
                              at<uint32_t>(ws, L.o_ghist),
                              at<unsigned long long>(ws, L.o_stat_e), tickets, af, halt));
        SPLATCT_LAUNCH_CK();
        for (int p = 0; p < L.passes; ++p) {
            const size_t ki = p % 2 ? L.o_k1 : L.o_k0, vi = p % 2 ? L.o_v1 : L.o_v0;
            const size_t ko = p % 2 ? L.o_k0 : L.o_k1, vo = p % 2 ? L.o_v0 : L.o_v1;
            SPLATCT_CK(launch_pdl(
                k_onesweep, dim3((unsigned)L.sort_blocks), dim3(SORT_NT), 0, s,
                at<uint32_t>(ws, ki), at<uint32_t>(ws, vi), at<uint32_t>(ws, ko),
                at<uint32_t>(ws, vo), npairs, 8 * p, at<uint32_t>(ws, L.o_ghist) + p * RADIX,
                at<unsigned long long>(ws, L.o_stat_s) + (size_t)p * RADIX * L.sort_blocks,
                tickets + 2 + p, halt));
            SPLATCT_LAUNCH_CK();
        }
    }
    {   // tile offsets from the sorted keys: no atomics
        const size_t ko = L.final_buf ? L.o_k1 : L.o_k0;
        const int64_t npk = n > 0 ? L.np : 0;
        // both masks: pocc .. the end of fcov (each w*h u64)
        const int64_t mwords =
            L.ntz <= 64 ? (int64_t)((L.o_fcov - L.o_pocc) / 8) + (int64_t)w * h : 0;
        SPLATCT_CK(launch_pdl(k_tile_starts, dim3((unsigned)((npk + 1 + 255) / 256)), dim3(256),
                              0, s, n > 0 ? at<uint32_t>(ws, ko) : nullptr,
                              n > 0 ? npairs : nullptr, L.nt, ybits,
                              at<uint32_t>(ws, L.o_tstart), at<uint32_t>(ws, L.o_tcount),
                              at<unsigned long long>(ws, L.o_pocc), mwords, halt));
        SPLATCT_LAUNCH_CK();
    }
    return SPLATCT_OK;
}

int splatct_fvr_bin(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                    int hy, int hz, void* ws, size_t ws_bytes, const int* halt, void* stream) {
    return fvr_bin_impl(params, n, w, h, c, z0, hx, hy, hz, ws, ws_bytes, halt, stream, false);
}

int splatct_fvr_bin_row_ordered(const double* params, int64_t n, int w, int h, int c, int z0,
                                int hx, int hy, int hz, void* ws, size_t ws_bytes,
                                const int* halt, void* stream) {
    return fvr_bin_impl(params, n, w, h, c, z0, hx, hy, hz, ws, ws_bytes, halt, stream, true);
}

int splatct_fvr_adam_bin(double* params, const double* grads, double* m1, double* m2,
                         const double* adam, double sigma_floor, double sigma_ceiling, int64_t n,
                         int w, int h, int c, int z0, int hx, int hy, int hz, void* ws,
                         size_t ws_bytes, int row_ordered, const int* halt, void* stream) {
    SPLATCT_REQUIRE(grads && m1 && m2 && adam, "adam_bin needs grads, moments and scalars");
    if (n == 0) return fvr_bin_impl(params, n, w, h, c, z0, hx, hy, hz, ws, ws_bytes, halt,
                                    stream, row_ordered != 0);
    const AdamFuse af{grads, m1, m2, adam, sigma_floor, sigma_ceiling};
    return fvr_bin_impl(params, n, w, h, c, z0, hx, hy, hz, ws, ws_bytes, halt, stream,
                        row_ordered != 0, af);
}

// TMA descriptor of the (h, w, c) volume for 16^3 boxes with the 64-byte
// swizzle (false: no driver entry point or unsupported strides -- the kernel
// then stores with plain vector stores)
static bool volume_tensor_map(CUtensorMap* m, const float* vol, int w, int h, int c,
                              int bz = 16, int bx = 16, int by = 16, bool swizzle = true) {
    if ((c & 3) != 0) {
        memset(m, 0, sizeof(*m));
        return false;
    }
    const cuuint64_t dim[3] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h};
    const cuuint64_t stride[2] = {(cuuint64_t)c * 4, (cuuint64_t)c * w * 4};
    const cuuint32_t box[3] = {(cuuint32_t)bz, (cuuint32_t)bx, (cuuint32_t)by};
    return encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, vol, dim, stride, box,
                        swizzle ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE);
}

static int fvr_forward_impl(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                            int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                            const int* halt, void* stream, bool masks) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    if (int e = check_args(n, w, h, c, hx, hy, hz, ws_bytes, L)) return e;
    const size_t vo = L.final_buf ? L.o_v1 : L.o_v0;
    const int64_t grid = L.nt < 148 * FWD_MINB ? L.nt : 148 * FWD_MINB;   // persistent: all resident
    int64_t fetch = L.nt / (8 * grid);                       // >= 8 claims per CTA
    fetch = fetch < 1 ? 1 : (fetch > 32 ? 32 : fetch);
    // the bins zeroed the tile counter and the masks; the default kernel
    // leaves its counter at zero again, so repeated forwards need no memset
    unsigned int* counter = at<uint32_t>(ws, L.o_tcount);
    const char* kern = getenv("SPLATCT_FWD_KERNEL");   // "mma" / "ff": the other kernels
    const bool tc_path = kern && !strcmp(kern, "tc") && L.nt <= (int64_t)148 * TC_LIST_CAP;
    const bool ff_path = kern && !strcmp(kern, "ff");
    if ((tc_path || ff_path) && masks && L.ntz <= 64)   // they may follow another forward
        SPLATCT_CK(cudaMemsetAsync(at<char>(ws, L.o_pocc), 0,
                                   L.o_fcov + sizeof(unsigned long long) * (size_t)w * h - L.o_pocc,
                                   as_stream(stream)));
    // (the tensor-core kernel keeps each CTA's tile list in shared memory:
    // volumes beyond 148 x 7680 tiles of 16^3 take the mma.sync kernel)
    if (tc_path) {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t g3 = L.nt < (int64_t)nsm ? L.nt : (int64_t)nsm;
        // one CTA per SM (it allocates all 512 TMEM columns): a dynamic
        // shared-memory reservation above half the SM keeps a second one off
        constexpr int kPad = TC_LIST_CAP * 16;   // the tile list; > half an SM: 1 CTA / SM
        auto go = [&](auto mk) {
            auto kern_fn = k_fvr_fwd_tc<decltype(mk)::value>;
            cudaFuncSetAttribute(kern_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kPad);
            return launch_pdl(kern_fn, dim3((unsigned)g3), dim3(TC_THREADS), kPad, as_stream(stream), at<GRec>(ws, L.o_rec), w, h,
                              c, z0, hx, hy, hz, L.ntx, L.nty, L.nt, L.Sl,
                              at<uint32_t>(ws, L.o_tstart), at<uint32_t>(ws, vo), vol_yxz,
                              at<unsigned long long>(ws, L.o_pocc),
                              at<unsigned long long>(ws, L.o_fcov), halt);
        };
        if (masks) SPLATCT_CK(go(std::true_type{}));
        else SPLATCT_CK(go(std::false_type{}));
        SPLATCT_LAUNCH_CK();
        return SPLATCT_OK;
    }
    if (ff_path) {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t g2 = L.nt < (int64_t)nsm * 8 ? L.nt : (int64_t)nsm * 8;
        int64_t f2 = L.nt / (8 * g2);
        f2 = f2 < 1 ? 1 : (f2 > 32 ? 32 : f2);
        auto go = [&](auto mk) {
            return launch_pdl(k_fvr_fwd_ff<decltype(mk)::value>, dim3((unsigned)g2),
                              dim3(FF_THREADS), 0, as_stream(stream), at<GRec>(ws, L.o_rec), w, h,
                              c, z0, hx, hy, hz, L.ntx, L.nty, L.nt, L.Sl,
                              at<uint32_t>(ws, L.o_tstart), at<uint32_t>(ws, vo), vol_yxz,
                              counter, (int)f2, at<unsigned long long>(ws, L.o_pocc),
                              at<unsigned long long>(ws, L.o_fcov), halt);
        };
        SPLATCT_CK(cudaMemsetAsync(counter, 0, sizeof(unsigned int), as_stream(stream)));
        if (masks) SPLATCT_CK(go(std::true_type{}));
        else SPLATCT_CK(go(std::false_type{}));
        SPLATCT_LAUNCH_CK();
        SPLATCT_CK(cudaMemsetAsync(counter, 0, sizeof(unsigned int), as_stream(stream)));
        return SPLATCT_OK;
    }
    CUtensorMap tmap;
    const int use_tma = volume_tensor_map(&tmap, vol_yxz, w, h, c) ? 1 : 0;
    SPLATCT_CK(launch_pdl(k_fvr_fwd, dim3((unsigned)grid), dim3(256), 0, as_stream(stream),
                          at<GRec>(ws, L.o_rec), w, h, c, z0, hx, hy, hz, L.ntx, L.nty, L.nt, L.Sl,
        at<uint32_t>(ws, L.o_tstart), at<uint32_t>(ws, vo), vol_yxz, counter, (int)fetch,
        masks ? at<unsigned long long>(ws, L.o_pocc) : nullptr,
        masks ? at<unsigned long long>(ws, L.o_fcov) : nullptr, tmap, use_tma, halt));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_fvr_forward(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                        int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                        const int* halt, void* stream) {
    return fvr_forward_impl(params, n, w, h, c, z0, hx, hy, hz, ws, ws_bytes, vol_yxz, halt,
                            stream, false);
}

int splatct_fvr_forward_masked(const double* params, int64_t n, int w, int h, int c, int z0,
                               int hx, int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                               const int* halt, void* stream) {
    return fvr_forward_impl(params, n, w, h, c, z0, hx, hy, hz, ws, ws_bytes, vol_yxz, halt,
                            stream, true);
}

int splatct_fvr_forward_plain(const double* params, int64_t n, int w, int h, int c, int z0,
                              int hx, int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                              void* stream) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    if (int e = check_args(n, w, h, c, hx, hy, hz, ws_bytes, L)) return e;
    const size_t vo = L.final_buf ? L.o_v1 : L.o_v0;
    k_fvr_fwd_plain<<<(unsigned)L.nt, 256, 0, as_stream(stream)>>>(
        at<GRec>(ws, L.o_rec), w, h, c, z0, hx, hy, hz, L.ntx, L.nty, L.Sl,
        at<uint32_t>(ws, L.o_tstart), at<uint32_t>(ws, vo), vol_yxz);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_fvr_backward(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                         int hy, int hz, void* ws, size_t ws_bytes, const float* up_yxz,
                         double* grads, double* accum, const int* halt, void* stream) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    if (int e = check_args(n, w, h, c, hx, hy, hz, ws_bytes, L)) return e;
    if (n == 0) return SPLATCT_OK;
    cudaStream_t s = as_stream(stream);
    const unsigned grid = (unsigned)((n + BG_WARPS - 1) / BG_WARPS);
    const bool fast = 2 * hx + 1 <= 17 && 2 * hz + 1 <= 17;
    // SPLATCT_BWD_KERNEL=warp|ts2|ts|sp forces a kernel (measurement knob).  By
    // default the asynchronous tile-staged kernel takes dense clouds: staging a
    // tile column's slabs pays once tiles hold enough first-tile Gaussians, and
    // when the upstream outgrows L2 it is read ~4x instead of ~19x.  Measured on
    // the C5 sweep: 256^3/400k 0.97 -> 0.72 ms, 512^3/2M
    // 5.18 -> 3.42 ms, C4 1.07 -> 0.90 ms; sparse or L2-resident light clouds
    // (C2, 1024^3/<=2M, 128^3) stay on the per-Gaussian warp kernel.
    const char* kern = getenv("SPLATCT_BWD_KERNEL");
    const double per_tile = (double)n / (double)L.nt;
    const bool big_up = 4.0 * w * h * c > 96.0 * (1 << 20);
    const bool dense = L.nt >= 4096 && (per_tile >= 48.0 || (big_up && per_tile >= 8.0));
    const bool use_ts2 = kern ? !strcmp(kern, "ts2") : dense;
    if (fast && 2 * hy + 1 <= 17 && use_ts2) {
        CUtensorMap smap;
        if (volume_tensor_map(&smap, up_yxz, w, h, c, 16, 32, 32, true)) {
            SPLATCT_CK(cudaMemsetAsync(grads, 0, sizeof(double) * 5 * (size_t)n, s));
            unsigned int* counter = at<uint32_t>(ws, L.o_tcount) + 1;
            SPLATCT_CK(cudaMemsetAsync(counter, 0, sizeof(unsigned int), s));
            int dev = 0, nsm = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            const size_t dyn = 3 * (size_t)BT_SLAB_BYTES;
            cudaFuncSetAttribute(k_fvr_bwd_ts2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            const size_t vs = L.final_buf ? L.o_v1 : L.o_v0;
            SPLATCT_CK(launch_pdl(k_fvr_bwd_ts2, dim3(nsm), dim3(BT2Z_THREADS), dyn, s, params, n,
                                  (const uint32_t*)at<uint32_t>(ws, vs),
                                  (const uint32_t*)at<uint32_t>(ws, L.o_tstart), L.ntx, L.nty,
                                  L.ntz, L.Sl, (const int32_t*)at<int32_t>(ws, L.o_fp),
                                  (const GRec*)at<GRec>(ws, L.o_rec), w, h, c, z0, up_yxz, smap,
                                  counter, grads, accum, halt));
            SPLATCT_LAUNCH_CK();
            return SPLATCT_OK;
        }
    }
    if (fast && 2 * hy + 1 <= 17 && kern && !strcmp(kern, "ts")) {
        CUtensorMap smap;
        if (volume_tensor_map(&smap, up_yxz, w, h, c, 16, 32, 32, true)) {   // 64 B swizzle
            // unlisted Gaussians (footprint outside the volume) are never visited
            SPLATCT_CK(cudaMemsetAsync(grads, 0, sizeof(double) * 5 * (size_t)n, s));
            unsigned int* counter = at<uint32_t>(ws, L.o_tcount) + 1;
            SPLATCT_CK(cudaMemsetAsync(counter, 0, sizeof(unsigned int), s));
            int dev = 0, nsm = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            const size_t dyn = 3 * (size_t)BT_SLAB_BYTES;
            cudaFuncSetAttribute(k_fvr_bwd_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            const size_t vs = L.final_buf ? L.o_v1 : L.o_v0;    // sorted values
            SPLATCT_CK(launch_pdl(k_fvr_bwd_ts, dim3(nsm), dim3(32 * BT_WARPS), dyn, s, params, n,
                                  (const uint32_t*)at<uint32_t>(ws, vs),
                                  (const uint32_t*)at<uint32_t>(ws, L.o_tstart), L.ntx, L.nty,
                                  L.ntz, L.Sl, (const int32_t*)at<int32_t>(ws, L.o_fp),
                                  (const GRec*)at<GRec>(ws, L.o_rec), w, h, c, z0, up_yxz, smap,
                                  counter, grads, accum, halt));
            SPLATCT_LAUNCH_CK();
            return SPLATCT_OK;
        }
    }
    if (fast && kern && !strcmp(kern, "sp")) {
        // spatially ordered persistent kernel; Gaussians with no pair (footprint
        // outside the volume) are never visited: their gradients are zero
        SPLATCT_CK(cudaMemsetAsync(grads, 0, sizeof(double) * 5 * (size_t)n, s));
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const size_t vs = L.final_buf ? L.o_v1 : L.o_v0;    // sorted values
        auto go = [&](auto kc) {
            return launch_pdl(k_fvr_bwd_sp<decltype(kc)::value>, dim3(nsm), dim3(32 * BS_WARPS), 0,
                              s, params, n, (const uint32_t*)at<uint32_t>(ws, vs),
                              (const uint32_t*)at<uint32_t>(ws, L.o_tstart), L.nt, L.Sl,
                              (const int32_t*)at<int32_t>(ws, L.o_fp),
                              (const GRec*)at<GRec>(ws, L.o_rec), w, h, c, z0, up_yxz, grads,
                              accum, halt);
        };
        if (c == 256) SPLATCT_CK(go(std::integral_constant<int, 256>{}));
        else if (c == 512) SPLATCT_CK(go(std::integral_constant<int, 512>{}));
        else if (c == 1024) SPLATCT_CK(go(std::integral_constant<int, 1024>{}));
        else if (c == 128) SPLATCT_CK(go(std::integral_constant<int, 128>{}));
        else SPLATCT_CK(go(std::integral_constant<int, 0>{}));
        SPLATCT_LAUNCH_CK();
        return SPLATCT_OK;
    }
    // per-Gaussian-warp kernel (boxes > 17, or SPLATCT_BWD_KERNEL=warp):
    // an upstream larger than ~half of L2 is read from HBM: visit the
    // Gaussians in tile order so neighbouring warps share DRAM pages / lines
    // (index order spreads concurrent warps out, best while L2-resident)
    bool ord = (int64_t)w * h * c * 4 > ((int64_t)64 << 20);
    if (const char* e = getenv("SPLATCT_BWD_ORDER")) ord = atoi(e) != 0;
    uint32_t* order = at<uint32_t>(ws, L.o_order);
    if (ord) {
        const size_t vs = L.final_buf ? L.o_v1 : L.o_v0;    // sorted values
        uint32_t* flags = at<uint32_t>(ws, L.o_flag);
        uint32_t* pos = at<uint32_t>(ws, L.o_pos);
        const unsigned gb = (unsigned)((L.np + 1 + 255) / 256);
        k_first_flags<<<gb, 256, 0, s>>>(at<uint32_t>(ws, vs), at<uint32_t>(ws, L.o_tstart), L.nt,
                                         L.np, L.Sl, flags);
        SPLATCT_LAUNCH_CK();
        if (int e = exclusive_scan_u32(flags, pos, L.np + 1, at<void>(ws, L.o_scan2), s)) return e;
        k_order_scatter<<<gb, 256, 0, s>>>(at<uint32_t>(ws, vs), flags, pos, L.np, L.Sl, order);
        SPLATCT_LAUNCH_CK();
        SPLATCT_CK(cudaMemsetAsync(grads, 0, sizeof(double) * 5 * (size_t)n, s));   // unlisted
    }
    CUtensorMap utmap, utmap2;
    int use_tma = 0;
    if (fast && !getenv("SPLATCT_BWD_NO_TMA"))
        use_tma = volume_tensor_map(&utmap, up_yxz, w, h, c, BT_ZB, 17, 1, false) &&
                          volume_tensor_map(&utmap2, up_yxz, w, h, c, BT_ZB, 17, BT2_ROWS, false)
                      ? 1 : 0;
    if (!use_tma) {
        memset(&utmap, 0, sizeof(utmap));
        memset(&utmap2, 0, sizeof(utmap2));
    }
    auto launch = [&](auto fast_c, auto ord_c) {
        return launch_pdl(k_fvr_bwd<decltype(fast_c)::value, decltype(ord_c)::value>,
                          dim3(grid), dim3(32 * BG_WARPS), 0, s, params, n,
                          (const uint32_t*)order, (const int32_t*)at<int32_t>(ws, L.o_fp),
                          (const GRec*)at<GRec>(ws, L.o_rec), w, h, c, z0, up_yxz, grads, accum,
                          utmap, utmap2, use_tma, halt);
    };
    using T = std::true_type;
    using F = std::false_type;
    if (fast && ord) SPLATCT_CK(launch(T{}, T{}));
    else if (fast) SPLATCT_CK(launch(T{}, F{}));
    else if (ord) SPLATCT_CK(launch(F{}, T{}));
    else SPLATCT_CK(launch(F{}, F{}));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_fvr_pixel_occupancy_offset(int64_t n, int w, int h, int c, int hx, int hy, int hz,
                                       size_t* offset) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    SPLATCT_REQUIRE(offset != nullptr, "null offset");
    *offset = L.ntz <= 64 ? L.o_pocc : (size_t)-1;
    return SPLATCT_OK;
}

int splatct_fvr_footprint_coverage_offset(int64_t n, int w, int h, int c, int hx, int hy, int hz,
                                          size_t* offset) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    SPLATCT_REQUIRE(offset != nullptr, "null offset");
    *offset = L.ntz <= 64 ? L.o_fcov : (size_t)-1;
    return SPLATCT_OK;
}

int splatct_grad_norm_accum(const double* grads, int64_t n, double* accum, const int* halt,
                            void* stream) {
    if (n <= 0) return SPLATCT_OK;
    k_grad_norm_accum<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(grads, n, accum,
                                                                                 halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_fvr_export_bins(const void* ws, size_t ws_bytes, int64_t n, int w, int h, int c,
                            int hx, int hy, int hz, int32_t* fp, int32_t* tile_start,
                            int32_t* items, int64_t* npairs, int64_t* n_tiles, void* stream) {
    FvrLayout L = make_layout(n, w, h, c, hx, hy, hz);
    if (int e = check_args(n, w, h, c, hx, hy, hz, ws_bytes, L)) return e;
    cudaStream_t s = as_stream(stream);
    uint32_t total = 0;
    SPLATCT_CK(cudaMemcpyAsync(&total, at<uint32_t>(ws, L.o_tstart) + L.nt, sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    *npairs = total;
    *n_tiles = L.nt;
    if (fp)
        SPLATCT_CK(cudaMemcpyAsync(fp, at<int32_t>(ws, L.o_fp), sizeof(int32_t) * 6 * n,
                                   cudaMemcpyDeviceToDevice, s));
    if (tile_start)
        SPLATCT_CK(cudaMemcpyAsync(tile_start, at<uint32_t>(ws, L.o_tstart),
                                   sizeof(int32_t) * (L.nt + 1), cudaMemcpyDeviceToDevice, s));
    if (items && total > 0) {
        const size_t vo = L.final_buf ? L.o_v1 : L.o_v0;
        k_export_items<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(at<uint32_t>(ws, vo),
                                                                        total, L.Sl, items);
        SPLATCT_LAUNCH_CK();
    }
    return SPLATCT_OK;
}

}  // extern "C"
