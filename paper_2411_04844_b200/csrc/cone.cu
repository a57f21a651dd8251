// cone.cu -- circular cone-beam projector and its exact adjoint (SURVEY §8(f)
// N3: named by the north star, absent from the reference, parity unpinned).
//
// Model.  For view a and detector column u the xy
// path is the reference's fan ray (_kernels.py:232-259; raygeom.cuh): source
// S, unit direction, length L = |P - S|, clipped to [-1,w]x[-1,h], samples
// t_k = t0 + (k + 1/2) step, k < int((t1 - t0) / step), bilinear weights
// merged per pixel exactly as the per-slice operator does (march_ray).  Each
// merged (column, pixel) entry also carries tau = tbar / L, tbar the
// weight-averaged sample distance of its samples.  Detector row v (height v
// at the detector) reads the pixel's z-column at z = cz + v tau (linear
// interpolation, zero outside the volume):
//     p(a, u, v) = step sqrt(1 + (v/L)^2) sum_e w_e lerp(vol[pix_e], cz + v tau_e)
// The centre row (v = 0) of an odd-c volume is therefore exactly the fan
// projection of slice cz (same merged weights).
//
// B200 design.  Setup (once per geometry): the f64 march into a
// column-major entry list {pixel, w, tau} and its per-pixel transpose
// {column, w, tau, 1/tau} sorted by (column, entry).  Forward: one CTA per
// detector column (16 warps x 32 rows), the column's entries staged once in
// shared memory and broadcast to every row; the lanes' two z-taps hit a short
// contiguous stretch of the pixel's (yxz) z-column.  Adjoint: one warp per (pixel, z window), lanes
// over the detector rows of each entry (coalesced dL/dpred loads); each row
// adds its two tap contributions into per-warp shared-memory z accumulators,
// one per (row residue mod P, tap) class with P tau sv > 1, so no two lanes
// of an instruction touch the same word: plain read-modify-writes, fixed
// order, deterministic, no atomics.  Slabs: zc is the centre height in the
// slab's local coordinates, so slab projections are partial line integrals
// that sum to the full one.
#include "common.cuh"
#include "raygeom.cuh"

namespace splatct {

struct __align__(16) ConeColEntry {   // column-major (forward)
    int pix;
    float w;        // merged bilinear weight of the pixel's samples
    float tau;      // tbar / L
    float pad;
};

struct __align__(16) ConeEntry {      // pixel-major (adjoint)
    uint32_t col;   // detector column (view * nu + u)
    float w, tau;
    float inv_tau;  // 1 / tau (row-range setup of the adjoint)
};

__device__ __forceinline__ double column_length(const Geom& g, int r) {
    const int a = r / g.n_det, d = r % g.n_det;
    const double u = (d - 0.5 * (g.n_det - 1)) * g.spacing;
    const double dx = (g.rd + g.rs) * g.cos_t[a] - u * g.sin_t[a];
    const double dy = (g.rd + g.rs) * g.sin_t[a] + u * g.cos_t[a];
    return sqrt(dx * dx + dy * dy);
}

__global__ void k_cone_count(Geom g, int64_t* __restrict__ cnt, float* __restrict__ invL) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= g.m * g.n_det) return;
    int64_t c = 0;
    march_ray(g, r, [&](int, double, double) { ++c; });
    cnt[r] = c;
    invL[r] = (float)(1.0 / column_length(g, r));
}

__global__ void k_cone_fill(Geom g, const int64_t* __restrict__ cptr,
                            ConeColEntry* __restrict__ CE) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= g.m * g.n_det) return;
    const double inv_len = 1.0 / column_length(g, r);
    int64_t j = cptr[r];
    march_ray(g, r, [&](int pix, double w, double wt) {
        ConeColEntry e;
        e.pix = pix;
        e.w = (float)w;
        e.tau = (float)(wt / w * inv_len);
        e.pad = 0.f;
        CE[j++] = e;
    });
}

// Pixel-major transpose: count, atomic fill, per-pixel rank sort by the
// entry's global index (column-major order) -- deterministic gather order.
__global__ void k_cone_ecount(const ConeColEntry* __restrict__ CE, int64_t n,
                              unsigned long long* __restrict__ cnt) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < n) atomicAdd(&cnt[CE[j].pix], 1ull);
}

__global__ void k_cone_efill(const ConeColEntry* __restrict__ CE, const int64_t* __restrict__ cptr,
                             int nrays, unsigned long long* __restrict__ cursor,
                             ConeEntry* __restrict__ E, uint64_t* __restrict__ key) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrays) return;
    for (int64_t j = cptr[r]; j < cptr[r + 1]; ++j) {
        const ConeColEntry c = CE[j];
        const unsigned long long pos = atomicAdd(&cursor[c.pix], 1ull);
        ConeEntry e;
        e.col = (uint32_t)r;
        e.w = c.w;
        e.tau = c.tau;
        e.inv_tau = 1.f / c.tau;
        E[pos] = e;
        key[pos] = (uint64_t)j;
    }
}

__global__ void k_cone_esort(int64_t npix, const int64_t* __restrict__ eptr,
                             const ConeEntry* __restrict__ in, const uint64_t* __restrict__ key,
                             ConeEntry* __restrict__ out) {
    const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= npix) return;
    const int64_t b = eptr[p], e = eptr[p + 1];
    for (int64_t i = b + lane; i < e; i += 32) {
        const uint64_t k = key[i];
        int64_t rank = 0;
        for (int64_t j = b; j < e; ++j) rank += key[j] < k;
        out[b + rank] = in[i];
    }
}

// Integer cell and fraction of a z coordinate without the conversion pipe:
// (z - 1/2) rounded to nearest by the 1.5*2^23 trick.  The cell is floor(z)
// except at exact integers, where it may be z - 1 with fraction 1 -- the same
// interpolated value (the adjoint's floor cell gives the same nonzero taps).
// |z| < 2^22.
__device__ __forceinline__ int zcell(float z, float& fz) {
    const float t = __fadd_rn(__fadd_rn(z, -0.5f), 12582912.0f);
    fz = __fadd_rn(z, -__fadd_rn(t, -12582912.0f));
    return __float_as_int(t) - 0x4B400000;
}

// --------------------------------------------------------------------------
// forward: one CTA per (column, up to CONE_WARPS x 32 detector rows); the
// column's entries are staged in shared memory once per CTA (every row of the
// column reads the same entries) and each warp walks them for its 32 rows
// --------------------------------------------------------------------------
constexpr int CONE_WARPS = 16;
constexpr int CONE_BATCH = 512;   // entries staged per round

__global__ void __launch_bounds__(32 * CONE_WARPS) k_cone_fwd(
    const ConeColEntry* __restrict__ CE, const int64_t* __restrict__ cptr,
    const float* __restrict__ invL, int nrays, int nv, float sv, float step, int cl, float zc,
    const float* __restrict__ vol, const unsigned long long* __restrict__ occ,
    float* __restrict__ sino, const int* halt) {
    if (halted(halt)) return;
    __shared__ float4 sb[CONE_BATCH];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int chunks = (nv + 31) / 32;
    const int cgroups = (chunks + CONE_WARPS - 1) / CONE_WARPS;
    const int64_t r = blockIdx.x / cgroups;
    const int chunk = (int)(blockIdx.x % cgroups) * CONE_WARPS + wid;
    const int dv = chunk * 32 + lane;
    const float vmid = 0.5f * (float)(nv - 1);
    const float v = ((float)dv - vmid) * sv;
    const int64_t b = cptr[r], e = cptr[r + 1];
    float acc = 0.f;
    bool any = false;
    if (b < e) {   // rows whose z-path misses the slab entirely skip the arithmetic
        const float ta = CE[b].tau, tb = CE[e - 1].tau;
        const float za = __fmaf_rn(v, ta, zc), zb = __fmaf_rn(v, tb, zc);
        const bool hit = dv < nv && !(fmaxf(za, zb) < -1.f || fminf(za, zb) >= (float)cl);
        any = __any_sync(0xffffffffu, hit);
    }
    static_assert(CONE_BATCH == 32 * CONE_WARPS, "one staged entry per thread");
    __shared__ int s_wcnt[CONE_WARPS];
    for (int64_t j0 = b; j0 < e; j0 += CONE_BATCH) {
        __syncthreads();
        // stage this batch, compacted to the entries whose pixel column has an
        // occupied tile (the others read only zeros); order is kept
        const int t = threadIdx.x;
        float4 en_t = make_float4(0.f, 0.f, 0.f, 0.f);
        bool keep = j0 + t < e;
        if (keep) {
            en_t = *reinterpret_cast<const float4*>(CE + j0 + t);
            if (occ) keep = occ[__float_as_int(en_t.x)] != 0ull;   // pixel column occupancy
        }
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_wcnt[wid] = __popc(km);
        __syncthreads();
        int base = 0, cnt = 0;
#pragma unroll
        for (int q = 0; q < CONE_WARPS; ++q) {
            const int v = s_wcnt[q];
            base += q < wid ? v : 0;
            cnt += v;
        }
        if (keep) sb[base + __popc(km & ((1u << lane) - 1u))] = en_t;
        __syncthreads();
        if (!any) continue;
#pragma unroll 4
        for (int jj = 0; jj < cnt; ++jj) {
            const float4 en = sb[jj];
            // z taps, clamped into the slab with zero weight outside it
            float fz;
            const int zi = zcell(__fmaf_rn(v, en.z, zc), fz);
            const float* col = vol + (int64_t)__float_as_int(en.x) * cl + zi;
            const float a0 = (unsigned)zi < (unsigned)cl ? __ldg(col) : 0.f;
            const float a1 = (unsigned)(zi + 1) < (unsigned)cl ? __ldg(col + 1) : 0.f;
            acc = fmaf(en.y, fmaf(fz, a1 - a0, a0), acc);
        }
    }
    if (dv < nv) {
        const float slope = v * invL[r];
        sino[r * nv + dv] = acc * (step * __fsqrt_rn(__fmaf_rn(slope, slope, 1.f)));
    }
}

// g_s[col][v] = g[col][v] * step * sqrt(1 + (v/L)^2): the per-row arc length
// of the forward, folded into the adjoint's input once
__global__ void k_cone_gscale(const float* __restrict__ g, const float* __restrict__ invL,
                              int64_t nrays, int nv, float sv, float step,
                              float* __restrict__ gs, const int* halt) {
    if (halted(halt)) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrays * nv) return;
    const int dv = (int)(i % nv);
    const float v = ((float)dv - 0.5f * (float)(nv - 1)) * sv;
    const float slope = v * invL[i / nv];
    gs[i] = g[i] * (step * __fsqrt_rn(__fmaf_rn(slope, slope, 1.f)));
}

// --------------------------------------------------------------------------
// adjoint: warp per (pixel, window of <= CA_ZW slices)
// --------------------------------------------------------------------------
constexpr int CA_ZW = 256;
constexpr int CA_PMAX = 3;   // residue classes held in shared memory (P tau sv > 1)
constexpr int CA_WARPS = 4;
constexpr int CA_LEN = CA_ZW + 4;   // slot 0 = slice zb - 1, slots zn + 1.. = spill-over

__global__ void __launch_bounds__(32 * CA_WARPS) k_cone_adj(
    const ConeEntry* __restrict__ E, const int64_t* __restrict__ eptr, int64_t npix, int nv,
    float sv, int cl, float zc, const float* __restrict__ gs, float* __restrict__ out,
    int accumulate, const unsigned long long* __restrict__ occ, int w, const int* halt) {
    if (halted(halt)) return;
    __shared__ float zacc[CA_WARPS][2 * CA_PMAX][CA_LEN];
    __shared__ float4 eb[CA_WARPS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int lm2 = lane & 1, lm3 = lane % 3;
    const int nwin = (cl + CA_ZW - 1) / CA_ZW;
    const int64_t gw = blockIdx.x * (int64_t)CA_WARPS + wid;
    const int64_t p = gw / nwin;
    if (p >= npix) return;
    const int zb = (int)(gw % nwin) * CA_ZW, zn = min(CA_ZW, cl - zb);
    if (occ) {   // training step: output read only inside occupied tiles
        const int tlo = zb >> 4, thi = (zb + zn - 1) >> 4;
        const unsigned long long zm =
            (thi >= 63 ? ~0ull : ((1ull << (thi + 1)) - 1ull)) & ~((1ull << tlo) - 1ull);
        // footprint coverage (the backward reads every footprint voxel, including
        // exact zeros, so the value-based pixel occupancy would not do)
        if ((occ[p] & zm) == 0ull) return;   // warp-uniform
    }
    for (int k = 0; k < 2 * CA_PMAX; ++k)
        for (int i = lane; i < zn + 3; i += 32) zacc[wid][k][i] = 0.f;
    const float vmid = 0.5f * (float)(nv - 1);
    const float inv_sv = 1.f / sv;
    const int64_t b = eptr[p], e = eptr[p + 1];
    for (int64_t j0 = b; j0 < e; j0 += 32) {
        __syncwarp();
        if (j0 + lane < e) eb[wid][lane] = *reinterpret_cast<const float4*>(E + j0 + lane);
        __syncwarp();
        const int cnt = (int)min((int64_t)32, e - j0);
        for (int jj = 0; jj < cnt; ++jj) {
            const float4 en = eb[wid][jj];
            const uint32_t col = __float_as_uint(en.x);
            const float wxy = en.y, tau = en.z;
            // rows with z in [zb - 1, zb + zn] (one row of margin for rounding)
            const float inv = en.w * inv_sv;
            const int d0 = max((int)floorf(((float)(zb - 1) - zc) * inv + vmid) - 1, 0);
            const int d1 = min((int)ceilf(((float)(zb + zn) - zc) * inv + vmid) + 1, nv - 1);
            const float* grow = gs + (int64_t)col * nv;
            // rows P apart are > 1 slice apart, so lanes of one residue class
            // mod P never share a voxel within an instruction
            const int P = (int)floorf(inv) + 1;
            if (P <= CA_PMAX) {   // one array pair per class: no barriers inside
                const int cls = P == 1 ? 0 : (P == 2 ? lm2 : lm3);
                float* ra = &zacc[wid][2 * cls][1];        // slot of slice z0 (local)
                float* rb = &zacc[wid][2 * cls + 1][2];    // slot of slice z0 + 1
                // the upstream rows come from L2: keep two chunks of loads in
                // flight ahead of the shared-memory read-modify-writes
                float g1 = d0 + lane <= d1 ? __ldg(grow + d0 + lane) : 0.f;
                float g2 = d0 + 32 + lane <= d1 ? __ldg(grow + d0 + 32 + lane) : 0.f;
                for (int dd = d0; dd <= d1; dd += 32) {
                    const int d = dd + lane;
                    const float gc = g1;
                    g1 = g2;
                    g2 = d + 64 <= d1 ? __ldg(grow + d + 64) : 0.f;
                    const float v = ((float)d - vmid) * sv;
                    // floor cell: at exact integers this picks the forward's other
                    // (zero-weight) neighbour, so the taps -- and the transpose -- agree
                    const float z = __fmaf_rn(v, tau, zc);
                    const float zf = floorf(z);
                    const int z0 = (int)zf - zb;
                    // taps of slices -1 .. zn land in padded slots, dropped at the end
                    const bool ok = d <= d1 && (unsigned)(z0 + 1) <= (unsigned)zn;
                    const float g = ok ? wxy * gc : 0.f;
                    const float tb = g * (z - zf);
                    if (ok) {
                        ra[z0] += g - tb;
                        rb[z0] += tb;
                    }
                    __syncwarp();
                }
            } else {              // very dense rows: classes in sequence
                const int cls = lane % P;
                for (int dd = d0; dd <= d1; dd += 32) {
                    const int d = dd + lane;
                    const float v = ((float)d - vmid) * sv;
                    const float z = __fmaf_rn(v, tau, zc);
                    const float zf = floorf(z);
                    const int z0 = (int)zf - zb;
                    const bool ok = d <= d1 && (unsigned)(z0 + 1) <= (unsigned)zn;
                    const float g = ok ? wxy * __ldg(grow + d) : 0.f;
                    const float tb = g * (z - zf);
                    for (int ph = 0; ph < P; ++ph) {
                        if (ok && cls == ph) zacc[wid][0][z0 + 1] += g - tb;
                        __syncwarp();
                        if (ok && cls == ph) zacc[wid][1][z0 + 2] += tb;
                        __syncwarp();
                    }
                }
            }
        }
    }
    __syncwarp();
    float* o = out + p * cl + zb;
    for (int i = lane; i < zn; i += 32) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * CA_PMAX; ++k) s += zacc[wid][k][i + 1];
        o[i] = accumulate ? o[i] + s : s;
    }
}

static Geom cone_geom(const double* cos_t, const double* sin_t, int m, int nu, double su,
                      double rs, double rd, int w, int h, double step) {
    Geom g;
    g.cos_t = cos_t;
    g.sin_t = sin_t;
    g.m = m;
    g.n_det = nu;
    g.spacing = su;
    g.step = step;
    g.is_fan = true;
    g.rs = rs;
    g.rd = rd;
    g.w = w;
    g.h = h;
    return g;
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_cone_setup_scratch_bytes(int m, int nu, int w, int h, size_t* bytes) {
    const int64_t n = (int64_t)m * nu + 1, np = (int64_t)w * h + 1;
    const int64_t big = n > np ? n : np;
    *bytes = align_up(sizeof(unsigned long long) * big) * 2 + scan_temp_bytes(big) + 256;
    return SPLATCT_OK;
}

int splatct_cone_count(const double* cos_t, const double* sin_t, int m, int nu, double su,
                       double rs, double rd, int w, int h, double step, int64_t* cptr,
                       float* invL, void* scratch, size_t scratch_bytes, int64_t* nentries,
                       void* stream) {
    SPLATCT_REQUIRE(m > 0 && nu > 0 && w > 0 && h > 0 && step > 0, "invalid cone geometry");
    size_t need = 0;
    splatct_cone_setup_scratch_bytes(m, nu, w, h, &need);
    SPLATCT_REQUIRE(scratch_bytes >= need, "cone scratch too small");
    cudaStream_t s = as_stream(stream);
    const int nr = m * nu;
    const int64_t big = (int64_t)nr + 1 > (int64_t)w * h + 1 ? (int64_t)nr + 1 : (int64_t)w * h + 1;
    int64_t* cnt = reinterpret_cast<int64_t*>(scratch);
    void* tmp = (char*)scratch + 2 * align_up(sizeof(unsigned long long) * big);
    SPLATCT_CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (nr + 1), s));
    const Geom g = cone_geom(cos_t, sin_t, m, nu, su, rs, rd, w, h, step);
    k_cone_count<<<(nr + 127) / 128, 128, 0, s>>>(g, cnt, invL);
    SPLATCT_LAUNCH_CK();
    if (int e = exclusive_scan_i64(cnt, cptr, nr + 1, tmp, s)) return e;
    SPLATCT_CK(cudaMemcpyAsync(nentries, cptr + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    return SPLATCT_OK;
}

int splatct_cone_fill(const double* cos_t, const double* sin_t, int m, int nu, double su,
                      double rs, double rd, int w, int h, double step, const int64_t* cptr,
                      void* col_entries, void* stream) {
    cudaStream_t s = as_stream(stream);
    const int nr = m * nu;
    const Geom g = cone_geom(cos_t, sin_t, m, nu, su, rs, rd, w, h, step);
    k_cone_fill<<<(nr + 127) / 128, 128, 0, s>>>(g, cptr,
                                                 reinterpret_cast<ConeColEntry*>(col_entries));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_cone_entry_count(const void* col_entries, const int64_t* cptr, int nrays, int w,
                             int h, int64_t* eptr, void* scratch, size_t scratch_bytes,
                             int64_t* nentries, void* stream) {
    const int64_t np = (int64_t)w * h;
    SPLATCT_REQUIRE(scratch_bytes >= align_up(sizeof(int64_t) * (np + 1)) * 2 +
                                          scan_temp_bytes(np + 1),
                    "cone entry scratch too small");
    cudaStream_t s = as_stream(stream);
    int64_t n = 0;
    SPLATCT_CK(cudaMemcpyAsync(&n, cptr + nrays, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(scratch);
    void* tmp = (char*)scratch + 2 * align_up(sizeof(int64_t) * (np + 1));
    SPLATCT_CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (np + 1), s));
    if (n > 0) {
        k_cone_ecount<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
            reinterpret_cast<const ConeColEntry*>(col_entries), n, cnt);
        SPLATCT_LAUNCH_CK();
    }
    if (int e = exclusive_scan_i64(reinterpret_cast<int64_t*>(cnt), eptr, np + 1, tmp, s))
        return e;
    SPLATCT_CK(cudaMemcpyAsync(nentries, eptr + np, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    return SPLATCT_OK;
}

int splatct_cone_entry_scratch_bytes(int64_t nentries, int w, int h, size_t* bytes) {
    const int64_t np = (int64_t)w * h;
    const size_t n1 = nentries > 0 ? (size_t)nentries : 1;
    *bytes = align_up(sizeof(ConeEntry) * n1) + align_up(sizeof(uint64_t) * n1) +
             align_up(sizeof(unsigned long long) * (np + 1));
    return SPLATCT_OK;
}

int splatct_cone_entry_fill(const void* col_entries, const int64_t* cptr, int nrays, int w,
                            int h, const int64_t* eptr, int64_t nentries, void* entries,
                            void* scratch, size_t scratch_bytes, void* stream) {
    size_t need = 0;
    splatct_cone_entry_scratch_bytes(nentries, w, h, &need);
    SPLATCT_REQUIRE(scratch_bytes >= need, "cone entry scratch too small");
    cudaStream_t s = as_stream(stream);
    const int64_t np = (int64_t)w * h;
    const size_t n1 = nentries > 0 ? (size_t)nentries : 1;
    ConeEntry* tmpE = reinterpret_cast<ConeEntry*>(scratch);
    uint64_t* key = reinterpret_cast<uint64_t*>((char*)scratch + align_up(sizeof(ConeEntry) * n1));
    unsigned long long* cursor = reinterpret_cast<unsigned long long*>(
        (char*)scratch + align_up(sizeof(ConeEntry) * n1) + align_up(sizeof(uint64_t) * n1));
    SPLATCT_CK(cudaMemcpyAsync(cursor, eptr, sizeof(int64_t) * (np + 1), cudaMemcpyDeviceToDevice,
                               s));
    k_cone_efill<<<(nrays + 127) / 128, 128, 0, s>>>(
        reinterpret_cast<const ConeColEntry*>(col_entries), cptr, nrays, cursor, tmpE, key);
    SPLATCT_LAUNCH_CK();
    k_cone_esort<<<(unsigned)((np * 32 + 255) / 256), 256, 0, s>>>(
        np, eptr, tmpE, key, reinterpret_cast<ConeEntry*>(entries));
    SPLATCT_LAUNCH_CK();
    SPLATCT_CK(cudaStreamSynchronize(s));   // scratch may be freed by the caller after return
    return SPLATCT_OK;
}

int splatct_cone_forward(const void* col_entries, const int64_t* cptr, const float* invL,
                         int nrays, int nv, double sv, double step, int w, int h, int c_local,
                         double zc, const float* vol_yxz, const uint64_t* col_occ, float* sino,
                         const int* halt, void* stream) {
    SPLATCT_REQUIRE(nrays >= 0 && nv > 0 && c_local > 0 && w > 0 && h > 0,
                    "invalid cone forward sizes");
    SPLATCT_REQUIRE(col_occ == nullptr || c_local <= 64 * 16, "occupancy needs <= 64 z tiles");
    const int chunks = (nv + 31) / 32;
    const int64_t blocks = (int64_t)nrays * ((chunks + CONE_WARPS - 1) / CONE_WARPS);
    if (blocks == 0) return SPLATCT_OK;
    k_cone_fwd<<<(unsigned)blocks, 32 * CONE_WARPS, 0, as_stream(stream)>>>(reinterpret_cast<const ConeColEntry*>(col_entries), cptr,
                                      invL, nrays, nv, (float)sv, (float)step, c_local,
                                      (float)zc, vol_yxz,
                                      reinterpret_cast<const unsigned long long*>(col_occ), sino,
                                      halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_cone_adjoint(const void* entries, const int64_t* eptr, const float* invL, int nrays,
                         int nv, double sv, double step, int w, int h, int c_local, double zc,
                         const float* gsino, float* gscaled, float* out_yxz, int accumulate,
                         const uint64_t* col_occ, const int* halt, void* stream) {
    SPLATCT_REQUIRE(nv > 0 && c_local > 0 && w > 0 && h > 0, "invalid cone adjoint sizes");
    SPLATCT_REQUIRE(col_occ == nullptr || c_local <= 64 * 16, "occupancy needs <= 64 z tiles");
    cudaStream_t s = as_stream(stream);
    const int64_t ng = (int64_t)nrays * nv;
    if (ng > 0) {
        k_cone_gscale<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(gsino, invL, nrays, nv,
                                                                   (float)sv, (float)step,
                                                                   gscaled, halt);
        SPLATCT_LAUNCH_CK();
    }
    const int64_t np = (int64_t)w * h;
    const int64_t warps = np * ((c_local + CA_ZW - 1) / CA_ZW);
    k_cone_adj<<<(unsigned)((warps + CA_WARPS - 1) / CA_WARPS), 32 * CA_WARPS, 0, s>>>(
        reinterpret_cast<const ConeEntry*>(entries), eptr, np, nv, (float)sv, c_local, (float)zc,
        gscaled, out_yxz, accumulate, reinterpret_cast<const unsigned long long*>(col_occ), w,
        halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
