// cone.cu -- circular cone-beam projector and its exact adjoint (SURVEY §8(f)
// N3: named by the north star, absent from the reference, parity unpinned).
//
// Model.  For view a and detector column u the xy
// path is the reference's fan ray (_kernels.py:232-259 via raygeom.cuh):
// source S, unit direction d, length L = |P - S|, clipped to [-1,w]x[-1,h],
// samples t_k = t0 + (k + 1/2) step, k < int((t1 - t0) / step).  Detector row
// v (height v at the detector) sees z(t) = cz + v t / L, so every row of a
// column shares the xy samples and bilinear weights; the value is
//     p(a, u, v) = step sqrt(1 + (v/L)^2) sum_k trilinear(vol; x_k, y_k, z_k)
// with zero outside the volume.  The centre row (v = 0) of an odd-c volume is
// exactly the fan projection of slice cz.
//
// B200 design.  The f64 xy march runs once per geometry into a per-column
// sample list {pixel, fx, fy, tau = t/L} (16 B).  Forward: one warp per
// (column, 32 rows), lanes over rows: each sample is a shared-memory
// broadcast, its four bilinear corners are warp-uniform, and the lanes'
// z-taps hit a short contiguous stretch of the corner's (yxz) z-column.
// Adjoint: the exact transpose as a gather (no atomics, deterministic): the
// samples are transposed once into per-pixel entry lists {column, tau, w_xy}
// sorted by (column, sample, corner); one warp per (pixel, 32 slices), each
// lane finds the detector rows whose z-taps land on its slice (the same f32
// z = fma(v, tau, zc) as the forward) and accumulates w_xy w_z g.
// Slabs: zc is the centre height in the slab's local coordinates, so
// per-slab projections are partial line integrals that sum to the full one.
#include "common.cuh"
#include "raygeom.cuh"

namespace splatct {

struct __align__(16) ConeSample {
    int pix;        // ((y0 + 1) << 16) | (x0 + 1), x0 in [-1, w], y0 in [-1, h]
    float fx, fy;   // bilinear fractions
    float tau;      // t / L
};

struct __align__(16) ConeEntry {
    uint32_t col;   // detector column (view * nu + u)
    float tau, wxy, pad;
};

struct ConeGeom {
    const double* cos_t;
    const double* sin_t;
    int m, nu;
    double su, step, rs, rd;
    int w, h;
};

__device__ __forceinline__ void cone_column(const ConeGeom& g, int r, double& ox, double& oy,
                                            double& dx, double& dy, double& t0, double& t1,
                                            double& len) {
    const int a = r / g.nu, d = r % g.nu;
    const double cx = 0.5 * (g.w - 1), cy = 0.5 * (g.h - 1);
    const double u = (d - 0.5 * (g.nu - 1)) * g.su;
    ray_geometry(g.cos_t[a], g.sin_t[a], u, true, g.rs, g.rd, cx, cy, g.w, g.h, ox, oy, dx, dy,
                 t0, t1);
    const double ddx = (g.rd + g.rs) * g.cos_t[a] - u * g.sin_t[a];
    const double ddy = (g.rd + g.rs) * g.sin_t[a] + u * g.cos_t[a];
    len = sqrt(ddx * ddx + ddy * ddy);
}

__global__ void k_cone_count(ConeGeom g, int64_t* __restrict__ cnt, float* __restrict__ invL) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= g.m * g.nu) return;
    double ox, oy, dx, dy, t0, t1, len;
    cone_column(g, r, ox, oy, dx, dy, t0, t1, len);
    cnt[r] = t1 > t0 ? (int64_t)((t1 - t0) / g.step) : 0;
    invL[r] = (float)(1.0 / len);
}

__global__ void k_cone_fill(ConeGeom g, const int64_t* __restrict__ rptr,
                            ConeSample* __restrict__ S) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= g.m * g.nu) return;
    double ox, oy, dx, dy, t0, t1, len;
    cone_column(g, r, ox, oy, dx, dy, t0, t1, len);
    const int64_t b = rptr[r], ns = rptr[r + 1] - b;
    for (int64_t k = 0; k < ns; ++k) {
        const double t = t0 + (k + 0.5) * g.step;
        const double sx = ox + t * dx, sy = oy + t * dy;
        const double fx0 = floor(sx), fy0 = floor(sy);
        ConeSample s;
        s.pix = (((int)fy0 + 1) << 16) | ((int)fx0 + 1);
        s.fx = (float)(sx - fx0);
        s.fy = (float)(sy - fy0);
        s.tau = (float)(t / len);
        S[b + k] = s;
    }
}

__device__ __forceinline__ float corner_weight(int q, float fx, float fy) {
    return __fmul_rn((q & 1) ? fx : 1.f - fx, (q & 2) ? fy : 1.f - fy);
}

// Pixel-entry transpose: count, atomic fill, per-pixel rank sort by key
// (column, sample, corner) -- deterministic order for the gather.
__global__ void k_cone_ecount(const ConeSample* __restrict__ S, const int64_t* __restrict__ rptr,
                              int nrays, int w, int h, unsigned long long* __restrict__ cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrays) return;
    for (int64_t j = rptr[r]; j < rptr[r + 1]; ++j) {
        const ConeSample s = S[j];
        const int x0 = (s.pix & 0xffff) - 1, y0 = (s.pix >> 16) - 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int px = x0 + (q & 1), py = y0 + (q >> 1);
            if (px < 0 || px >= w || py < 0 || py >= h || corner_weight(q, s.fx, s.fy) == 0.f)
                continue;
            atomicAdd(&cnt[(int64_t)py * w + px], 1ull);
        }
    }
}

__global__ void k_cone_efill(const ConeSample* __restrict__ S, const int64_t* __restrict__ rptr,
                             int nrays, int w, int h, unsigned long long* __restrict__ cursor,
                             ConeEntry* __restrict__ E, uint64_t* __restrict__ key) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrays) return;
    const int64_t b = rptr[r];
    for (int64_t j = b; j < rptr[r + 1]; ++j) {
        const ConeSample s = S[j];
        const int x0 = (s.pix & 0xffff) - 1, y0 = (s.pix >> 16) - 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int px = x0 + (q & 1), py = y0 + (q >> 1);
            const float wq = corner_weight(q, s.fx, s.fy);
            if (px < 0 || px >= w || py < 0 || py >= h || wq == 0.f) continue;
            const unsigned long long pos = atomicAdd(&cursor[(int64_t)py * w + px], 1ull);
            ConeEntry e;
            e.col = (uint32_t)r;
            e.tau = s.tau;
            e.wxy = wq;
            e.pad = 0.f;
            E[pos] = e;
            key[pos] = ((uint64_t)r << 34) | ((uint64_t)(j - b) << 2) | (uint64_t)q;
        }
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

// --------------------------------------------------------------------------
// forward: warp per (column, 32 detector rows)
// --------------------------------------------------------------------------
constexpr int CONE_WARPS = 8;

__global__ void __launch_bounds__(32 * CONE_WARPS) k_cone_fwd(
    const ConeSample* __restrict__ S, const int64_t* __restrict__ rptr,
    const float* __restrict__ invL, int nrays, int nv, float sv, float step, int w, int h, int cl,
    float zc, const float* __restrict__ vol, float* __restrict__ sino, const int* halt) {
    if (halted(halt)) return;
    __shared__ float4 sb[CONE_WARPS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int chunks = (nv + 31) / 32;
    const int64_t gw = blockIdx.x * (int64_t)CONE_WARPS + wid;
    const int64_t r = gw / chunks;
    if (r >= nrays) return;
    const int dv = (int)(gw % chunks) * 32 + lane;
    const float vmid = 0.5f * (float)(nv - 1);
    const float v = ((float)dv - vmid) * sv;
    const int64_t b = rptr[r], e = rptr[r + 1];
    float acc = 0.f;
    bool any = false;
    if (b < e) {   // rows whose z-path misses the slab entirely skip the march
        const float ta = S[b].tau, tb = S[e - 1].tau;
        const float za = __fmaf_rn(v, ta, zc), zb = __fmaf_rn(v, tb, zc);
        const bool hit = dv < nv && !(fmaxf(za, zb) < -1.f || fminf(za, zb) >= (float)cl);
        any = __any_sync(0xffffffffu, hit);
    }
    if (any) {
        for (int64_t j0 = b; j0 < e; j0 += 32) {
            __syncwarp();
            if (j0 + lane < e) sb[wid][lane] = *reinterpret_cast<const float4*>(S + j0 + lane);
            __syncwarp();
            const int cnt = (int)min((int64_t)32, e - j0);
            for (int jj = 0; jj < cnt; ++jj) {
                const float4 sm = sb[wid][jj];
                const int pix = __float_as_int(sm.x);
                const float z = __fmaf_rn(v, sm.w, zc);
                const float zf = floorf(z);
                const int z0 = (int)zf;
                const float fz = z - zf;
                if (z0 < -1 || z0 >= cl) continue;
                const bool ok0 = z0 >= 0, ok1 = z0 + 1 < cl;
                const int x0 = (pix & 0xffff) - 1, y0 = (pix >> 16) - 1;
                float s = 0.f;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int px = x0 + (q & 1), py = y0 + (q >> 1);
                    if (px < 0 || px >= w || py < 0 || py >= h) continue;   // warp-uniform
                    const float* col = vol + ((int64_t)py * w + px) * cl;
                    const float a0 = ok0 ? __ldg(col + z0) : 0.f;
                    const float a1 = ok1 ? __ldg(col + z0 + 1) : 0.f;
                    s = fmaf(corner_weight(q, sm.y, sm.z), fmaf(fz, a1 - a0, a0), s);
                }
                acc += s;
            }
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
// adjoint: warp per (pixel, 32 slices), gather over the pixel's entries
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * CONE_WARPS) k_cone_adj(
    const ConeEntry* __restrict__ E, const int64_t* __restrict__ eptr, int64_t npix, int nv,
    float sv, int cl, float zc, const float* __restrict__ gs, float* __restrict__ out,
    int accumulate, const int* halt) {
    if (halted(halt)) return;
    __shared__ float4 eb[CONE_WARPS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int zchunks = (cl + 31) / 32;
    const int64_t gw = blockIdx.x * (int64_t)CONE_WARPS + wid;
    const int64_t p = gw / zchunks;
    if (p >= npix) return;
    const int zl = (int)(gw % zchunks) * 32 + lane;
    const float vmid = 0.5f * (float)(nv - 1);
    const float zrel = (float)zl - zc;
    const int64_t b = eptr[p], e = eptr[p + 1];
    float acc = 0.f;
    for (int64_t j0 = b; j0 < e; j0 += 32) {
        __syncwarp();
        if (j0 + lane < e) eb[wid][lane] = *reinterpret_cast<const float4*>(E + j0 + lane);
        __syncwarp();
        const int cnt = (int)min((int64_t)32, e - j0);
        for (int jj = 0; jj < cnt; ++jj) {
            const float4 en = eb[wid][jj];
            const uint32_t col = __float_as_uint(en.x);
            const float tau = en.y, wxy = en.z;
            // rows whose forward tap z = fma(v, tau, zc) lies in [zl - 1, zl + 1)
            const float inv = 1.f / (tau * sv);
            const int d0 = max((int)floorf((zrel - 1.f) * inv + vmid) - 1, 0);
            const int d1 = min((int)ceilf((zrel + 1.f) * inv + vmid) + 1, nv - 1);
            const float* grow = gs + (int64_t)col * nv;
            float s = 0.f;
            for (int d = d0; d <= d1; ++d) {
                const float v = ((float)d - vmid) * sv;
                const float z = __fmaf_rn(v, tau, zc);
                const float zf = floorf(z);
                const int z0 = (int)zf;
                const float fz = z - zf;
                const float wz = z0 == zl ? 1.f - fz : (z0 + 1 == zl ? fz : 0.f);
                if (wz != 0.f) s = fmaf(wz, __ldg(grow + d), s);
            }
            acc = fmaf(wxy, s, acc);
        }
    }
    if (zl < cl) {
        float* o = out + p * cl + zl;
        *o = accumulate ? *o + acc : acc;
    }
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
                       double rs, double rd, int w, int h, double step, int64_t* rptr,
                       float* invL, void* scratch, size_t scratch_bytes, int64_t* nsamples,
                       void* stream) {
    SPLATCT_REQUIRE(m > 0 && nu > 0 && w > 0 && h > 0 && step > 0, "invalid cone geometry");
    SPLATCT_REQUIRE(w < 65534 && h < 32766, "cone sample packing needs w < 65534, h < 32766");
    size_t need = 0;
    splatct_cone_setup_scratch_bytes(m, nu, w, h, &need);
    SPLATCT_REQUIRE(scratch_bytes >= need, "cone scratch too small");
    cudaStream_t s = as_stream(stream);
    const int nr = m * nu;
    int64_t* cnt = reinterpret_cast<int64_t*>(scratch);
    void* tmp = (char*)scratch + 2 * align_up(sizeof(unsigned long long) *
                                              ((int64_t)nr + 1 > (int64_t)w * h + 1
                                                   ? (int64_t)nr + 1 : (int64_t)w * h + 1));
    SPLATCT_CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (nr + 1), s));
    ConeGeom g{cos_t, sin_t, m, nu, su, step, rs, rd, w, h};
    k_cone_count<<<(nr + 127) / 128, 128, 0, s>>>(g, cnt, invL);
    SPLATCT_LAUNCH_CK();
    if (int e = exclusive_scan_i64(cnt, rptr, nr + 1, tmp, s)) return e;
    SPLATCT_CK(cudaMemcpyAsync(nsamples, rptr + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    return SPLATCT_OK;
}

int splatct_cone_fill(const double* cos_t, const double* sin_t, int m, int nu, double su,
                      double rs, double rd, int w, int h, double step, const int64_t* rptr,
                      void* samples, void* stream) {
    cudaStream_t s = as_stream(stream);
    const int nr = m * nu;
    ConeGeom g{cos_t, sin_t, m, nu, su, step, rs, rd, w, h};
    k_cone_fill<<<(nr + 127) / 128, 128, 0, s>>>(g, rptr, reinterpret_cast<ConeSample*>(samples));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_cone_entry_count(const void* samples, const int64_t* rptr, int nrays, int w, int h,
                             int64_t* eptr, void* scratch, size_t scratch_bytes,
                             int64_t* nentries, void* stream) {
    const int64_t np = (int64_t)w * h;
    SPLATCT_REQUIRE(scratch_bytes >= align_up(sizeof(int64_t) * (np + 1)) * 2 +
                                          scan_temp_bytes(np + 1),
                    "cone entry scratch too small");
    cudaStream_t s = as_stream(stream);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(scratch);
    void* tmp = (char*)scratch + 2 * align_up(sizeof(int64_t) * (np + 1));
    SPLATCT_CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (np + 1), s));
    k_cone_ecount<<<(nrays + 127) / 128, 128, 0, s>>>(
        reinterpret_cast<const ConeSample*>(samples), rptr, nrays, w, h, cnt);
    SPLATCT_LAUNCH_CK();
    if (int e = exclusive_scan_i64(reinterpret_cast<int64_t*>(cnt), eptr, np + 1, tmp, s))
        return e;
    SPLATCT_CK(cudaMemcpyAsync(nentries, eptr + np, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    return SPLATCT_OK;
}

int splatct_cone_entry_scratch_bytes(int64_t nentries, int w, int h, size_t* bytes) {
    const int64_t np = (int64_t)w * h;
    *bytes = align_up(sizeof(ConeEntry) * (size_t)(nentries > 0 ? nentries : 1)) +
             align_up(sizeof(uint64_t) * (size_t)(nentries > 0 ? nentries : 1)) +
             align_up(sizeof(unsigned long long) * (np + 1));
    return SPLATCT_OK;
}

int splatct_cone_entry_fill(const void* samples, const int64_t* rptr, int nrays, int w, int h,
                            const int64_t* eptr, int64_t nentries, void* entries, void* scratch,
                            size_t scratch_bytes, void* stream) {
    size_t need = 0;
    splatct_cone_entry_scratch_bytes(nentries, w, h, &need);
    SPLATCT_REQUIRE(scratch_bytes >= need, "cone entry scratch too small");
    cudaStream_t s = as_stream(stream);
    const int64_t np = (int64_t)w * h;
    const size_t n1 = nentries > 0 ? nentries : 1;
    ConeEntry* tmpE = reinterpret_cast<ConeEntry*>(scratch);
    uint64_t* key = reinterpret_cast<uint64_t*>((char*)scratch + align_up(sizeof(ConeEntry) * n1));
    unsigned long long* cursor = reinterpret_cast<unsigned long long*>(
        (char*)scratch + align_up(sizeof(ConeEntry) * n1) + align_up(sizeof(uint64_t) * n1));
    SPLATCT_CK(cudaMemcpyAsync(cursor, eptr, sizeof(int64_t) * (np + 1), cudaMemcpyDeviceToDevice,
                               s));
    k_cone_efill<<<(nrays + 127) / 128, 128, 0, s>>>(reinterpret_cast<const ConeSample*>(samples),
                                                     rptr, nrays, w, h, cursor, tmpE, key);
    SPLATCT_LAUNCH_CK();
    k_cone_esort<<<(unsigned)((np * 32 + 255) / 256), 256, 0, s>>>(
        np, eptr, tmpE, key, reinterpret_cast<ConeEntry*>(entries));
    SPLATCT_LAUNCH_CK();
    SPLATCT_CK(cudaStreamSynchronize(s));   // scratch may be freed by the caller after return
    return SPLATCT_OK;
}

int splatct_cone_forward(const void* samples, const int64_t* rptr, const float* invL, int nrays,
                         int nv, double sv, double step, int w, int h, int c_local, double zc,
                         const float* vol_yxz, float* sino, const int* halt, void* stream) {
    SPLATCT_REQUIRE(nrays >= 0 && nv > 0 && c_local > 0, "invalid cone forward sizes");
    const int64_t warps = (int64_t)nrays * ((nv + 31) / 32);
    if (warps == 0) return SPLATCT_OK;
    k_cone_fwd<<<(unsigned)((warps + CONE_WARPS - 1) / CONE_WARPS), 32 * CONE_WARPS, 0,
                 as_stream(stream)>>>(reinterpret_cast<const ConeSample*>(samples), rptr, invL,
                                      nrays, nv, (float)sv, (float)step, w, h, c_local,
                                      (float)zc, vol_yxz, sino, halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_cone_adjoint(const void* entries, const int64_t* eptr, const float* invL, int nrays,
                         int nv, double sv, double step, int w, int h, int c_local, double zc,
                         const float* gsino, float* gscaled, float* out_yxz, int accumulate,
                         const int* halt, void* stream) {
    SPLATCT_REQUIRE(nv > 0 && c_local > 0 && w > 0 && h > 0, "invalid cone adjoint sizes");
    cudaStream_t s = as_stream(stream);
    const int64_t ng = (int64_t)nrays * nv;
    if (ng > 0) {
        k_cone_gscale<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(gsino, invL, nrays, nv,
                                                                   (float)sv, (float)step,
                                                                   gscaled, halt);
        SPLATCT_LAUNCH_CK();
    }
    const int64_t np = (int64_t)w * h;
    const int64_t warps = np * ((c_local + 31) / 32);
    k_cone_adj<<<(unsigned)((warps + CONE_WARPS - 1) / CONE_WARPS), 32 * CONE_WARPS, 0, s>>>(
        reinterpret_cast<const ConeEntry*>(entries), eptr, np, nv, (float)sv, c_local,
        (float)zc, gscaled, out_yxz, accumulate, halt);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
