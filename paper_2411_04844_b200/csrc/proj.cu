// proj.cu -- per-slice parallel/fan projector and its exact adjoint on B200.
//
// Reference (/root/reference/pkg/src/splatct/_kernels.py):
//   _clip_ray      :208-229   ray vs bilinear support box [-1,w] x [-1,h]
//   _ray_geometry  :232-259   origin, unit direction, [t0,t1] (f64)
//   project_forward:262-303   n_steps = int((t1-t0)/step); sample k at
//                             t0+(k+1/2)step; 4 bilinear taps with per-tap
//                             bounds checks; * step
//   project_adjoint:306-357   the same samples scattered with the same weights
//
// B200 design: the geometry is identical for every
// slice, so the f64 ray march is done ONCE per geometry and its sample
// weights are merged per (ray, pixel) into a CSR operator A (ray-major) and
// its exact transpose A^T (pixel-major, rows sorted by ray id).  Every
// iteration then is a CSR x (pixel-column z-vectors) product: one warp per
// row, the row's (index, weight) pairs broadcast by shuffles, 16-byte
// vector loads of contiguous z-vectors (yxz volume / (m,n,p) sinogram), all
// slices of the z-slab handled by one weight fetch.  The adjoint also fuses
// the TV subgradient and TV value of loss.tv_loss (loss.py:183-207).
#include <stdlib.h>

#include "common.cuh"
#include "raygeom.cuh"

namespace splatct {

// The march is one sequential f64 chain per ray: a thread per ray leaves
// ~5 warps per SM at C2.  It runs as PSEG segments per ray (march_ray_seg),
// a thread each; segment (r, s) is CSR sub-row r * PSEG + s, so a ray's
// entries are its segments' in order (SPLATCT_MARCH_SEGMENTS=1: whole rays).
constexpr int PSEG = 16;

static int march_segments() {
    const char* e = getenv("SPLATCT_MARCH_SEGMENTS");
    const int n = e ? atoi(e) : PSEG;
    return n < 1 ? 1 : (n > PSEG ? PSEG : n);
}

__global__ void k_proj_count(Geom g, int nseg, int64_t* __restrict__ cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)g.m * g.n_det * nseg) return;
    int64_t c = 0;
    march_ray_seg(g, (int)(i / nseg), (int)(i % nseg), nseg, [&](int, double, double) { ++c; });
    cnt[i] = c;
}

__global__ void k_proj_fill(Geom g, int nseg, const int64_t* __restrict__ sub_ptr,
                            int32_t* __restrict__ a_col, float* __restrict__ a_val) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)g.m * g.n_det * nseg) return;
    int64_t j = sub_ptr[i];
    const double step = g.step;
    march_ray_seg(g, (int)(i / nseg), (int)(i % nseg), nseg, [&](int pix, double w, double) {
        a_col[j] = pix;
        a_val[j] = (float)(step * w);
        ++j;
    });
}

// a_ptr[r] = sub_ptr[r * nseg] (r = 0 .. rays)
__global__ void k_ray_ptr(const int64_t* __restrict__ sub_ptr, int rays, int nseg,
                          int64_t* __restrict__ a_ptr) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r <= rays) a_ptr[r] = sub_ptr[(int64_t)r * nseg];
}

__global__ void k_col_count(const int32_t* __restrict__ a_col, int64_t nnz,
                            unsigned long long* __restrict__ cnt) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < nnz) atomicAdd(&cnt[a_col[j]], 1ull);
}

// warp per ray (the slot order inside a pixel row is arbitrary: k_row_sort
// orders it by ray next)
__global__ void k_transpose_fill(int n_rays, const int64_t* __restrict__ a_ptr,
                                 const int32_t* __restrict__ a_col, const float* __restrict__ a_val,
                                 unsigned long long* __restrict__ cursor,
                                 int32_t* __restrict__ t_ray, float* __restrict__ t_val) {
    const int r = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (r >= n_rays) return;
    for (int64_t j = a_ptr[r] + (threadIdx.x & 31); j < a_ptr[r + 1]; j += 32) {
        const unsigned long long pos = atomicAdd(&cursor[a_col[j]], 1ull);
        t_ray[pos] = r;
        t_val[pos] = a_val[j];
    }
}

// Warp per pixel row: rank sort of the (ray, weight) pairs by ray id (ray
// ids within a row are distinct, so ranks are a permutation).
__global__ void k_row_sort(int64_t nrows, const int64_t* __restrict__ ptr,
                           const int32_t* __restrict__ in_ray, const float* __restrict__ in_val,
                           int32_t* __restrict__ out_ray, float* __restrict__ out_val) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= nrows) return;
    const int64_t b = ptr[row], e = ptr[row + 1];
    for (int64_t i = b + lane; i < e; i += 32) {
        const int32_t key = in_ray[i];
        int64_t rank = 0;
        for (int64_t j = b; j < e; ++j) rank += in_ray[j] < key;
        out_ray[b + rank] = key;
        out_val[b + rank] = in_val[i];
    }
}

// ---------------------------------------------------------------------------
// CSR x z-vectors.  Warp per row; lane covers V consecutive slices per chunk,
// NCH chunks of 32*V slices starting at zoff.
// ---------------------------------------------------------------------------
template <int V>
struct VecT;
template <>
struct VecT<1> { using T = float; };
template <>
struct VecT<2> { using T = float2; };
template <>
struct VecT<4> { using T = float4; };

template <int V>
__device__ __forceinline__ void ldv(const float* p, float (&o)[V]) {
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
__device__ __forceinline__ void stv(float* p, const float (&o)[V]) {
    if constexpr (V == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
    } else {
        p[0] = o[0];
    }
}

struct TvArgs {
    const float* vol;      // yxz, local slab
    const float* halo_lo;  // plane z = -1 ([h*w]) or null
    const float* halo_hi;  // plane z = c ([h*w]) or null
    double coef;           // lambda_tv / tv_count
    double* partial;       // per-row sum |forward diffs| (or null)
    int w, h;
};

__device__ __forceinline__ float tv_at(const TvArgs& a, int64_t row, int z, int c, float v0,
                                       double& tvsum) {
    const int y = (int)(row / a.w), x = (int)(row % a.w);
    const float* vol = a.vol;
    int g = 0;
    auto sgn = [](float d) { return (d > 0.f) - (d < 0.f); };
    if (x + 1 < a.w) {
        const float v1 = __ldg(vol + (row + 1) * c + z);
        tvsum += fabs((double)v1 - (double)v0);
        g -= sgn(v1 - v0);
    }
    if (x > 0) g += sgn(v0 - __ldg(vol + (row - 1) * c + z));
    if (y + 1 < a.h) {
        const float v1 = __ldg(vol + (row + a.w) * c + z);
        tvsum += fabs((double)v1 - (double)v0);
        g -= sgn(v1 - v0);
    }
    if (y > 0) g += sgn(v0 - __ldg(vol + (row - a.w) * c + z));
    const float* zn = nullptr;
    if (z + 1 < c) zn = vol + row * c + z + 1;
    else if (a.halo_hi) zn = a.halo_hi + row;
    if (zn) {
        const float v1 = __ldg(zn);
        tvsum += fabs((double)v1 - (double)v0);
        g -= sgn(v1 - v0);
    }
    const float* zp = nullptr;
    if (z > 0) zp = vol + row * c + z - 1;
    else if (a.halo_lo) zp = a.halo_lo + row;
    if (zp) g += sgn(v0 - __ldg(zp));
    return (float)g;
}

template <int V, int NCH, bool TV>
__global__ void __launch_bounds__(256) k_csr_spmm(const int64_t* __restrict__ ptr,
                                                  const int32_t* __restrict__ col,
                                                  const float* __restrict__ val, int64_t nrows,
                                                  const float* __restrict__ X,
                                                  float* __restrict__ Y, int c, int zoff,
                                                  TvArgs tv, const int* halt) {
    if (halted(halt)) return;
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= nrows) return;
    float acc[NCH][V];
#pragma unroll
    for (int q = 0; q < NCH; ++q)
#pragma unroll
        for (int e = 0; e < V; ++e) acc[q][e] = 0.f;
    bool zok[NCH];
    int zb[NCH];
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        zb[q] = zoff + q * 32 * V + lane * V;
        zok[q] = zb[q] < c;   // c % V == 0 by construction
    }
    const int64_t b = ptr[row], e = ptr[row + 1];
    for (int64_t j0 = b; j0 < e; j0 += 32) {
        const int64_t jl = j0 + lane;
        const int cl = jl < e ? __ldg(col + jl) : 0;
        const float vl = jl < e ? __ldg(val + jl) : 0.f;
        const int cnt = (int)min((int64_t)32, e - j0);
        int jj = 0;
        for (; jj + 4 <= cnt; jj += 4) {
            int p[4];
            float wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                p[u] = __shfl_sync(0xffffffffu, cl, jj + u);
                wv[u] = __shfl_sync(0xffffffffu, vl, jj + u);
            }
            float x[4][NCH][V];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < NCH; ++q) {
                    if (zok[q]) ldv<V>(X + (int64_t)p[u] * c + zb[q], x[u][q]);
                    else
#pragma unroll
                        for (int t = 0; t < V; ++t) x[u][q][t] = 0.f;
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < NCH; ++q)
#pragma unroll
                    for (int t = 0; t < V; ++t) acc[q][t] = fmaf(wv[u], x[u][q][t], acc[q][t]);
        }
        for (; jj < cnt; ++jj) {
            const int p = __shfl_sync(0xffffffffu, cl, jj);
            const float wv = __shfl_sync(0xffffffffu, vl, jj);
#pragma unroll
            for (int q = 0; q < NCH; ++q) {
                if (!zok[q]) continue;
                float x[V];
                ldv<V>(X + (int64_t)p * c + zb[q], x);
#pragma unroll
                for (int t = 0; t < V; ++t) acc[q][t] = fmaf(wv, x[t], acc[q][t]);
            }
        }
    }
    double tvsum = 0.0;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        if (!zok[q]) continue;
        float o[V];
#pragma unroll
        for (int t = 0; t < V; ++t) {
            if constexpr (TV) {
                const float v0 = __ldg(tv.vol + row * c + zb[q] + t);
                const float gt = tv_at(tv, row, zb[q] + t, c, v0, tvsum);
                o[t] = (float)fma((double)gt, tv.coef, (double)acc[q][t]);
            } else {
                o[t] = acc[q][t];
            }
        }
        stv<V>(Y + row * c + zb[q], o);
    }
    if constexpr (TV) {
        if (tv.partial) {
            tvsum = warp_sum(tvsum);
            if (lane == 0) {
                if (zoff == 0) tv.partial[row] = tvsum;
                else tv.partial[row] += tvsum;
            }
        }
    }
}

template <int V, bool TV>
static int launch_spmm_v(const int64_t* ptr, const int32_t* col, const float* val, int64_t nrows,
                         const float* X, float* Y, int c, const TvArgs& tv, const int* halt,
                         cudaStream_t s) {
    const unsigned grid = (unsigned)((nrows + 7) / 8);
    const int per_chunk = 32 * V;
    int zoff = 0;
    while (zoff < c) {
        const int rem = c - zoff;
        if (rem > 2 * per_chunk) {
            k_csr_spmm<V, 4, TV><<<grid, 256, 0, s>>>(ptr, col, val, nrows, X, Y, c, zoff, tv, halt);
            zoff += 4 * per_chunk;
        } else if (rem > per_chunk) {
            k_csr_spmm<V, 2, TV><<<grid, 256, 0, s>>>(ptr, col, val, nrows, X, Y, c, zoff, tv, halt);
            zoff += 2 * per_chunk;
        } else {
            k_csr_spmm<V, 1, TV><<<grid, 256, 0, s>>>(ptr, col, val, nrows, X, Y, c, zoff, tv, halt);
            zoff += per_chunk;
        }
        SPLATCT_LAUNCH_CK();
    }
    return SPLATCT_OK;
}

template <bool TV>
static int launch_spmm(const int64_t* ptr, const int32_t* col, const float* val, int64_t nrows,
                       const float* X, float* Y, int c, const TvArgs& tv, const int* halt,
                       cudaStream_t s) {
    const bool al16 = ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
    const bool al8 = ((uintptr_t)X % 8 == 0) && ((uintptr_t)Y % 8 == 0);
    // V = 4 wants >= 128 slices per chunk to keep lanes busy; small slabs use V = 2/1.
    if (c % 4 == 0 && al16 && c >= 128) return launch_spmm_v<4, TV>(ptr, col, val, nrows, X, Y, c, tv, halt, s);
    if (c % 2 == 0 && al8 && c >= 64) return launch_spmm_v<2, TV>(ptr, col, val, nrows, X, Y, c, tv, halt, s);
    return launch_spmm_v<1, TV>(ptr, col, val, nrows, X, Y, c, tv, halt, s);
}

// ---------------------------------------------------------------------------
// Direct ray-marching forward projection (no matrix): warp per ray, lanes
// over slices, the same f64 sample enumeration as _kernels.py:284-303.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_march_fwd(Geom g, int c, const float* __restrict__ vol,
                                                   float* __restrict__ sino) {
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= g.m * g.n_det) return;
    const int v = r / g.n_det, d = r % g.n_det;
    const double cx = 0.5 * (g.w - 1), cy = 0.5 * (g.h - 1);
    const double u = (d - 0.5 * (g.n_det - 1)) * g.spacing;
    double ox, oy, dx, dy, t0, t1;
    ray_geometry(g.cos_t[v], g.sin_t[v], u, g.is_fan, g.rs, g.rd, cx, cy, g.w, g.h, ox, oy, dx, dy,
                 t0, t1);
    const int64_t ns = t1 > t0 ? (int64_t)((t1 - t0) / g.step) : 0;
    for (int zb = 0; zb < c; zb += 32) {
        const int z = zb + lane;
        double acc = 0.0;
        for (int64_t k = 0; k < ns; ++k) {
            const double t = t0 + (k + 0.5) * g.step;
            const double sx = ox + t * dx, sy = oy + t * dy;
            const int64_t x0 = (int64_t)floor(sx), y0 = (int64_t)floor(sy);
            const double fx = sx - (double)x0, fy = sy - (double)y0;
            if (z < c) {
                auto tap = [&](int64_t xx, int64_t yy, double wgt) {
                    if (xx >= 0 && xx < g.w && yy >= 0 && yy < g.h)
                        acc += wgt * (double)__ldg(vol + (yy * g.w + xx) * c + z);
                };
                tap(x0, y0, (1 - fx) * (1 - fy));
                tap(x0 + 1, y0, fx * (1 - fy));
                tap(x0, y0 + 1, (1 - fx) * fy);
                tap(x0 + 1, y0 + 1, fx * fy);
            }
        }
        if (z < c) sino[(int64_t)r * c + z] = (float)(acc * g.step);
    }
}

static Geom make_geom(const double* cos_t, const double* sin_t, int m, int n_det, double spacing,
                      double step, int is_fan, double rs, double rd, int w, int h) {
    Geom g;
    g.cos_t = cos_t; g.sin_t = sin_t; g.m = m; g.n_det = n_det; g.spacing = spacing;
    g.step = step; g.is_fan = is_fan != 0; g.rs = rs; g.rd = rd; g.w = w; g.h = h;
    return g;
}

struct ProjScratch {
    size_t o_cnt, o_cursor, o_sub, o_scan, o_tray, o_tval, total;
};
static ProjScratch proj_scratch(int m, int n_det, int w, int h, int64_t nnz) {
    ProjScratch S{};
    const int64_t rays = (int64_t)m * n_det, pix = (int64_t)w * h;
    const int64_t big = rays > pix ? rays : pix;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += align_up(b > 0 ? b : 1); return o; };
    const int64_t nsub = rays * PSEG;   // march segments (sub-rows)
    const int64_t cnt_n = (big > nsub ? big : nsub) + 1;
    S.o_cnt = take(sizeof(int64_t) * cnt_n);
    S.o_cursor = take(sizeof(int64_t) * (pix + 1));
    S.o_sub = take(sizeof(int64_t) * (nsub + 1));
    S.o_scan = take(scan_temp_bytes(cnt_n));
    S.o_tray = take(sizeof(int32_t) * (size_t)nnz);
    S.o_tval = take(sizeof(float) * (size_t)nnz);
    S.total = off;
    return S;
}

// per-segment entry counts of the march -> exclusive offsets sub[0 .. rays * nseg]
static int march_offsets(const Geom& g, int nseg, const ProjScratch& S, void* scratch,
                         int64_t* sub, cudaStream_t s) {
    const int64_t nsub = (int64_t)g.m * g.n_det * nseg;
    int64_t* cnt = reinterpret_cast<int64_t*>((char*)scratch + S.o_cnt);
    SPLATCT_CK(cudaMemsetAsync(cnt + nsub, 0, sizeof(int64_t), s));
    k_proj_count<<<(unsigned)((nsub + 127) / 128), 128, 0, s>>>(g, nseg, cnt);
    SPLATCT_LAUNCH_CK();
    return exclusive_scan_i64(cnt, sub, nsub + 1, (char*)scratch + S.o_scan, s);
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_proj_scratch_bytes(int m, int n_det, int w, int h, int64_t nnz, size_t* bytes) {
    *bytes = proj_scratch(m, n_det, w, h, nnz).total;
    return SPLATCT_OK;
}

int splatct_proj_count(const double* cos_t, const double* sin_t, int m, int n_det,
                       double spacing, double step, int is_fan, double rs, double rd, int w,
                       int h, int64_t* a_ptr, void* scratch, size_t scratch_bytes,
                       int64_t* nnz, void* stream) {
    SPLATCT_REQUIRE(m > 0 && n_det > 0 && w > 0 && h > 0 && step > 0, "invalid projector sizes");
    ProjScratch S = proj_scratch(m, n_det, w, h, 0);
    SPLATCT_REQUIRE(scratch_bytes >= S.total, "projector scratch too small");
    cudaStream_t s = as_stream(stream);
    Geom g = make_geom(cos_t, sin_t, m, n_det, spacing, step, is_fan, rs, rd, w, h);
    const int rays = m * n_det;
    int64_t* sub = reinterpret_cast<int64_t*>((char*)scratch + S.o_sub);
    const int nseg = march_segments();
    if (int e = march_offsets(g, nseg, S, scratch, sub, s)) return e;
    k_ray_ptr<<<(rays + 1 + 255) / 256, 256, 0, s>>>(sub, rays, nseg, a_ptr);
    SPLATCT_LAUNCH_CK();
    SPLATCT_CK(cudaMemcpyAsync(nnz, a_ptr + rays, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    return SPLATCT_OK;
}

int splatct_proj_fill(const double* cos_t, const double* sin_t, int m, int n_det,
                      double spacing, double step, int is_fan, double rs, double rd, int w,
                      int h, const int64_t* a_ptr, int32_t* a_col, float* a_val,
                      int64_t* at_ptr, int32_t* at_ray, float* at_val, void* scratch,
                      size_t scratch_bytes, void* stream) {
    cudaStream_t s = as_stream(stream);
    const int rays = m * n_det;
    const int64_t pix = (int64_t)w * h;
    int64_t nnz = 0;
    SPLATCT_CK(cudaMemcpyAsync(&nnz, a_ptr + rays, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPLATCT_CK(cudaStreamSynchronize(s));
    ProjScratch S = proj_scratch(m, n_det, w, h, nnz);
    SPLATCT_REQUIRE(scratch_bytes >= S.total, "projector scratch too small (%zu < %zu)",
                    scratch_bytes, S.total);
    Geom g = make_geom(cos_t, sin_t, m, n_det, spacing, step, is_fan, rs, rd, w, h);
    // the segments' offsets again (the count's scratch is not kept), then the fill
    int64_t* sub = reinterpret_cast<int64_t*>((char*)scratch + S.o_sub);
    const int nseg = march_segments();
    if (int e = march_offsets(g, nseg, S, scratch, sub, s)) return e;
    const int64_t nsub = (int64_t)rays * nseg;
    k_proj_fill<<<(unsigned)((nsub + 127) / 128), 128, 0, s>>>(g, nseg, sub, a_col, a_val);
    SPLATCT_LAUNCH_CK();
    // transpose: per-pixel counts -> offsets -> scatter -> per-row sort by ray
    auto* cnt = reinterpret_cast<unsigned long long*>((char*)scratch + S.o_cnt);
    auto* cursor = reinterpret_cast<unsigned long long*>((char*)scratch + S.o_cursor);
    auto* tray = reinterpret_cast<int32_t*>((char*)scratch + S.o_tray);
    auto* tval = reinterpret_cast<float*>((char*)scratch + S.o_tval);
    SPLATCT_CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (pix + 1), s));
    if (nnz > 0) {
        k_col_count<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(a_col, nnz, cnt);
        SPLATCT_LAUNCH_CK();
    }
    if (int e = exclusive_scan_i64(reinterpret_cast<int64_t*>(cnt), at_ptr, pix + 1,
                                   (char*)scratch + S.o_scan, s))
        return e;
    SPLATCT_CK(cudaMemcpyAsync(cursor, at_ptr, sizeof(int64_t) * (pix + 1),
                               cudaMemcpyDeviceToDevice, s));
    k_transpose_fill<<<(unsigned)(((int64_t)rays * 32 + 255) / 256), 256, 0, s>>>(
        rays, a_ptr, a_col, a_val, cursor, tray, tval);
    SPLATCT_LAUNCH_CK();
    k_row_sort<<<(unsigned)((pix * 32 + 255) / 256), 256, 0, s>>>(pix, at_ptr, tray, tval, at_ray,
                                                                  at_val);
    SPLATCT_LAUNCH_CK();
    SPLATCT_CK(cudaStreamSynchronize(s));   // scratch may be freed by the caller after return
    return SPLATCT_OK;
}

int splatct_proj_forward(const int64_t* a_ptr, const int32_t* a_col, const float* a_val,
                         int n_rays, const float* vol_yxz, float* sino, int c,
                         const int* halt, void* stream) {
    SPLATCT_REQUIRE(n_rays >= 0 && c > 0, "invalid sizes");
    TvArgs tv{};
    return launch_spmm<false>(a_ptr, a_col, a_val, n_rays, vol_yxz, sino, c, tv, halt,
                              as_stream(stream));
}

int splatct_proj_adjoint(const int64_t* at_ptr, const int32_t* at_ray, const float* at_val,
                         int w, int h, int c, const float* gsino, const float* vol_yxz,
                         const float* halo_lo, const float* halo_hi, double lambda_tv,
                         double tv_count, float* out_yxz, double* tv_partial, const int* halt,
                         void* stream) {
    SPLATCT_REQUIRE(w > 0 && h > 0 && c > 0, "invalid sizes");
    TvArgs tv{};
    tv.vol = vol_yxz; tv.halo_lo = halo_lo; tv.halo_hi = halo_hi;
    tv.coef = tv_count > 0.0 ? lambda_tv / tv_count : 0.0;
    tv.partial = tv_partial; tv.w = w; tv.h = h;
    const int64_t pix = (int64_t)w * h;
    cudaStream_t s = as_stream(stream);
    if (vol_yxz != nullptr && lambda_tv > 0.0) {
        SPLATCT_REQUIRE(tv_count > 0.0, "tv_count must be positive");
        return launch_spmm<true>(at_ptr, at_ray, at_val, pix, gsino, out_yxz, c, tv, halt, s);
    }
    return launch_spmm<false>(at_ptr, at_ray, at_val, pix, gsino, out_yxz, c, tv, halt, s);
}

int splatct_proj_march_forward(const double* cos_t, const double* sin_t, int m, int n_det,
                               double spacing, double step, int is_fan, double rs, double rd,
                               int w, int h, int c, const float* vol_yxz, float* sino,
                               void* stream) {
    Geom g = make_geom(cos_t, sin_t, m, n_det, spacing, step, is_fan, rs, rd, w, h);
    const int rays = m * n_det;
    k_march_fwd<<<(rays + 7) / 8, 256, 0, as_stream(stream)>>>(g, c, vol_yxz, sino);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
