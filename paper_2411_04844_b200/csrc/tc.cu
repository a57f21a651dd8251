// tc.cu -- self-test of the tcgen05 conventions in tc.cuh (TMEM layouts of A
// and D, the K-major no-swizzle B descriptor, the TF32 instruction
// descriptor, commit -> mbarrier).  One CTA computes D = A B^T for
// A [128 x 8], B [16 x 8] (row-major f32 inputs, D [128 x 16] out):
//   mode 0: one TF32 MMA on the inputs as given;
//   mode 1: the 3xTF32 split the voxelizer uses, hi = x & ~0x1fff,
//           lo = x - hi: D = Ahi Bhi + Ahi Blo + Alo Bhi (fp32-level result).
#include "common.cuh"
#include "tc.cuh"

namespace splatct {

__global__ void __launch_bounds__(128) k_tc_selftest(const float* __restrict__ A,
                                                    const float* __restrict__ B,
                                                    float* __restrict__ D, int mode) {
    __shared__ __align__(128) uint32_t sb[2][16 * 8];   // B hi / lo, canonical K-major
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 64);
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::mbar_init_fence();
    }
    // B: element (n, k) at byte (n % 8) * 16 + (n / 8) * 128 + (k / 4) * 256 + (k % 4) * 4
    {
        const int n = tid >> 3, k = tid & 7;   // 128 threads = 16 x 8 elements
        const float v = B[n * 8 + k];
        const uint32_t hi = mode ? (__float_as_uint(v) & 0xffffe000u) : __float_as_uint(v);
        const uint32_t lo = __float_as_uint(v - __uint_as_float(hi));
        const int off = ((n & 7) * 16 + (n >> 3) * 128 + (k >> 2) * 256 + (k & 3) * 4) / 4;
        sb[0][off] = hi;
        sb[1][off] = lo;
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t t0 = tbase;
    // TMEM columns: D at 0..15, A hi at 32..39, A lo at 40..47
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    {
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float v = A[tid * 8 + k];
            hi[k] = mode ? (__float_as_uint(v) & 0xffffe000u) : __float_as_uint(v);
            lo[k] = __float_as_uint(v - __uint_as_float(hi[k]));
        }
        tc::st_x8(t0 + lane_base + 32, hi);
        tc::st_x8(t0 + lane_base + 40, lo);
        tc::wait_st();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (mode >= 2) {   // timing: `mode` MMAs (M128 N16 K8), 1 or 2 accumulators
        if (tid == 0) {
            const uint32_t id = tc::idesc_tf32(128, 16);
            const uint64_t bh = tc::smem_desc(tc::smem_u32(sb[0]), 256, 128);
            const long long c0 = clock64();
            for (int i = 0; i < mode; ++i)
                tc::mma_tf32_ts(t0 + (A[0] > 100.f ? 16 * (i & 1) : 0), t0 + 32, bh, id, i > 1);
            tc::commit(&bar);
            tc::mbar_wait(&bar, 0);
            const long long c1 = clock64();
            D[0] = (float)(c1 - c0);
        }
        __syncthreads();
        if (warp == 0) tc::tmem_free(t0, 64);
        return;
    }
    if (tid == 0) {
        const uint32_t id = tc::idesc_tf32(128, 16);
        const uint64_t bh = tc::smem_desc(tc::smem_u32(sb[0]), 256, 128);
        const uint64_t bl = tc::smem_desc(tc::smem_u32(sb[1]), 256, 128);
        if (mode == 0) {
            tc::mma_tf32_ts(t0, t0 + 32, bh, id, 0);
        } else {   // small terms first
            tc::mma_tf32_ts(t0, t0 + 40, bh, id, 0);
            tc::mma_tf32_ts(t0, t0 + 32, bl, id, 1);
            tc::mma_tf32_ts(t0, t0 + 32, bh, id, 1);
        }
        tc::commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after();
    uint32_t d[16];
    tc::ld_x16(t0 + lane_base, d);
    tc::wait_ld();
#pragma unroll
    for (int n = 0; n < 16; ++n) D[tid * 16 + n] = __uint_as_float(d[n]);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free(t0, 64);
}

}  // namespace splatct

using namespace splatct;

extern "C" int splatct_tc_selftest(const float* a, const float* b, float* d, int mode,
                                   void* stream) {
    k_tc_selftest<<<1, 128, 0, as_stream(stream)>>>(a, b, d, mode);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}
