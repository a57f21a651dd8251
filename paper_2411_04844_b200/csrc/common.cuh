// common.cuh -- shared helpers for the splatct sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/splatct.h"

namespace splatct {

// Thread-local last-error message (the C-ABI's only global state).
void set_error_msg(const char* fmt, ...);

#define SPLATCT_CK(expr)                                                          \
    do {                                                                          \
        cudaError_t e_ = (expr);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            ::splatct::set_error_msg("%s:%d %s: %s", __FILE__, __LINE__, #expr,   \
                                     cudaGetErrorString(e_));                     \
            return SPLATCT_ERR_CUDA;                                              \
        }                                                                         \
    } while (0)

// Every kernel launch goes through SPLATCT_LAUNCH_CK, which also counts it
// (splatct_launch_count(): the evidence for bench.py's gpu_launches).
void count_launch();
#define SPLATCT_LAUNCH_CK()            \
    do {                               \
        ::splatct::count_launch();     \
        SPLATCT_CK(cudaGetLastError()); \
    } while (0)

#define SPLATCT_REQUIRE(cond, ...)                                                \
    do {                                                                          \
        if (!(cond)) {                                                            \
            ::splatct::set_error_msg(__VA_ARGS__);                                \
            return SPLATCT_ERR_INVALID;                                           \
        }                                                                         \
    } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: the training-step kernels are launched with
// programmatic stream serialization, so a kernel's CTAs are resident (and its
// launch latency hidden) while its predecessor drains; every such kernel
// starts with griddep_wait(), which returns once the predecessor grid has
// completed and its memory is visible (a no-op for an ordinary launch).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     cudaStream_t s, Args... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

static inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Early-out for kernels inside a training iteration once a non-finite loss
// has been recorded (mirrors optim.py:356-366 aborting before the update).
__device__ __forceinline__ bool halted(const int* halt) {
    return halt != nullptr && *(volatile const int*)halt != 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One Adam step of parameter element idx (row = idx / n: 3 = sigma, clamped to
// [sfloor, sceil]; 4 = intensity, >= 0), optim.py:109-144; shared by k_adam and
// the Adam-fused binning pass so both compute it identically.
__device__ __forceinline__ void adam_elem(double* __restrict__ P, const double* __restrict__ G,
                                          double* __restrict__ M1, double* __restrict__ M2,
                                          int64_t idx, int row, double lr, double bc1, double bc2,
                                          double sfloor, double sceil) {
    const double g = G[idx];
    const double m = 0.9 * M1[idx] + (1.0 - 0.9) * g;
    const double v = 0.999 * M2[idx] + (1.0 - 0.999) * g * g;
    double p = P[idx] - lr * (m / bc1) / (sqrt(v / bc2) + 1e-8);
    if (row == 3) p = fmin(fmax(p, sfloor), sceil);
    if (row == 4) p = fmax(p, 0.0);
    M1[idx] = m;
    M2[idx] = v;
    P[idx] = p;
}

// Block-wide sum of a double into lane 0 of warp 0 (deterministic order).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= NT/32 */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < NT / 32 ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// Sum of in[0, n) by one 1024-thread block, fixed order (8 independent
// accumulators per thread, then block_sum): bitwise the same wherever it runs.
__device__ __forceinline__ double block_reduce_f64(const double* __restrict__ in, int64_t n,
                                                   double* sh) {
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int64_t i = threadIdx.x;
    for (; i + 7 * 1024 < n; i += 8 * 1024) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] += in[i + k * 1024];
    }
    for (int k = 0; i < n; i += 1024, ++k) a[k & 7] += in[i];
    const double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    return block_sum<1024>(acc, sh);
}

// Packed FP32 FMA (sm_100 FFMA2): d = a * b + c on both halves; with b a
// broadcast scalar the compiler uses the .F32 operand form, so one issue slot
// does two FMAs.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
          "l"(*reinterpret_cast<const unsigned long long*>(&b)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}

// Device-wide exclusive scan helpers (scan.cu).
size_t scan_temp_bytes(int64_t n);
int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp, cudaStream_t s);
int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* temp, cudaStream_t s);

// Sum of n doubles in fixed order into out[0] (one CTA).
int reduce_sum_f64(const double* in, int64_t n, double* out, cudaStream_t s);

}  // namespace splatct
