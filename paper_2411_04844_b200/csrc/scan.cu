// scan.cu -- device-wide exclusive scans and fixed-order reductions, plus the
// C-ABI error plumbing.  Used by the voxelizer's radix sort / tile offsets
// and by the projector's CSR construction.
#include <atomic>

#include "common.cuh"

#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

namespace splatct {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error_msg(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

constexpr int SCAN_NT = 256;
constexpr int SCAN_PER_THREAD = 16;
constexpr int64_t SCAN_CHUNK = SCAN_NT * SCAN_PER_THREAD;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Exclusive block scan of one value per thread; returns the exclusive prefix
// and writes the block total to *total.
template <typename T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T s = lane < NT / 32 ? sh[lane] : T(0);
        s = warp_incl_scan(s);
        if (lane < NT / 32) sh[lane] = s;
    }
    __syncthreads();
    T wprefix = wid > 0 ? sh[wid - 1] : T(0);
    *total = sh[NT / 32 - 1];
    __syncthreads();
    return wprefix + inc - v;
}

size_t scan_temp_bytes(int64_t n) {
    int64_t nb = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
    return align_up((size_t)(nb > 0 ? nb : 1) * sizeof(int64_t)) + 256;   // + tile counter
}

// Single-pass scan with decoupled look-back: each CTA takes the next tile id
// from a counter (so predecessors are always already running), publishes its
// aggregate, then walks back over predecessors' aggregates until one
// publishes an inclusive prefix.  Status words: 2-bit flag | 62-bit value
// (the scanned arrays are non-negative counts).
constexpr unsigned long long ST_A = 1ull << 62, ST_P = 2ull << 62, ST_V = ST_A - 1;

template <typename T>
__global__ void __launch_bounds__(SCAN_NT) k_scan_lookback(const T* __restrict__ in,
                                                           T* __restrict__ out, int64_t n,
                                                           unsigned long long* status,
                                                           unsigned int* counter) {
    __shared__ T sh[SCAN_NT / 32];
    __shared__ unsigned int s_tile;
    __shared__ T s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SCAN_CHUNK + (int64_t)threadIdx.x * SCAN_PER_THREAD;
    T v[SCAN_PER_THREAD];
    T acc = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        v[k] = base + k < n ? in[base + k] : T(0);
        acc += v[k];
    }
    T tot;
    T off = block_excl_scan<T, SCAN_NT>(acc, sh, &tot);
    if (threadIdx.x == 0) {
        T excl = 0;
        if (tile == 0) {
            atomicExch(&status[0], ST_P | (unsigned long long)tot);
        } else {
            atomicExch(&status[tile], ST_A | (unsigned long long)tot);
            for (int64_t pred = tile - 1;; --pred) {
                unsigned long long st;
                do {
                    st = atomicAdd(&status[pred], 0ull);
                } while ((st >> 62) == 0);
                excl += (T)(st & ST_V);
                if ((st >> 62) == 2) break;
            }
            atomicExch(&status[tile], ST_P | (unsigned long long)(excl + tot));
        }
        s_excl = excl;
    }
    __syncthreads();
    off += s_excl;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        if (base + k < n) out[base + k] = off;
        off += v[k];
    }
}

// Whole array in one CTA (n <= SMALL_SCAN): one launch instead of three.
constexpr int64_t SMALL_SCAN = 1 << 13;

template <typename T>
__global__ void __launch_bounds__(1024) k_scan_small(const T* __restrict__ in, T* __restrict__ out,
                                                     int64_t n) {
    __shared__ T sh[32];
    const int64_t per = (n + 1023) / 1024;
    const int64_t beg = threadIdx.x * per;
    const int64_t end = beg + per < n ? beg + per : n;
    T acc = 0;
    for (int64_t i = beg; i < end; ++i) acc += in[i];
    T tot;
    T off = block_excl_scan<T, 1024>(acc, sh, &tot);
    for (int64_t i = beg; i < end; ++i) {
        const T v = in[i];
        out[i] = off;
        off += v;
    }
}

template <typename T>
static int exclusive_scan(const T* in, T* out, int64_t n, void* temp, cudaStream_t s) {
    if (n <= 0) return SPLATCT_OK;
    if (n <= SMALL_SCAN) {
        k_scan_small<T><<<1, 1024, 0, s>>>(in, out, n);
        SPLATCT_LAUNCH_CK();
        return SPLATCT_OK;
    }
    const int64_t nb = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(temp);
    unsigned int* counter = reinterpret_cast<unsigned int*>(
        reinterpret_cast<char*>(temp) + align_up((size_t)nb * sizeof(int64_t)));
    SPLATCT_CK(cudaMemsetAsync(temp, 0, align_up((size_t)nb * sizeof(int64_t)) + 256, s));
    k_scan_lookback<T><<<(unsigned)nb, SCAN_NT, 0, s>>>(in, out, n, status, counter);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* temp, cudaStream_t s) {
    return exclusive_scan<int64_t>(in, out, n, temp, s);
}
int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* temp,
                       cudaStream_t s) {
    return exclusive_scan<uint32_t>(in, out, n, temp, s);
}

__global__ void __launch_bounds__(1024) k_reduce_sum(const double* __restrict__ in, int64_t n,
                                                     double* __restrict__ out) {
    griddep_wait();
    __shared__ double sh[32];
    // 8 independent loads in flight per thread (a fixed order: deterministic);
    // the strided single loop was latency-bound (~17 us for the C2 TV partials)
    const double r = block_reduce_f64(in, n, sh);
    if (threadIdx.x == 0) out[0] = r;
}

int reduce_sum_f64(const double* in, int64_t n, double* out, cudaStream_t s) {
    SPLATCT_CK(launch_pdl(k_reduce_sum, dim3(1), dim3(1024), 0, s, in, n, out));
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // namespace splatct

extern "C" {

int splatct_abi_version(void) { return SPLATCT_ABI_VERSION; }

const char* splatct_last_error(void) { return splatct::g_err; }

unsigned long long splatct_launch_count(void) { return splatct::g_launches.load(); }

int splatct_reduce_sum(const double* in, int64_t n, double* out, void* stream) {
    return splatct::reduce_sum_f64(in, n, out, splatct::as_stream(stream));
}

// Host copy into page-locked staging memory with non-temporal stores: the
// lines go to DRAM instead of staying dirty in the CPU caches, so the DMA
// that follows reads them without snooping (SPLATCT_STAGE_NT=0: memcpy).
static void stage_copy(char* dst, const char* src, size_t len, bool nt) {
#if defined(__x86_64__)
    if (nt && ((uintptr_t)dst & 15) == 0) {
        size_t i = 0;
        for (; i + 64 <= len; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
            const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
        }
        if (i < len) memcpy(dst + i, src + i, len - i);
        _mm_sfence();
        return;
    }
#endif
    (void)nt;
    memcpy(dst, src, len);
}

int splatct_stage_upload(void* dst, const void* src, void* pinned, size_t bytes, int nthreads,
                         void* stream) {
    // nthreads host threads each copy one slice into the page-locked buffer
    // and queue that slice's DMA at once, so the copies and the DMAs overlap
    SPLATCT_REQUIRE(dst && src && pinned, "null pointer");
    if (bytes == 0) return SPLATCT_OK;
    const int k = nthreads < 1 ? 1 : (nthreads > 32 ? 32 : nthreads);
    const size_t slice = ((bytes + k - 1) / k + 4095) & ~(size_t)4095;
    cudaStream_t s = splatct::as_stream(stream);
    const char* env = getenv("SPLATCT_STAGE_NT");
    const bool nt = !(env && !strcmp(env, "0"));
    std::vector<std::thread> th;
    std::vector<cudaError_t> err(k, cudaSuccess);
    for (int i = 0; i < k; ++i) {
        const size_t off = (size_t)i * slice;
        if (off >= bytes) break;
        const size_t len = bytes - off < slice ? bytes - off : slice;
        th.emplace_back([=, &err]() {
            stage_copy(static_cast<char*>(pinned) + off, static_cast<const char*>(src) + off, len,
                       nt);
            err[i] = cudaMemcpyAsync(static_cast<char*>(dst) + off,
                                     static_cast<const char*>(pinned) + off, len,
                                     cudaMemcpyHostToDevice, s);
        });
    }
    for (auto& t : th) t.join();
    for (int i = 0; i < k; ++i) SPLATCT_CK(err[i]);
    return SPLATCT_OK;
}

}  // extern "C"
