// fbp.cu -- filtered back projection used once to initialise the cloud
// (projector.fbp, projector.py:154-206; optim.init_cloud_fbp optim.py:158-200).
// Not on the per-iteration path.  Rows are filtered by direct convolution
// with the real-space kernel of the zero-padded FFT ramp filter (exactly the
// circular convolution _filter_rows performs, projector.py:134-141; the
// kernel itself is built on the host from _ramp_response), then
// back-projected pixel-driven (_kernels.py:360-419), all slices of a pixel
// column handled by consecutive threads.
#include "common.cuh"

namespace splatct {

// filtered[v][i][z] = sum_j kernel[i - j + n - 1] * det_weight[j] * sino[v][j][z]
__global__ void k_fbp_filter(const float* __restrict__ sino, int m, int n, int p,
                             const double* __restrict__ kern, const double* __restrict__ wdet,
                             double* __restrict__ out) {
    const int z = blockIdx.x * 32 + (threadIdx.x & 31);
    const int i = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int v = blockIdx.z;
    if (z >= p || i >= n) return;
    const float* row = sino + (int64_t)v * n * p + z;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
        double x = (double)row[(int64_t)j * p];
        if (wdet) x *= wdet[j];
        acc += kern[i - j + n - 1] * x;
    }
    out[((int64_t)v * n + i) * p + z] = acc;
}

__global__ void k_fbp_bp(const double* __restrict__ F, const double* __restrict__ cos_t,
                         const double* __restrict__ sin_t, int m, int n, int p, int w, int h,
                         double spacing, double dbeta, int is_fan, double rs,
                         float* __restrict__ out) {
    const int z = blockIdx.x * 32 + (threadIdx.x & 31);
    const int64_t pix = blockIdx.y * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (z >= p || pix >= (int64_t)w * h) return;
    const int y = (int)(pix / w), x = (int)(pix % w);
    const double cx = 0.5 * (w - 1), cy = 0.5 * (h - 1);
    const double rx = x - cx, ry = y - cy;
    const double u0 = -0.5 * (n - 1) * spacing;
    double acc = 0.0;
    for (int v = 0; v < m; ++v) {
        const double c = cos_t[v], s = sin_t[v];
        double q, wgt = 1.0;
        if (is_fan) {
            const double along = rs + rx * c + ry * s;
            if (along <= 1e-6) continue;
            const double u_iso = rs * (-rx * s + ry * c) / along;
            q = (u_iso - u0) / spacing;
            wgt = (rs * rs) / (along * along);
        } else {
            const double u = -rx * s + ry * c;
            q = (u - u0) / spacing;
        }
        const int j = (int)floor(q);
        if (j < 0 || j >= n - 1) continue;
        const double f = q - j;
        const double* row = F + (int64_t)v * n * p + z;
        const double val = (1 - f) * row[(int64_t)j * p] + f * row[(int64_t)(j + 1) * p];
        acc += is_fan ? val * wgt : val;
    }
    out[pix * p + z] = (float)(acc * dbeta);
}

}  // namespace splatct

using namespace splatct;

extern "C" {

int splatct_fbp_filter(const float* sino, int m, int n, int p, const double* kernel,
                       const double* det_weight, double* filtered, void* stream) {
    SPLATCT_REQUIRE(m > 0 && n > 0 && p > 0, "invalid sizes");
    dim3 grid((p + 31) / 32, (n + 7) / 8, m);
    k_fbp_filter<<<grid, 256, 0, as_stream(stream)>>>(sino, m, n, p, kernel, det_weight, filtered);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

int splatct_fbp_backproject(const double* filtered, const double* cos_t, const double* sin_t,
                            int m, int n, int p, int w, int h, double spacing, double dbeta,
                            int is_fan, double rs, float* out_yxz, void* stream) {
    SPLATCT_REQUIRE(m > 0 && n > 0 && p > 0 && w > 0 && h > 0, "invalid sizes");
    const int64_t pix = (int64_t)w * h;
    dim3 grid((p + 31) / 32, (unsigned)((pix + 7) / 8));
    k_fbp_bp<<<grid, 256, 0, as_stream(stream)>>>(filtered, cos_t, sin_t, m, n, p, w, h, spacing,
                                                  dbeta, is_fan, rs, out_yxz);
    SPLATCT_LAUNCH_CK();
    return SPLATCT_OK;
}

}  // extern "C"
