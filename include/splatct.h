/*
 * splatct.h -- C ABI of libsplatct.so, the B200 (sm_100a) hot path of DGR
 * Fast Volume Reconstruction (arXiv 2411.04844).
 *
 * Every entry point is extern "C", takes plain device pointers, explicit
 * sizes and a CUDA stream (as void*), never allocates, never synchronises
 * (except the two *_count setup calls, which return a size to the host), and
 * returns 0 on success or a SPLATCT_ERR_* code; splatct_last_error() then
 * holds a thread-local message.  Validation of domain invariants stays in the
 * Python layer (as in the reference, fvr.py:123-139).
 *
 * Each function names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/splatct/).
 *
 * Device layouts (chosen for B200):
 *   params  double[5][n]  rows mu_x, mu_y, mu_z, sigma, intensity
 *           (GaussianCloud, core.py:211-235; kept in f64 like the reference
 *           so floor(mu) -- the footprint -- is bit-exact)
 *   grads   double[5][n]  d_mu_x, d_mu_y, d_mu_z, d_sigma, d_intensity
 *           (ParamGradients, core.py:278-303)
 *   volume  float[h][w][c]   "yxz": slice index fastest, i.e. one contiguous
 *           c-vector per (y, x) pixel column.  The reference's VolumeGrid is
 *           (c,h,w) x-fastest (core.py:9-11); the Python layer transposes at
 *           the API edge.
 *   sinogram float[m][n][p]  identical to the reference (core.py:12-13):
 *           one contiguous p-vector per (view, detector) ray.
 */
#ifndef SPLATCT_H
#define SPLATCT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPLATCT_OK 0
#define SPLATCT_ERR_INVALID 1
#define SPLATCT_ERR_CUDA 2

#define SPLATCT_ABI_VERSION 1

int splatct_abi_version(void);
const char* splatct_last_error(void);
/* Number of kernels this library has launched (process lifetime). */
unsigned long long splatct_launch_count(void);

/* ---------------------------------------------------------------------------
 * Voxelizer ("FVR"): fvr.reconstruct / fvr.backward (fvr.py:148-167,
 * 227-273) replacing _kernels.splat_decomposed (_kernels.py:22-78) and
 * _kernels.splat_backward (_kernels.py:132-205).
 * Tiles are SPLATCT_TILE^3 voxels; a Gaussian's footprint is
 * [floor(mu_a)-h_a, floor(mu_a)+h_a] intersect [0, dim_a) (_kernels.py:45-78).
 * (w, h, c) are the dims of the local volume; z0 is its origin in the global
 * volume (0 unless the volume is a z-slab of a sharded volume): local voxel
 * z holds global slice z0 + z, and footprints are clipped to the slab.
 * ------------------------------------------------------------------------- */
#define SPLATCT_TILE 16

/* Bytes of the caller-provided voxelizer workspace (footprints, GRec records,
 * sort buffers and tile starts, empty-space masks, tile counters, the
 * backward's visiting order) for n Gaussians on a (w,h,c) grid with box
 * halves. */
int splatct_fvr_workspace_bytes(int64_t n, int w, int h, int c, int hx, int hy, int hz,
                                size_t* bytes);

/* Footprints + radix-sorted (tile, Gaussian) bin lists into ws.  Replaces the
 * implicit per-Gaussian box loop of _kernels.py:42-78 (no reference
 * counterpart for tiles).  halt: optional device flag; non-zero skips work. */
int splatct_fvr_bin(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                    int hy, int hz, void* ws, size_t ws_bytes, const int* halt, void* stream);
/* Same bins, each tile's list ordered by the Gaussians' first footprint row
 * relative to the tile (quantised into the radix key's spare bits, no extra
 * pass), then by Gaussian: the forward then skips whole k8 steps per warp
 * more often.  The lists hold the same pairs; the forward's per-voxel sums run
 * in a different (still deterministic) order, so volumes agree with the
 * canonical bins to f32 rounding.  The training step uses these. */
int splatct_fvr_bin_row_ordered(const double* params, int64_t n, int w, int h, int c, int z0,
                                int hx, int hy, int hz, void* ws, size_t ws_bytes,
                                const int* halt, void* stream);
/* splatct_adam (params, m1, m2 updated in place with the scalars adam =
 * {lr, 1-b1^t, 1-b2^t}, sigma clamped, intensity >= 0) followed by the bins of
 * the updated params (row-ordered when row_ordered != 0), in one pass: each
 * thread updates its own Gaussian and bins it.  The training step's form. */
int splatct_fvr_adam_bin(double* params, const double* grads, double* m1, double* m2,
                         const double* adam, double sigma_floor, double sigma_ceiling, int64_t n,
                         int w, int h, int c, int z0, int hx, int hy, int hz, void* ws,
                         size_t ws_bytes, int row_ordered, const int* halt, void* stream);

/* V = sum_i I_i ex_i (x) ey_i (x) ez_i over box intersect volume; one CTA per
 * tile accumulating in registers/shared memory, each voxel written once
 * (no memset, no float atomics; persistent CTAs take tiles from a counter in
 * ws).  Requires a prior splatct_fvr_bin on the same params.  Replaces _kernels.splat_decomposed(mu, sigma, intensity,
 * hx, hy, hz, w, h, c, bufs) (_kernels.py:23) + fvr.py:163-167. */
int splatct_fvr_forward(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                        int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                        const int* halt, void* stream);
/* The same, also recording the two empty-space masks of the volume (pixel
 * occupancy, footprint coverage; see splatct_fvr_pixel_occupancy_offset) --
 * the training step's variant (the masks cost ~5-10 % of the splat). */
int splatct_fvr_forward_masked(const double* params, int64_t n, int w, int h, int c, int z0,
                               int hx, int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                               const int* halt, void* stream);

/* The non-decomposed splat on the same bins (fvr.reconstruct_nodecomp ->
 * _kernels.splat_plain, _kernels.py:81-129): one exponential per box voxel;
 * the comparator of the decomposition.  Call after
 * splatct_fvr_bin; every voxel of vol_yxz is written. */
int splatct_fvr_forward_plain(const double* params, int64_t n, int w, int h, int c, int z0,
                              int hx, int hy, int hz, void* ws, size_t ws_bytes, float* vol_yxz,
                              void* stream);

/* Per-Gaussian gradients from dL/dV (yxz), fvr.py:227-273: one warp per
 * Gaussian sums its box's five moments in a fixed order (deterministic, no
 * partial buffers), the upstream rows arriving by TMA (c % 4 == 0; full 17^3
 * boxes two rows per load) or direct loads, then the f64 chain rule.  The
 * general path never reads upstream outside the footprint (the masked
 * adjoint leaves it unwritten).
 * grads: double[5][n] (overwritten).  accum: optional double[n]; if non-NULL
 * accum[i] += |d_mu_i| (fvr.py:266-273).  Requires the bins of
 * splatct_fvr_bin on the same params.  Replaces _kernels.splat_backward(mu,
 * sigma, intensity, hx, hy, hz, w, h, c, upstream, d_mu, d_sigma,
 * d_intensity) (_kernels.py:133-134). */
int splatct_fvr_backward(const double* params, int64_t n, int w, int h, int c, int z0, int hx,
                         int hy, int hz, void* ws, size_t ws_bytes, const float* up_yxz,
                         double* grads, double* accum, const int* halt, void* stream);

/* accum[i] += |(grads[0][i], grads[1][i], grads[2][i])| -- the densification
 * statistic of fvr.py:266-273, applied after the cross-slab gradient
 * all-reduce when the volume is sharded. */
/* Empty-space masks inside the splatct_fvr_bin workspace, written by
 * splatct_fvr_forward_masked (one uint64 per pixel column, w * h words; SIZE_MAX
 * offset when the volume has more than 64 z tiles):
 *  - pixel occupancy: bit tz = the column's 16-slice segment in z tile tz holds
 *    a non-zero voxel (value-based; the projector forwards' skip test);
 *  - footprint coverage: bit tz = a Gaussian footprint covers the column in z
 *    tile tz (what splatct_fvr_backward reads; the adjoints' skip test). */
int splatct_fvr_pixel_occupancy_offset(int64_t n, int w, int h, int c, int hx, int hy, int hz,
                                       size_t* offset);
int splatct_fvr_footprint_coverage_offset(int64_t n, int w, int h, int c, int hx, int hy, int hz,
                                          size_t* offset);
int splatct_grad_norm_accum(const double* grads, int64_t n, double* accum, const int* halt,
                            void* stream);

/* Copy the bins out for the bit-exact check against the CPU restatement.
 * fp: int32[n][6] {xlo,xhi,ylo,yhi,zlo,zhi} (empty axis: lo>hi);
 * tile_start: int32[n_tiles+1]; items: int32[npairs] Gaussian ids, per tile
 * ascending.  *npairs and *n_tiles are written to host memory (synchronous). */
int splatct_fvr_export_bins(const void* ws, size_t ws_bytes, int64_t n, int w, int h, int c,
                            int hx, int hy, int hz, int32_t* fp, int32_t* tile_start,
                            int32_t* items, int64_t* npairs, int64_t* n_tiles, void* stream);

/* ---------------------------------------------------------------------------
 * Projector: forward_project / back_project (projector.py:59-111) replacing
 * _kernels.project_forward (_kernels.py:262-303) and project_adjoint
 * (_kernels.py:306-357).  The per-slice geometry is slice-invariant, so the
 * ray march (_ray_geometry/_clip_ray, _kernels.py:208-259, in f64) runs once
 * per geometry and produces the exact sample weights merged per (ray, pixel):
 * A (ray-major CSR) and its exact transpose A^T (pixel-major CSR).  Each
 * iteration then applies them to the z-vectors of the yxz volume / sinogram.
 * cos_t, sin_t: device double[m] (projector.py:50-52, f64 on host).
 * ------------------------------------------------------------------------- */

/* Scratch bytes for splatct_proj_count (nnz = 0) and splatct_proj_fill
 * (nnz = the count returned by splatct_proj_count). */
int splatct_proj_scratch_bytes(int m, int n_det, int w, int h, int64_t nnz, size_t* bytes);

/* Pass 1 (synchronous): a_ptr (device int64[m*n_det+1]) = row offsets of A;
 * *nnz (host) = number of merged (ray, pixel) weights. */
int splatct_proj_count(const double* cos_t, const double* sin_t, int m, int n_det,
                       double spacing, double step, int is_fan, double rs, double rd, int w,
                       int h, int64_t* a_ptr, void* scratch, size_t scratch_bytes,
                       int64_t* nnz, void* stream);

/* Pass 2: fills A (a_col = pixel y*w+x, a_val = step * merged bilinear
 * weight) and A^T (at_ptr int64[w*h+1], at_ray, at_val; rows sorted by ray). */
int splatct_proj_fill(const double* cos_t, const double* sin_t, int m, int n_det,
                      double spacing, double step, int is_fan, double rs, double rd, int w,
                      int h, const int64_t* a_ptr, int32_t* a_col, float* a_val,
                      int64_t* at_ptr, int32_t* at_ray, float* at_val, void* scratch,
                      size_t scratch_bytes, void* stream);

/* sino[r][z] = sum_j a_val[j] * vol[a_col[j]][z]  for r < n_rays, z < c. */
int splatct_proj_forward(const int64_t* a_ptr, const int32_t* a_col, const float* a_val,
                         int n_rays, const float* vol_yxz, float* sino, int c,
                         const int* halt, void* stream);

/* out[p][z] = f32( sum_j at_val[j] * gsino[at_ray[j]][z] + lambda_tv * tvgrad(p,z) )
 * with tvgrad the anisotropic TV subgradient of vol / tv_count
 * (loss.tv_loss, loss.py:183-207) fused in; tv_partial (optional, double[w*h])
 * receives per-pixel-column sums of |forward differences| of vol.
 * halo_lo / halo_hi (optional, float[h*w]) are the neighbouring z-planes
 * z = -1 and z = c of a z-slab (NULL at the global volume edges); the
 * forward difference into halo_hi is counted by this slab.
 * Pass vol = NULL / lambda_tv = 0 for the plain adjoint. */
int splatct_proj_adjoint(const int64_t* at_ptr, const int32_t* at_ray, const float* at_val,
                         int w, int h, int c, const float* gsino, const float* vol_yxz,
                         const float* halo_lo, const float* halo_hi, double lambda_tv,
                         double tv_count, float* out_yxz, double* tv_partial, const int* halt,
                         void* stream);

/* Row-blocked form of a CSR operator (proj_blocked.cu).  kind 0 groups rows
 * 4g..4g+3 and kind 2 rows 8g..8g+7 (consecutive rays of A); kind 1 groups
 * the 2x2 pixel quad (2qx+dx, 2qy+dy), k = 2*dy + dx, of A^T on a w x h
 * slice.  A group entry is (column, w[R]) with the R member rows' weights (0
 * where absent), columns ascending -- or, with order_dir (device
 * float[ngroups][2], the group's ray direction; ray groups only), in march
 * order along that direction so concurrent warps sweep the slice together.
 * kinds 3 / 4 are bands of 8 / 16 consecutive rays (forward only, w * h <=
 * 2^27, at most 8192 weights per band): an entry is a sliding 4-ray window,
 * (k0 << 27 | pixel, w[4]) for band rays k0..k0+3, one per window of a
 * pixel's run of rays, entries ordered by (k0, pixel); order_dir is ignored.
 * count (synchronous) -> gptr[ngroups+1] and *nb; fill -> gidx, gval
 * (float[nb][R], R = 8 for kind 2 and 4 otherwise, 16-byte aligned).  fill
 * takes the scratch its count used (the count leaves the largest group's
 * size there; a mismatch is an error, not a wrong operator).  Rows already
 * sorted by column (A^T from splatct_proj_fill) are merged without a sort. */
int splatct_proj_block_scratch_bytes(int nrows, int kind, int w, int h, size_t* bytes);
int splatct_proj_block_count(const int64_t* ptr, const int32_t* idx, int nrows, int kind, int w,
                             int h, const float* order_dir, int64_t* gptr, void* scratch,
                             size_t scratch_bytes, int64_t* nb, void* stream);
int splatct_proj_block_fill(const int64_t* ptr, const int32_t* idx, const float* val, int nrows,
                            int kind, int w, int h, const float* order_dir, const int64_t* gptr,
                            int32_t* gidx, float* gval, void* scratch, size_t scratch_bytes,
                            void* stream);

/* Length (doubles) of the tv_partial buffer splatct_proj_adjoint_blocked
 * writes for a w x h x c slab: one slot per (2 x 2 pixel quad, 32*V-slice
 * chunk), each written exactly once (reduce the whole buffer in a fixed
 * order). */
int splatct_proj_tv_partial_len(int w, int h, int c, int64_t* len);

/* Blocked applications: same results as splatct_proj_forward /
 * splatct_proj_adjoint (up to f32 summation order), one z-column load per
 * group entry feeding the group's rows (forward: kind 0, 2, 3 or 4 groups;
 * bands store each ray once as their 4-ray window slides past it). */
/* col_occ (optional, NULL = off): the voxelizer's PIXEL-column occupancy of
 * vol_yxz (splatct_fvr_pixel_occupancy_offset into the bins workspace, valid
 * after splatct_fvr_forward); entries whose pixel column is zero in a warp's
 * z range are skipped -- they would add exact zeros.  w, h: volume width and
 * height (pixel = y * w + x). */
int splatct_proj_forward_blocked(const int64_t* gptr, const int32_t* gidx, const float* gval,
                                 int n_rays, int kind, const float* vol_yxz, float* sino, int c,
                                 const uint64_t* col_occ, int w, int h, const int* halt,
                                 void* stream);
/* The forward's launch shape for a c-slice volume: *ctas CTAs over ngroups x
 * *zsplit (group, z-chunk) warp tasks, 4 per CTA, CTA b taking tasks
 * 4b..4b+3.  *ordered: 1 = tasks are group-major (task t: group t / zsplit,
 * chunk t % zsplit); 2 = z-chunk-major, used once the volume outgrows ~3/4 of
 * L2 (group t % ngroups, chunk t / ngroups) -- an order should then keep each
 * chunk's CTAs together, so the warps in flight keep sharing one chunk;
 * 0 = bands, which take no order. */
int splatct_proj_forward_ctas(int n_rays, int kind, int w, int h, int c, int64_t* ctas,
                              int* zsplit, int* ordered);
/* splatct_proj_forward_blocked with cta_order (device int32[*ctas], a
 * permutation, or NULL): CTA b runs CTA cta_order[b]'s tasks.  Listing the
 * CTAs with the most entries first shortens the grid's tail; the results are
 * bitwise those of the default order. */
int splatct_proj_forward_blocked_ordered(const int64_t* gptr, const int32_t* gidx,
                                         const float* gval, int n_rays, int kind,
                                         const float* vol_yxz, float* sino, int c,
                                         const uint64_t* col_occ, int w, int h,
                                         const int32_t* cta_order, const int* halt,
                                         void* stream);
/* col_occ (optional, NULL = dense): the voxelizer's footprint coverage of
 * vol_yxz (splatct_fvr_footprint_coverage_offset).  A 2x2-pixel quad x
 * z-chunk whose one-voxel neighbourhood no footprint covers is skipped: its
 * TV terms are zero (the volume is zero there) and its out_yxz values are
 * LEFT UNWRITTEN -- only for callers that read the result inside footprints
 * (the training step's voxelizer backward).  Its tv_partial slots are 0. */
int splatct_proj_adjoint_blocked(const int64_t* gptr, const int32_t* gidx, const float* gval,
                                 int w, int h, int c, const float* gsino, const float* vol_yxz,
                                 const float* halo_lo, const float* halo_hi, double lambda_tv,
                                 double tv_count, float* out_yxz, double* tv_partial,
                                 const uint64_t* col_occ, const int* halt, void* stream);

/* Direct ray-marching forward projection (no matrix), same f64 ray setup and
 * sample enumeration as _kernels.py:262-303; used as a cross-check and for
 * one-off projections. */
int splatct_proj_march_forward(const double* cos_t, const double* sin_t, int m, int n_det,
                               double spacing, double step, int is_fan, double rs, double rd,
                               int w, int h, int c, const float* vol_yxz, float* sino,
                               void* stream);

/* ---------------------------------------------------------------------------
 * Loss: loss.total_loss_detailed (loss.py:210-239): L1 (loss.py:64-74) and
 * valid-window SSIM (loss.py:77-180) of pred vs ref, both (m,n,p), with the
 * analytic gradient written as f32 (optim.py:368 quantisation).
 * ------------------------------------------------------------------------- */

int splatct_loss_workspace_bytes(int m, int n, int p, size_t* bytes);

/* out[0] = max(x) over all bins (double) -- the SSIM dynamic range L.
 * out must hold 1 + SPLATCT_SQDIFF_BLOCKS doubles (the tail is scratch). */
int splatct_sino_max(const float* x, int64_t count, double* out, void* stream);

/* grad_pred = lambda1*sign(pred-ref)/l1_count - lambda2*dSSIM/dpred/ssim_slices.
 * sums (device double[2]) receive sum|pred-ref| and sum over local slices of
 * mean-SSIM.  lmax: global max(ref) (<=0 -> 1).  l1_count and ssim_slices are
 * GLOBAL counts (they differ from m*n*p under z-slab sharding). */
int splatct_loss_fused(const float* pred, const float* ref, int m, int n, int p, double lmax,
                       double lambda1, double lambda2, double l1_count, double ssim_slices,
                       float* grad_pred, void* ws, size_t ws_bytes, double* sums,
                       const int* halt, void* stream);

/* The measured sinogram is constant over a run: splatct_loss_prepare_ref
 * stores its per-window SSIM moments (mean_y, E[y^2]) in ws once, and
 * splatct_loss_fused_prepared (same arguments as splatct_loss_fused, same ref
 * and ws) then carries only the three pred-dependent moments per iteration. */
int splatct_loss_prepare_ref(const float* ref, int m, int n, int p, void* ws, size_t ws_bytes,
                             void* stream);
int splatct_loss_fused_prepared(const float* pred, const float* ref, int m, int n, int p,
                                double lmax, double lambda1, double lambda2, double l1_count,
                                double ssim_slices, float* grad_pred, void* ws, size_t ws_bytes,
                                double* sums, const int* halt, void* stream);
/* The same, leaving the l1 and SSIM sums as block partials in ws (sums[0] and
 * sums[1] are not written, except sums[1] = 0 when lambda2 = 0):
 * splatct_iter_finalize_partials reduces them.  splatct_loss_partials gives
 * their addresses and counts (n_ssim = 0 when lambda2 = 0). */
int splatct_loss_fused_prepared_deferred(const float* pred, const float* ref, int m, int n, int p,
                                         double lmax, double lambda1, double lambda2,
                                         double l1_count, double ssim_slices, float* grad_pred,
                                         void* ws, size_t ws_bytes, double* sums,
                                         const int* halt, void* stream);
int splatct_loss_partials(int m, int n, int p, double lambda2, void* ws, size_t ws_bytes,
                          const double** l1_part, int64_t* n_l1, const double** ssim_part,
                          int64_t* n_ssim);

/* out[0] = sum (x-y)^2 over count elements (f64, fixed order); ws holds
 * SPLATCT_SQDIFF_BLOCKS doubles.  Used for PSNR (metrics.psnr, metrics.py:24-38). */
#define SPLATCT_SQDIFF_BLOCKS 592
int splatct_sum_sq_diff(const float* x, const float* y, int64_t count, double* ws, double* out,
                        void* stream);

/* Sum n doubles in a fixed order into out[0] (deterministic reductions). */
int splatct_reduce_sum(const double* in, int64_t n, double* out, void* stream);

/* Host -> device upload through a page-locked staging buffer of >= bytes:
 * nthreads host threads each copy a slice of src into pinned and queue that
 * slice's DMA on stream (returns once every slice is queued; the DMAs run in
 * stream order).  The measured sinogram's upload in run_reconstruction; the
 * call releases the GIL (ctypes), so the caller overlaps it with other host work. */
int splatct_stage_upload(void* dst, const void* src, void* pinned, size_t bytes, int nthreads,
                         void* stream);

/* TV terms across a z-slab boundary after an adjoint that ran without halo
 * planes (the halo exchange then overlaps it), loss.py:183-207: plane c-1 gets
 * -lambda/count * sign(hi - v) and |hi - v| is added to *tv_sum (this slab
 * owns that difference); plane 0 gets +lambda/count * sign(v - lo).  NULL
 * halo = volume edge.  Deterministic (one block, fixed order). */
int splatct_tv_halo_fixup(const float* vol_yxz, float* dl_yxz, const float* halo_lo,
                          const float* halo_hi, int w, int h, int c, double lambda_tv,
                          double tv_count, double* tv_sum, const int* halt, void* stream);
/* Iteration bookkeeping (optim.py:350-386): from the global sums
 * {l1_sum, ssim_sum, tv_sum} compute the loss parts
 * (zero-weight terms -> NaN, loss.py:216-239), write
 * trace[4*it .. 4*it+3] = {loss, l1, ssim, tv} with it = *iter, set *halt if
 * the loss is non-finite (optim.py:356), else write the Adam scalars
 * adam[0..2] = {lr, 1-b1^t, 1-b2^t} for the pre-increment *step
 * (optim.py:88-90,123-126) and advance *step and *iter. */
int splatct_iter_finalize(const double* sums, double lambda1, double lambda2, double lambda3,
                          double l1_count, double ssim_count, double tv_count, double lr0,
                          double lrf, int64_t max_iters, int64_t* step, int64_t* iter,
                          double* trace, int64_t trace_cap, double* adam, int* halt,
                          void* stream);
/* The same, first reducing sums[0..2] = {l1, ssim, tv} from block partials
 * (32 blocks sum fixed slices, the last one to finish combines them in block
 * order: deterministic); a part with n = 0 keeps sums[f] as given.  scratch:
 * SPLATCT_FIN_SCRATCH_DOUBLES doubles, zero before the first call (the kernel
 * leaves its ticket word at zero again).  sched (optional, sched_len rows):
 * the Adam scalars {lr, 1-b1^t, 1-b2^t} per pre-increment step, computed on
 * the host like the reference; steps beyond it use device pow.  Replaces the
 * three separate reductions of the single-device training step. */
#define SPLATCT_FIN_SCRATCH_DOUBLES 97
int splatct_iter_finalize_partials(double* sums, const double* l1_part, int64_t n_l1,
                                   const double* ssim_part, int64_t n_ssim,
                                   const double* tv_part, int64_t n_tv, double* scratch,
                                   const double* sched, int64_t sched_len, double lambda1,
                                   double lambda2, double lambda3, double l1_count,
                                   double ssim_count, double tv_count, double lr0, double lrf,
                                   int64_t max_iters, int64_t* step, int64_t* iter,
                                   double* trace, int64_t trace_cap, double* adam, int* halt,
                                   void* stream);

/* ---------------------------------------------------------------------------
 * Adam: optim.adam_step (optim.py:109-144): bias-corrected Adam on the
 * params block with scalars adam = {lr, bc1, bc2} from splatct_iter_finalize
 * (device), then sigma clamped to [sigma_floor, sigma_ceiling], intensity >= 0.
 * ------------------------------------------------------------------------- */
int splatct_adam(double* params, const double* grads, double* m1, double* m2, int64_t n,
                 const double* adam, double sigma_floor, double sigma_ceiling,
                 const int* halt, void* stream);

/* ---------------------------------------------------------------------------
 * FBP initialiser (projector.fbp, projector.py:154-206; out of the iteration
 * loop): filtered rows (host-filtered or device) are back-projected
 * pixel-driven, _kernels.backproject_parallel_beam / backproject_fan_beam
 * (_kernels.py:360-419).  filtered: (m, n, p) like the sinogram; out yxz.
 * ------------------------------------------------------------------------- */
int splatct_fbp_filter(const float* sino, int m, int n, int p, const double* kernel,
                       const double* det_weight, double* filtered, void* stream);
int splatct_fbp_backproject(const double* filtered, const double* cos_t, const double* sin_t,
                            int m, int n, int p, int w, int h, double spacing, double dbeta,
                            int is_fan, double rs, float* out_yxz, void* stream);

/* ---------------------------------------------------------------------------
 * Cone-beam extension (no reference counterpart, parity
 * unpinned; model in cone.cu / DESIGN.md "Cone beam").  Setup, once per
 * geometry: splatct_cone_count (per-column merged-entry counts -> cptr[m*nu+1],
 * 1/L per column; returns the total) and splatct_cone_fill (16-byte column
 * entries {pixel, w, tau}); splatct_cone_entry_count / _fill transpose them
 * into per-pixel entry lists (16 B each, eptr[w*h+1]) for the gather adjoint.
 * Per iteration: splatct_cone_forward (vol yxz slab [h][w][c_local] -> sino
 * (m*nu, nv); zc = (c_global-1)/2 - z0, so slab results are partial
 * projections that sum to the full one) and splatct_cone_adjoint (exact
 * transpose; gscaled is an (m*nu*nv) f32 scratch; accumulate != 0 adds into
 * out).  Optional occupancy (NULL = dense): the forward's col_occ is the
 * voxelizer's PIXEL-column occupancy (splatct_fvr_pixel_occupancy_offset;
 * entries whose column is all zero are skipped, exact); the adjoint's is the
 * FOOTPRINT coverage (splatct_fvr_footprint_coverage_offset): pixel x
 * z-windows no footprint covers are left UNWRITTEN (training step only: its
 * consumer, splatct_fvr_backward, reads inside Gaussian footprints).
 * ------------------------------------------------------------------------- */
int splatct_cone_setup_scratch_bytes(int m, int nu, int w, int h, size_t* bytes);
int splatct_cone_count(const double* cos_t, const double* sin_t, int m, int nu, double su,
                       double rs, double rd, int w, int h, double step, int64_t* rptr,
                       float* inv_len, void* scratch, size_t scratch_bytes, int64_t* nsamples,
                       void* stream);
int splatct_cone_fill(const double* cos_t, const double* sin_t, int m, int nu, double su,
                      double rs, double rd, int w, int h, double step, const int64_t* rptr,
                      void* samples, void* stream);
int splatct_cone_entry_count(const void* samples, const int64_t* rptr, int nrays, int w, int h,
                             int64_t* eptr, void* scratch, size_t scratch_bytes,
                             int64_t* nentries, void* stream);
int splatct_cone_entry_scratch_bytes(int64_t nentries, int w, int h, size_t* bytes);
int splatct_cone_entry_fill(const void* samples, const int64_t* rptr, int nrays, int w, int h,
                            const int64_t* eptr, int64_t nentries, void* entries, void* scratch,
                            size_t scratch_bytes, void* stream);
int splatct_cone_forward(const void* samples, const int64_t* rptr, const float* inv_len,
                         int nrays, int nv, double sv, double step, int w, int h, int c_local,
                         double zc, const float* vol_yxz, const uint64_t* col_occ, float* sino,
                         const int* halt, void* stream);
int splatct_cone_adjoint(const void* entries, const int64_t* eptr, const float* inv_len,
                         int nrays, int nv, double sv, double step, int w, int h, int c_local,
                         double zc, const float* gsino, float* gscaled, float* out_yxz,
                         int accumulate, const uint64_t* col_occ, const int* halt, void* stream);

/* ---------------------------------------------------------------------------
 * Densification on the device: densify.densify_and_prune,
 * reference densify.py:86-147, plus the Adam-moment remap optim.py:92-106.
 * params / m1 / m2 are [5, n] f64 (x, y, z, sigma, intensity rows).
 *  - classify: cls[n] = 0 keep | 1 prune | 2 clone candidate | 3 split
 *    candidate (densify.py:97-110, avg = accum / iters; sigma_prune = 3 x box
 *    size); keys[n] = bit pattern of avg; counts[3] = (prune, clone cand.,
 *    split cand.) -- the host reads them to size the budgets.
 *  - select: mark (cls += 2) the k highest-avg members of class `which`
 *    (_limit, densify.py:73-83; ties at the cut: lower index first).
 *  - apply: new cloud [kept | clones | split children] of n_new rows; noise
 *    is the reference's rng.standard_normal((2 * n_split, 3)) (optim.py:394),
 *    row-major f64 on the device; cbrt2 = numpy.cbrt(2.0).
 * ------------------------------------------------------------------------- */
int splatct_densify_workspace_bytes(int64_t n, size_t* bytes);
int splatct_densify_classify(const double* params, const double* accum, int64_t n, double iters,
                             double tau, double theta, double sigma_prune, int grad_prune,
                             uint8_t* cls, uint64_t* keys, uint64_t* counts, void* stream);
int splatct_densify_select(uint8_t* cls, const uint64_t* keys, int64_t n, int which, int64_t k,
                           int64_t count, void* ws, size_t ws_bytes, void* stream);
int splatct_densify_apply(const double* params, const double* m1, const double* m2,
                          const uint8_t* cls, const double* noise, int64_t n, int64_t n_new,
                          double cbrt2, double* new_params, double* new_m1, double* new_m2,
                          void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Tensor-core self-test (no reference counterpart; validates the tcgen05
 * conventions the voxelizer forward builds on): D[128][16] = A[128][8] B[16][8]^T
 * with A in TMEM, B in shared memory, D in TMEM (kind::tf32, cta_group::1).
 * mode 0: one TF32 MMA; mode 1: the 3xTF32 split. Device f32 pointers.
 * ------------------------------------------------------------------------- */
int splatct_tc_selftest(const float* a, const float* b, float* d, int mode, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLATCT_H */
