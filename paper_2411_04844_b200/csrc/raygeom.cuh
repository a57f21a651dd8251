// raygeom.cuh -- the reference's per-ray 2D setup (_clip_ray + _ray_geometry,
// /root/reference/pkg/src/splatct/_kernels.py:208-259), f64 with the same
// operation order; shared by the per-slice projector (proj.cu) and the
// cone-beam extension (cone.cu), whose xy march is the fan's.
#pragma once
#include "common.cuh"

namespace splatct {

// _clip_ray + _ray_geometry, f64, same operation order as the reference.
__device__ __forceinline__ void ray_geometry(double cos_a, double sin_a, double u, bool is_fan,
                                             double rs, double rd, double cx, double cy, int w,
                                             int h, double& ox, double& oy, double& dx,
                                             double& dy, double& t0, double& t1) {
    if (is_fan) {
        const double sx = cx - rs * cos_a, sy = cy - rs * sin_a;
        const double px = cx + rd * cos_a - u * sin_a, py = cy + rd * sin_a + u * cos_a;
        double ddx = px - sx, ddy = py - sy;
        const double len = sqrt(ddx * ddx + ddy * ddy);
        dx = ddx / len;
        dy = ddy / len;
        t0 = 0.0;
        t1 = len;
        ox = sx;
        oy = sy;
    } else {
        ox = cx - u * sin_a;
        oy = cy + u * cos_a;
        dx = cos_a;
        dy = sin_a;
        const double reach = hypot((double)w, (double)h);
        t0 = -reach;
        t1 = reach;
    }
    const double xlo = -1.0, xhi = (double)w, ylo = -1.0, yhi = (double)h;
    if (dx != 0.0) {
        double ta = (xlo - ox) / dx, tb = (xhi - ox) / dx;
        if (ta > tb) { double q = ta; ta = tb; tb = q; }
        t0 = fmax(t0, ta);
        t1 = fmin(t1, tb);
    } else if (ox < xlo || ox > xhi) {
        t0 = 1.0; t1 = 0.0;
        return;
    }
    if (dy != 0.0) {
        double ta = (ylo - oy) / dy, tb = (yhi - oy) / dy;
        if (ta > tb) { double q = ta; ta = tb; tb = q; }
        t0 = fmax(t0, ta);
        t1 = fmin(t1, tb);
    } else if (oy < ylo || oy > yhi) {
        t0 = 1.0; t1 = 0.0;
    }
}

struct Geom {
    const double* cos_t;
    const double* sin_t;
    int m, n_det;
    double spacing, step;
    bool is_fan;
    double rs, rd;
    int w, h;
};

// March one ray; call emit(pixel, merged_weight, merged_weight_times_t) for
// every distinct pixel it touches with non-zero weight, in order of closing
// (t = distance of the sample from the ray origin; the cone-beam extension
// uses the weight-averaged t of a pixel's samples).
// A pixel's support is the open square (x-1,x+1)x(y-1,y+1); the samples
// inside it are a contiguous k-range, so a pixel untouched by sample k is
// final (the "open set" never holds more than 8 entries).
//
// Segment seg of nseg: the samples [ns*seg/nseg, ns*(seg+1)/nseg) open
// pixels; the segment owns the pixels it opens and keeps marching past its
// end until they are all closed, while pixels still open from the previous
// sample at its start belong to an earlier segment and are skipped.  Every
// pixel is therefore summed by exactly one segment, over the same samples in
// the same order as by the whole-ray march (identical merged weights); only
// the order of emission across segment boundaries differs.
template <typename Emit>
__device__ void march_ray_seg(const Geom& g, int r, int seg, int nseg, Emit emit) {
    const int v = r / g.n_det, d = r % g.n_det;
    const double cx = 0.5 * (g.w - 1), cy = 0.5 * (g.h - 1);
    const double u = (d - 0.5 * (g.n_det - 1)) * g.spacing;
    double ox, oy, dx, dy, t0, t1;
    ray_geometry(g.cos_t[v], g.sin_t[v], u, g.is_fan, g.rs, g.rd, cx, cy, g.w, g.h, ox, oy, dx,
                 dy, t0, t1);
    if (!(t1 > t0)) return;
    const int64_t ns = (int64_t)((t1 - t0) / g.step);
    const int64_t kb = ns * seg / nseg, ke = ns * (seg + 1) / nseg;
    if (kb >= ke) return;
    // the 4 bilinear taps of sample k: pixel (or -1: outside / zero weight), weight
    auto taps = [&](int64_t k, double& t, int (&px)[4], double (&tw)[4]) {
        t = t0 + (k + 0.5) * g.step;
        const double sx = ox + t * dx, sy = oy + t * dy;
        const double fx0 = floor(sx), fy0 = floor(sy);
        const int64_t x0 = (int64_t)fx0, y0 = (int64_t)fy0;
        const double fx = sx - (double)x0, fy = sy - (double)y0;
        const int64_t tx[4] = {x0, x0 + 1, x0, x0 + 1};
        const int64_t ty[4] = {y0, y0, y0 + 1, y0 + 1};
        tw[0] = (1 - fx) * (1 - fy);
        tw[1] = fx * (1 - fy);
        tw[2] = (1 - fx) * fy;
        tw[3] = fx * fy;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            px[q] = (tx[q] < 0 || tx[q] >= g.w || ty[q] < 0 || ty[q] >= g.h || tw[q] == 0.0)
                        ? -1 : (int)(ty[q] * g.w + tx[q]);
    };
    int pre[4] = {-1, -1, -1, -1};   // pixels an earlier segment still has open
    if (kb > 0) {
        double t, tw[4];
        taps(kb - 1, t, pre, tw);
    }
    int opix[8];
    double ow[8], owt[8];
    bool otouch[8];
    int nopen = 0;
    for (int64_t k = kb; k < ns; ++k) {
        const bool opening = k < ke;
        if (!opening && nopen == 0) break;
        double t, tw[4];
        int px[4];
        taps(k, t, px, tw);
        for (int q = 0; q < nopen; ++q) otouch[q] = false;
        bool ptouch[4] = {false, false, false, false};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int pix = px[q];
            if (pix < 0) continue;
            bool earlier = false;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (pre[e] == pix) { ptouch[e] = true; earlier = true; }
            if (earlier) continue;
            int f = -1;
            for (int e = 0; e < nopen; ++e)
                if (opix[e] == pix) f = e;
            if (f < 0) {
                if (!opening) continue;   // a later segment's pixel
                f = nopen++;
                opix[f] = pix;
                ow[f] = 0.0;
                owt[f] = 0.0;
            }
            ow[f] += tw[q];
            owt[f] += tw[q] * t;
            otouch[f] = true;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (!ptouch[e]) pre[e] = -1;   // closed: it cannot be touched again
        int keep = 0;
        for (int e = 0; e < nopen; ++e) {
            if (!otouch[e]) {
                emit(opix[e], ow[e], owt[e]);
            } else {
                opix[keep] = opix[e];
                ow[keep] = ow[e];
                owt[keep] = owt[e];
                otouch[keep] = true;
                ++keep;
            }
        }
        nopen = keep;
    }
    for (int e = 0; e < nopen; ++e) emit(opix[e], ow[e], owt[e]);
}

template <typename Emit>
__device__ void march_ray(const Geom& g, int r, Emit emit) {
    march_ray_seg(g, r, 0, 1, emit);
}

}  // namespace splatct
