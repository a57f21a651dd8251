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

}  // namespace splatct
