// Ray-driven cone-beam projector with trilinear volume sampling -- the
// reference's comparison baseline `ct_project_linear` (baseline.py:52-98),
// which the backprojector calibration runs on every call
// (calibrate_bp_normalization, pipeline.py:245-257).
//
// One thread per ray (view, u, v).  The ray geometry, slab clipping against
// the volume cube, the N midpoint samples and the trilinear weights follow
// the reference's float64 arithmetic; volume values are float32 and the sum
// is accumulated in float64.
#include "../../include/cbnufft_b200.h"
#include "cbn_plan.h"

namespace cbn {
namespace {

struct RayGeom {
    double so, sd, pu, pv, half, voxel;
    int nu, nv, n_views, n;
};

__global__ void __launch_bounds__(256)
k_ct_project_linear(const float* __restrict__ vol, RayGeom g, int64_t rays,
                    float* __restrict__ frames) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rays) return;
    const int iv = (int)(r % g.nv);
    const int iu = (int)((r / g.nv) % g.nu);
    const int k = (int)(r / ((int64_t)g.nu * g.nv));
    const double a = 2.0 * kPi * (double)k / (double)g.n_views;       // geometry.py:59-60
    const double ca = cos(a), sa = sin(a);
    const double sh[3] = {ca, sa, 0.0}, uh[3] = {-sa, ca, 0.0}, vh[3] = {0.0, 0.0, 1.0};
    // detector_axes_physical (baseline.py:20-25)
    const double u = ((double)iu - (double)g.nu / 2.0 + 0.5) * g.pu;
    const double v = ((double)iv - (double)g.nv / 2.0 + 0.5) * g.pv;
    double src[3], d[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        src[q] = g.so * sh[q];
        const double pt = ((-g.sd * sh[q]) + src[q]) + u * uh[q] + v * vh[q];
        d[q] = pt - src[q];
    }
    const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
    for (int q = 0; q < 3; ++q) d[q] /= nrm;
    // slab intersection with [-half, half]^3
    double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double safe = fabs(d[q]) < 1e-300 ? 1e-300 : d[q];
        const double ta = (-g.half - src[q]) / safe;
        const double tb = (g.half - src[q]) / safe;
        t0 = fmax(t0, fmin(ta, tb));
        t1 = fmin(t1, fmax(ta, tb));
    }
    const double span = fmax(t1 - t0, 0.0);
    const double step = span / (double)g.n;
    double acc = 0.0;
    if (span > 0.0) {
        const double c0 = (double)g.n / 2.0 - 0.5;
        const int n = g.n;
        for (int s = 0; s < n; ++s) {
            const double tau = t0 + ((double)s + 0.5) * step;
            double idx[3];
            int lo[3];
            double fr[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                idx[q] = (src[q] + tau * d[q]) / g.voxel + c0;
                const double fl = floor(idx[q]);
                lo[q] = (int)fl;
                fr[q] = idx[q] - fl;
            }
#pragma unroll
            for (int corner = 0; corner < 8; ++corner) {
                const int o0 = corner & 1, o1 = (corner >> 1) & 1, o2 = (corner >> 2) & 1;
                const int x = lo[0] + o0, y = lo[1] + o1, z = lo[2] + o2;
                if (x < 0 || x >= n || y < 0 || y >= n || z < 0 || z >= n) continue;
                const double w = (o0 ? fr[0] : 1.0 - fr[0]) * (o1 ? fr[1] : 1.0 - fr[1]) *
                                 (o2 ? fr[2] : 1.0 - fr[2]);
                acc += w * (double)__ldg(vol + ((int64_t)x * n + y) * n + z);
            }
        }
    }
    frames[r] = (float)(acc * step);
}

}  // namespace
}  // namespace cbn

using namespace cbn;

extern "C" int cbn_ct_project_linear(const cbn_geometry* geom, const float* vol, int32_t n,
                                     double voxel_mm, float* frames, void* stream) {
    try {
        CBN_REQUIRE(geom && vol && frames, "null argument");
        CBN_REQUIRE(n >= 1 && voxel_mm > 0, "bad volume");
        CBN_REQUIRE(geom->nu >= 1 && geom->nv >= 1 && geom->n_views >= 1, "bad geometry");
        RayGeom g;
        g.so = geom->so_mm;
        g.sd = geom->sd_mm;
        g.pu = geom->det_width_mm / geom->nu;
        g.pv = geom->det_height_mm / geom->nv;
        g.voxel = voxel_mm;
        g.half = 0.5 * (double)n * voxel_mm;
        g.nu = geom->nu;
        g.nv = geom->nv;
        g.n_views = geom->n_views;
        g.n = n;
        const int64_t rays = (int64_t)geom->n_views * geom->nu * geom->nv;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        k_ct_project_linear<<<blocks_for(rays, 256), 256, 0, s>>>(vol, g, rays, frames);
        CBN_LAUNCH_CHECK();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
