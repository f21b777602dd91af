// Elementwise radial-line stages of the transform API (radon_fourier.py):
// per-rho complex weights (spectral_rho_derivative, ramp_filter_radial, the
// 2D FBP ramp), node phases exp(+-i w.shift) (_center_phase) and the
// trilinear sinc^2 transfer on the radial node set.  All are one streaming
// pass over the data (HBM-bound, one thread per element, grid-stride).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "cbn_plan.h"
#include "cbn_runtime.h"

namespace cbn {

// data viewed as [outer][n][inner] complex64; element (o, k, i) *= w[k]
__global__ void k_line_weight(float2* __restrict__ data, int64_t total, int64_t n, int64_t inner,
                              const double2* __restrict__ w) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = (e / inner) % n;
        const double2 c = w[k];
        const float2 v = data[e];
        // complex128 product rounded once to complex64 (the reference multiplies in float64)
        const double re = (double)v.x * c.x - (double)v.y * c.y;
        const double im = (double)v.x * c.y + (double)v.y * c.x;
        data[e] = make_float2((float)re, (float)im);
    }
}

// y[i] = y[i] * exp(sgn * i * sum_d nodes[i, d] * shift[d]) * (w ? w[i / w_inner] : 1)
__global__ void k_node_phase(float2* __restrict__ y, const double* __restrict__ nodes, int64_t m,
                             int d, double s0, double s1, double s2, double sgn,
                             const double* __restrict__ w, int64_t w_inner) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double* p = nodes + i * d;
        double a = p[0] * s0;
        if (d > 1) a += p[1] * s1;
        if (d > 2) a += p[2] * s2;
        double sn, cs;
        sincos(sgn * a, &sn, &cs);
        if (w) {
            const double g = w[i / w_inner];
            sn *= g;
            cs *= g;
        }
        const float2 v = y[i];
        y[i] = make_float2((float)((double)v.x * cs - (double)v.y * sn),
                           (float)((double)v.x * sn + (double)v.y * cs));
    }
}

__device__ __forceinline__ double sinc_pi(double x) {
    // numpy.sinc: sin(pi x) / (pi x), 1 at 0
    if (x == 0.0) return 1.0;
    const double px = CUDART_PI * x;
    return sinpi(x) / px;
}

// out[phi][theta][rho] = prod_d sinc(node_d / 2pi)^2 at the unwrapped radial
// node w_rho * voxel * (cos phi sin theta, sin phi sin theta, cos theta)
__global__ void k_trilinear_transfer(double* __restrict__ out, int n_rho, int n_theta, int n_phi,
                                     double delta_rho, double voxel) {
    const int64_t total = (int64_t)n_rho * n_theta * n_phi;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % n_rho);
        const int t = (int)((e / n_rho) % n_theta);
        const int f = (int)(e / ((int64_t)n_rho * n_theta));
        // radial_omega (radon_fourier.py:46-49), polar angles (geometry.py:162-168)
        const double om = 2.0 * CUDART_PI * (double)(r - n_rho / 2) / ((double)n_rho * delta_rho) * voxel;
        const double th = (double)t * CUDART_PI / (double)n_theta;
        const double ph = 2.0 * CUDART_PI * (double)f / (double)n_phi;
        const double st = sin(th);
        const double x = om * (cos(ph) * st), y = om * (sin(ph) * st), z = om * cos(th);
        const double inv = 1.0 / (2.0 * CUDART_PI);
        const double p = sinc_pi(x * inv) * sinc_pi(y * inv) * sinc_pi(z * inv);
        out[e] = p * p;
    }
}

// out[o][k] = (in[o][k] * w[k], 0)  (real lines -> complex, per-column weight)
__global__ void k_lines_real_in(const float* __restrict__ in, int64_t total, int64_t n,
                                const double* __restrict__ w, float2* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x)
        out[e] = make_float2((float)((double)in[e] * w[e % n]), 0.f);
}

// out[o][k] = Re(in[o][k]) * w[k]
__global__ void k_lines_real_out(const float2* __restrict__ in, int64_t total, int64_t n,
                                 const double* __restrict__ w, float* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x)
        out[e] = (float)((double)in[e].x * w[e % n]);
}

// g -= mean of the outermost ring of an nu x nv frame (grangeat.py:167-169):
// one block sums the ring in float64, then every element is shifted
__global__ void k_ring_mean(const float* __restrict__ g, int nu, int nv, double* __restrict__ mean) {
    const int nring = (nu == 1 || nv == 1) ? nu * nv : 2 * nu + 2 * nv - 4;
    double acc = 0.0;
    for (int r = threadIdx.x; r < nring; r += blockDim.x) {
        int u, v;
        if (nu == 1 || nv == 1) {
            u = r / nv;
            v = r % nv;
        } else if (r < nv) {
            u = 0;
            v = r;
        } else if (r < 2 * nv) {
            u = nu - 1;
            v = r - nv;
        } else {
            const int k = r - 2 * nv;
            u = 1 + k / 2;
            v = (k & 1) ? nv - 1 : 0;
        }
        acc += (double)g[(int64_t)u * nv + v];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        mean[0] = t / nring;
    }
}

__global__ void k_sub_mean(float* __restrict__ g, int64_t n, const double* __restrict__ mean) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        g[e] = (float)((double)g[e] - mean[0]);
}

static unsigned stream_grid(int64_t total) {
    const int64_t b = (total + 255) / 256;
    return (unsigned)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace cbn

using namespace cbn;

extern "C" {

int cbn_line_weight(void* data, int64_t outer, int64_t n, int64_t inner, const double* w,
                    void* stream) {
    try {
        CBN_REQUIRE(data && w && outer >= 1 && n >= 1 && inner >= 1, "bad argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<double2> wd;
        wd.upload(reinterpret_cast<const double2*>(w), (size_t)n, s);
        const int64_t total = outer * n * inner;
        k_line_weight<<<stream_grid(total), 256, 0, s>>>(static_cast<float2*>(data), total, n, inner,
                                                         wd.p);
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));  // wd is freed on return
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_node_phase(void* values, const double* nodes, int64_t m, int32_t d, const double* shift,
                   int32_t conj, const double* w, int64_t w_inner, void* stream) {
    try {
        CBN_REQUIRE(values && nodes && shift && m >= 1 && d >= 1 && d <= 3, "bad argument");
        CBN_REQUIRE(!w || w_inner >= 1, "bad weight stride");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<double> nd, wd;
        nd.upload(nodes, (size_t)(m * d), s);
        if (w) wd.upload(w, (size_t)((m + w_inner - 1) / w_inner), s);
        const double s0 = shift[0], s1 = d > 1 ? shift[1] : 0.0, s2 = d > 2 ? shift[2] : 0.0;
        k_node_phase<<<stream_grid(m), 256, 0, s>>>(static_cast<float2*>(values), nd.p, m, d, s0, s1,
                                                    s2, conj ? -1.0 : 1.0, w ? wd.p : nullptr,
                                                    w ? w_inner : 1);
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_trilinear_transfer(int32_t n_rho, int32_t n_theta, int32_t n_phi, double delta_rho,
                           double voxel_mm, double* out, void* stream) {
    try {
        CBN_REQUIRE(out && n_rho >= 1 && n_theta >= 1 && n_phi >= 1 && delta_rho > 0.0,
                    "bad argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int64_t total = (int64_t)n_rho * n_theta * n_phi;
        k_trilinear_transfer<<<stream_grid(total), 256, 0, s>>>(out, n_rho, n_theta, n_phi,
                                                                delta_rho, voxel_mm);
        CBN_LAUNCH_CHECK();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_lines_real_in(const float* in, int64_t outer, int64_t n, const double* w, void* out,
                      void* stream) {
    try {
        CBN_REQUIRE(in && w && out && outer >= 1 && n >= 1, "bad argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<double> wd;
        wd.upload(w, (size_t)n, s);
        const int64_t total = outer * n;
        k_lines_real_in<<<stream_grid(total), 256, 0, s>>>(in, total, n, wd.p,
                                                          static_cast<float2*>(out));
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_lines_real_out(const void* in, int64_t outer, int64_t n, const double* w, float* out,
                       void* stream) {
    try {
        CBN_REQUIRE(in && w && out && outer >= 1 && n >= 1, "bad argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<double> wd;
        wd.upload(w, (size_t)n, s);
        const int64_t total = outer * n;
        k_lines_real_out<<<stream_grid(total), 256, 0, s>>>(static_cast<const float2*>(in), total,
                                                           n, wd.p, out);
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_frame_ring_center(float* g, int32_t nu, int32_t nv, void* stream) {
    try {
        CBN_REQUIRE(g && nu >= 1 && nv >= 1, "bad argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<double> mean(1);
        k_ring_mean<<<1, 256, 0, s>>>(g, nu, nv, mean.p);
        CBN_LAUNCH_CHECK();
        k_sub_mean<<<stream_grid((int64_t)nu * nv), 256, 0, s>>>(g, (int64_t)nu * nv, mean.p);
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
