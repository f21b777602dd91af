// Stand-alone resampling plan and centred radial FFT, for the module-level API
// of the reference (resampling.py:79-196, radon_fourier.py:117-135).
//
// cbn_resample mirrors ResamplePlan.  Method B (cbn_resample_create_b) keeps
// only the targets and runs the truncated periodic-sinc gather / spread of
// cbn_dirichlet.cuh on the padded lattice.  Method A: arbitrary fractional lattice
// targets, a generic NUFFT plan on the rho-padded lattice with nodes
// -2 pi pos / padded (resampling.py:97-102), and
//   apply:     pad(origin_avg(x)) -> fftn -> fftshift / size -> type 2   (146-148)
//   transpose: type 1 -> ifftshift -> ifftn -> crop rho -> origin_avg   (170-196)
// The reference multiplies by plan.phase and by _centered_shift_phase, whose
// product is exactly 1 (SURVEY finding 9); both are omitted.  Arrays use the
// reference layout (rho, theta, phi), rho slowest.
#include <mutex>

#include "cbn_dirichlet.cuh"
#include "cbn_plan.h"

extern "C" {
struct cbn_nufft_s;
int cbn_nufft_create(cbn_nufft_s** plan, int ndim, const int64_t* dims, const int32_t* taps,
                     double oversample_factor, const double* nodes, int64_t m,
                     const int64_t* ls_rows, int64_t n_ls, void* stream);
int cbn_nufft_destroy(cbn_nufft_s* plan);
int cbn_nufft_set_phase(cbn_nufft_s* plan, int32_t on);
int cbn_nufft_type2(cbn_nufft_s* plan, const void* x, void* y, void* stream);
int cbn_nufft_type1(cbn_nufft_s* plan, const void* y, void* x, void* stream);
}

namespace cbn {
namespace {

// x (n_rho, L) with L = n_theta * n_phi  ->  origin-averaged, rho-padded
// (n_rho + 2 pad, L); mean = average of row n_rho / 2
__global__ void k_rs_pad(const float2* __restrict__ x, int n_rho, int64_t L, int pad,
                         const double* __restrict__ mean, float2* __restrict__ out) {
    const int64_t total = (int64_t)(n_rho + 2 * pad) * L;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int r = (int)(e / L) - pad;
    const int64_t c = e % L;
    float2 v = make_float2(0.f, 0.f);
    if (r >= 0 && r < n_rho)
        v = (r == n_rho / 2) ? make_float2((float)mean[0], (float)mean[1]) : x[(int64_t)r * L + c];
    out[e] = v;
}

// row mean (complex, float64) of row `row` of a (rows, L) array, single block
__global__ void k_row_mean(const float2* __restrict__ x, int64_t L, int row, double scale,
                           double* __restrict__ out) {
    double re = 0, im = 0;
    for (int64_t c = threadIdx.x; c < L; c += blockDim.x) {
        float2 v = x[(int64_t)row * L + c];
        re += v.x;
        im += v.y;
    }
    __shared__ double sr[32], si[32];
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sr[threadIdx.x >> 5] = re;
        si[threadIdx.x >> 5] = im;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += sr[w];
            b += si[w];
        }
        out[0] = a * scale / (double)L;
        out[1] = b * scale / (double)L;
    }
}

// 3D (i)fftshift copy with scale: out[k] = in[(k + sh) mod n] per axis
__global__ void k_shift3(const float2* __restrict__ in, float2* __restrict__ out, int n0, int n1,
                         int n2, int s0, int s1, int s2, float scale) {
    const int64_t total = (int64_t)n0 * n1 * n2;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int k2 = (int)(e % n2);
    const int k1 = (int)((e / n2) % n1);
    const int k0 = (int)(e / ((int64_t)n1 * n2));
    const int j0 = (k0 + s0) % n0, j1 = (k1 + s1) % n1, j2 = (k2 + s2) % n2;
    const float2 v = in[((int64_t)j0 * n1 + j1) * n2 + j2];
    out[e] = make_float2(v.x * scale, v.y * scale);
}

// rho crop of a (n_rho + 2 pad, L) array with scale, then the origin row is
// replaced by its mean in a second pass
__global__ void k_rs_crop(const float2* __restrict__ in, int n_rho, int64_t L, int pad,
                          float scale, float2* __restrict__ out) {
    const int64_t total = (int64_t)n_rho * L;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const float2 v = in[e + (int64_t)pad * L];
    out[e] = make_float2(v.x * scale, v.y * scale);
}

__global__ void k_set_row(float2* __restrict__ x, int64_t L, int row,
                          const double* __restrict__ mean) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < L) x[(int64_t)row * L + c] = make_float2((float)mean[0], (float)mean[1]);
}

// centred FFT / IFFT along the fastest axis: pre ifftshift, transform, post fftshift, scale
__global__ void k_line_shift(const float2* __restrict__ in, float2* __restrict__ out, int n,
                             int64_t total, int shift, float scale) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int j = (int)(e % n);
    const int64_t line = e / n;
    const float2 v = in[line * n + (j + shift) % n];
    out[e] = make_float2(v.x * scale, v.y * scale);
}

}  // namespace
}  // namespace cbn

using namespace cbn;

struct cbn_resample_s {
    int n_rho = 0, n_theta = 0, n_phi = 0, pad = 0, dr = 0;
    int64_t m = 0;
    int method = 0;                 // 0: A (NUFFT), 1: B (truncated periodic sinc)
    int taps = 3;                   // method B: side_lobes + 1
    DevBuf<double> targets;         // method B: (m, 3) fractional indices
    cbn_nufft_s* plan = nullptr;
    FFTCache fft;
    DevBuf<float2> a, b;
    DevBuf<double> mean;
    ~cbn_resample_s() {
        if (plan) cbn_nufft_destroy(plan);
    }
};

static std::mutex g_fft_mu;
static FFTCache* g_fft = nullptr;

extern "C" {

int cbn_resample_create(cbn_resample_s** out, int32_t n_rho, int32_t n_theta, int32_t n_phi,
                        int32_t rho_pad, const int32_t* taps, double oversample_factor,
                        const double* targets, int64_t m, const int64_t* ls_rows, int64_t n_ls,
                        void* stream) {
    try {
        CBN_REQUIRE(out && taps && targets && m >= 1, "bad argument");
        CBN_REQUIRE(n_rho >= 2 && n_rho % 2 == 0 && n_theta >= 1 && n_phi >= 1, "bad radial spec");
        CBN_REQUIRE(rho_pad >= 0, "rho_pad must be >= 0");
        auto p = std::make_unique<cbn_resample_s>();
        p->n_rho = n_rho;
        p->n_theta = n_theta;
        p->n_phi = n_phi;
        p->pad = rho_pad;
        p->dr = n_rho + 2 * rho_pad;
        p->m = m;
        const double padded[3] = {(double)p->dr, (double)n_theta, (double)n_phi};
        std::vector<double> nodes((size_t)m * 3);
        for (int64_t i = 0; i < m; ++i)
            for (int d = 0; d < 3; ++d) {
                double pos = targets[i * 3 + d] + (d == 0 ? (double)rho_pad : 0.0);
                nodes[i * 3 + d] = (-2.0 * kPi) * pos / padded[d];   // resampling.py:99-101
            }
        const int64_t dims[3] = {p->dr, n_theta, n_phi};
        int st = cbn_nufft_create(&p->plan, 3, dims, taps, oversample_factor, nodes.data(), m,
                                  ls_rows, n_ls, stream);
        if (st != CBN_OK) return st;
        cbn_nufft_set_phase(p->plan, 0);
        const size_t big = (size_t)p->dr * n_theta * n_phi;
        p->a.alloc(big);
        p->b.alloc(big);
        p->mean.alloc(2);
        *out = p.release();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_resample_create_b(cbn_resample_s** out, int32_t n_rho, int32_t n_theta, int32_t n_phi,
                          int32_t rho_pad, int32_t side_lobes, const double* targets, int64_t m,
                          void* stream) {
    try {
        CBN_REQUIRE(out && targets && m >= 1, "bad argument");
        CBN_REQUIRE(n_rho >= 2 && n_rho % 2 == 0 && n_theta >= 1 && n_phi >= 1, "bad radial spec");
        CBN_REQUIRE(rho_pad >= 0, "rho_pad must be >= 0");
        CBN_REQUIRE(side_lobes >= 0 && side_lobes + 1 <= kMaxDirTaps, "side_lobes must be 0..7");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto p = std::make_unique<cbn_resample_s>();
        p->n_rho = n_rho;
        p->n_theta = n_theta;
        p->n_phi = n_phi;
        p->pad = rho_pad;
        p->dr = n_rho + 2 * rho_pad;
        p->m = m;
        p->method = 1;
        p->taps = side_lobes + 1;
        p->targets.upload(targets, (size_t)m * 3, s);
        const size_t big = (size_t)p->dr * n_theta * n_phi;
        p->a.alloc(big);
        p->mean.alloc(2);
        CBN_CUDA(cudaStreamSynchronize(s));
        *out = p.release();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_resample_destroy(cbn_resample_s* p) {
    delete p;
    return CBN_OK;
}

int cbn_resample_apply(cbn_resample_s* p, const void* data, void* values, void* stream) {
    try {
        CBN_REQUIRE(p && data && values, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int64_t L = (int64_t)p->n_theta * p->n_phi;
        const int64_t tot = (int64_t)p->dr * L;
        const float2* x = static_cast<const float2*>(data);
        k_row_mean<<<1, 256, 0, s>>>(x, L, p->n_rho / 2, 1.0, p->mean.p);
        CBN_LAUNCH_CHECK();
        k_rs_pad<<<blocks_for(tot, 256), 256, 0, s>>>(x, p->n_rho, L, p->pad, p->mean.p, p->a.p);
        CBN_LAUNCH_CHECK();
        if (p->method == 1) {
            const DirGrid g{{p->dr, p->n_theta, p->n_phi}, {L, (int64_t)p->n_phi, 1}};
            const ExplicitPos src{p->targets.p, p->pad};
            dispatch_taps(p->taps, [&](auto tc) {
                k_dir_gather<decltype(tc)::value><<<blocks_for(p->m, 256), 256, 0, s>>>(
                    p->a.p, g, src, p->m, static_cast<float2*>(values), nullptr, nullptr, 1);
                return 0;
            });
            CBN_LAUNCH_CHECK();
            return CBN_OK;
        }
        long long dims[3] = {p->dr, p->n_theta, p->n_phi};
        p->fft.exec(p->fft.get(3, dims, 1), p->a.p, p->a.p, CUFFT_FORWARD, s);
        // spectrum = fftshift(F) / size: out[k] = F[(k - n//2) mod n] = F[(k + n - n//2) mod n]
        k_shift3<<<blocks_for(tot, 256), 256, 0, s>>>(p->a.p, p->b.p, p->dr, p->n_theta, p->n_phi,
                                                      p->dr - p->dr / 2, p->n_theta - p->n_theta / 2,
                                                      p->n_phi - p->n_phi / 2, (float)(1.0 / (double)tot));
        CBN_LAUNCH_CHECK();
        return cbn_nufft_type2(p->plan, p->b.p, values, stream);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_resample_transpose(cbn_resample_s* p, const void* values, void* data, void* stream) {
    try {
        CBN_REQUIRE(p && data && values, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int64_t L = (int64_t)p->n_theta * p->n_phi;
        const int64_t tot = (int64_t)p->dr * L;
        if (p->method == 1) {
            CBN_CUDA(cudaMemsetAsync(p->a.p, 0, sizeof(float2) * tot, s));
            const DirGrid g{{p->dr, p->n_theta, p->n_phi}, {L, (int64_t)p->n_phi, 1}};
            const ExplicitPos src{p->targets.p, p->pad};
            dispatch_taps(p->taps, [&](auto tc) {
                k_dir_spread<decltype(tc)::value><<<blocks_for(p->m, 256), 256, 0, s>>>(
                    p->a.p, nullptr, g, src, p->m, static_cast<const float2*>(values), nullptr);
                return 0;
            });
            CBN_LAUNCH_CHECK();
            float2* out = static_cast<float2*>(data);
            const int64_t nout = (int64_t)p->n_rho * L;
            k_rs_crop<<<blocks_for(nout, 256), 256, 0, s>>>(p->a.p, p->n_rho, L, p->pad, 1.0f, out);
            CBN_LAUNCH_CHECK();
            k_row_mean<<<1, 256, 0, s>>>(out, L, p->n_rho / 2, 1.0, p->mean.p);
            CBN_LAUNCH_CHECK();
            k_set_row<<<blocks_for(L, 256), 256, 0, s>>>(out, L, p->n_rho / 2, p->mean.p);
            CBN_LAUNCH_CHECK();
            return CBN_OK;
        }
        int st = cbn_nufft_type1(p->plan, values, p->a.p, stream);
        if (st != CBN_OK) return st;
        // ifftshift: out[k] = in[(k + n//2) mod n]
        k_shift3<<<blocks_for(tot, 256), 256, 0, s>>>(p->a.p, p->b.p, p->dr, p->n_theta, p->n_phi,
                                                      p->dr / 2, p->n_theta / 2, p->n_phi / 2, 1.0f);
        CBN_LAUNCH_CHECK();
        long long dims[3] = {p->dr, p->n_theta, p->n_phi};
        p->fft.exec(p->fft.get(3, dims, 1), p->b.p, p->b.p, CUFFT_INVERSE, s);
        float2* out = static_cast<float2*>(data);
        const int64_t nout = (int64_t)p->n_rho * L;
        k_rs_crop<<<blocks_for(nout, 256), 256, 0, s>>>(p->b.p, p->n_rho, L, p->pad,
                                                        (float)(1.0 / (double)tot), out);
        CBN_LAUNCH_CHECK();
        k_row_mean<<<1, 256, 0, s>>>(out, L, p->n_rho / 2, 1.0, p->mean.p);
        CBN_LAUNCH_CHECK();
        k_set_row<<<blocks_for(L, 256), 256, 0, s>>>(out, L, p->n_rho / 2, p->mean.p);
        CBN_LAUNCH_CHECK();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// centred FFT (inverse = 0) or IFFT (inverse = 1) of `lines` contiguous lines of
// length n, times `scale` (radon_fourier.py:117-135: radial_fft scale = d_rho,
// radial_ifft scale = 1 / d_rho; the IFFT's 1/n is included here)
int cbn_radial_fft(void* data, int64_t n, int64_t lines, int32_t inverse, double scale,
                   void* stream) {
    try {
        CBN_REQUIRE(data && n >= 1 && lines >= 1, "bad argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int64_t tot = n * lines;
        DevBuf<float2> tmp((size_t)tot);
        float2* x = static_cast<float2*>(data);
        k_line_shift<<<blocks_for(tot, 256), 256, 0, s>>>(x, tmp.p, (int)n, tot, (int)(n / 2), 1.0f);
        CBN_LAUNCH_CHECK();
        {
            std::lock_guard<std::mutex> lk(g_fft_mu);
            if (!g_fft) g_fft = new FFTCache();
            long long nn[1] = {n};
            g_fft->exec(g_fft->get(1, nn, lines), tmp.p, tmp.p, inverse ? CUFFT_INVERSE : CUFFT_FORWARD, s);
        }
        const double sc = inverse ? scale / (double)n : scale;
        k_line_shift<<<blocks_for(tot, 256), 256, 0, s>>>(tmp.p, x, (int)n, tot, (int)(n - n / 2),
                                                          (float)sc);
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));   // tmp is freed on return
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
