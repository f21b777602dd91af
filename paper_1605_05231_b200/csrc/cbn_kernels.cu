// Non-template kernels shared by the plans: scaling fit and remap tables.
#include "cbn_kernels.cuh"

namespace cbn {

__global__ void k_ls_fit(const double* __restrict__ frac, const double* __restrict__ wts, int n,
                         LSParams p, double* __restrict__ s_raw, int s_stride) {
    const int d = blockIdx.y;
    const int k = blockIdx.x;
    if (k >= p.N[d]) return;
    const int N = p.N[d], K = p.K[d], J = p.J[d];
    // nu = (k - N//2) / K cycles per oversampled sample (nufft.py:122)
    const double nu = (double)(k - N / 2) / (double)K;
    double er[kLSMaxJ], ei[kLSMaxJ];
    for (int q = 0; q < J; ++q) sincospi(-2.0 * q * nu, &ei[q], &er[q]);
    double num = 0.0, den = 0.0;
    for (int s = threadIdx.x; s < n; s += blockDim.x) {
        const double* ws = wts + ((size_t)d * n + s) * kLSMaxJ;
        double rr = 0.0, ri = 0.0;
        for (int q = 0; q < J; ++q) {
            rr += ws[q] * er[q];
            ri += ws[q] * ei[q];
        }
        den += rr * rr + ri * ri;
        double sn, cs;
        sincospi(2.0 * frac[(size_t)d * n + s] * nu, &sn, &cs);
        // sum_p w_p cos(2 pi (frac - p) nu) = Re(e^{2 pi i frac nu} * resp)
        num += cs * rr - sn * ri;
    }
    __shared__ double sh_num[32], sh_den[32];
    for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sh_num[warp] = num;
        sh_den[warp] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += sh_num[w];
            b += sh_den[w];
        }
        s_raw[(size_t)d * s_stride + k] = a / fmax(b, 1e-300);
    }
}

__global__ void k_ls_finish(double* s_raw, int s_stride, LSParams p, float* s32, int s32_stride) {
    const int d = blockIdx.x;
    const int N = p.N[d];
    double* s = s_raw + (size_t)d * s_stride;
    double mx = -1e308;
    for (int k = threadIdx.x; k < N; k += blockDim.x) mx = fmax(mx, s[k]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = sh[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
        sh[0] = m;
    }
    __syncthreads();
    const double floor_v = 1e-8 * sh[0];
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double v = fmax(s[k], floor_v);
        s[k] = v;
        s32[(size_t)d * s32_stride + k] = (float)(v * p.i0beta[d]);
    }
}

__global__ void k_build_table(int mode, int N, int K, const float* __restrict__ s32, int* idx,
                              float* scale) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int h = N / 2;
    if (mode == kTabPad || mode == kTabPadShift) {
        if (e >= K) return;
        int n = -1;
        if (e < N - h) n = e + h;
        else if (e >= K - h) n = e - K + h;
        if (n < 0) {
            idx[e] = -1;
            scale[e] = 0.f;
            return;
        }
        int src = n;
        if (mode == kTabPadShift) src = ((n - h) % N + N) % N;
        idx[e] = src;
        scale[e] = s32 ? s32[n] : 1.f;
    } else {
        if (e >= N) return;
        int n = e;
        if (mode == kTabCropShift) n = (e + h) % N;
        int g = ((n - h) % K + K) % K;
        idx[e] = g;
        scale[e] = s32 ? s32[n] : 1.f;
    }
}

__global__ void k_remap_herm3(const float2* __restrict__ src, float2* __restrict__ dst,
                              RemapAxis a0, RemapAxis a1, RemapAxis a2, float gain) {
    const int h2 = a2.n / 2 + 1;
    const int e2 = blockIdx.x * blockDim.x + threadIdx.x;
    if (e2 >= h2) return;
    const int e[3] = {(int)blockIdx.z, (int)blockIdx.y, e2};
    const RemapAxis ax[3] = {a0, a1, a2};
    float2 v[2];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        float sc = gain;
        int64_t so = 0;
        bool zero = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int k = e[d];
            if (side) k = k == 0 ? 0 : ax[d].n - k;     // (-k) mod n
            const int id = ax[d].idx[k];
            zero |= id < 0;
            so += (int64_t)id * ax[d].sstride;
            sc *= ax[d].scale[k];
        }
        const float2 g = zero ? make_float2(0.f, 0.f) : src[so];
        v[side] = make_float2(g.x * sc, g.y * sc);
    }
    // conj(P[e]) + P[-e], halved
    dst[((size_t)e[0] * a1.n + e[1]) * h2 + e2] =
        make_float2(0.5f * (v[0].x + v[1].x), 0.5f * (v[1].y - v[0].y));
}

// k_remap_herm3_list through 32 x 32 (axis 0 x axis 2) shared-memory tiles per
// axis-1 cell, for sources whose axis 0 is the contiguous one (a0.sstride ==
// 1): loads run along axis 0, stores along axis 2.  Grid (ceil(n2l / 32),
// ceil(n0l / 32), n1l), block (32, 8).
__global__ void k_remap_herm3_tile(const float2* __restrict__ src, float2* __restrict__ dst,
                                   RemapAxis a0, RemapAxis a1, RemapAxis a2,
                                   const int* __restrict__ l0, const int* __restrict__ l1,
                                   const int* __restrict__ l2, int n0l, int n2l, float gain) {
    __shared__ float2 tile[2][32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int q00 = blockIdx.y * 32, q20 = blockIdx.x * 32;
    const int e1 = l1[blockIdx.z];
    const int h2 = a2.n / 2 + 1;
    const int e1m = e1 == 0 ? 0 : a1.n - e1;
    const int id1[2] = {a1.idx[e1], a1.idx[e1m]};
    const float sc1[2] = {gain * a1.scale[e1], gain * a1.scale[e1m]};
    // load: tx along axis 0 (contiguous source), ty over axis-2 rows
    const int q0 = q00 + tx;
    int e0 = 0, k0[2] = {0, 0};
    if (q0 < n0l) {
        e0 = l0[q0];
        k0[0] = e0;
        k0[1] = e0 == 0 ? 0 : a0.n - e0;
    }
    for (int r = ty; r < 32; r += blockDim.y) {
        const int q2 = q20 + r;
        if (q0 >= n0l || q2 >= n2l) continue;
        const int e2 = l2[q2];
        const int k2[2] = {e2, e2 == 0 ? 0 : a2.n - e2};
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const int i0 = a0.idx[k0[side]], i2 = a2.idx[k2[side]];
            float2 g = make_float2(0.f, 0.f);
            if (i0 >= 0 && id1[side] >= 0 && i2 >= 0) {
                const float sc = sc1[side] * a0.scale[k0[side]] * a2.scale[k2[side]];
                const float2 x = src[(int64_t)i0 + (int64_t)id1[side] * a1.sstride +
                                     (int64_t)i2 * a2.sstride];
                g = make_float2(x.x * sc, x.y * sc);
            }
            tile[side][r][tx] = g;
        }
    }
    __syncthreads();
    // store: tx along axis 2, conj(P[e]) + P[-e], halved
    const int q2 = q20 + tx;
    if (q2 >= n2l) return;
    const int e2 = l2[q2];
    for (int r = ty; r < 32; r += blockDim.y) {
        const int qq0 = q00 + r;
        if (qq0 >= n0l) break;
        const float2 v0 = tile[0][tx][r], v1 = tile[1][tx][r];
        dst[((size_t)l0[qq0] * a1.n + e1) * h2 + e2] =
            make_float2(0.5f * (v0.x + v1.x), 0.5f * (v1.y - v0.y));
    }
}

__global__ void k_remap_herm3_list(const float2* __restrict__ src, float2* __restrict__ dst,
                                   RemapAxis a0, RemapAxis a1, RemapAxis a2,
                                   const int* __restrict__ l0, const int* __restrict__ l1,
                                   const int* __restrict__ l2, int n2l, float gain) {
    const int q2 = blockIdx.x * blockDim.x + threadIdx.x;
    if (q2 >= n2l) return;
    const int h2 = a2.n / 2 + 1;
    const int e[3] = {l0[blockIdx.z], l1[blockIdx.y], l2[q2]};
    const RemapAxis ax[3] = {a0, a1, a2};
    float2 v[2];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        float sc = gain;
        int64_t so = 0;
        bool zero = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int k = e[d];
            if (side) k = k == 0 ? 0 : ax[d].n - k;     // (-k) mod n
            const int id = ax[d].idx[k];
            zero |= id < 0;
            so += (int64_t)id * ax[d].sstride;
            sc *= ax[d].scale[k];
        }
        const float2 g = zero ? make_float2(0.f, 0.f) : src[so];
        v[side] = make_float2(g.x * sc, g.y * sc);
    }
    dst[((size_t)e[0] * a1.n + e[1]) * h2 + e[2]] =
        make_float2(0.5f * (v[0].x + v[1].x), 0.5f * (v[1].y - v[0].y));
}

std::vector<int> pad_positions(int N, int K, bool mirror, bool half) {
    std::vector<char> on((size_t)K, 0);
    const int h = N / 2;
    for (int n = 0; n < N; ++n) {
        const int k = ((n - h) % K + K) % K;
        on[(size_t)k] = 1;
        if (mirror) on[(size_t)((K - k) % K)] = 1;
    }
    std::vector<int> out;
    for (int k = 0; k < K; ++k)
        if (on[(size_t)k] && (!half || k <= K / 2)) out.push_back(k);
    return out;
}

std::vector<std::pair<int, int>> pad_runs(int N, int K, bool mirror) {
    std::vector<std::pair<int, int>> runs;
    for (int k : pad_positions(N, K, mirror, false)) {
        if (!runs.empty() && runs.back().second == k) runs.back().second = k + 1;
        else runs.emplace_back(k, k + 1);
    }
    return runs;
}

}  // namespace cbn
