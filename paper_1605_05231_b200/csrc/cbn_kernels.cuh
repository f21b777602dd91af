// Templated NUFFT kernels shared by the generic plan and the projector.
//
// Node sources (`Src`) generate the wrapped float64 node of row i on the fly
// (explicit arrays, radial-line tables, umbrella planes), so the reference's
// dense (m, J^d) interpolation matrix (nufft.py:188-213) is never formed:
// only the integer first tap and the fp32 KB weights are computed per point.
//
// Src concept:
//   struct Aux;                                     // per-row side data
//   __device__ void node(int64_t i, double (&w)[D], Aux&) const;   // wrapped node
// Gather epilogue:  __device__ void put(int64_t i, float2 v, const double (&w)[D], const Aux&) const;
// Spread values:    __device__ float2 value(int64_t i, const double (&w)[D], const Aux&) const;
#pragma once

#include <vector>

#include "cbn_common.cuh"

namespace cbn {

struct KBSet {
    KBAxis ax[kMaxDim];
};

template <int D>
struct TapIndex {
    int first[D];
    double u[D];
};

template <int D, int J>
CBN_D void tap_setup(const KBSet& kb, const double (&w)[D], int (&first)[D], float (&wt)[D][J]) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
        double u = axis_coord(w[d], kb.ax[d].K, 0.5 * (double)kb.ax[d].J, first[d]);
        kb_weights<J>(kb.ax[d], u, first[d], wt[d]);
    }
}

// kb_weights from a precomputed polynomial argument y and edge-tap decision
// (point records of the projector's radial node sets)
template <int J>
CBN_D void kb_weights_y(const KBAxis& kb, float y, bool drop0, float (&w)[J]) {
#pragma unroll
    for (int p = 0; p < J; ++p) w[p] = kb.pp[p][kPPDeg];
#pragma unroll
    for (int k = kPPDeg - 1; k >= 0; --k)
#pragma unroll
        for (int p = 0; p < J; ++p) w[p] = fmaf(w[p], y, kb.pp[p][k]);
    if (drop0) w[0] = 0.0f;
}


CBN_D int wrapc(int c, int K) {
    c = c < 0 ? c + K : c;
    return c >= K ? c - K : c;
}

// e / d by multiply-shift for the small shared-memory region indices: exact
// while e * (m d - 2^20) < 2^20 and e * m < 2^32 (regions of < 8K cells, d >= 16
// or e < 4096)
struct FastDiv {
    unsigned m;
    int d;
    CBN_D explicit FastDiv(int d_) : m(((1u << 20) + (unsigned)d_ - 1) / (unsigned)d_), d(d_) {}
    CBN_D int div(int e) const { return (int)(((unsigned)e * m) >> 20); }
};

// the nonzero taps of w and of its mirror wm are mirror images (mod K): same
// count, and the mirror's lowest nonzero tap is minus the node's highest.  The
// reference's exact support test can drop the edge tap on one side only
// (u - J/2 an integer on one side, a rounding ulp off it on the other).
CBN_D bool mirror_taps_match(int K, int J, double w, double wm) {
    int f, fm;
    const double u = axis_coord(w, K, 0.5 * J, f);
    const double um = axis_coord(wm, K, 0.5 * J, fm);
    const double edge = 0.5 * J * (1.0 - 1e-12);
    const int e0 = (u - f) >= edge && !kb_inside(u - f, J) ? 1 : 0;
    const int e0m = (um - fm) >= edge && !kb_inside(um - fm, J) ? 1 : 0;
    return e0 == e0m && wrap_index(fm + e0m + f + J - 1, K) == 0;
}


// ------------------------------------------------------------------ gather
// y_i = sum_taps w0 w1 w2 G[c0, c1, c2]  (SparseInterpolator.apply, nufft.py:68-74)
template <int D, int J, class Src, class Epi>
__global__ void __launch_bounds__(256)
k_gather(const float2* __restrict__ grid, KBSet kb, Src src, Epi epi, int64_t m) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double w[D];
    typename Src::Aux aux;
    src.node(i, w, aux);
    int first[D];
    float wt[D][J];
    tap_setup<D, J>(kb, w, first, wt);
    float2 acc = make_float2(0.f, 0.f);
    if constexpr (D == 1) {
        const int K0 = kb.ax[0].K;
#pragma unroll
        for (int a = 0; a < J; ++a) {
            float2 g = __ldg(grid + wrapc(first[0] + a, K0));
            acc.x = fmaf(wt[0][a], g.x, acc.x);
            acc.y = fmaf(wt[0][a], g.y, acc.y);
        }
    } else if constexpr (D == 2) {
        const int K0 = kb.ax[0].K, K1 = kb.ax[1].K;
        int c1[J];
#pragma unroll
        for (int b = 0; b < J; ++b) c1[b] = wrapc(first[1] + b, K1);
#pragma unroll
        for (int a = 0; a < J; ++a) {
            const float2* row = grid + (size_t)wrapc(first[0] + a, K0) * K1;
            float2 r = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < J; ++b) {
                float2 g = __ldg(row + c1[b]);
                r.x = fmaf(wt[1][b], g.x, r.x);
                r.y = fmaf(wt[1][b], g.y, r.y);
            }
            acc.x = fmaf(wt[0][a], r.x, acc.x);
            acc.y = fmaf(wt[0][a], r.y, acc.y);
        }
    } else {
        const int K0 = kb.ax[0].K, K1 = kb.ax[1].K, K2 = kb.ax[2].K;
        int c2[J];
#pragma unroll
        for (int c = 0; c < J; ++c) c2[c] = wrapc(first[2] + c, K2);
#pragma unroll
        for (int a = 0; a < J; ++a) {
            const float2* plane = grid + (size_t)wrapc(first[0] + a, K0) * K1 * K2;
            float2 pa = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < J; ++b) {
                const float2* row = plane + (size_t)wrapc(first[1] + b, K1) * K2;
                float2 r = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < J; ++c) {
                    float2 g = __ldg(row + c2[c]);
                    r.x = fmaf(wt[2][c], g.x, r.x);
                    r.y = fmaf(wt[2][c], g.y, r.y);
                }
                pa.x = fmaf(wt[1][b], r.x, pa.x);
                pa.y = fmaf(wt[1][b], r.y, pa.y);
            }
            acc.x = fmaf(wt[0][a], pa.x, acc.x);
            acc.y = fmaf(wt[0][a], pa.y, acc.y);
        }
    }
    epi.put(i, acc, w, aux);
}

// ------------------------------------------------------------------ spread
// G[c] += w0 w1 w2 y_i   (SparseInterpolator.apply_adjoint, nufft.py:76-85)
template <int D, int J, class Src>
__global__ void __launch_bounds__(256)
k_spread(float2* __restrict__ grid, KBSet kb, Src src, int64_t m) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double w[D];
    typename Src::Aux aux;
    src.node(i, w, aux);
    float2 v = src.value(i, w, aux);
    if (v.x == 0.f && v.y == 0.f) return;
    int first[D];
    float wt[D][J];
    tap_setup<D, J>(kb, w, first, wt);
    if constexpr (D == 1) {
        const int K0 = kb.ax[0].K;
#pragma unroll
        for (int a = 0; a < J; ++a)
            atomicAdd(grid + wrapc(first[0] + a, K0), cscale(v, wt[0][a]));
    } else if constexpr (D == 2) {
        const int K0 = kb.ax[0].K, K1 = kb.ax[1].K;
#pragma unroll
        for (int a = 0; a < J; ++a) {
            float2* row = grid + (size_t)wrapc(first[0] + a, K0) * K1;
            float2 va = cscale(v, wt[0][a]);
#pragma unroll
            for (int b = 0; b < J; ++b) atomicAdd(row + wrapc(first[1] + b, K1), cscale(va, wt[1][b]));
        }
    } else {
        const int K0 = kb.ax[0].K, K1 = kb.ax[1].K, K2 = kb.ax[2].K;
        int c2[J];
#pragma unroll
        for (int c = 0; c < J; ++c) c2[c] = wrapc(first[2] + c, K2);
#pragma unroll
        for (int a = 0; a < J; ++a) {
            float2* plane = grid + (size_t)wrapc(first[0] + a, K0) * K1 * K2;
            float2 va = cscale(v, wt[0][a]);
#pragma unroll
            for (int b = 0; b < J; ++b) {
                float2* row = plane + (size_t)wrapc(first[1] + b, K1) * K2;
                float2 vb = cscale(va, wt[1][b]);
#pragma unroll
                for (int c = 0; c < J; ++c) atomicAdd(row + c2[c], cscale(vb, wt[2][c]));
            }
        }
    }
}

// ------------------------------------------------------ least-squares scaling
// _ls_scaling (nufft.py:111-134) on the plan's sampled rows (nufft.py:163-168).
constexpr int kLSMaxJ = 16;

struct LSParams {
    int ndim;
    int N[kMaxDim];
    int K[kMaxDim];
    int J[kMaxDim];
    double beta[kMaxDim];
    double i0beta[kMaxDim];
};

// per sampled row and axis: frac = u - first and the float64 KB weights
template <int D, class Src>
__global__ void k_ls_samples(Src src, const int64_t* __restrict__ rows, int n, LSParams p,
                             double* __restrict__ frac, double* __restrict__ wts) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    double w[D];
    typename Src::Aux aux;
    src.node(rows[s], w, aux);
#pragma unroll
    for (int d = 0; d < D; ++d) {
        int first;
        double u = axis_coord(w[d], p.K[d], 0.5 * (double)p.J[d], first);
        frac[d * n + s] = dsub(u, (double)first);
        for (int q = 0; q < p.J[d]; ++q)
            wts[((size_t)d * n + s) * kLSMaxJ + q] =
                kb_value_f64(dsub(u, (double)(first + q)), p.J[d], p.beta[d]);
    }
}

// one block per (frequency n, axis): num / den reductions over the samples
__global__ void k_ls_fit(const double* __restrict__ frac, const double* __restrict__ wts, int n,
                         LSParams p, double* __restrict__ s_raw, int s_stride);

// one block per axis: clip at 1e-8 max, write float64 and scaled float32 copies
__global__ void k_ls_finish(double* s_raw, int s_stride, LSParams p, float* s32, int s32_stride);

// ----------------------------------------------------------- separable remap
// dst[e] = gain * prod_d scale_d[e_d] * src[sum_d idx_d[e_d] * sstride_d]
// (zero when any idx is negative).  Implements deapodise+pad (nufft.py:226-230),
// crop+deapodise (nufft.py:245-247) and the resampler's fftshift/ifftshift
// index maps (resampling.py:146,175) as one table-driven pass.
struct RemapAxis {
    const int* idx;
    const float* scale;
    int n;            // destination extent
    int64_t sstride;  // source stride (elements)
};

enum RemapMode { kStoreC = 0, kAccumC = 1, kStoreRe = 2 };

template <int D, class SrcT, int MODE>
__global__ void k_remap(const SrcT* __restrict__ src, void* __restrict__ dst, RemapAxis a0,
                        RemapAxis a1, RemapAxis a2, float gain) {
    // D == 3: (x: a2 fastest, y: a1, z: a0); D == 2: (x: a1, y: a0); D == 1: x: a0
    int e_last = blockIdx.x * blockDim.x + threadIdx.x;
    RemapAxis ax[3] = {a0, a1, a2};
    const RemapAxis& fast = ax[D - 1];
    if (e_last >= fast.n) return;
    int e[3] = {0, 0, 0};
    e[D - 1] = e_last;
    if (D >= 2) e[D - 2] = blockIdx.y;
    if (D >= 3) e[0] = blockIdx.z;
    float sc = gain;
    int64_t so = 0;
    bool zero = false;
    size_t doff = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        int id = ax[d].idx[e[d]];
        zero |= id < 0;
        so += (int64_t)id * ax[d].sstride;
        sc *= ax[d].scale[e[d]];
        doff = doff * (size_t)ax[d].n + (size_t)e[d];
    }
    float2 v = make_float2(0.f, 0.f);
    if (!zero) {
        if constexpr (sizeof(SrcT) == sizeof(float)) {
            v.x = sc * (float)src[so];
        } else {
            float2 g = src[so];
            v = make_float2(g.x * sc, g.y * sc);
        }
    }
    if constexpr (MODE == kStoreC) {
        static_cast<float2*>(dst)[doff] = v;
    } else if constexpr (MODE == kAccumC) {
        float2* p = static_cast<float2*>(dst) + doff;
        float2 o = *p;
        *p = make_float2(o.x + v.x, o.y + v.y);
    } else {
        static_cast<float*>(dst)[doff] = v.x;
    }
}

// 3D pad to the half spectrum of a real transform: out[e0][e1][e2], e2 <=
// n2 / 2, holds conj of the Hermitian part of the padded grid P,
// (conj(P[e]) + P[-e]) / 2, so that a complex-to-real FFT of it gives
// Re(forward FFT of P) (the only part the resample gather reads).
__global__ void k_remap_herm3(const float2* __restrict__ src, float2* __restrict__ dst,
                              RemapAxis a0, RemapAxis a1, RemapAxis a2, float gain);

// The same remaps restricted to the destination cells a pad table can make
// non-zero (compact per-axis index lists `l`, lengths nl; the caller zeroes
// the rest of the destination first; grid (nl2 / 256, nl1, nl0)): k_remap (3D, kStoreRe / kStoreC) and
// k_remap_herm3 (list on the half axis limited to <= n2 / 2).
template <class SrcT, int MODE>
__global__ void k_remap_list3(const SrcT* __restrict__ src, void* __restrict__ dst, RemapAxis a0,
                              RemapAxis a1, RemapAxis a2, const int* __restrict__ l0,
                              const int* __restrict__ l1, const int* __restrict__ l2, int n2l,
                              float gain) {
    // grid (n2l / 256, n1l, n0l)
    const int q2 = blockIdx.x * blockDim.x + threadIdx.x;
    if (q2 >= n2l) return;
    const int e0 = l0[blockIdx.z], e1 = l1[blockIdx.y], e2 = l2[q2];
    const int id0 = a0.idx[e0], id1 = a1.idx[e1], id2 = a2.idx[e2];
    const size_t doff = ((size_t)e0 * a1.n + e1) * a2.n + e2;
    float2 v = make_float2(0.f, 0.f);
    if (id0 >= 0 && id1 >= 0 && id2 >= 0) {
        const float sc = gain * a0.scale[e0] * a1.scale[e1] * a2.scale[e2];
        const int64_t so = (int64_t)id0 * a0.sstride + (int64_t)id1 * a1.sstride + (int64_t)id2 * a2.sstride;
        if constexpr (sizeof(SrcT) == sizeof(float)) {
            v.x = sc * (float)src[so];
        } else {
            const float2 g = src[so];
            v = make_float2(g.x * sc, g.y * sc);
        }
    }
    if constexpr (MODE == kStoreRe) static_cast<float*>(dst)[doff] = v.x;
    else static_cast<float2*>(dst)[doff] = v;
}

__global__ void k_remap_herm3_tile(const float2* __restrict__ src, float2* __restrict__ dst,
                                   RemapAxis a0, RemapAxis a1, RemapAxis a2,
                                   const int* __restrict__ l0, const int* __restrict__ l1,
                                   const int* __restrict__ l2, int n0l, int n2l, float gain);
__global__ void k_remap_herm3_list(const float2* __restrict__ src, float2* __restrict__ dst,
                                   RemapAxis a0, RemapAxis a1, RemapAxis a2,
                                   const int* __restrict__ l0, const int* __restrict__ l1,
                                   const int* __restrict__ l2, int n2l, float gain);

// destination indices a pad table (kTabPad / kTabPadShift: source n, output
// k = (n - N//2) mod K) can fill, with their mirrors -k when `mirror`, and
// only k <= K/2 when `half` (host)
std::vector<int> pad_positions(int N, int K, bool mirror, bool half);
// pad_positions(N, K, mirror, false) as sorted runs [a, b)
std::vector<std::pair<int, int>> pad_runs(int N, int K, bool mirror);

// Table modes for k_build_table.
enum TableMode {
    kTabPad = 0,      // g in [0,K): source n of the rolled placement (n - N//2) mod K, scale s[n]
    kTabCrop = 1,     // n in [0,N): source g = (n - N//2) mod K, scale s[n]
    kTabPadShift = 2, // as kTabPad, but the source is the unshifted FFT: f = (n - N//2) mod N
    kTabCropShift = 3 // k in [0,N): n = (k + N//2) mod N, source g = (n - N//2) mod K, scale s[n]
};

__global__ void k_build_table(int mode, int N, int K, const float* __restrict__ s32, int* idx,
                              float* scale);

// Host-side launch helper for k_remap.
template <class SrcT, int MODE>
void launch_remap(int D, const SrcT* src, void* dst, const RemapAxis* ax, float gain,
                  cudaStream_t s) {
    RemapAxis z{nullptr, nullptr, 1, 0};
    RemapAxis a0 = ax[0], a1 = D > 1 ? ax[1] : z, a2 = D > 2 ? ax[2] : z;
    int fastn = ax[D - 1].n;
    dim3 block(256);
    dim3 grid((fastn + 255) / 256, D >= 2 ? ax[D - 2].n : 1, D >= 3 ? ax[0].n : 1);
    if (D == 1) k_remap<1, SrcT, MODE><<<grid, block, 0, s>>>(src, dst, a0, a1, a2, gain);
    else if (D == 2) k_remap<2, SrcT, MODE><<<grid, block, 0, s>>>(src, dst, a0, a1, a2, gain);
    else k_remap<3, SrcT, MODE><<<grid, block, 0, s>>>(src, dst, a0, a1, a2, gain);
}

}  // namespace cbn
