// Host-side plan helpers: per-axis KB parameters and the on-device
// least-squares scaling fit (nufft.py:111-134,159-186).
#pragma once

#include "cbn_kernels.cuh"
#include "cbn_runtime.h"

namespace cbn {

struct AxisPlan {
    int N = 0, K = 0, J = 0;
    double beta = 0.0, i0beta = 1.0;
    KBAxis kb{};
};

// Beatty's rule (nufft.py:53-56), same float64 expression order.
double beatty_beta(int j, double alpha);
// K = N * ceil(sigma - 1e-12) (nufft.py:159); beta from K/N; KB polynomial.
AxisPlan make_axis(int N, int J, double sigma);
void fit_kb_pieces(KBAxis& kb, int J, double beta, double i0beta);
int oversample_mult(double sigma);

// Scratch for one scaling fit of up to kMaxLS rows.
constexpr int kMaxLS = 8192;
struct LSScratch {
    DevBuf<double> frac, wts, s64;
    void ensure(int nrows, int ndim, int stride) {
        frac.ensure((size_t)ndim * nrows);
        wts.ensure((size_t)ndim * nrows * kLSMaxJ);
        s64.ensure((size_t)ndim * stride);
    }
};

inline LSParams ls_params(int D, const AxisPlan* ax) {
    LSParams p{};
    p.ndim = D;
    for (int d = 0; d < D; ++d) {
        p.N[d] = ax[d].N;
        p.K[d] = ax[d].K;
        p.J[d] = ax[d].J;
        p.beta[d] = ax[d].beta;
        p.i0beta[d] = ax[d].i0beta;
    }
    return p;
}

// Fit the per-axis scalings for the node source `src` at sampled rows
// (device array), writing float64 into scratch.s64 (stride) and float32
// scaled by I0(beta) into s32 (stride) on the device.
template <int D, class Src>
void ls_fit(const Src& src, const int64_t* rows_dev, int nrows, const AxisPlan* ax,
            LSScratch& sc, float* s32, int stride, cudaStream_t s) {
    CBN_REQUIRE(nrows > 0 && nrows <= kMaxLS, "scaling fit needs 1..8192 rows");
    sc.ensure(nrows, D, stride);
    LSParams p = ls_params(D, ax);
    k_ls_samples<D, Src><<<(nrows + 127) / 128, 128, 0, s>>>(src, rows_dev, nrows, p, sc.frac.p,
                                                             sc.wts.p);
    CBN_LAUNCH_CHECK();
    int maxN = 0;
    for (int d = 0; d < D; ++d) maxN = ax[d].N > maxN ? ax[d].N : maxN;
    k_ls_fit<<<dim3(maxN, D), 256, 0, s>>>(sc.frac.p, sc.wts.p, nrows, p, sc.s64.p, stride);
    CBN_LAUNCH_CHECK();
    k_ls_finish<<<D, 256, 0, s>>>(sc.s64.p, stride, p, s32, stride);
    CBN_LAUNCH_CHECK();
}

// Remap tables for one axis (device arrays inside `idx`/`scale` at offset).
void build_table(int mode, int N, int K, const float* s32, int* idx, float* scale, cudaStream_t s);

template <class F>
auto dispatch_j(int J, F&& f) {
    switch (J) {
        case 2: return f(std::integral_constant<int, 2>{});
        case 3: return f(std::integral_constant<int, 3>{});
        case 4: return f(std::integral_constant<int, 4>{});
        case 5: return f(std::integral_constant<int, 5>{});
        case 6: return f(std::integral_constant<int, 6>{});
        case 7: return f(std::integral_constant<int, 7>{});
        case 8: return f(std::integral_constant<int, 8>{});
        default: throw Error(CBN_EUNSUPPORTED, "tap count must be 2..8 on the device path");
    }
}

inline unsigned blocks_for(int64_t m, int threads) { return (unsigned)((m + threads - 1) / threads); }

}  // namespace cbn
