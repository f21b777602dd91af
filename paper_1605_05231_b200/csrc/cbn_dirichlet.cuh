// Resample method B (resampling.py:126-196, nufft.py:285-298): truncated
// centred periodic-sinc interpolation directly on the rho-padded lattice --
// T = side_lobes + 1 taps per axis, complex weights, no FFT and no plan state
// beyond the targets.
//
//   first = ceil(pos - T/2)                 (resampling.py:128, exact integer)
//   t     = pos - (first + k)
//   w     = dirichlet(t, n) * exp(-2 pi i (n//2) t / n)
//   dirichlet(t, n) = exp(i pi t (n-1)/n) * sin(pi t) / (n sin(pi t / n)),
//                     cos(pi t) / cos(pi t / n) where |n sin(pi t / n)| < 1e-9
//   cols  = (first + k) mod n
//
// apply:      y = sum_abc w0[a] w1[b] w2[c] x[c0[a], c1[b], c2[c]]   (152-160)
// transpose:  x[...] += conj(w0 w1 w2) y                              (176-189)
// Weights are evaluated in float64 and applied in float32 complex.
#pragma once

#include <type_traits>

#include "cbn_common.cuh"
#include "cbn_runtime.h"

namespace cbn {

constexpr int kMaxDirTaps = 8;

template <int T>
CBN_D void dirichlet_taps(double pos, int n, int (&cols)[T], float2 (&w)[T]) {
    const double first = ceil(pos - (double)T / 2.0);
    const double nd = (double)n;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const double off = first + (double)k;
        const double t = pos - off;
        const double pt = kPi * t;
        const double den = nd * sin(pt / nd);
        const double ratio = fabs(den) < 1e-9 ? cos(pt) / cos(pt / nd) : sin(pt) / den;
        // exp(i pi t (n-1)/n) * exp(-2 pi i (n//2) t / n)
        const double ang = pt * (nd - 1.0) / nd - 2.0 * kPi * (double)(n / 2) * t / nd;
        double sn, cs;
        sincos(ang, &sn, &cs);
        w[k] = make_float2((float)(ratio * cs), (float)(ratio * sn));
        long long c = (long long)off % n;
        cols[k] = (int)(c < 0 ? c + n : c);
    }
}

// positions straight from a (m, 3) fractional target array (rho, theta, phi),
// rho shifted by the padding (resampling.py:143-144)
struct ExplicitPos {
    const double* tg;
    int pad;
    CBN_D void position(int64_t i, double (&pos)[3], bool& valid) const {
        pos[0] = tg[i * 3 + 0] + (double)pad;
        pos[1] = tg[i * 3 + 1];
        pos[2] = tg[i * 3 + 2];
        valid = true;
    }
};

// axis extents (rho padded, theta, phi) and element strides of the padded lattice
struct DirGrid {
    int n[3];
    int64_t st[3];
};

// apply (gather).  Out: complex values, or Re() * tscale[i % n_t] zeroed where
// the target is invalid (the forward projector's store, pipeline.py:136-137)
template <int T, class Pos>
__global__ void __launch_bounds__(256)
k_dir_gather(const float2* __restrict__ x, DirGrid g, Pos src, int64_t m,
             float2* __restrict__ cout, float* __restrict__ rout,
             const float* __restrict__ tscale, int n_t) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double pos[3];
    bool valid;
    src.position(i, pos, valid);
    int c0[T], c1[T], c2[T];
    float2 w0[T], w1[T], w2[T];
    dirichlet_taps<T>(pos[0], g.n[0], c0, w0);
    dirichlet_taps<T>(pos[1], g.n[1], c1, w1);
    dirichlet_taps<T>(pos[2], g.n[2], c2, w2);
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int a = 0; a < T; ++a) {
#pragma unroll
        for (int b = 0; b < T; ++b) {
            const float2 wab = cmul(w0[a], w1[b]);
            const float2* row = x + c0[a] * g.st[0] + c1[b] * g.st[1];
#pragma unroll
            for (int c = 0; c < T; ++c) {
                const float2 wk = cmul(wab, w2[c]);
                const float2 v = __ldg(row + c2[c] * g.st[2]);
                acc.x = fmaf(wk.x, v.x, fmaf(-wk.y, v.y, acc.x));
                acc.y = fmaf(wk.x, v.y, fmaf(wk.y, v.x, acc.y));
            }
        }
    }
    if (cout) cout[i] = acc;
    if (rout) {
        float r = valid ? acc.x : 0.f;
        if (tscale) r *= tscale[i % n_t];
        rout[i] = r;
    }
}

// transpose (spread).  Values complex (cin) or real (rin, invalid targets
// skipped); with `den`, also the transposed validity mask (value 1)
template <int T, class Pos>
__global__ void __launch_bounds__(256)
k_dir_spread(float2* __restrict__ x, float2* __restrict__ den, DirGrid g, Pos src, int64_t m,
             const float2* __restrict__ cin, const float* __restrict__ rin) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double pos[3];
    bool valid;
    src.position(i, pos, valid);
    if (!valid) return;
    const float2 y = !x ? make_float2(0.f, 0.f) : (cin ? cin[i] : make_float2(rin[i], 0.f));
    if (y.x == 0.f && y.y == 0.f && !den) return;
    int c0[T], c1[T], c2[T];
    float2 w0[T], w1[T], w2[T];
    dirichlet_taps<T>(pos[0], g.n[0], c0, w0);
    dirichlet_taps<T>(pos[1], g.n[1], c1, w1);
    dirichlet_taps<T>(pos[2], g.n[2], c2, w2);
#pragma unroll
    for (int a = 0; a < T; ++a) {
#pragma unroll
        for (int b = 0; b < T; ++b) {
            const float2 wab = cmul(w0[a], w1[b]);
            const int64_t row = c0[a] * g.st[0] + c1[b] * g.st[1];
#pragma unroll
            for (int c = 0; c < T; ++c) {
                const float2 wk = cmul(wab, w2[c]);     // conj(wk) * y
                const int64_t e = row + c2[c] * g.st[2];
                if (x && (y.x != 0.f || y.y != 0.f))
                    atomicAdd(x + e, make_float2(wk.x * y.x + wk.y * y.y, wk.x * y.y - wk.y * y.x));
                if (den) atomicAdd(den + e, make_float2(wk.x, -wk.y));
            }
        }
    }
}

template <class F>
auto dispatch_taps(int T, F&& f) {
    switch (T) {
        case 1: return f(std::integral_constant<int, 1>{});
        case 2: return f(std::integral_constant<int, 2>{});
        case 3: return f(std::integral_constant<int, 3>{});
        case 4: return f(std::integral_constant<int, 4>{});
        case 5: return f(std::integral_constant<int, 5>{});
        case 6: return f(std::integral_constant<int, 6>{});
        case 7: return f(std::integral_constant<int, 7>{});
        case 8: return f(std::integral_constant<int, 8>{});
        default: throw Error(CBN_EINVAL, "side_lobes must give 1..8 taps per axis");
    }
}

}  // namespace cbn
