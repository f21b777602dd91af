// Common device helpers for the B200 NUFFT cone-beam projector.
//
// * Bit-exact float64 index math of the reference plan (nufft.py:104-108,
//   171-179): every operation on that path is an explicit round-to-nearest
//   intrinsic so nvcc can never contract it into an FMA, which would change
//   the last bit and with it the integer first-tap index.
// * Kaiser-Bessel weights (nufft.py:36-41) evaluated in fp32 as a positive-
//   coefficient polynomial in t = 1 - (2x/J)^2, normalised by I0(beta); the
//   per-axis deapodisation absorbs the I0(beta) factor.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define CBN_HD __host__ __device__ __forceinline__
#define CBN_D __device__ __forceinline__

// Device-side checks of the check build (make check -> libcbnufft_b200_check.so,
// -DCBN_BOUNDS_CHECK): every binned kernel asserts that a point's first tap
// lies in its bin's tile (so all J^d taps stay inside the shared-memory
// region), the window gather asserts its buffer indices, the cell gather its
// row ids.  compute-sanitizer is not available on this GPU pool; this build
// plus the parity tests is the memory check.  Off (no code) otherwise.
#ifdef CBN_BOUNDS_CHECK
#include <cstdio>
#define CBN_DCHECK(cond, what)                                                            \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("CBN_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                          \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define CBN_DCHECK(cond, what) \
    do {                       \
    } while (0)
#endif

namespace cbn {

// numpy's float64 pi and 2*pi (exact doubles)
constexpr double kPi = 3.141592653589793115997963468544185161590576171875;
constexpr double kTwoPi = 6.28318530717958623199592693708837032318115234375;

constexpr int kMaxPoly = 48;   // KB polynomial degree cap
constexpr int kMaxDim = 3;

// ---------------------------------------------------------------- complex
CBN_HD float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
CBN_HD float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
CBN_HD float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
CBN_HD float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// --------------------------------------------------- exact float64 helpers
CBN_D double dadd(double a, double b) { return __dadd_rn(a, b); }
CBN_D double dsub(double a, double b) { return __dsub_rn(a, b); }
CBN_D double dmul(double a, double b) { return __dmul_rn(a, b); }
CBN_D double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Exact fmod(a, b) for b > 0 and |a / b| well inside 2^52: with q = trunc(a/b)
// the remainder a - q b is exactly representable, so one fma returns it
// exactly; q from a * (1/b) can be off by one only when a/b is within an ulp
// of an integer, which the range checks detect and fix.  Bit-identical to
// fmod (checked against numpy in tests/test_gpu_nufft.py) at a fraction of
// libdevice fmod's cost.
CBN_D double fmod_pos(double a, double b, double inv_b) {
    const double q = trunc(a * inv_b);
    double r = fma(-q, b, a);
    if (a >= 0.0) {
        if (r < 0.0) r = fma(-(q - 1.0), b, a);
        else if (r >= b) r = fma(-(q + 1.0), b, a);
    } else {
        if (r > 0.0) r = fma(-(q + 1.0), b, a);
        else if (r <= -b) r = fma(-(q - 1.0), b, a);
    }
    return r;
}

// numpy.remainder for float64 with a positive divisor (npy_divmod):
// fmod, then move to the divisor's sign; zero becomes +0.
CBN_D double np_mod_pos(double a, double b, double inv_b) {
    double m = fmod_pos(a, b, inv_b);
    if (m != 0.0) {
        if (m < 0.0) m = dadd(m, b);
    } else {
        m = 0.0;
    }
    return m;
}

CBN_D double np_mod(double a, double b) { return np_mod_pos(a, b, 1.0 / b); }

constexpr double kInvTwoPi = 0.15915494309189534561;   // only steers the quotient guess

// mod(x + pi, 2 pi) - pi   (nufft.py:104-108)
CBN_D double wrap_pi(double x) { return dsub(np_mod_pos(dadd(x, kPi), kTwoPi, kInvTwoPi), kPi); }

// u = mod(w, 2 pi) * K / (2 pi); snap |u - rint(u)| < 1e-9; first = ceil(u - J/2)
// (nufft.py:173-176).  Returns u; first through the reference.
CBN_D double axis_coord(double w, int K, double half_j, int& first) {
    double u = ddiv(dmul(np_mod_pos(w, kTwoPi, kInvTwoPi), (double)K), kTwoPi);
    double r = rint(u);
    if (fabs(dsub(u, r)) < 1e-9) u = r;
    first = (int)ceil(dsub(u, half_j));
    return u;
}

CBN_HD int wrap_index(int c, int K) {
    c %= K;
    return c < 0 ? c + K : c;
}

// ------------------------------------------------------------ KB kernel
constexpr int kMaxJ = 8;
constexpr int kPPDeg = 15;     // piecewise-polynomial degree (fitted to < 2e-8 of the peak)

struct KBAxis {
    int J;          // taps
    int K;          // oversampled length
    // Tap p's weight I0(beta sqrt(1 - (2x/J)^2)) / I0(beta) at x = frac - p,
    // frac = u - first in (J/2 - 1, J/2], as a polynomial in
    // y = 2 (frac - J/2 + 1) - 1 in (-1, 1]: pp[p][k] y^k.
    float pp[kMaxJ][kPPDeg + 1];
};

// Exact support decision of the reference: arg = 1 - ((2x)/J)^2 > 0.
// |2x| < J - margin is certainly inside, |2x| >= J certainly outside;
// the thin band between uses the reference's exact float64 sequence.
CBN_D bool kb_inside(double x, int J) {
    double ax2 = fabs(dmul(2.0, x));
    double jj = (double)J;
    if (ax2 < jj * (1.0 - 1e-12)) return true;
    if (ax2 >= jj) return false;
    double q = ddiv(dmul(2.0, x), jj);
    return dsub(1.0, dmul(q, q)) > 0.0;
}

// Weights of the J taps first..first+J-1 for grid coordinate u (fp64).
// All taps share one Horner sweep (J independent FMA chains, coefficients are
// compile-time offsets into the kernel-parameter bank).  Only tap 0 can reach
// the support edge (x = J/2 when u - J/2 is an integer); there the reference's
// exact float64 support test decides (nufft.py:39-41).
// J (the template) is the plan's largest per-axis tap count: an axis with
// fewer taps (kb.J < J, nufft.py:137 takes per-axis j) has zero polynomials
// for taps kb.J..J-1 (fit_kb_pieces), so those weights vanish; the
// polynomial argument and the support test use the axis's own tap count.
template <int J>
CBN_D void kb_weights(const KBAxis& kb, double u, int first, float (&w)[J]) {
    const double fr = dsub(u, (double)first);
    const int Ja = kb.J;
    const float y = (float)(2.0 * (fr - (0.5 * Ja - 1.0)) - 1.0);
#pragma unroll
    for (int p = 0; p < J; ++p) w[p] = kb.pp[p][kPPDeg];
#pragma unroll
    for (int k = kPPDeg - 1; k >= 0; --k)
#pragma unroll
        for (int p = 0; p < J; ++p) w[p] = fmaf(w[p], y, kb.pp[p][k]);
    if (fr >= 0.5 * Ja * (1.0 - 1e-12) && !kb_inside(fr, Ja)) w[0] = 0.0f;
}

// float64 I0 by its (all-positive) power series; |z| <= ~25 here.
CBN_HD double i0_series(double z) {
    double y = 0.25 * z * z;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 200; ++k) {
        term *= y / ((double)k * (double)k);
        sum += term;
        if (term < 1e-17 * sum) break;
    }
    return sum;
}

// float64 KB value exactly as the reference decides its support (nufft.py:36-41)
CBN_D double kb_value_f64(double x, int J, double beta) {
    double q = ddiv(dmul(2.0, x), (double)J);
    double arg = dsub(1.0, dmul(q, q));
    if (!(arg > 0.0)) return 0.0;
    return i0_series(beta * sqrt(arg));
}

}  // namespace cbn
