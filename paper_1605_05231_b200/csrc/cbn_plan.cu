#include <cmath>

#include "cbn_plan.h"

namespace cbn {

double beatty_beta(int j, double alpha) {
    // np.pi * np.sqrt(max((j / alpha) ** 2 * (alpha - 0.5) ** 2 - 0.8, 0.0))
    double arg = std::pow((double)j / alpha, 2.0) * std::pow(alpha - 0.5, 2.0) - 0.8;
    return kPi * std::sqrt(arg > 0.0 ? arg : 0.0);
}

int oversample_mult(double sigma) { return (int)std::ceil(sigma - 1e-12); }

AxisPlan make_axis(int N, int J, double sigma) {
    AxisPlan a;
    a.N = N;
    a.J = J;
    a.K = N * oversample_mult(sigma);
    a.beta = beatty_beta(J, (double)a.K / (double)N);
    a.i0beta = i0_series(a.beta);
    a.kb.J = J;
    a.kb.K = a.K;
    fit_kb_pieces(a.kb, J, a.beta, a.i0beta);
    return a;
}

// Chebyshev interpolation of each tap's weight on its unit interval, converted
// to monomials in y in (-1, 1]; checked against the float64 series on a fine grid.
void fit_kb_pieces(KBAxis& kb, int J, double beta, double i0b) {
    CBN_REQUIRE(J >= 1 && J <= kMaxJ, "tap count must be 1..8");
    constexpr int n = kPPDeg + 1;
    auto weight = [&](int p, double y) {
        double x = 0.5 * (y + 1.0) + 0.5 * J - 1.0 - p;
        double q = 2.0 * x / J;
        double t = 1.0 - q * q;
        return t > 0.0 ? i0_series(beta * std::sqrt(t)) / i0b : (t == 0.0 ? 1.0 / i0b : 0.0);
    };
    for (int p = 0; p < kMaxJ; ++p)
        for (int k = 0; k < n; ++k) kb.pp[p][k] = 0.f;
    double worst = 0.0;
    for (int p = 0; p < J; ++p) {
        double f[n], c[n];
        for (int i = 0; i < n; ++i) f[i] = weight(p, std::cos(kPi * (i + 0.5) / n));
        for (int k = 0; k < n; ++k) {
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += f[i] * std::cos(kPi * k * (i + 0.5) / n);
            c[k] = (k == 0 ? 1.0 : 2.0) * s / n;
        }
        // Chebyshev series -> monomials: T_k via the recurrence on coefficient vectors
        double mono[n] = {0}, tkm1[n] = {0}, tk[n] = {0}, tkp1[n];
        tkm1[0] = 1.0;        // T0
        tk[1] = 1.0;          // T1
        mono[0] += c[0];
        for (int j = 0; j < n; ++j) mono[j] += c[1] * tk[j];
        for (int k = 2; k < n; ++k) {
            for (int j = 0; j < n; ++j) tkp1[j] = (j ? 2.0 * tk[j - 1] : 0.0) - tkm1[j];
            for (int j = 0; j < n; ++j) mono[j] += c[k] * tkp1[j];
            for (int j = 0; j < n; ++j) {
                tkm1[j] = tk[j];
                tk[j] = tkp1[j];
            }
        }
        for (int k = 0; k < n; ++k) kb.pp[p][k] = (float)mono[k];
        for (int i = 0; i <= 2000; ++i) {
            double y = -1.0 + 2.0 * i / 2000.0;
            double acc = 0.0;
            for (int k = n - 1; k >= 0; --k) acc = acc * y + (double)kb.pp[p][k];
            worst = std::max(worst, std::fabs(acc - weight(p, y)));
        }
    }
    CBN_REQUIRE(worst < 5e-7, "KB piecewise fit too coarse: " + std::to_string(worst));
}

void build_table(int mode, int N, int K, const float* s32, int* idx, float* scale, cudaStream_t s) {
    int n = (mode == kTabPad || mode == kTabPadShift) ? K : N;
    k_build_table<<<(n + 255) / 256, 256, 0, s>>>(mode, N, K, s32, idx, scale);
    CBN_LAUNCH_CHECK();
}

}  // namespace cbn
