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
    // I0(beta sqrt(t)) / I0(beta) = sum_k (beta^2/4)^k / (k!)^2 t^k / I0(beta)
    const double y = 0.25 * a.beta * a.beta;
    double term = 1.0;
    int deg = 0;
    a.kb.poly[0] = (float)(1.0 / a.i0beta);
    for (int k = 1; k <= kMaxPoly; ++k) {
        term *= y / ((double)k * (double)k);
        a.kb.poly[k] = (float)(term / a.i0beta);
        deg = k;
        if (k > y && term / a.i0beta < 1e-10) break;
    }
    a.kb.deg = deg;
    return a;
}

void build_table(int mode, int N, int K, const float* s32, int* idx, float* scale, cudaStream_t s) {
    int n = (mode == kTabPad || mode == kTabPadShift) ? K : N;
    k_build_table<<<(n + 255) / 256, 256, 0, s>>>(mode, N, K, s32, idx, scale);
    CBN_LAUNCH_CHECK();
}

}  // namespace cbn
