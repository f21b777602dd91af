// Host-side dtype conversion for the drop-in operators (plumbing, no numerics):
// the reference API is float64 numpy in and out, the device computes in
// float32, so every call converts on the host between the caller's arrays and
// the plan's pinned staging buffers.  Done here with OpenMP threads (outside the
// Python interpreter lock) at memory bandwidth: per-frame numpy calls from a
// Python thread pool spent most of their time in task dispatch.
#include <immintrin.h>
#include <omp.h>

#include <cstdint>
#include <cstdlib>

#include "cbn_runtime.h"

namespace {

// Conversion team: all cores but two by default.  The calling thread spins on
// CUDA events, a second host thread feeds the copies, and the driver has its
// own threads; with one conversion thread per core, a descheduled team member
// stalled whole calls (20 drop-in forward calls at config 2 on 16 cores:
// median 13.3 ms, worst 17-31 ms with 16 threads; median 12.8-13.0 ms, worst
// 13.2 ms with 14).  OMP_NUM_THREADS below that still wins.
int team(int32_t threads) {
    if (threads > 0) return threads;
    static const int n = [] {
        const int hw = omp_get_num_procs(), m = omp_get_max_threads();
        const int want = hw > 4 ? hw - 2 : hw;
        return m < want ? (m > 0 ? m : 1) : want;
    }();
    return n;
}

// float32 -> float64 with non-temporal stores: the result (2x the input) is
// written once and not read back by this code, so the lines skip the
// read-for-ownership (measured 1.5-1.9x on the 94 MB -> 189 MB frames)
__attribute__((target("avx2"))) void widen_stream_avx2(const float* s, double* d, int64_t n) {
    int64_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31)) {
        d[i] = (double)s[i];
        ++i;
    }
    for (; i + 8 <= n; i += 8) {
        const __m256 v = _mm256_loadu_ps(s + i);
        _mm256_stream_pd(d + i, _mm256_cvtps_pd(_mm256_castps256_ps128(v)));
        _mm256_stream_pd(d + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)));
    }
    for (; i < n; ++i) d[i] = (double)s[i];
    _mm_sfence();
}

// float64 -> float32 with non-temporal stores (the pinned staging buffer is
// written once and read by the DMA engine, not by this code)
__attribute__((target("avx2"))) void narrow_stream_avx2(const double* s, float* d, int64_t n) {
    int64_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31)) {
        d[i] = (float)s[i];
        ++i;
    }
    for (; i + 8 <= n; i += 8) {
        const __m128 a = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i));
        const __m128 b = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i + 4));
        _mm256_stream_ps(d + i, _mm256_set_m128(b, a));
    }
    for (; i < n; ++i) d[i] = (float)s[i];
    _mm_sfence();
}

bool narrow_stream_on() {
    static const bool on = [] {
        // on by default (drop-in forward call 12.76 / 12.94 -> 12.46 / 12.43 ms on
        // the GPU box's 16 cores); CBN_NT_NARROW=0 keeps the plain loop
        const char* e = std::getenv("CBN_NT_NARROW");
        return !(e && e[0] == '0') && __builtin_cpu_supports("avx2");
    }();
    return on;
}

// tasks 0..tasks-1 over the team.  Calls of a few million elements (the
// chunks and view blocks of the projector calls, ~1 ms each) take tasks
// dynamically: a thread that loses its core for a moment then holds back one
// 16 Ki task, not a fixed share of the array (it removed the stalled calls of
// the drop-in operators).  Large arrays (config 4's 10^8 values) keep the
// static split, whose long contiguous runs per thread stream faster (800-830
// against 630 Msamples/s through the numpy API).
constexpr int64_t kDynamicBelowTasks = 2048;   // 32 Mi elements

template <class Body>
void for_tasks(int64_t tasks, int32_t threads, Body body) {
    if (tasks < kDynamicBelowTasks) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(team(threads))
        for (int64_t t = 0; t < tasks; ++t) body(t);
    } else {
#pragma omp parallel for schedule(static) num_threads(team(threads))
        for (int64_t t = 0; t < tasks; ++t) body(t);
    }
}

}  // namespace

extern "C" {

// dst[k * elems + i] = (float)src[k][i] for the n_src arrays src[0..n_src)
int cbn_host_gather_f64_to_f32(const double* const* src, int64_t n_src, int64_t elems, float* dst,
                               int32_t threads) {
    try {
        CBN_REQUIRE(src && dst && n_src >= 0 && elems >= 0, "bad argument");
        for (int64_t k = 0; k < n_src; ++k) CBN_REQUIRE(src[k], "null source array");
        // blocks of 16 Ki elements across all arrays, so a few large frames
        // and many small ones both spread evenly over the team
        constexpr int64_t B = 1 << 14;
        const int64_t per = (elems + B - 1) / B;
        const int64_t tasks = n_src * per;
        const bool stream = narrow_stream_on();
        for_tasks(tasks, threads, [=](int64_t t) {
            const int64_t k = t / per, b = t - k * per;
            const int64_t lo = b * B, hi = lo + B < elems ? lo + B : elems;
            const double* s = src[k];
            float* d = dst + k * elems;
            if (stream) {
                narrow_stream_avx2(s + lo, d + lo, hi - lo);
                return;
            }
            for (int64_t i = lo; i < hi; ++i) d[i] = (float)s[i];
        });
        return CBN_OK;
    } catch (const std::exception& e) {
        return cbn::fail(e);
    }
}

// dst[i] = (double)src[i]  (float32 result -> float64 numpy)
int cbn_host_f32_to_f64(const float* src, double* dst, int64_t n, int32_t threads) {
    try {
        CBN_REQUIRE(src && dst && n >= 0, "bad argument");
        constexpr int64_t B = 1 << 14;
        const int64_t tasks = (n + B - 1) / B;
        static const bool avx2 = __builtin_cpu_supports("avx2");
        for_tasks(tasks, threads, [=](int64_t t) {
            const int64_t lo = t * B, hi = lo + B < n ? lo + B : n;
            if (avx2) {
                widen_stream_avx2(src + lo, dst + lo, hi - lo);
                return;
            }
            for (int64_t i = lo; i < hi; ++i) dst[i] = (double)src[i];
        });
        return CBN_OK;
    } catch (const std::exception& e) {
        return cbn::fail(e);
    }
}

// dst[i] = (float)src[i]  (float64 numpy -> float32 staging)
int cbn_host_f64_to_f32(const double* src, float* dst, int64_t n, int32_t threads) {
    return cbn_host_gather_f64_to_f32(&src, 1, n, dst, threads);
}

}  // extern "C"
