// Host-side runtime for the C-ABI library: status codes, exceptions mapped to
// codes at the boundary, device buffers, and a cuFFT plan cache whose plans
// share one workspace (plans on one stream run back to back).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/cbnufft_b200.h"

namespace cbn {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
int fail(const std::exception& e);

#define CBN_REQUIRE(cond, msg)                                                   \
    do {                                                                         \
        if (!(cond)) throw ::cbn::Error(CBN_EINVAL, (msg));                      \
    } while (0)

#define CBN_CUDA(expr)                                                           \
    do {                                                                         \
        cudaError_t e_ = (expr);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            int code_ = e_ == cudaErrorMemoryAllocation ? CBN_ENOMEM : CBN_ECUDA; \
            throw ::cbn::Error(code_, std::string(#expr ": ") + cudaGetErrorString(e_)); \
        }                                                                        \
    } while (0)

#define CBN_CUFFT(expr)                                                          \
    do {                                                                         \
        cufftResult r_ = (expr);                                                 \
        if (r_ != CUFFT_SUCCESS) {                                               \
            int code_ = r_ == CUFFT_ALLOC_FAILED ? CBN_ENOMEM : CBN_ECUDA;       \
            throw ::cbn::Error(code_, std::string(#expr ": cufft error ") + std::to_string((int)r_)); \
        }                                                                        \
    } while (0)

extern std::atomic<long long> g_launches;
#define CBN_LAUNCH_CHECK()                                                       \
    do {                                                                         \
        ::cbn::g_launches.fetch_add(1, std::memory_order_relaxed);               \
        CBN_CUDA(cudaGetLastError());                                            \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count == n && p) return;
        release();
        if (count) CBN_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void upload(const T* host, size_t count, cudaStream_t s) {
        ensure(count);
        CBN_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    size_t bytes() const { return n * sizeof(T); }
};

// C2C float FFT plans keyed by geometry; one shared workspace per cache.
class FFTCache {
public:
    ~FFTCache();
    // rank-r transform of `batch` contiguous arrays of shape n[0..r-1] (row-major)
    cufftHandle get(int rank, const long long* n, long long batch);
    // 1D transforms of length n over `batch` lines with element stride / distance
    cufftHandle get_strided(long long n, long long batch, long long stride, long long dist);
    void exec(cufftHandle h, void* in, void* out, int direction, cudaStream_t s);
    // real-to-complex 1D transforms of `batch` contiguous lines of length n
    // (n/2 + 1 complex outputs per line, out of place)
    cufftHandle get_r2c(long long n, long long batch);
    void exec_r2c(cufftHandle h, const float* in, void* out, cudaStream_t s);
    // complex-to-real 3D transform of a [n0][n1][n2/2+1] half spectrum to
    // [n0][n1][n2] real (out of place)
    cufftHandle get_c2r3(const long long* n);
    // complex-to-real 2D transforms of `batch` [n0][n1/2+1] half spectra to
    // [n0][n1] real (out of place, contiguous batches)
    cufftHandle get_c2r2(const long long* n, long long batch);
    // real-to-complex 2D transforms of `batch` [n0][n1] reals to [n0][n1/2+1]
    // (out of place, contiguous batches; run with exec_r2c3)
    cufftHandle get_r2c2(const long long* n, long long batch);
    // real-to-complex 3D transform [n0][n1][n2] -> [n0][n1][n2/2+1] (out of place)
    cufftHandle get_r2c3(const long long* n);
    void exec_r2c3(cufftHandle h, const float* in, void* out, cudaStream_t s);
    void exec_c2r(cufftHandle h, const void* in, float* out, cudaStream_t s);
    void clear();

private:
    using Key = std::tuple<int, long long, long long, long long, long long, long long, long long>;
    std::map<Key, cufftHandle> plans_;
    DevBuf<char> work_;
    cufftHandle make(int rank, long long* n, long long batch, long long stride, long long dist,
                     cufftType type = CUFFT_C2C);
};

// [a, b) runs of grid indices taken from a remap table idx[0..n) (device array,
// copied to the host): positions=true -> the k with idx[k] >= 0 (a pad table's
// written cells); false -> the distinct values idx[k] >= 0 (a crop table's reads)
std::vector<std::pair<int, int>> index_runs(const int* idx_dev, int n, bool positions, cudaStream_t s);

// 3D C2C FFT of nbatch contiguous grids kd[0] x kd[1] x kd[2] when only the
// slowest-axis planes in `planes` matter on the sparse side: forward, the
// other planes are zero on input (2D FFTs of the listed planes, then the 1D
// FFT along the slowest axis); inverse, only the listed planes are read
// afterwards (1D FFT along the slowest axis, then 2D FFTs of those planes).
void fft3_pruned(FFTCache& fft, float2* g, const long long* kd, long long nbatch,
                 const std::vector<std::pair<int, int>>& planes, int direction, cudaStream_t s);

// Per-stage CUDA-event timing (enabled per plan; off by default).
class StageTimer {
public:
    ~StageTimer();
    bool on = false;
    void begin(const char* name, cudaStream_t s);
    void end(cudaStream_t s);
    // synchronises, folds recorded pairs into per-name totals
    void collect();
    void reset();
    std::vector<std::pair<std::string, double>> totals;   // name -> ms
    // algorithmic bytes per stage (roofline of the bench): compulsory HBM
    // bytes and on-chip tap bytes of the work the stage's kernels did,
    // accumulated while timing is on (DESIGN.md section 4 gives each formula)
    void add_bytes(const char* name, double hbm, double chip);
    struct Bytes { double hbm = 0, chip = 0; };
    std::vector<std::pair<std::string, Bytes>> bytes;
private:
    struct Rec { std::string name; cudaEvent_t a, b; };
    std::vector<Rec> recs_;
    std::vector<cudaEvent_t> pool_;
    cudaEvent_t get();
};

struct StageScope {
    StageTimer& t;
    cudaStream_t s;
    StageScope(StageTimer& t_, const char* name, cudaStream_t s_) : t(t_), s(s_) {
        if (t.on) t.begin(name, s);
    }
    ~StageScope() {
        if (t.on) t.end(s);
    }
};

}  // namespace cbn
