#include <cstdlib>

#include "cbn_runtime.h"

#include <algorithm>
#include <cstring>

namespace cbn {

static thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

void set_last_error(const std::string& msg) { g_last_error = msg; }

int fail(const std::exception& e) {
    set_last_error(e.what());
    if (auto* ce = dynamic_cast<const Error*>(&e)) return ce->code;
    if (dynamic_cast<const std::bad_alloc*>(&e)) return CBN_ENOMEM;
    return CBN_ECUDA;
}

FFTCache::~FFTCache() { clear(); }

void FFTCache::clear() {
    for (auto& kv : plans_) cufftDestroy(kv.second);
    plans_.clear();
    work_.release();
}

cufftHandle FFTCache::make(int rank, long long* n, long long batch, long long stride, long long dist,
                           cufftType type) {
    cufftHandle h;
    CBN_CUFFT(cufftCreate(&h));
    static const bool auto_ws = [] {
        const char* e = std::getenv("CBN_FFT_AUTOALLOC");
        return e && e[0] == '1';
    }();
    if (!auto_ws) CBN_CUFFT(cufftSetAutoAllocation(h, 0));
    size_t ws = 0;
    long long* embed = nullptr;
    long long emb[3];
    if (stride != 1 || rank == 1) {
        for (int i = 0; i < rank; ++i) emb[i] = n[i];
        embed = emb;
    }
    cufftResult r;
    if (type == CUFFT_R2C && rank >= 2) {
        r = cufftMakePlanMany64(h, rank, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_R2C, batch, &ws);
    } else if (type == CUFFT_C2R) {
        r = cufftMakePlanMany64(h, rank, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_C2R, batch, &ws);
    } else if (type == CUFFT_R2C) {
        long long ie[1] = {n[0]}, oe[1] = {n[0] / 2 + 1};
        r = cufftMakePlanMany64(h, 1, n, ie, 1, n[0], oe, 1, n[0] / 2 + 1, CUFFT_R2C, batch, &ws);
    } else {
        r = cufftMakePlanMany64(h, rank, n, embed, stride, dist, embed, stride, dist, CUFFT_C2C,
                                batch, &ws);
    }
    if (r != CUFFT_SUCCESS) {
        cufftDestroy(h);
        throw Error(r == CUFFT_ALLOC_FAILED ? CBN_ENOMEM : CBN_ECUDA,
                    "cufftMakePlanMany64 failed: " + std::to_string((int)r));
    }
    if (auto_ws) return h;
    if (ws > work_.n) {
        work_.alloc(ws);
        for (auto& kv : plans_) CBN_CUFFT(cufftSetWorkArea(kv.second, work_.p));
    }
    CBN_CUFFT(cufftSetWorkArea(h, work_.p));
    return h;
}

cufftHandle FFTCache::get(int rank, const long long* n, long long batch) {
    CBN_REQUIRE(rank >= 1 && rank <= 3, "fft rank must be 1..3");
    long long dims[3] = {0, 0, 0};
    long long total = 1;
    for (int i = 0; i < rank; ++i) {
        dims[i] = n[i];
        total *= n[i];
    }
    Key key{rank, dims[0], dims[1], dims[2], batch, 1, total};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    cufftHandle h = make(rank, dims, batch, 1, total);
    plans_[key] = h;
    return h;
}

cufftHandle FFTCache::get_strided(long long n, long long batch, long long stride, long long dist) {
    Key key{-1, n, 0, 0, batch, stride, dist};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    long long dims[1] = {n};
    cufftHandle h = make(1, dims, batch, stride, dist);
    plans_[key] = h;
    return h;
}

cufftHandle FFTCache::get_r2c(long long n, long long batch) {
    Key key{-2, n, 0, 0, batch, 1, n};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    long long dims[1] = {n};
    cufftHandle h = make(1, dims, batch, 1, n, CUFFT_R2C);
    plans_[key] = h;
    return h;
}

cufftHandle FFTCache::get_c2r3(const long long* n) {
    Key key{-3, n[0], n[1], n[2], 1, 1, 0};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    long long dims[3] = {n[0], n[1], n[2]};
    cufftHandle h = make(3, dims, 1, 1, 0, CUFFT_C2R);
    plans_[key] = h;
    return h;
}

cufftHandle FFTCache::get_c2r2(const long long* n, long long batch) {
    Key key{-5, n[0], n[1], 0, batch, 1, 0};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    long long dims[2] = {n[0], n[1]};
    cufftHandle h = make(2, dims, batch, 1, 0, CUFFT_C2R);
    plans_[key] = h;
    return h;
}

cufftHandle FFTCache::get_r2c2(const long long* n, long long batch) {
    Key key{-6, n[0], n[1], 0, batch, 1, 0};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    long long dims[2] = {n[0], n[1]};
    cufftHandle h = make(2, dims, batch, 1, 0, CUFFT_R2C);
    plans_[key] = h;
    return h;
}

cufftHandle FFTCache::get_r2c3(const long long* n) {
    Key key{-4, n[0], n[1], n[2], 1, 1, 0};
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
    long long dims[3] = {n[0], n[1], n[2]};
    cufftHandle h = make(3, dims, 1, 1, 0, CUFFT_R2C);
    plans_[key] = h;
    return h;
}

void FFTCache::exec_r2c3(cufftHandle h, const float* in, void* out, cudaStream_t s) {
    CBN_CUFFT(cufftSetStream(h, s));
    CBN_CUFFT(cufftExecR2C(h, const_cast<cufftReal*>(in), static_cast<cufftComplex*>(out)));
}

void FFTCache::exec_c2r(cufftHandle h, const void* in, float* out, cudaStream_t s) {
    CBN_CUFFT(cufftSetStream(h, s));
    CBN_CUFFT(cufftExecC2R(h, const_cast<cufftComplex*>(static_cast<const cufftComplex*>(in)), out));
}

void FFTCache::exec_r2c(cufftHandle h, const float* in, void* out, cudaStream_t s) {
    CBN_CUFFT(cufftSetStream(h, s));
    CBN_CUFFT(cufftExecR2C(h, const_cast<cufftReal*>(in), static_cast<cufftComplex*>(out)));
}

void FFTCache::exec(cufftHandle h, void* in, void* out, int direction, cudaStream_t s) {
    CBN_CUFFT(cufftSetStream(h, s));
    CBN_CUFFT(cufftExecC2C(h, static_cast<cufftComplex*>(in), static_cast<cufftComplex*>(out),
                           direction));
}

std::vector<std::pair<int, int>> index_runs(const int* idx_dev, int n, bool positions, cudaStream_t s) {
    std::vector<int> h((size_t)n);
    CBN_CUDA(cudaMemcpyAsync(h.data(), idx_dev, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    std::vector<int> ks;
    for (int k = 0; k < n; ++k)
        if (h[(size_t)k] >= 0) ks.push_back(positions ? k : h[(size_t)k]);
    std::sort(ks.begin(), ks.end());
    ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
    std::vector<std::pair<int, int>> runs;
    for (int k : ks) {
        if (!runs.empty() && runs.back().second == k) ++runs.back().second;
        else runs.emplace_back(k, k + 1);
    }
    return runs;
}

void fft3_pruned(FFTCache& fft, float2* g, const long long* kd, long long nbatch,
                 const std::vector<std::pair<int, int>>& planes, int direction, cudaStream_t s) {
    const long long plane = kd[1] * kd[2], total = kd[0] * plane;
    const long long k2[2] = {kd[1], kd[2]};
    cufftHandle col = fft.get_strided(kd[0], plane, plane, 1);
    for (long long b = 0; b < nbatch; ++b) {
        float2* gb = g + b * total;
        if (direction == CUFFT_FORWARD) {
            for (const auto& r : planes)
                fft.exec(fft.get(2, k2, r.second - r.first), gb + r.first * plane,
                         gb + r.first * plane, direction, s);
            fft.exec(col, gb, gb, direction, s);
        } else {
            fft.exec(col, gb, gb, direction, s);
            for (const auto& r : planes)
                fft.exec(fft.get(2, k2, r.second - r.first), gb + r.first * plane,
                         gb + r.first * plane, direction, s);
        }
    }
}

StageTimer::~StageTimer() {
    for (auto& r : recs_) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : pool_) cudaEventDestroy(e);
}

cudaEvent_t StageTimer::get() {
    if (!pool_.empty()) {
        cudaEvent_t e = pool_.back();
        pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    CBN_CUDA(cudaEventCreate(&e));
    return e;
}

void StageTimer::begin(const char* name, cudaStream_t s) {
    Rec r{name, get(), nullptr};
    CBN_CUDA(cudaEventRecord(r.a, s));
    recs_.push_back(r);
}

void StageTimer::end(cudaStream_t s) {
    for (auto it = recs_.rbegin(); it != recs_.rend(); ++it) {
        if (!it->b) {
            it->b = get();
            CBN_CUDA(cudaEventRecord(it->b, s));
            return;
        }
    }
}

void StageTimer::collect() {
    for (auto& r : recs_) {
        if (!r.b) continue;
        CBN_CUDA(cudaEventSynchronize(r.b));
        float ms = 0.f;
        CBN_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        bool found = false;
        for (auto& kv : totals)
            if (kv.first == r.name) {
                kv.second += ms;
                found = true;
            }
        if (!found) totals.emplace_back(r.name, (double)ms);
        pool_.push_back(r.a);
        pool_.push_back(r.b);
    }
    recs_.clear();
}

void StageTimer::reset() {
    collect();
    totals.clear();
    bytes.clear();
}

void StageTimer::add_bytes(const char* name, double hbm, double chip) {
    if (!on) return;
    for (auto& kv : bytes)
        if (kv.first == name) {
            kv.second.hbm += hbm;
            kv.second.chip += chip;
            return;
        }
    Bytes b;
    b.hbm = hbm;
    b.chip = chip;
    bytes.emplace_back(name, b);
}

}  // namespace cbn

extern "C" long long cbn_launch_count(void) { return cbn::g_launches.load(); }

extern "C" const char* cbn_last_error(void) { return cbn::g_last_error.c_str(); }
