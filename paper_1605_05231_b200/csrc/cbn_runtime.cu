#include "cbn_runtime.h"

#include <cstring>

namespace cbn {

static thread_local std::string g_last_error;

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

cufftHandle FFTCache::make(int rank, long long* n, long long batch, long long stride, long long dist) {
    cufftHandle h;
    CBN_CUFFT(cufftCreate(&h));
    CBN_CUFFT(cufftSetAutoAllocation(h, 0));
    size_t ws = 0;
    long long* embed = nullptr;
    long long emb[3];
    if (stride != 1 || rank == 1) {
        for (int i = 0; i < rank; ++i) emb[i] = n[i];
        embed = emb;
    }
    cufftResult r = cufftMakePlanMany64(h, rank, n, embed, stride, dist, embed, stride, dist,
                                        CUFFT_C2C, batch, &ws);
    if (r != CUFFT_SUCCESS) {
        cufftDestroy(h);
        throw Error(r == CUFFT_ALLOC_FAILED ? CBN_ENOMEM : CBN_ECUDA,
                    "cufftMakePlanMany64 failed: " + std::to_string((int)r));
    }
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

void FFTCache::exec(cufftHandle h, void* in, void* out, int direction, cudaStream_t s) {
    CBN_CUFFT(cufftSetStream(h, s));
    CBN_CUFFT(cufftExecC2C(h, static_cast<cufftComplex*>(in), static_cast<cufftComplex*>(out),
                           direction));
}

}  // namespace cbn

extern "C" const char* cbn_last_error(void) { return cbn::g_last_error.c_str(); }
