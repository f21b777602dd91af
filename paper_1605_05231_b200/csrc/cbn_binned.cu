#include <algorithm>
#include <vector>

#include "cbn_binned.cuh"

#include <cstdlib>

#include <cub/device/device_scan.cuh>

namespace cbn {

int spread_warps_override() {
    static const int w = [] {
        const char* e = std::getenv("CBN_SPREAD_W");
        return e ? std::atoi(e) : 0;
    }();
    return w;
}

bool bulk_flush_enabled() {
    static const bool on = [] {
        // off by default: measured 3.15 -> 3.28 ms on the config-2 backprojector
        // spread and 40.8 -> 40.9 ms on config 4
        const char* e = std::getenv("CBN_BULK_FLUSH");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

bool bulk_fill_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CBN_BULK_FILL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

__global__ void k_bin_scatter(const int* __restrict__ keys, int64_t m, int* __restrict__ cursor,
                              int* __restrict__ perm) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    perm[atomicAdd(cursor + keys[i], 1)] = (int)i;
}

void finish_bins(BinPlan& bp, DevBuf<int>& keys, DevBuf<int>& counts, int64_t nbins, int max_sub,
                 cudaStream_t s) {
    std::vector<int> h((size_t)nbins);
    CBN_CUDA(cudaMemcpyAsync(h.data(), counts.p, sizeof(int) * nbins, cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    std::vector<SubProblem> subs;
    int64_t off = 0;
    for (int64_t b = 0; b < nbins; ++b) {
        const int c = h[(size_t)b];
        for (int st = 0; st < c; st += max_sub)
            subs.push_back(SubProblem{(int)b, (int)(off + st), std::min(max_sub, c - st), 0});
        h[(size_t)b] = (int)off;   // exclusive scan in place -> scatter cursors
        off += c;
    }
    CBN_REQUIRE(off == bp.m, "bin counts do not add up");
    CBN_CUDA(cudaMemcpyAsync(counts.p, h.data(), sizeof(int) * nbins, cudaMemcpyHostToDevice, s));
    bp.perm.alloc((size_t)bp.m);
    k_bin_scatter<<<(unsigned)((bp.m + 255) / 256), 256, 0, s>>>(keys.p, bp.m, counts.p, bp.perm.p);
    CBN_LAUNCH_CHECK();
    bp.nsubs = (int)subs.size();
    bp.subs.alloc(subs.size());
    CBN_CUDA(cudaMemcpyAsync(bp.subs.p, subs.data(), sizeof(SubProblem) * subs.size(),
                             cudaMemcpyHostToDevice, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    bp.ready = true;
}

__global__ void k_sub_counts(const int* __restrict__ counts, int64_t nbins, int max_sub,
                             int* __restrict__ nsub) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nbins) nsub[b] = (counts[b] + max_sub - 1) / max_sub;
}

__global__ void k_fill_subs(const int* __restrict__ counts, const int* __restrict__ offs,
                            const int* __restrict__ suboff, int64_t nbins, int max_sub,
                            SubProblem* __restrict__ subs) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbins) return;
    const int c = counts[b];
    int q = suboff[b];
    for (int st = 0; st < c; st += max_sub)
        subs[q++] = SubProblem{(int)b, offs[b] + st, min(max_sub, c - st), 0};
}

void device_bins_finish(BinPlan& bp, DeviceSortScratch& sc, int64_t nbins, int max_sub,
                        cudaStream_t s) {
    CBN_REQUIRE(nbins < (1LL << 31) && bp.m < (1LL << 31), "device sort: too many bins or points");
    const int64_t cap = nbins + (bp.m + max_sub - 1) / max_sub;
    sc.offs.ensure((size_t)nbins);
    sc.nsub.ensure((size_t)nbins);
    sc.suboff.ensure((size_t)nbins);
    size_t need = 0;
    CBN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, sc.counts.p, sc.offs.p, (int)nbins, s));
    if (need > sc.temp_bytes) {
        sc.temp.alloc(need);
        sc.temp_bytes = need;
    }
    const unsigned nb = (unsigned)((nbins + 255) / 256);
    k_sub_counts<<<nb, 256, 0, s>>>(sc.counts.p, nbins, max_sub, sc.nsub.p);
    CBN_LAUNCH_CHECK();
    CBN_CUDA(cub::DeviceScan::ExclusiveSum(sc.temp.p, need, sc.counts.p, sc.offs.p, (int)nbins, s));
    CBN_CUDA(cub::DeviceScan::ExclusiveSum(sc.temp.p, need, sc.nsub.p, sc.suboff.p, (int)nbins, s));
    if (bp.subs.n < (size_t)cap) bp.subs.alloc((size_t)cap);
    CBN_CUDA(cudaMemsetAsync(bp.subs.p, 0, sizeof(SubProblem) * cap, s));
    k_fill_subs<<<nb, 256, 0, s>>>(sc.counts.p, sc.offs.p, sc.suboff.p, nbins, max_sub, bp.subs.p);
    CBN_LAUNCH_CHECK();
    if (bp.perm.n < (size_t)bp.m) bp.perm.alloc((size_t)bp.m);
    // the scatter advances offs as cursors (k_fill_subs has read them)
    k_bin_scatter<<<(unsigned)((bp.m + 255) / 256), 256, 0, s>>>(sc.keys.p, bp.m, sc.offs.p, bp.perm.p);
    CBN_LAUNCH_CHECK();
    bp.nsubs = (int)cap;
    bp.ready = true;
}

}  // namespace cbn
