#include <algorithm>
#include <vector>

#include "cbn_binned.cuh"

#include <cstdlib>

namespace cbn {

int spread_warps_override() {
    static const int w = [] {
        const char* e = std::getenv("CBN_SPREAD_W");
        return e ? std::atoi(e) : 0;
    }();
    return w;
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

}  // namespace cbn
