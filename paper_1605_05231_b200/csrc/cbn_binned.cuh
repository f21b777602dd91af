// Bin-sorted KB gather / spread with shared-memory grid subproblems.
//
// Points are counting-sorted once per plan by the tile of the oversampled grid
// that holds their first tap (the integer index of nufft.py:176, so the bins
// are exactly the reference's tap blocks).  A subproblem is <= max_sub points
// of one bin; its CTA works on the tile plus the J-1 halo, (T+J-1)^D cells,
// staged in shared memory:
//  * gather: the region is loaded once (wrapped, coalesced along the fastest
//    axis), then one thread per point reads its J^D taps from shared memory;
//  * spread: each warp owns a private copy of the region and processes one
//    point at a time with its lanes covering the J^D taps, so shared-memory
//    updates are plain load/add/store (sm_100a has no native shared fp32
//    atomic add -- it lowers to a CAS loop); the copies are summed and
//    flushed with one global RED per non-zero cell.
#pragma once

#include "cbn_kernels.cuh"

namespace cbn {

struct SubProblem {
    int bin;
    int start;
    int count;
    int pad;
};

template <int D>
struct TileGeom {
    int T[3];        // tile edge per axis
    int R[3];        // region edge per axis (T + J - 1)
    int nb[3];       // bins per axis
    int K[3];        // grid extent per axis
};

template <int D>
CBN_D void bin_origin(const TileGeom<D>& tg, int bin, int (&o)[3]) {
    if constexpr (D == 3) {
        o[2] = (bin % tg.nb[2]) * tg.T[2];
        bin /= tg.nb[2];
        o[1] = (bin % tg.nb[1]) * tg.T[1];
        o[0] = (bin / tg.nb[1]) * tg.T[0];
    } else {
        o[1] = (bin % tg.nb[1]) * tg.T[1];
        o[0] = (bin / tg.nb[1]) * tg.T[0];
        o[2] = 0;
    }
}

// bin of each point (first tap mod K, divided by the tile edge)
template <int D, int J, class Src>
__global__ void k_bin_keys(Src src, KBSet kb, TileGeom<D> tg, int64_t m, int* __restrict__ keys,
                           int* __restrict__ counts) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double w[D];
    typename Src::Aux aux;
    src.node(i, w, aux);
    int key = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        int f;
        axis_coord(w[d], kb.ax[d].K, 0.5 * (double)J, f);
        key = key * tg.nb[d] + wrapc(f, kb.ax[d].K) / tg.T[d];
    }
    keys[i] = key;
    atomicAdd(counts + key, 1);
}

__global__ void k_bin_scatter(const int* __restrict__ keys, int64_t m, int* __restrict__ cursor,
                              int* __restrict__ perm);

// ---------------------------------------------------------------- gather
template <int D, int J, class Src, class Epi>
__global__ void __launch_bounds__(256)
k_gather_binned(const float2* __restrict__ grid, KBSet kb, TileGeom<D> tg, Src src, Epi epi,
                const int* __restrict__ perm, const SubProblem* __restrict__ subs) {
    extern __shared__ float2 tile[];
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<D>(tg, sp.bin, o);
    const int R0 = tg.R[0], R1 = tg.R[1], R2 = D == 3 ? tg.R[2] : 1;
    const int nreg = R0 * R1 * R2;
    for (int e = threadIdx.x; e < nreg; e += blockDim.x) {
        const int r2 = e % R2, r01 = e / R2, r1 = r01 % R1, r0 = r01 / R1;
        size_t g;
        if constexpr (D == 3)
            g = ((size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1])) * tg.K[2] +
                wrapc(o[2] + r2, tg.K[2]);
        else
            g = (size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1]);
        // asynchronous 8-byte copy global -> shared (LDGSTS): all of a thread's
        // halo loads are in flight at once
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(tile + e)),
                     "l"(grid + g));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        const int64_t i = perm[sp.start + k];
        double w[D];
        typename Src::Aux aux;
        src.node(i, w, aux);
        int first[D];
        float wt[D][J];
        tap_setup<D, J>(kb, w, first, wt);
        int l[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < D; ++d) l[d] = wrapc(first[d], tg.K[d]) - o[d];
        float2 acc = make_float2(0.f, 0.f);
        if constexpr (D == 3) {
#pragma unroll
            for (int a = 0; a < J; ++a) {
                float2 pa = make_float2(0.f, 0.f);
#pragma unroll
                for (int b = 0; b < J; ++b) {
                    const float2* row = tile + ((l[0] + a) * R1 + l[1] + b) * R2 + l[2];
                    float2 r = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < J; ++c) {
                        float2 g = row[c];
                        r.x = fmaf(wt[2][c], g.x, r.x);
                        r.y = fmaf(wt[2][c], g.y, r.y);
                    }
                    pa.x = fmaf(wt[1][b], r.x, pa.x);
                    pa.y = fmaf(wt[1][b], r.y, pa.y);
                }
                acc.x = fmaf(wt[0][a], pa.x, acc.x);
                acc.y = fmaf(wt[0][a], pa.y, acc.y);
            }
        } else {
#pragma unroll
            for (int a = 0; a < J; ++a) {
                const float2* row = tile + (l[0] + a) * R1 + l[1];
                float2 r = make_float2(0.f, 0.f);
#pragma unroll
                for (int b = 0; b < J; ++b) {
                    float2 g = row[b];
                    r.x = fmaf(wt[1][b], g.x, r.x);
                    r.y = fmaf(wt[1][b], g.y, r.y);
                }
                acc.x = fmaf(wt[0][a], r.x, acc.x);
                acc.y = fmaf(wt[0][a], r.y, acc.y);
            }
        }
        epi.put(i, acc, w, aux);
    }
}

// ---------------------------------------------------------------- spread
// WARPS warps per CTA, each with a private region copy + a weight scratch of
// 32 points x D x J floats.
template <int D, int J>
constexpr int spread_taps() {
    return D == 3 ? J * J * J : J * J;
}

template <int D, int J, int WARPS, class Src>
__global__ void __launch_bounds__(WARPS * 32)
k_spread_binned(float2* __restrict__ grid, KBSet kb, TileGeom<D> tg, Src src,
                const int* __restrict__ perm, const SubProblem* __restrict__ subs) {
    extern __shared__ float2 smem[];
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<D>(tg, sp.bin, o);
    const int R0 = tg.R[0], R1 = tg.R[1], R2 = D == 3 ? tg.R[2] : 1;
    const int nreg = R0 * R1 * R2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* copy = smem + (size_t)warp * nreg;
    float* scratch = reinterpret_cast<float*>(smem + (size_t)WARPS * nreg) + warp * 32 * D * J;
    for (int e = threadIdx.x; e < WARPS * nreg; e += blockDim.x) smem[e] = make_float2(0.f, 0.f);
    __syncthreads();
    constexpr int NT = spread_taps<D, J>();
    for (int base = warp * 32; base < sp.count; base += WARPS * 32) {
        // each lane prepares one point: local first, weights (to scratch), value
        const int k = base + lane;
        int l0 = 0, l1 = 0, l2 = 0;
        float2 v = make_float2(0.f, 0.f);
        if (k < sp.count) {
            const int64_t i = perm[sp.start + k];
            double w[D];
            typename Src::Aux aux;
            src.node(i, w, aux);
            v = src.value(i, w, aux);
            int first[D];
            float wt[D][J];
            tap_setup<D, J>(kb, w, first, wt);
            l0 = wrapc(first[0], tg.K[0]) - o[0];
            l1 = wrapc(first[1], tg.K[1]) - o[1];
            if constexpr (D == 3) l2 = wrapc(first[2], tg.K[2]) - o[2];
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int p = 0; p < J; ++p) scratch[(lane * D + d) * J + p] = wt[d][p];
        }
        __syncwarp();
        const int npts = min(32, sp.count - base);
        for (int j = 0; j < npts; ++j) {
            const int a0 = __shfl_sync(0xffffffffu, l0, j);
            const int a1 = __shfl_sync(0xffffffffu, l1, j);
            const int a2 = __shfl_sync(0xffffffffu, l2, j);
            const float vx = __shfl_sync(0xffffffffu, v.x, j);
            const float vy = __shfl_sync(0xffffffffu, v.y, j);
            const float* ws = scratch + j * D * J;
            if (vx != 0.f || vy != 0.f) {
#pragma unroll
                for (int t0 = 0; t0 < NT; t0 += 32) {
                    const int t = t0 + lane;
                    if (t < NT) {
                        float wk;
                        int cell;
                        if constexpr (D == 3) {
                            const int a = t / (J * J), b = (t / J) % J, c = t % J;
                            wk = ws[a] * ws[J + b] * ws[2 * J + c];
                            cell = ((a0 + a) * R1 + a1 + b) * R2 + a2 + c;
                        } else {
                            const int a = t / J, b = t % J;
                            wk = ws[a] * ws[J + b];
                            cell = (a0 + a) * R1 + a1 + b;
                        }
                        float2 cur = copy[cell];
                        cur.x = fmaf(wk, vx, cur.x);
                        cur.y = fmaf(wk, vy, cur.y);
                        copy[cell] = cur;
                    }
                }
            }
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nreg; e += blockDim.x) {
        float2 s = smem[e];
#pragma unroll
        for (int wi = 1; wi < WARPS; ++wi) {
            float2 x = smem[(size_t)wi * nreg + e];
            s.x += x.x;
            s.y += x.y;
        }
        if (s.x == 0.f && s.y == 0.f) continue;
        const int r2 = e % R2, r01 = e / R2, r1 = r01 % R1, r0 = r01 / R1;
        size_t g;
        if constexpr (D == 3)
            g = ((size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1])) * tg.K[2] +
                wrapc(o[2] + r2, tg.K[2]);
        else
            g = (size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1]);
        atomicAdd(grid + g, s);
    }
}

template <int D, int J, int WARPS>
constexpr size_t spread_smem_bytes(int nreg) {
    return (size_t)WARPS * nreg * sizeof(float2) + (size_t)WARPS * 32 * D * J * sizeof(float);
}

}  // namespace cbn

#include "cbn_runtime.h"

namespace cbn {

// Sorted point order + subproblem list of one fixed node set (plan data).
struct BinPlan {
    bool ready = false;
    int D = 0, J = 0;
    TileGeom<3> tg{};
    int64_t m = 0;
    int nreg = 0;
    DevBuf<int> perm;
    DevBuf<SubProblem> subs;
    int nsubs = 0;
    template <int D_>
    TileGeom<D_> geom() const {
        TileGeom<D_> g;
        for (int d = 0; d < 3; ++d) {
            g.T[d] = tg.T[d];
            g.R[d] = tg.R[d];
            g.nb[d] = tg.nb[d];
            g.K[d] = tg.K[d];
        }
        return g;
    }
};

// counts -> offsets and subproblems on the host (one-time plan step), then the
// device scatter of the sorted order
void finish_bins(BinPlan& bp, DevBuf<int>& keys, DevBuf<int>& counts, int64_t nbins, int max_sub,
                 cudaStream_t s);

template <int D, int J, class Src>
void build_bins(BinPlan& bp, const Src& src, const KBSet& kb, int64_t m, const int* tile,
                int max_sub, cudaStream_t s) {
    bp.D = D;
    bp.J = J;
    bp.m = m;
    int64_t nbins = 1;
    bp.nreg = 1;
    for (int d = 0; d < 3; ++d) {
        if (d < D) {
            bp.tg.K[d] = kb.ax[d].K;
            bp.tg.T[d] = std::min(tile[d], kb.ax[d].K);
            bp.tg.R[d] = bp.tg.T[d] + J - 1;
            bp.tg.nb[d] = (bp.tg.K[d] + bp.tg.T[d] - 1) / bp.tg.T[d];
            nbins *= bp.tg.nb[d];
            bp.nreg *= bp.tg.R[d];
        } else {
            bp.tg.K[d] = bp.tg.T[d] = bp.tg.R[d] = bp.tg.nb[d] = 1;
        }
    }
    DevBuf<int> keys((size_t)m), counts((size_t)nbins);
    CBN_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int) * nbins, s));
    TileGeom<D> tg = bp.geom<D>();
    k_bin_keys<D, J, Src><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(src, kb, tg, m, keys.p, counts.p);
    CBN_LAUNCH_CHECK();
    finish_bins(bp, keys, counts, nbins, max_sub, s);
}

}  // namespace cbn
