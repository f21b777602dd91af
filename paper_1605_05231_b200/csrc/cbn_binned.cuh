// Bin-sorted KB gather / spread with shared-memory grid subproblems.
//
// Points are counting-sorted once per plan by the tile of the oversampled grid
// that holds their first tap (the integer index of nufft.py:176, so the bins
// are exactly the reference's tap blocks).  A subproblem is <= max_sub points
// of one bin; its CTA works on the tile plus the J-1 halo, (T+J-1)^D cells,
// staged in shared memory:
//  * gather: the region is loaded once (wrapped, coalesced along the fastest
//    axis), then one thread per point reads its J^D taps from shared memory;
//  * spread (2D): each warp owns a private copy of the region and processes
//    one point at a time with its lanes covering the J^D taps, so
//    shared-memory updates are plain load/add/store (sm_100a has no native
//    shared fp32 atomic add -- it lowers to a CAS loop); the copies are
//    summed and flushed with one global RED per non-zero cell;
//  * spread (3D): one region copy per CTA, cells owned by warp: warp w
//    updates only the region rows (axis 0) congruent to w mod W, so every
//    warp walks every point of the subproblem but touches only its rows --
//    no atomics, no private copies, and W x 32 threads share one region.
// The 3D region's fastest axis is stored with a pitch P = J (mod 16) so that
// 16 lanes covering consecutive (b, c) tap pairs hit 16 distinct bank pairs.
// Within a subproblem the points are interleaved by the bank residue of
// their region offset (k_bin_interleave), so the 16 lanes of a half-warp in
// the thread-per-point gather read 16 distinct bank pairs at every tap.
#pragma once

#include <type_traits>

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
    int P;           // shared-memory pitch of the last axis (>= R[D-1])
    int bulk;        // 3D: bit 0 = spread flushes region rows with TMA bulk reductions,
                     // bit 1 = gather fills its tile with TMA bulk copies
};

// Shared -> global bulk reduction of one contiguous run of floats (TMA,
// UBLKRED): the run is added element-wise into global memory by the async
// proxy; 16-byte aligned on both sides, size a multiple of 16 bytes.
CBN_D void bulk_red_add_f32(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes)
                 : "memory");
}

// Global -> shared bulk copy (TMA, UBLKCP) completing on an mbarrier: 16-byte
// aligned on both sides, size a multiple of 16 bytes.
CBN_D void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
CBN_D void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)), "r"(bytes)
                 : "memory");
}
CBN_D void bulk_copy_g2s(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc), "r"(bytes),
        "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}
CBN_D void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
        "r"(phase)
        : "memory");
}

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
        axis_coord(w[d], kb.ax[d].K, 0.5 * (double)kb.ax[d].J, f);
        key = key * tg.nb[d] + wrapc(f, kb.ax[d].K) / tg.T[d];
    }
    keys[i] = key;
    atomicAdd(counts + key, 1);
}

__global__ void k_bin_scatter(const int* __restrict__ keys, int64_t m, int* __restrict__ cursor,
                              int* __restrict__ perm);

// Sources that keep their coordinates in bin-sorted order expose
// node_at(pos, i, ...) (pos = sorted position, i = original index); the binned
// kernels prefer it, so coordinates stream instead of gathering by perm.
template <class Src, class = void>
struct has_node_at : std::false_type {};
template <class Src>
struct has_node_at<Src, std::void_t<decltype(&Src::node_at)>> : std::true_type {};

// Sources that carry per-plan point records (sorted order) expose
// stage<J>(kb, pos, v, l, wt): value, bin-local first taps and KB weights of
// the point at sorted position pos, with no node generation per step.
template <class Src, class = void>
struct has_stage : std::false_type {};
template <class Src>
struct has_stage<Src, std::void_t<typename Src::is_record_src>> : std::true_type {};

template <class Src, int D>
CBN_D void src_node(const Src& src, int64_t pos, int64_t i, double (&w)[D], typename Src::Aux& a) {
    if constexpr (has_node_at<Src>::value) src.node_at(pos, i, w, a);
    else src.node(i, w, a);
}

// ---------------------------------------------------------------- gather
// HALF (3D): `grid` is the [K0][K1][K2/2+1] half spectrum of a real input
// (R2C); cells with k2 > K2/2 are read as conj(G[-k]).
template <int D, int J, class Src, class Epi, bool HALF = false>
__global__ void __launch_bounds__(256, 3)   // <= 80 registers: 3 CTAs per SM
k_gather_binned(const float2* __restrict__ grid, KBSet kb, TileGeom<D> tg, Src src, Epi epi,
                const int* __restrict__ perm, const SubProblem* __restrict__ subs) {
    extern __shared__ float4 smem4[];   // 16-byte aligned: the bulk copies need it
    float2* tile = reinterpret_cast<float2*>(smem4);
    const SubProblem sp = subs[blockIdx.x];
    if (sp.count == 0) return;   // unused slot of a device-sorted plan
    int o[3];
    bin_origin<D>(tg, sp.bin, o);
    const int R0 = tg.R[0], R1 = D == 3 ? tg.R[1] : tg.P;
    const int P2 = D == 3 ? tg.P : 1;
    const int R2 = D == 3 ? tg.R[2] : 1;
    const int nreg = R0 * R1 * P2;
    // cell -> (r0, r1, r2) by multiply-shift division (FastDiv)
    const FastDiv dP(P2), dR(R1);
    unsigned negmask = 0;   // HALF: region columns r2 read as conj(G[-k])
    if constexpr (D == 3 && HALF) {
        const int lane = threadIdx.x & 31;
        const bool neg = lane < R2 && wrapc(o[2] + lane, tg.K[2]) >= tg.K[2] / 2 + 1;
        negmask = __ballot_sync(0xffffffffu, neg);
    }
    bool filled = false;
    if constexpr (D == 3 && !HALF) {
        if (tg.bulk & 2) {
            // Tile rows (r0, r1) are contiguous runs of P2 cells in shared memory
            // and, up to the wrap of the last axis, in the grid: one TMA bulk copy
            // per run (two at the wrap) completing on an mbarrier, instead of one
            // 8-byte cp.async per cell with its index arithmetic.
            __shared__ unsigned long long fill_bar;
            const int rows = R0 * R1;
            if (threadIdx.x == 0) {
                mbar_init(&fill_bar, 1);
                mbar_expect_tx(&fill_bar, (unsigned)rows * (unsigned)P2 * 8u);
            }
            __syncthreads();
            const int n1 = min(P2, tg.K[2] - o[2]);   // cells before the wrap
            for (int row = threadIdx.x; row < rows; row += blockDim.x) {
                const int r0 = dR.div(row), r1 = row - r0 * R1;
                const float2* grow = grid + ((size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] +
                                             wrapc(o[1] + r1, tg.K[1])) * tg.K[2];
                float2* srow = tile + row * P2;
                bulk_copy_g2s(srow, grow + o[2], (unsigned)n1 * 8u, &fill_bar);
                if (n1 < P2) bulk_copy_g2s(srow + n1, grow, (unsigned)(P2 - n1) * 8u, &fill_bar);
            }
            mbar_wait(&fill_bar, 0);
            filled = true;
        }
    }
    for (int e = threadIdx.x; e < (filled ? 0 : nreg); e += blockDim.x) {
        const int r01 = dP.div(e), r2 = e - r01 * P2;
        const int r0 = dR.div(r01), r1 = r01 - r0 * R1;
        if (r2 >= R2 || (D == 2 && r1 >= tg.R[1])) continue;
        size_t g;
        if constexpr (D == 3 && HALF) {
            int i0 = wrapc(o[0] + r0, tg.K[0]), i1 = wrapc(o[1] + r1, tg.K[1]);
            int i2 = wrapc(o[2] + r2, tg.K[2]);
            const int h2 = tg.K[2] / 2 + 1;
            if ((negmask >> r2) & 1u) {   // conjugated after the copy
                i0 = i0 ? tg.K[0] - i0 : 0;
                i1 = i1 ? tg.K[1] - i1 : 0;
                i2 = tg.K[2] - i2;
            }
            g = ((size_t)i0 * tg.K[1] + i1) * h2 + i2;
        } else if constexpr (D == 3)
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
    if constexpr (D == 3 && HALF) {
        // each thread conjugates the mirrored cells it copied itself
        if (negmask)
            for (int e = threadIdx.x; e < nreg; e += blockDim.x) {
                const int r01 = dP.div(e), r2 = e - r01 * P2;
                if (r2 < R2 && ((negmask >> r2) & 1u)) tile[e].y = -tile[e].y;
            }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        const int64_t i = perm[sp.start + k];
        double w[D];
        typename Src::Aux aux;
        src_node(src, sp.start + k, i, w, aux);
        int first[D];
        float wt[D][J];
        tap_setup<D, J>(kb, w, first, wt);
        int l[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < D; ++d) {
            l[d] = wrapc(first[d], tg.K[d]) - o[d];
            CBN_DCHECK(l[d] >= 0 && l[d] < tg.T[d], "gather: point outside its bin tile");
        }
        float2 acc = make_float2(0.f, 0.f);
        if constexpr (D == 3) {
#pragma unroll
            for (int a = 0; a < J; ++a) {
                float2 pa = make_float2(0.f, 0.f);
#pragma unroll
                for (int b = 0; b < J; ++b) {
                    const float2* row = tile + ((l[0] + a) * R1 + l[1] + b) * P2 + l[2];
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
    static_assert(D == 2, "3D spreads use k_spread_owned");
    extern __shared__ float2 smem[];
    const SubProblem sp = subs[blockIdx.x];
    if (sp.count == 0) return;   // unused slot of a device-sorted plan
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
            src_node(src, sp.start + k, i, w, aux);
            v = src.value(i, w, aux);
            int first[D];
            float wt[D][J];
            tap_setup<D, J>(kb, w, first, wt);
            l0 = wrapc(first[0], tg.K[0]) - o[0];
            l1 = wrapc(first[1], tg.K[1]) - o[1];
            if constexpr (D == 3) l2 = wrapc(first[2], tg.K[2]) - o[2];
            CBN_DCHECK(l0 >= 0 && l0 < tg.T[0] && l1 >= 0 && l1 < tg.T[1] && l2 >= 0 &&
                           (D == 2 || l2 < tg.T[2]),
                       "spread: point outside its bin tile");
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


// ------------------------------------------------------ owner-computes spread
// 3D spread with one shared region per CTA.  Round structure: every thread
// stages one point (local first taps, D x J weights, value), then each warp
// walks all staged points and applies the taps of the region rows it owns
// (row = l0 + a, owned by warp (l0 + a) mod W).  Lanes cover consecutive
// (b, c) tap pairs of a row.  Cells of distinct warps are disjoint and a warp
// applies one point at a time, so the read-add-write needs no atomics.
template <int J>
constexpr int owned_stage_stride() {
    return (3 * J) | 1;   // odd: conflict-free staging writes
}

// J = 8 with four warps stages each point as a 16-byte aligned block -- header
// (value, packed first taps), the x weights as (a, a + 4) pairs by owning
// warp, the y weights as (b, b + 4) pairs -- plus the z weights at an odd
// stride: a warp reads a point's header, its x pair, its y pair and its z
// weight with one instruction each, 4 instead of 7 staging reads per point and
// warp (type 1 of config 4: 41.3 -> 37.8 ms).  The same packing at J = 6 / two
// warps (header and the warp's three x weights as 16-byte broadcasts) was
// slower, 3.16 -> 3.68 ms on the config-2 backprojector: it stays scalar.
template <int J, int W>
constexpr bool owned_packed() {
    return J == 8 && W == 4;
}
template <int J>
constexpr int owned_block_floats() {   // aligned block per staged point
    return 20;
}
template <int J>
constexpr int owned_rest_stride() {    // odd stride of the z weights
    return 9;
}

template <int J, int W>
constexpr size_t spread_owned_smem_bytes(int nreg) {
    if (owned_packed<J, W>())
        return (size_t)((nreg + 1) & ~1) * sizeof(float2) +
               (size_t)W * 32 * (owned_block_floats<J>() + owned_rest_stride<J>()) * sizeof(float) + 16;
    return (size_t)nreg * sizeof(float2) + (size_t)W * 32 * owned_stage_stride<J>() * sizeof(float) +
           (size_t)W * 32 * (sizeof(float2) + sizeof(int)) + 8;
}

template <int J, int W, class Src>
__global__ void __launch_bounds__(W * 32)
k_spread_owned(float2* __restrict__ grid, KBSet kb, TileGeom<3> tg, Src src,
               const int* __restrict__ perm, const SubProblem* __restrict__ subs) {
    constexpr int NP = W * 32;
    constexpr int SW = owned_stage_stride<J>();
    constexpr int ROWS = (J + W - 1) / W;           // max rows per warp per point
    constexpr int JJ = J * J;
    constexpr int ITERS = (ROWS * JJ + 31) / 32;
    extern __shared__ float4 smem4[];
    const SubProblem sp = subs[blockIdx.x];
    if (sp.count == 0) return;   // unused slot of a device-sorted plan
    int o[3];
    bin_origin<3>(tg, sp.bin, o);
    const int R0 = tg.R[0], R1 = tg.R[1], R2 = tg.R[2], P = tg.P;
    const int nreg = R0 * R1 * P;
    constexpr bool PACK = owned_packed<J, W>();
    constexpr int BF = owned_block_floats<J>(), RS = owned_rest_stride<J>();
    float2* reg = reinterpret_cast<float2*>(smem4);
    float* stw = reinterpret_cast<float*>(reg + nreg);
    float2* stv = reinterpret_cast<float2*>(stw + ((NP * SW + 1) & ~1));
    int* stl = reinterpret_cast<int*>(stv + NP);
    // packed staging: aligned blocks, then the odd-stride rest
    float4* blk = reinterpret_cast<float4*>(reg + ((nreg + 1) & ~1));
    float* rest = reinterpret_cast<float*>(blk) + NP * BF;
    for (int e = threadIdx.x; e < nreg; e += NP) reg[e] = make_float2(0.f, 0.f);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // this lane's taps of a warp's rows: row index, cell offset, weight slots
    const int row_stride = R1 * P;
    int t_row[ITERS], t_off[ITERS], t_wy[ITERS], t_wz[ITERS];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
        const int t = it * 32 + lane;
        const int r = t / JJ, pq = t % JJ, b = pq / J, c = pq % J;
        t_row[it] = t < ROWS * JJ ? r : J;
        t_off[it] = r * W * row_stride + b * P + c;
        t_wy[it] = J + b;
        t_wz[it] = 2 * J + c;
    }
    for (int base = 0; base < sp.count; base += NP) {
        __syncthreads();   // region zeroed / previous round's points consumed
        const int k = base + threadIdx.x;
        if (k < sp.count) {
            float2 v;
            float wt[3][J];
            int l0, l1, l2;
            if constexpr (has_stage<Src>::value) {
                int l[3];
                src.template stage<J>(kb, (int64_t)sp.start + k, v, l, wt);
                l0 = l[0];
                l1 = l[1];
                l2 = l[2];
            } else {
                const int64_t i = perm[sp.start + k];
                double w[3];
                typename Src::Aux aux;
                src_node(src, sp.start + k, i, w, aux);
                v = src.value(i, w, aux);
                int first[3];
                tap_setup<3, J>(kb, w, first, wt);
                l0 = wrapc(first[0], tg.K[0]) - o[0];
                l1 = wrapc(first[1], tg.K[1]) - o[1];
                l2 = wrapc(first[2], tg.K[2]) - o[2];
            }
            CBN_DCHECK(l0 >= 0 && l0 < tg.T[0] && l1 >= 0 && l1 < tg.T[1] && l2 >= 0 &&
                           l2 < tg.T[2],
                       "owned spread: point outside its bin tile");
            const int pl = (l0 << 24) | ((l0 * R1 + l1) * P + l2);
            if constexpr (PACK) {
                float4* b4 = blk + threadIdx.x * (BF / 4);
                float* rs = rest + threadIdx.x * RS;
                b4[0] = make_float4(v.x, v.y, __int_as_float(pl), 0.f);
                // (a, a + 4) x pairs by owning warp, (b, b + 4) y pairs
                b4[1] = make_float4(wt[0][0], wt[0][4], wt[0][1], wt[0][5]);
                b4[2] = make_float4(wt[0][2], wt[0][6], wt[0][3], wt[0][7]);
                b4[3] = make_float4(wt[1][0], wt[1][4], wt[1][1], wt[1][5]);
                b4[4] = make_float4(wt[1][2], wt[1][6], wt[1][3], wt[1][7]);
#pragma unroll
                for (int q = 0; q < 8; ++q) rs[q] = wt[2][q];
            } else {
                stl[threadIdx.x] = pl;
                stv[threadIdx.x] = v;
#pragma unroll
                for (int d = 0; d < 3; ++d)
#pragma unroll
                    for (int p = 0; p < J; ++p) stw[threadIdx.x * SW + d * J + p] = wt[d][p];
            }
        }
        __syncthreads();
        const int npts = min(NP, sp.count - base);
        if constexpr (J == 8 && W == 4) {
            // J = 8, four warps, two rows each: lane = tap pairs (b, c) and
            // (b + 4, c), b = lane / 8, c = lane % 8, fixed over both rows, so
            // wy * wz is formed once per point and each row costs one
            // broadcast x weight; all four cell loads issue before the stores
            const int fb = lane >> 3, fc = lane & 7;
            const int off0 = fb * P + fc, off1 = (fb + 4) * P + fc;
            for (int j = 0; j < npts; ++j) {
                const float4 h = blk[j * (BF / 4)];
                const float2 v = make_float2(h.x, h.y);
                if (v.x == 0.f && v.y == 0.f) continue;     // uniform over the CTA
                const int pl = __float_as_int(h.z);
                const int l0 = pl >> 24;
                const float2* pairs = reinterpret_cast<const float2*>(blk + j * (BF / 4) + 1);
                const int a0 = (warp - l0) & 3;
                float2* row0 = reg + (pl & 0xffffff) + a0 * row_stride;
                float2* row1 = row0 + W * row_stride;
                const float wz = rest[j * RS + fc];
                const float2 wy = pairs[4 + fb], wx = pairs[a0];
                const float wyz0 = wy.x * wz, wyz1 = wy.y * wz;
                const float wx0 = wx.x, wx1 = wx.y;
                float2 cur[4] = {row0[off0], row0[off1], row1[off0], row1[off1]};
                const float wk[4] = {wx0 * wyz0, wx0 * wyz1, wx1 * wyz0, wx1 * wyz1};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    cur[r].x = fmaf(wk[r], v.x, cur[r].x);
                    cur[r].y = fmaf(wk[r], v.y, cur[r].y);
                }
                row0[off0] = cur[0];
                row0[off1] = cur[1];
                row1[off0] = cur[2];
                row1[off1] = cur[3];
                __syncwarp();
            }
            continue;
        }
        if constexpr (J == 6 && W == 2) {
            // J = 6, two warps, three rows each: lane = tap pair (b, c) =
            // (lane / 6, lane % 6) of pq = lane < 32, fixed over the three
            // rows, so wy * wz is formed once per point and each row costs
            // one broadcast x weight; the 4 left-over pairs of each row
            // (b = 5, c = 2..5) go to lanes 0..11 of a fourth pass
            const int fb = lane / 6, fc = lane % 6;
            const int f_off = fb * P + fc;
            const int lr = lane >> 2, lc = 2 + (lane & 3);
            const int l_off = lr * W * row_stride + 5 * P + lc;
            for (int j = 0; j < npts; ++j) {
                const float2 v = stv[j];
                if (v.x == 0.f && v.y == 0.f) continue;     // uniform over the CTA
                const int pl = stl[j];
                const int l0 = pl >> 24;
                const float* ws = stw + j * SW;
                const int a0 = (warp - l0) & 1;
                float2* base_row = reg + (pl & 0xffffff) + a0 * row_stride;
                const float wyz = ws[J + fb] * ws[2 * J + fc];
                float wl = 0.f;
                if (lane < 12) wl = ws[a0 + lr * W] * ws[J + 5] * ws[2 * J + lc];
                // the four cells are distinct: all loads issue before any store
                float2* cell[4];
                float2 cur[4];
                float wk[4];
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    cell[r] = base_row + r * W * row_stride + f_off;
                    wk[r] = ws[a0 + r * W] * wyz;
                }
                cell[3] = base_row + l_off;
                wk[3] = wl;
#pragma unroll
                for (int r = 0; r < 3; ++r) cur[r] = *cell[r];
                if (lane < 12) cur[3] = *cell[3];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    cur[r].x = fmaf(wk[r], v.x, cur[r].x);
                    cur[r].y = fmaf(wk[r], v.y, cur[r].y);
                }
#pragma unroll
                for (int r = 0; r < 3; ++r) *cell[r] = cur[r];
                if (lane < 12) *cell[3] = cur[3];
                __syncwarp();
            }
            continue;
        }
        for (int j = 0; j < npts; ++j) {
            const float2 v = stv[j];
            if (v.x == 0.f && v.y == 0.f) continue;     // uniform over the CTA
            const int pl = stl[j];
            const int l0 = pl >> 24;
            const float* ws = stw + j * SW;
            int a0 = (W & (W - 1)) == 0 ? (warp - l0) & (W - 1) : ((warp - l0) % W + W) % W;
            const int nrows = J % W == 0 ? J / W : (a0 < J ? (J - 1 - a0) / W + 1 : 0);
            float2* base_row = reg + (pl & 0xffffff) + a0 * row_stride;
            // a lane's cells are distinct: all loads issue before any store
            float2 cur[ITERS];
            float wk[ITERS];
#pragma unroll
            for (int it = 0; it < ITERS; ++it) {
                if (t_row[it] < nrows) {
                    wk[it] = ws[a0 + t_row[it] * W] * ws[t_wy[it]] * ws[t_wz[it]];
                    cur[it] = base_row[t_off[it]];
                }
            }
#pragma unroll
            for (int it = 0; it < ITERS; ++it) {
                if (t_row[it] < nrows) {
                    cur[it].x = fmaf(wk[it], v.x, cur[it].x);
                    cur[it].y = fmaf(wk[it], v.y, cur[it].y);
                    base_row[t_off[it]] = cur[it];
                }
            }
            __syncwarp();
        }
    }
    const FastDiv dP(P), dR1(R1);
    if (tg.bulk & 1) {
        // Region rows (r0, r1) are contiguous runs of P cells in shared memory
        // and, up to the axis-2 wrap, in the grid (the pad cells past R2 are
        // zero): one TMA bulk reduction per run instead of one RED per cell.
        // The generic-proxy tap writes are fenced to the async proxy first.
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (lane == 0) {
            const int n1 = min(P, tg.K[2] - o[2]);   // cells before the wrap
            for (int r = warp; r < R0 * R1; r += W) {
                const int r0 = dR1.div(r), r1 = r - r0 * R1;
                float2* grow = grid + ((size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] +
                                       wrapc(o[1] + r1, tg.K[1])) * tg.K[2];
                const float2* srow = reg + r * P;
                bulk_red_add_f32(grow + o[2], srow, (unsigned)n1 * 8u);
                if (n1 < P) bulk_red_add_f32(grow, srow + n1, (unsigned)(P - n1) * 8u);
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            // the region must stay allocated until the engine has read it
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        }
        return;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nreg; e += NP) {
        const int r01 = dP.div(e), r2 = e - r01 * P;
        if (r2 >= R2) continue;
        const int r0 = dR1.div(r01), r1 = r01 - r0 * R1;
        const float2 s = reg[e];
        if (s.x == 0.f && s.y == 0.f) continue;
        const size_t g = ((size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1])) *
                             tg.K[2] + wrapc(o[2] + r2, tg.K[2]);
        atomicAdd(grid + g, s);
    }
}

// J = 8, W = 8: one row per warp per point, lanes on (b, c) = (lane / 8, lane % 8)
// and (b + 4, c).  The staging packs each point's value and packed first taps
// into one 16-byte header and stores the y weights as (b, b + 4) pairs, so a
// warp reads 4 shared-memory wavefronts of point data per point instead of 6.
constexpr int kOwned8Stride = 26;   // floats per staged point: 8 x, 8 y pairs, 8 z, 2 pad

inline constexpr size_t spread_owned8_smem_bytes(int nreg) {
    return (size_t)nreg * sizeof(float2) + 256 * (sizeof(float4) + kOwned8Stride * sizeof(float));
}

template <class Src>
__global__ void __launch_bounds__(256)
k_spread_owned8(float2* __restrict__ grid, KBSet kb, TileGeom<3> tg, Src src,
                const int* __restrict__ perm, const SubProblem* __restrict__ subs) {
    constexpr int J = 8, NP = 256, SW = kOwned8Stride;
    extern __shared__ float4 smem4[];
    const SubProblem sp = subs[blockIdx.x];
    if (sp.count == 0) return;   // unused slot of a device-sorted plan
    int o[3];
    bin_origin<3>(tg, sp.bin, o);
    const int R0 = tg.R[0], R1 = tg.R[1], R2 = tg.R[2], P = tg.P;
    const int nreg = R0 * R1 * P;
    float2* reg = reinterpret_cast<float2*>(smem4);
    float4* hdr = reinterpret_cast<float4*>(reg + ((nreg + 1) & ~1));
    float* stw = reinterpret_cast<float*>(hdr + NP);
    for (int e = threadIdx.x; e < nreg; e += NP) reg[e] = make_float2(0.f, 0.f);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row_stride = R1 * P;
    const int b = lane >> 3, c = lane & 7;
    const int off0 = b * P + c, off1 = (b + 4) * P + c;
    for (int base = 0; base < sp.count; base += NP) {
        __syncthreads();   // region zeroed / previous round's points consumed
        const int k = base + threadIdx.x;
        if (k < sp.count) {
            const int64_t i = perm[sp.start + k];
            double w[3];
            typename Src::Aux aux;
            src_node(src, sp.start + k, i, w, aux);
            const float2 v = src.value(i, w, aux);
            int first[3];
            float wt[3][J];
            tap_setup<3, J>(kb, w, first, wt);
            const int l0 = wrapc(first[0], tg.K[0]) - o[0];
            const int l1 = wrapc(first[1], tg.K[1]) - o[1];
            const int l2 = wrapc(first[2], tg.K[2]) - o[2];
            CBN_DCHECK(l0 >= 0 && l0 < tg.T[0] && l1 >= 0 && l1 < tg.T[1] && l2 >= 0 &&
                           l2 < tg.T[2],
                       "owned spread: point outside its bin tile");
            hdr[threadIdx.x] = make_float4(v.x, v.y, __int_as_float((l0 << 24) | ((l0 * R1 + l1) * P + l2)),
                                           0.f);
            float* ws = stw + threadIdx.x * SW;
#pragma unroll
            for (int p = 0; p < 8; ++p) ws[p] = wt[0][p];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ws[8 + 2 * q] = wt[1][q];
                ws[9 + 2 * q] = wt[1][q + 4];
            }
#pragma unroll
            for (int p = 0; p < 8; ++p) ws[16 + p] = wt[2][p];
        }
        __syncthreads();
        const int npts = min(NP, sp.count - base);
        for (int j = 0; j < npts; ++j) {
            const float4 h = hdr[j];
            if (h.x == 0.f && h.y == 0.f) continue;     // uniform over the CTA
            const int pl = __float_as_int(h.z);
            const int a0 = (warp - (pl >> 24)) & 7;
            const float* ws = stw + j * SW;
            const float wx = ws[a0];
            const float2 wy = *reinterpret_cast<const float2*>(ws + 8 + 2 * b);
            const float wz = ws[16 + c];
            float2* row = reg + (pl & 0xffffff) + a0 * row_stride;
            const float wk0 = wx * wy.x * wz, wk1 = wx * wy.y * wz;
            float2 c0 = row[off0], c1 = row[off1];
            c0.x = fmaf(wk0, h.x, c0.x);
            c0.y = fmaf(wk0, h.y, c0.y);
            c1.x = fmaf(wk1, h.x, c1.x);
            c1.y = fmaf(wk1, h.y, c1.y);
            row[off0] = c0;
            row[off1] = c1;
            __syncwarp();
        }
    }
    __syncthreads();
    const FastDiv dP(P), dR1(R1);
    for (int e = threadIdx.x; e < nreg; e += NP) {
        const int r01 = dP.div(e), r2 = e - r01 * P;
        if (r2 >= R2) continue;
        const int r0 = dR1.div(r01), r1 = r01 - r0 * R1;
        const float2 sv = reg[e];
        if (sv.x == 0.f && sv.y == 0.f) continue;
        const size_t g = ((size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1])) *
                             tg.K[2] + wrapc(o[2] + r2, tg.K[2]);
        atomicAdd(grid + g, sv);
    }
}

// ------------------------------------------- bank-residue interleaved order
// Reorders each subproblem's points (plan time) so consecutive points have
// distinct region-offset residues mod 16 for as long as the residue classes
// last: stable rank q within the class, then order by (q, residue).
constexpr int kInterleaveMax = 4096;

template <int D, int J, class Src>
__global__ void __launch_bounds__(256)
k_bin_interleave(Src src, KBSet kb, TileGeom<D> tg, int* __restrict__ perm,
                 const SubProblem* __restrict__ subs, const float* __restrict__ raw32 = nullptr,
                 float* __restrict__ sorted32 = nullptr) {
    __shared__ int ids[kInterleaveMax];
    __shared__ short rank[kInterleaveMax];
    __shared__ unsigned char res[kInterleaveMax];
    __shared__ int wcnt[8][16];
    __shared__ int cnt[16];
    const SubProblem sp = subs[blockIdx.x];
    if (sp.count == 0) return;   // unused slot of a device-sorted plan
    int o[3];
    bin_origin<D>(tg, sp.bin, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 16) cnt[threadIdx.x] = 0;
    for (int c0 = 0; c0 < sp.count; c0 += 256) {
        const int k = c0 + threadIdx.x;
        int r = -1;
        if (k < sp.count) {
            const int64_t i = perm[sp.start + k];
            double w[D];
            typename Src::Aux aux;
            src.node(i, w, aux);
            int l[3] = {0, 0, 0};
#pragma unroll
            for (int d = 0; d < D; ++d) {
                int f;
                axis_coord(w[d], kb.ax[d].K, 0.5 * (double)kb.ax[d].J, f);
                l[d] = wrapc(f, kb.ax[d].K) - o[d];
            }
            const int off = D == 3 ? (l[0] * tg.R[1] + l[1]) * tg.P + l[2] : l[0] * tg.P + l[1];
            r = off & 15;
            ids[k] = (int)i;
            res[k] = (unsigned char)r;
        }
        int q = 0;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            const unsigned m = __ballot_sync(0xffffffffu, r == rr);
            if (r == rr) q = __popc(m & ((1u << lane) - 1u));
            if (lane == 0) wcnt[warp][rr] = __popc(m);
        }
        __syncthreads();
        if (r >= 0) {
            q += cnt[r];
            for (int w2 = 0; w2 < warp; ++w2) q += wcnt[w2][r];
            rank[k] = (short)q;
        }
        __syncthreads();
        if (threadIdx.x < 16) {
            int add = 0;
            for (int w2 = 0; w2 < 8; ++w2) add += wcnt[w2][threadIdx.x];
            cnt[threadIdx.x] += add;
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < sp.count; k += 256) {
        const int q = rank[k], r = res[k];
        int pos = 0;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) pos += min(cnt[rr], q) + (rr < r && cnt[rr] > q ? 1 : 0);
        perm[sp.start + pos] = ids[k];
        // float32 node sets keep a bin-ordered copy of the coordinates: written
        // here, while the subproblem's nodes (read above) are still in L1 / L2,
        // instead of by a separate pass of random reads
        if (sorted32) {
#pragma unroll
            for (int d = 0; d < D; ++d)
                sorted32[(size_t)(sp.start + pos) * D + d] = __ldg(raw32 + (size_t)ids[k] * D + d);
        }
    }
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
        g.P = tg.P;
        g.bulk = tg.bulk;
        return g;
    }
};

// counts -> offsets and subproblems on the host (one-time plan step), then the
// device scatter of the sorted order
void finish_bins(BinPlan& bp, DevBuf<int>& keys, DevBuf<int>& counts, int64_t nbins, int max_sub,
                 cudaStream_t s);

// Device-only counting sort (no host round trip, graph-capturable): bin keys
// and counts -> exclusive scans (CUB) of the counts and of the per-bin
// subproblem counts -> subproblem list, written into a list of fixed capacity
// nbins + ceil(m / max_sub) whose unused entries have count 0 (the binned
// kernels return at once for those) -> scatter.  Scratch is kept for re-sorts.
struct DeviceSortScratch {
    DevBuf<int> keys, counts, offs, nsub, suboff;
    DevBuf<char> temp;
    size_t temp_bytes = 0;
};
void device_bins_finish(BinPlan& bp, DeviceSortScratch& sc, int64_t nbins, int max_sub,
                        cudaStream_t s);

bool bulk_flush_enabled();   // CBN_BULK_FLUSH=1: TMA bulk-reduction flush of the 3D spread (A/B)
bool bulk_fill_enabled();    // CBN_BULK_FILL=0: cp.async tile fill of the 3D gather instead of TMA bulk copies

// pitch_pad: store the last region axis with pitch = J (mod 16) (required by
// k_spread_owned; harmless for the gather)
template <int D, int J, class Src>
void build_bins(BinPlan& bp, const Src& src, const KBSet& kb, int64_t m, const int* tile,
                int max_sub, cudaStream_t s, bool pitch_pad = false,
                DeviceSortScratch* dev = nullptr, const float* raw32 = nullptr,
                float* sorted32 = nullptr) {
    CBN_REQUIRE(max_sub <= kInterleaveMax, "subproblem size above the interleave limit");
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
    bp.tg.P = bp.tg.R[D - 1];
    if (D == 3 && pitch_pad) bp.tg.P += (((J - bp.tg.P) % 16) + 16) % 16;
    bp.nreg = bp.nreg / bp.tg.R[D - 1] * bp.tg.P;
    // TMA bulk flush of the 3D spread: 16-byte aligned row runs on both sides
    // and at most one wrap along the last axis
    const bool bulk_ok = D == 3 && pitch_pad && bp.tg.P % 2 == 0 && bp.tg.T[2] % 2 == 0 &&
                         bp.tg.K[2] % 2 == 0 && bp.tg.P <= bp.tg.K[2] && bp.tg.K[2] % bp.tg.T[2] == 0;
    bp.tg.bulk = bulk_ok ? (bulk_flush_enabled() ? 1 : 0) | (bulk_fill_enabled() ? 2 : 0) : 0;
    if (dev) {
        DeviceSortScratch& sc = *dev;
        sc.keys.ensure((size_t)m);
        sc.counts.ensure((size_t)nbins);
        CBN_CUDA(cudaMemsetAsync(sc.counts.p, 0, sizeof(int) * nbins, s));
        k_bin_keys<D, J, Src><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(src, kb, bp.geom<D>(), m,
                                                                        sc.keys.p, sc.counts.p);
        CBN_LAUNCH_CHECK();
        device_bins_finish(bp, sc, nbins, max_sub, s);
        k_bin_interleave<D, J, Src><<<bp.nsubs, 256, 0, s>>>(src, kb, bp.geom<D>(), bp.perm.p,
                                                             bp.subs.p, raw32, sorted32);
        CBN_LAUNCH_CHECK();
        return;
    }
    DevBuf<int> keys((size_t)m), counts((size_t)nbins);
    CBN_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int) * nbins, s));
    TileGeom<D> tg = bp.geom<D>();
    k_bin_keys<D, J, Src><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(src, kb, tg, m, keys.p, counts.p);
    CBN_LAUNCH_CHECK();
    finish_bins(bp, keys, counts, nbins, max_sub, s);
    if (bp.nsubs > 0) {
        k_bin_interleave<D, J, Src><<<bp.nsubs, 256, 0, s>>>(src, kb, bp.geom<D>(), bp.perm.p, bp.subs.p,
                                                             raw32, sorted32);
        CBN_LAUNCH_CHECK();
    }
}

// warps per CTA of the 3D owner-computes spread: rows per warp x J^2 taps
// (measured on B200: J=8 -> 4 warps with fixed tap pairs per lane, 40.5 ms
// of type 1 on config 4 against 41.6 ms for k_spread_owned8 (CBN_SPREAD_W=8);
// J=6 -> 2 warps, 10.4 ms vs 12.7 ms at 3 on the config-2 backprojection)
template <int J>
constexpr int owned_warps() {
    return J == 6 ? 2 : (J < 8 ? J : (J == 8 ? 4 : 8));
}

template <int J, int W, class Src>
void launch_spread3_w(float2* grid, const KBSet& kb, const BinPlan& bb, const Src& src, cudaStream_t s,
                      int s0, int s1) {
    const size_t smem = spread_owned_smem_bytes<J, W>(bb.nreg);
    CBN_CUDA(cudaFuncSetAttribute(k_spread_owned<J, W, Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    if (s1 > s0)
        k_spread_owned<J, W><<<s1 - s0, W * 32, smem, s>>>(grid, kb, bb.geom<3>(), src, bb.perm.p,
                                                           bb.subs.p + s0);
    CBN_LAUNCH_CHECK();
}

int spread_warps_override();   // CBN_SPREAD_W (tuning experiments), 0 = default

// subproblems [s0, s1) of the plan (default: all)
template <int J, class Src>
void launch_spread3(float2* grid, const KBSet& kb, const BinPlan& bb, const Src& src, cudaStream_t s,
                    int s0 = 0, int s1 = -1) {
    CBN_REQUIRE(bb.D == 3 && bb.tg.P % 16 == J % 16, "3D spread needs a pitch-padded bin plan");
    if (s1 < 0) s1 = bb.nsubs;
    if constexpr (J == 8 && !has_stage<Src>::value) {
        if (spread_warps_override() == 8) {   // the one-row-per-warp kernel (A/B)
            const size_t smem = spread_owned8_smem_bytes(bb.nreg);
            CBN_CUDA(cudaFuncSetAttribute(k_spread_owned8<Src>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            if (s1 > s0)
                k_spread_owned8<<<s1 - s0, 256, smem, s>>>(grid, kb, bb.geom<3>(), src, bb.perm.p,
                                                           bb.subs.p + s0);
            CBN_LAUNCH_CHECK();
            return;
        }
    }
    switch (spread_warps_override()) {
        case 1: return launch_spread3_w<J, 1>(grid, kb, bb, src, s, s0, s1);
        case 2: return launch_spread3_w<J, 2>(grid, kb, bb, src, s, s0, s1);
        case 4: return launch_spread3_w<J, 4>(grid, kb, bb, src, s, s0, s1);
        default: return launch_spread3_w<J, owned_warps<J>()>(grid, kb, bb, src, s, s0, s1);
    }
}

}  // namespace cbn
