// Binned 2D KB spread / gather of the per-view Grangeat step over blocks of
// views (grangeat.py:131-170).  The polar detector-plane nodes are shared by
// all views (plan_grangeat), so per plan each node is sorted into a 2D tile,
// and its local first tap, the J + J KB weights and its complex factor
// (filter * phase) are precomputed once.  Per (subproblem, view group) a CTA
// then only streams the per-view values:
//   reverse: warp-private shared tiles, one view group of VG views per CTA,
//            lanes = taps, plain load/add/store, one RED per non-zero cell;
//   forward: the VG view tiles are staged in shared memory, one thread per
//            node reads its taps for each view.
#pragma once

#include "cbn_binned.cuh"
#include "cbn_sources.cuh"

namespace cbn {

template <int J>
struct GrPoint {
    short lu, lv;      // first tap relative to the bin origin
    int col;           // mu * n_t + (rolled t index) into the per-view t buffer
    float2 fac;        // complex factor (filter * phase), zero if the node is inert
    float w[2 * J];    // u weights, then v weights
};

struct GrFactor {
    int n_t;
    int reverse;               // 1: conj phases * (i q_t); 0: phases * pu pv * (i omega_t)
    int N[2];                  // detector dims (centre / plan phases, grangeat.py:119,140)
    const float* q;            // reverse: -sign(omega) taper dt c2 per t
    const double* omega;       // forward: omega_t
    float pupv;
};

template <int J>
__global__ void k_gr_points(KBSet kb, TileGeom<2> tg, PolarSrc src, GrFactor f,
                            const int* __restrict__ perm, const SubProblem* __restrict__ subs,
                            GrPoint<J>* __restrict__ out) {
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        const int i = perm[sp.start + k];
        double w[2];
        PolarSrc::Aux aux;
        src.node(i, w, aux);
        int first[2];
        float wt[2][J];
        tap_setup<2, J>(kb, w, first, wt);
        GrPoint<J> g;
        g.lu = (short)(wrapc(first[0], tg.K[0]) - o[0]);
        g.lv = (short)(wrapc(first[1], tg.K[1]) - o[1]);
        const int im = i / f.n_t;
        g.col = im * f.n_t + (aux.jt - f.n_t / 2 + f.n_t) % f.n_t;
        double sn, cs;
        if (f.reverse) {
            sincos(-centre_plan_angle<2>(aux.wc, w, f.N), &sn, &cs);
            const float q = f.q[aux.jt];
            g.fac = make_float2(-(float)sn * q, (float)cs * q);
        } else {
            sincos(centre_plan_angle<2>(aux.wc, w, f.N), &sn, &cs);
            const float om = (float)f.omega[aux.jt] * f.pupv;
            g.fac = make_float2(-(float)sn * om, (float)cs * om);
        }
#pragma unroll
        for (int p = 0; p < J; ++p) {
            g.w[p] = wt[0][p];
            g.w[J + p] = wt[1][p];
        }
        out[sp.start + k] = g;
    }
}

// reverse: grids[v] += sum_points w * (t[v][col] * fac)  for views [v0, v0 + nv)
template <int J, int VG, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
k_gr_spread_binned(float2* __restrict__ grids, size_t grid_stride, TileGeom<2> tg,
                   const GrPoint<J>* __restrict__ pts, const SubProblem* __restrict__ subs,
                   const float2* __restrict__ tf, size_t tf_stride, int nviews) {
    extern __shared__ float2 smem[];
    const SubProblem sp = subs[blockIdx.x];
    const int v0 = blockIdx.y * VG;
    const int nv = min(VG, nviews - v0);
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    const int R1 = tg.R[1];
    const int nreg = tg.R[0] * R1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* copy = smem + (size_t)warp * VG * nreg;
    for (int e = threadIdx.x; e < WARPS * VG * nreg; e += blockDim.x) smem[e] = make_float2(0.f, 0.f);
    __syncthreads();
    const int a = lane / J, b = lane % J;
    const bool active = lane < J * J;
    const float2* tfv = tf + (size_t)v0 * tf_stride;
    // PG points x VG views per step: one independent value load per lane, then
    // the warp walks the PG points with lanes = taps and shuffles the values in
    constexpr int PG = 32 / VG;
    for (int base = warp * PG; base < sp.count; base += WARPS * PG) {
        const int kl = base + lane / VG, vl = lane % VG;
        float2 y = make_float2(0.f, 0.f);
        if (kl < sp.count && vl < nv) {
            const GrPoint<J>& gl = pts[sp.start + kl];
            y = cmul(__ldg(tfv + vl * tf_stride + gl.col), gl.fac);
        }
        const int npg = min(PG, sp.count - base);
        for (int j = 0; j < npg; ++j) {
            const GrPoint<J>& g = pts[sp.start + base + j];
            const float wk = active ? g.w[a] * g.w[J + b] : 0.f;
            const int cell = (g.lu + a) * R1 + g.lv + b;
#pragma unroll
            for (int v = 0; v < VG; ++v) {
                const float yx = __shfl_sync(0xffffffffu, y.x, j * VG + v);
                const float yy = __shfl_sync(0xffffffffu, y.y, j * VG + v);
                if (active && (yx != 0.f || yy != 0.f)) {
                    float2 cur = copy[v * nreg + cell];
                    cur.x = fmaf(wk, yx, cur.x);
                    cur.y = fmaf(wk, yy, cur.y);
                    copy[v * nreg + cell] = cur;
                }
            }
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nv * nreg; e += blockDim.x) {
        float2 s = smem[e];
#pragma unroll
        for (int wi = 1; wi < WARPS; ++wi) {
            const float2 x = smem[(size_t)wi * VG * nreg + e];
            s.x += x.x;
            s.y += x.y;
        }
        if (s.x == 0.f && s.y == 0.f) continue;
        const int v = e / nreg, c = e % nreg;
        const int r0 = c / R1, r1 = c % R1;
        const size_t gi = (size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1]);
        atomicAdd(grids + (size_t)(v0 + v) * grid_stride + gi, s);
    }
}

// reverse, lanes = views: each warp walks its points, every lane adds its own
// view's value to a private [cell][32 views] shared tile (consecutive lanes,
// consecutive words: conflict-free, no shuffles); one RED per non-zero
// (cell, view) at the end.  nviews <= 32.
template <int J, int WARPS, int TILE>
__global__ void __launch_bounds__(WARPS * 32)
k_gr_spread_views(float2* __restrict__ grids, size_t grid_stride, TileGeom<2> tg,
                  const GrPoint<J>* __restrict__ pts, const SubProblem* __restrict__ subs,
                  const float2* __restrict__ tf, size_t tf_stride, int nviews) {
    extern __shared__ float2 smem[];
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    constexpr int R1 = TILE + J - 1;
    constexpr int nreg = R1 * R1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* copy = smem + (size_t)warp * nreg * 32;
    for (int e = threadIdx.x; e < WARPS * nreg * 32; e += blockDim.x) smem[e] = make_float2(0.f, 0.f);
    __syncthreads();
    const bool live = lane < nviews;
    const float2* tfl = tf + (size_t)lane * tf_stride;
    // CH points per step: lanes < CH fetch one point record each; then every
    // lane issues its CH view-value loads back to back (deep memory-level
    // parallelism at 4 warps / SM), and the CH points are applied from registers
    constexpr int CH = 16;
    for (int base0 = warp * CH; base0 < sp.count; base0 += WARPS * CH) {
        const int npts = min(CH, sp.count - base0);
        GrPoint<J> mine;
        if (lane < npts) mine = pts[sp.start + base0 + lane];
        else {
            mine.lu = mine.lv = 0;
            mine.col = 0;
            mine.fac = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 2 * J; ++q) mine.w[q] = 0.f;
        }
        float2 yv[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            const int col = __shfl_sync(0xffffffffu, mine.col, j);
            yv[j] = (live && j < npts) ? __ldg(tfl + col) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            const float fx = __shfl_sync(0xffffffffu, mine.fac.x, j);
            const float fy = __shfl_sync(0xffffffffu, mine.fac.y, j);
            if (fx == 0.f && fy == 0.f) continue;   // warp-uniform (also past npts)
            const int lu = __shfl_sync(0xffffffffu, (int)mine.lu, j);
            const int lv = __shfl_sync(0xffffffffu, (int)mine.lv, j);
            float w[2 * J];
#pragma unroll
            for (int q = 0; q < 2 * J; ++q) w[q] = __shfl_sync(0xffffffffu, mine.w[q], j);
            const float2 y = cmul(yv[j], make_float2(fx, fy));
            // the J x J cells are distinct: load all, update, store all
            float2* base = copy + (lu * R1 + lv) * 32 + lane;
            float2 cur[J][J];
#pragma unroll
            for (int a = 0; a < J; ++a)
#pragma unroll
                for (int b = 0; b < J; ++b) cur[a][b] = base[(a * R1 + b) * 32];
#pragma unroll
            for (int a = 0; a < J; ++a)
#pragma unroll
                for (int b = 0; b < J; ++b) {
                    const float wk = w[a] * w[J + b];
                    cur[a][b].x = fmaf(wk, y.x, cur[a][b].x);
                    cur[a][b].y = fmaf(wk, y.y, cur[a][b].y);
                }
#pragma unroll
            for (int a = 0; a < J; ++a)
#pragma unroll
                for (int b = 0; b < J; ++b) base[(a * R1 + b) * 32] = cur[a][b];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nreg * 32; e += blockDim.x) {
        const int v = e & 31, c = e >> 5;
        if (v >= nviews) continue;
        float2 s = smem[e];
#pragma unroll
        for (int wi = 1; wi < WARPS; ++wi) {
            const float2 x = smem[(size_t)wi * nreg * 32 + e];
            s.x += x.x;
            s.y += x.y;
        }
        if (s.x == 0.f && s.y == 0.f) continue;
        const int r0 = c / R1, r1 = c % R1;
        const size_t gi = (size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1]);
        atomicAdd(grids + (size_t)v * grid_stride + gi, s);
    }
}

// forward: out[v][col] = fac * sum_taps w * grid_v   for views [v0, v0 + nv)
template <int J, int VG>
__global__ void __launch_bounds__(256)
k_gr_gather_binned(const float2* __restrict__ grids, size_t grid_stride, TileGeom<2> tg,
                   const GrPoint<J>* __restrict__ pts, const SubProblem* __restrict__ subs,
                   float2* __restrict__ out, size_t out_stride, int nviews) {
    extern __shared__ float2 tile[];
    const SubProblem sp = subs[blockIdx.x];
    const int v0 = blockIdx.y * VG;
    const int nv = min(VG, nviews - v0);
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    const int R1 = tg.R[1];
    const int nreg = tg.R[0] * R1;
    for (int e = threadIdx.x; e < nv * nreg; e += blockDim.x) {
        const int v = e / nreg, c = e % nreg;
        const int r0 = c / R1, r1 = c % R1;
        const size_t gi = (size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(tile + e)),
                     "l"(grids + (size_t)(v0 + v) * grid_stride + gi));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        const GrPoint<J> g = pts[sp.start + k];
        for (int v = 0; v < nv; ++v) {
            const float2* t = tile + v * nreg;
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int a = 0; a < J; ++a) {
                const float2* row = t + (g.lu + a) * R1 + g.lv;
                float2 r = make_float2(0.f, 0.f);
#pragma unroll
                for (int b = 0; b < J; ++b) {
                    const float2 x = row[b];
                    r.x = fmaf(g.w[J + b], x.x, r.x);
                    r.y = fmaf(g.w[J + b], x.y, r.y);
                }
                acc.x = fmaf(g.w[a], r.x, acc.x);
                acc.y = fmaf(g.w[a], r.y, acc.y);
            }
            out[(size_t)(v0 + v) * out_stride + g.col] = cmul(acc, g.fac);
        }
    }
}

}  // namespace cbn
