// Binned 2D KB spread / gather of the per-view Grangeat step over blocks of
// views (grangeat.py:131-170).  The polar detector-plane nodes are shared by
// all views (plan_grangeat), so per plan each node is sorted into a 2D tile,
// and its local first tap, the J + J KB weights and its complex factor
// (filter * phase) are precomputed once.  Per subproblem a CTA then only
// streams the per-view values:
//   reverse: one [cell][32 views] shared region, rows owned by warps, lanes =
//            views (k_gr_spread_owned);
//   forward: the VG view tiles are staged in shared memory, one thread per
//            node reads its taps for each view.
#pragma once

#include "cbn_binned.cuh"
#include "cbn_sources.cuh"

namespace cbn {

template <int J>
struct GrPoint {
    short lu, lv;      // first tap relative to the bin origin
    // forward records: mu * n_t + (rolled t index) into the per-view C2C buffer;
    // reverse records: mu * (n_t/2 + 1) + k into the R2C half spectrum, stored
    // as ~index when the value is the conjugate of bin n_t - k (Hermitian half)
    int col;
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
        CBN_DCHECK(g.lu >= 0 && g.lu < tg.T[0] && g.lv >= 0 && g.lv < tg.T[1],
                   "grangeat: point outside its bin tile");
        const int im = i / f.n_t;
        const int kr = (aux.jt - f.n_t / 2 + f.n_t) % f.n_t;   // fftshift of the t FFT
        g.col = im * f.n_t + kr;
        double sn, cs;
        if (f.reverse) {
            // the reference rolls the line by n_t/2 before a C2C FFT; here the
            // unrolled real line goes through R2C, so bin kr picks up (-1)^kr
            // and bins above n_t/2 read the conjugate of bin n_t - kr
            const int nh = f.n_t / 2 + 1;
            g.col = kr < nh ? im * nh + kr : ~(im * nh + (f.n_t - kr));
            sincos(-centre_plan_angle<2>(aux.wc, w, f.N), &sn, &cs);
            const float q = (kr & 1) ? -f.q[aux.jt] : f.q[aux.jt];
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

// reverse, lanes = views, one [cell][32 views] region per CTA with rows owned
// by warps: J warps, warp w updates only region rows u = w (mod J), so each
// point's J x J taps are split one row per warp.  Chunks of 32 points are
// staged in shared memory (record: packed first taps, u / v weights, factor;
// value: t-spectrum * factor per view), then every warp applies every staged
// point to its row.  Lanes are views, so no two lanes share a word and warps
// share no cells: plain read-add-write, no syncs inside a chunk, and J x 32
// threads per region instead of one warp per private region.
template <int J, int TILE>
__global__ void __launch_bounds__(J * 32)
k_gr_spread_owned(float2* __restrict__ grids, size_t grid_stride, TileGeom<2> tg,
                  const GrPoint<J>* __restrict__ pts, const SubProblem* __restrict__ subs,
                  const float2* __restrict__ tf, size_t tf_stride, int nviews) {
    static_assert(J <= 8, "record layout holds up to 8 weights per axis");
    constexpr int W = J;
    constexpr int R1 = TILE + J - 1;
    constexpr int nreg = R1 * R1;
    constexpr int CH = 32;
    constexpr int SW = 16;            // [0, J): v weights, [8, 8 + J): u weights
    extern __shared__ float4 smem4[];
    float2* region = reinterpret_cast<float2*>(smem4);       // [nreg][32]
    float2* sy = region + nreg * 32;                         // [CH][32]
    float* sw = reinterpret_cast<float*>(sy + CH * 32);      // [CH][SW]
    float2* sfac = reinterpret_cast<float2*>(sw + CH * SW);  // [CH]
    int* sl = reinterpret_cast<int*>(sfac + CH);             // [CH] lu | lv << 16
    int* scol = sl + CH;                                     // [CH]
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < nreg * 32; e += W * 32) region[e] = make_float2(0.f, 0.f);
    const bool live = lane < nviews;
    const float2* tfl = tf + (size_t)lane * tf_stride;
    for (int base = 0; base < sp.count; base += CH) {
        const int npts = min(CH, sp.count - base);
        __syncthreads();   // region zeroed / previous chunk consumed
        if (threadIdx.x < npts) {
            const GrPoint<J>& g = pts[sp.start + base + threadIdx.x];
            float* w = sw + threadIdx.x * SW;
#pragma unroll
            for (int q = 0; q < J; ++q) {
                w[q] = g.w[J + q];
                w[8 + q] = g.w[q];
            }
            sfac[threadIdx.x] = g.fac;
            sl[threadIdx.x] = (int)(unsigned short)g.lu | ((int)g.lv << 16);
            scol[threadIdx.x] = g.col;
        }
        __syncthreads();
#pragma unroll
        for (int p0 = 0; p0 < CH; p0 += W) {
            const int p = p0 + warp;
            if (p < npts) {
                const float2 f = sfac[p];
                const int c = scol[p];
                float2 y = make_float2(0.f, 0.f);
                if (live) {
                    y = __ldg(tfl + (c >= 0 ? c : ~c));
                    y.y = c >= 0 ? y.y : -y.y;
                    y = cmul(y, f);
                }
                sy[p * 32 + lane] = y;
            }
        }
        __syncthreads();
        for (int p = 0; p < npts; ++p) {
            const float2 f = sfac[p];
            if (f.x == 0.f && f.y == 0.f) continue;   // inert node, uniform over the CTA
            const int pl = sl[p];
            const int lu = pl & 0xffff, lv = pl >> 16;
            int a0 = (warp - lu) % W;
            a0 += a0 < 0 ? W : 0;
            const float* w = sw + p * SW;
            const float wa = w[8 + a0];
            float wv[8];
            const float4 w03 = *reinterpret_cast<const float4*>(w);
            const float4 w47 = *reinterpret_cast<const float4*>(w + 4);
            wv[0] = w03.x; wv[1] = w03.y; wv[2] = w03.z; wv[3] = w03.w;
            wv[4] = w47.x; wv[5] = w47.y; wv[6] = w47.z; wv[7] = w47.w;
            const float2 y = sy[p * 32 + lane];
            float2* row = region + ((lu + a0) * R1 + lv) * 32 + lane;
            float2 cur[J];
#pragma unroll
            for (int b = 0; b < J; ++b) cur[b] = row[b * 32];
#pragma unroll
            for (int b = 0; b < J; ++b) {
                const float wk = wa * wv[b];
                cur[b].x = fmaf(wk, y.x, cur[b].x);
                cur[b].y = fmaf(wk, y.y, cur[b].y);
            }
#pragma unroll
            for (int b = 0; b < J; ++b) row[b * 32] = cur[b];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nreg * 32; e += W * 32) {
        const int v = e & 31, c = e >> 5;
        if (v >= nviews) continue;
        const float2 s = region[e];
        if (s.x == 0.f && s.y == 0.f) continue;
        const int r0 = c / R1, r1 = c % R1;
        const size_t gi = (size_t)wrapc(o[0] + r0, tg.K[0]) * tg.K[1] + wrapc(o[1] + r1, tg.K[1]);
        atomicAdd(grids + (size_t)v * grid_stride + gi, s);
    }
}

template <int J, int TILE>
constexpr size_t gr_spread_owned_smem() {
    return sizeof(float2) * ((size_t)(TILE + J - 1) * (TILE + J - 1) * 32 + 32 * 32) +
           sizeof(float) * 32 * 16 + sizeof(float2) * 32 + sizeof(int) * 64;
}

// ---------------------------------------------- reverse as a cell gather
// The reverse spread onto the detector grids is a sparse product with a
// geometry-only matrix (the polar nodes are shared by every view):
// grid_v[cell] = sum_p W[cell, p] y_v[p].  Per plan, each cell's (node,
// complex weight = w_u w_v fac) entries are listed (CSR); per call, one warp
// sums a cell's entries with lanes = views, reading each node's 32 view
// values as one 256-byte row of the view-fastest t-spectra.  No shared-memory
// read-modify-write, no atomics, and every grid cell is written once.
struct GrEntry {
    int id;         // row of the node-scaled t-spectra (GrNode table)
    float w;        // w_u[a] w_v[b] * pair factor
};

// One row of the node-scaled reverse t-spectra: fac * (conj?) R2C bin `src`.
// Rows [0, nspec) are the half-spectrum bins (the live node of that bin, or
// zero); rows past nspec hold the second node of bins whose two nodes (t and
// its mirror) both survive the pair merge.
struct GrNode {
    int src;        // R2C half-spectrum index
    int conj;       // 1: the node reads the conjugate of bin src
    float2 fac;     // node factor (filter * phase)
};

// Reverse Grangeat values are conjugate-symmetric in t (real detector lines,
// odd filter), so the spread grid is Hermitian and only Re of its inverse FFT
// is used: a node and its mirror (same mu, t -> -t) can be merged into one
// entry of doubled weight when they mirror exactly (no wrap jump, mirrored
// taps after the reference's edge test).  Returns the node's weight factor:
// 2 (kept side of a merged pair), 0 (dropped side) or 1.
CBN_D int gr_pair_factor(const PolarSrc& src, const KBSet& kb, int J, int i) {
    const int n_t = src.n_t;
    const int jt = i % n_t;
    if (jt == 0 || 2 * jt == n_t) return 1;
    double w[2], wm[2];
    PolarSrc::Aux a, am;
    src.node(i, w, a);
    src.node(i - jt + (n_t - jt), wm, am);
    bool ok = true;
#pragma unroll
    for (int d = 0; d < 2; ++d)
        ok = ok && fabs(w[d] + wm[d]) < 1e-12 && fabs(a.wc[d] + am.wc[d]) < 1e-12 &&
             mirror_taps_match(kb.ax[d].K, J, w[d], wm[d]);
    if (!ok) return 1;
    return 2 * jt < n_t ? 2 : 0;
}

// node rows: per live point (pts order) its GrNode row id, -1 if inert or
// dropped by the pair merge (see GrNode)
template <int J>
__global__ void k_gr_node_ids(const GrPoint<J>* __restrict__ pts, const int* __restrict__ perm,
                              int64_t m, PolarSrc src, KBSet kb, int nspec,
                              int* __restrict__ node_id, int* __restrict__ mult_out,
                              GrNode* __restrict__ tab, int* __restrict__ nextra) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    const GrPoint<J>& g = pts[q];
    int mult = 0;
    if (g.fac.x != 0.f || g.fac.y != 0.f) mult = gr_pair_factor(src, kb, J, perm[q]);
    int id = -1;
    if (mult) {
        const int half = g.col >= 0 ? g.col : ~g.col;
        // the direct node, or a kept conjugate node whose partner was merged in,
        // owns row `half`; a conjugate node beside a live partner takes a new row
        id = (g.col >= 0 || mult == 2) ? half : nspec + atomicAdd(nextra, 1);
        GrNode n;
        n.src = half;
        n.conj = g.col >= 0 ? 0 : 1;
        n.fac = g.fac;
        tab[id] = n;
    }
    node_id[q] = id;
    mult_out[q] = mult;
}

template <int J>
__global__ void k_gr_csr_count(TileGeom<2> tg, const GrPoint<J>* __restrict__ pts,
                               const SubProblem* __restrict__ subs,
                               const int* __restrict__ node_id, int* __restrict__ counts) {
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        if (node_id[sp.start + k] < 0) continue;
        const GrPoint<J>& g = pts[sp.start + k];
#pragma unroll
        for (int a = 0; a < J; ++a)
#pragma unroll
            for (int b = 0; b < J; ++b)
                atomicAdd(counts + (size_t)wrapc(o[0] + g.lu + a, tg.K[0]) * tg.K[1] +
                              wrapc(o[1] + g.lv + b, tg.K[1]),
                          1);
    }
}

template <int J>
__global__ void k_gr_csr_fill(TileGeom<2> tg, const GrPoint<J>* __restrict__ pts,
                              const SubProblem* __restrict__ subs,
                              const int* __restrict__ node_id, const int* __restrict__ mult,
                              int* __restrict__ cursor, GrEntry* __restrict__ ent) {
    const SubProblem sp = subs[blockIdx.x];
    int o[3];
    bin_origin<2>(tg, sp.bin, o);
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        const int id = node_id[sp.start + k];
        if (id < 0) continue;
        const GrPoint<J>& g = pts[sp.start + k];
        const float fm = (float)mult[sp.start + k];
#pragma unroll
        for (int a = 0; a < J; ++a)
#pragma unroll
            for (int b = 0; b < J; ++b) {
                const size_t cell = (size_t)wrapc(o[0] + g.lu + a, tg.K[0]) * tg.K[1] +
                                    wrapc(o[1] + g.lv + b, tg.K[1]);
                GrEntry e;
                e.id = id;
                e.w = g.w[a] * g.w[J + b] * fm;
                ent[atomicAdd(cursor + cell, 1)] = e;
            }
    }
}

// 32 consecutive cells per CTA, 8 warps x 4 cells, lanes = views; the
// [cell][view] results are transposed through shared memory so each view's 32
// cells are stored as one contiguous 256-byte row
constexpr int kGrRows = 8;    // value rows in flight per warp (16: 10.1 ms, 8: 8.3 ms per step at cfg 2)

// sum of CSR entries [e0, e1) with lanes = views (rows of the view-fastest
// node-scaled t-spectra `tl` = tfv + lane): 32 entry records per coalesced
// load, staged in the warp's shared slots `sb` and read back as broadcasts
// (one LDS per entry instead of two shuffles), kGrRows value rows in flight
CBN_D float2 gr_range_sum(int e0, int e1, const GrEntry* __restrict__ ent,
                          const float2* __restrict__ tl, int lane, GrEntry* sb) {
    float2 acc = make_float2(0.f, 0.f);
    for (int base = e0; base < e1; base += 32) {
        const int n = min(32, e1 - base);
        __syncwarp();
        sb[lane] = lane < n ? ent[base + lane] : GrEntry{0, 0.f};
        __syncwarp();
        for (int j0 = 0; j0 < n; j0 += kGrRows) {
            float2 y[kGrRows];
            float w[kGrRows];
#pragma unroll
            for (int j = 0; j < kGrRows; ++j) {
                const GrEntry e = sb[j0 + j];         // < 32; entries past n have w = 0
                w[j] = e.w;
                y[j] = __ldg(tl + (size_t)e.id * 32);
            }
#pragma unroll
            for (int j = 0; j < kGrRows; ++j) {
                acc.x = fmaf(w[j], y[j].x, acc.x);
                acc.y = fmaf(w[j], y[j].y, acc.y);
            }
        }
    }
    return acc;
}

// full-plane cell pair (k, -k) of half-plane cell c of [Ku][Kv/2+1]
CBN_D void gr_half_cells(int64_t c, int Ku, int Kv, int64_t& k, int64_t& km) {
    const int hv = Kv / 2 + 1;
    const int u = (int)(c / hv), v = (int)(c - (int64_t)u * hv);
    k = (int64_t)u * Kv + v;
    km = (int64_t)(u ? Ku - u : 0) * Kv + (v ? Kv - v : 0);
}

// Cell gather onto the Hermitian half plane [Ku][Kv/2+1]: half-plane cell c
// holds (G[k] + conj(G[-k])) / 2 of the full grid G, whose complex-to-real
// inverse FFT is Re(IFFT(G)) -- the only part the reverse Grangeat keeps
// (grangeat.py:166).  Lanes = views; no atomics, no memset.  Work items come
// costliest first (plan-time order; node density peaks at the origin):
//   item >= 0: 32 consecutive cells, 8 warps x 4 cells, results stored
//              view-major through a shared-memory transpose (heavy cells
//              skipped);
//   item <  0: one heavy cell -(item + 1), its two entry lists split over the
//              8 warps and reduced in shared memory.
static __global__ void __launch_bounds__(256)
k_gr_gather_cells(float2* __restrict__ grids, size_t grid_stride, int64_t ncell,
                  const int* __restrict__ col_ptr, const GrEntry* __restrict__ ent,
                  const float2* __restrict__ tfv, int nviews, int Ku, int Kv,
                  const int* __restrict__ order, const unsigned char* __restrict__ heavy) {
    __shared__ float2 tile[32][33];
    __shared__ GrEntry slots[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float2* tl = tfv + lane;
    GrEntry* sb = slots[warp];
    const int item = order[blockIdx.x];
    if (item < 0) {
        const int64_t c = -(int64_t)item - 1;
        int64_t k, km;
        gr_half_cells(c, Ku, Kv, k, km);
        const int a0 = col_ptr[k], a1 = col_ptr[k + 1], b0 = col_ptr[km], b1 = col_ptr[km + 1];
        const int la = a1 - a0, lb = b1 - b0;
        const float2 a = gr_range_sum(a0 + (int)((int64_t)la * warp / 8),
                                      a0 + (int)((int64_t)la * (warp + 1) / 8), ent, tl, lane, sb);
        const float2 b = gr_range_sum(b0 + (int)((int64_t)lb * warp / 8),
                                      b0 + (int)((int64_t)lb * (warp + 1) / 8), ent, tl, lane, sb);
        tile[warp][lane] = make_float2(a.x + b.x, a.y - b.y);
        __syncthreads();
        if (warp == 0) {
            float2 t = make_float2(0.f, 0.f);
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                t.x += tile[w][lane].x;
                t.y += tile[w][lane].y;
            }
            if (lane < nviews) grids[(size_t)lane * grid_stride + c] = make_float2(0.5f * t.x, 0.5f * t.y);
        }
        return;
    }
    const int64_t c0 = (int64_t)item * 32;
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
        const int cl = warp + 8 * q;
        const int64_t c = c0 + cl;
        float2 acc = make_float2(0.f, 0.f);
        if (c < ncell && !heavy[c]) {
            int64_t k, km;
            gr_half_cells(c, Ku, Kv, k, km);
            const float2 a = gr_range_sum(col_ptr[k], col_ptr[k + 1], ent, tl, lane, sb);
            const float2 b = gr_range_sum(col_ptr[km], col_ptr[km + 1], ent, tl, lane, sb);
            acc = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
        }
        tile[cl][lane] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int v = e >> 5, cl = e & 31;
        const int64_t c = c0 + cl;
        if (v < nviews && c < ncell && !heavy[c]) grids[(size_t)v * grid_stride + c] = tile[cl][v];
    }
}

// ----------------------------------------------------------------------
// Strip form of the reverse-Grangeat cell gather.  A node's 5 x 5 taps reach
// 5 consecutive cells along v in each of 5 rows, so the cell CSR lists every
// node row ~25 times and the gather reads each 256-byte row (32 views) once
// per cell: the kernel is bound by L1 wavefronts.  Grouping the half plane
// into strips of kGrStrip cells along v and merging a strip's cell lists by
// node (plan time, host) reads each row once per strip and applies it to the
// strip's cells with per-cell weights: half-plane cell i of the strip is
//   (G[k_i] + conj G[-k_i]) / 2 = sum_nodes (p_i Re y, q_i Im y)
// with p_i = (w_i + m_i) / 2 and q_i = (w_i - m_i) / 2, where w_i / m_i are
// the node's weights in the direct / mirrored cell lists (real weights).
constexpr int kGrStrip = 4;

CBN_D void gr_strip_sum(int e0, int e1, const int* __restrict__ sid, const float4* __restrict__ sp,
                        const float4* __restrict__ sq, const float2* __restrict__ tl, int lane,
                        int* s_id, float4* s_p, float4* s_q, float2 (&acc)[kGrStrip]) {
    for (int base = e0; base < e1; base += 32) {
        const int n = min(32, e1 - base);
        __syncwarp();
        if (lane < n) {
            s_id[lane] = sid[base + lane];
            s_p[lane] = sp[base + lane];
            s_q[lane] = sq[base + lane];
        } else {
            s_id[lane] = 0;
            s_p[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
            s_q[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncwarp();
        for (int j0 = 0; j0 < n; j0 += kGrRows) {
            float2 y[kGrRows];
#pragma unroll
            for (int j = 0; j < kGrRows; ++j) y[j] = __ldg(tl + (size_t)s_id[j0 + j] * 32);
#pragma unroll
            for (int j = 0; j < kGrRows; ++j) {
                const float4 p = s_p[j0 + j], q = s_q[j0 + j];
                acc[0].x = fmaf(p.x, y[j].x, acc[0].x);
                acc[0].y = fmaf(q.x, y[j].y, acc[0].y);
                acc[1].x = fmaf(p.y, y[j].x, acc[1].x);
                acc[1].y = fmaf(q.y, y[j].y, acc[1].y);
                acc[2].x = fmaf(p.z, y[j].x, acc[2].x);
                acc[2].y = fmaf(q.z, y[j].y, acc[2].y);
                acc[3].x = fmaf(p.w, y[j].x, acc[3].x);
                acc[3].y = fmaf(q.w, y[j].y, acc[3].y);
            }
        }
    }
}

// Work items (plan-time order, costliest first):
//   item >= 0: row u = item / ngrp, strips 8 g .. 8 g + 7 (g = item % ngrp),
//              one per warp, = half-plane cells 32 g .. 32 g + 31 of the row,
//              stored view-major through a shared-memory transpose (heavy
//              strips skipped);
//   item <  0: one heavy strip -(item + 1), its entries split over 8 warps.
static __global__ void __launch_bounds__(256)
k_gr_gather_strips(float2* __restrict__ grids, size_t grid_stride, int hv, int nsx, int ngrp,
                   const int* __restrict__ sptr, const int* __restrict__ sid,
                   const float4* __restrict__ sp, const float4* __restrict__ sq,
                   const float2* __restrict__ tfv, int nviews, const int* __restrict__ order,
                   const unsigned char* __restrict__ heavy) {
    __shared__ float2 tile[32][33];
    __shared__ int s_id[8][32];
    __shared__ float4 s_p[8][32], s_q[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float2* tl = tfv + lane;
    const int item = order[blockIdx.x];
    float2 acc[kGrStrip];
#pragma unroll
    for (int i = 0; i < kGrStrip; ++i) acc[i] = make_float2(0.f, 0.f);
    if (item < 0) {
        const int64_t st = -(int64_t)item - 1;
        const int a0 = sptr[st], a1 = sptr[st + 1], la = a1 - a0;
        gr_strip_sum(a0 + (int)((int64_t)la * warp / 8), a0 + (int)((int64_t)la * (warp + 1) / 8),
                     sid, sp, sq, tl, lane, s_id[warp], s_p[warp], s_q[warp], acc);
#pragma unroll
        for (int i = 0; i < kGrStrip; ++i) tile[warp * kGrStrip + i][lane] = acc[i];
        __syncthreads();
        if (warp < kGrStrip) {
            float2 t = make_float2(0.f, 0.f);
            for (int w = 0; w < 8; ++w) {
                t.x += tile[w * kGrStrip + warp][lane].x;
                t.y += tile[w * kGrStrip + warp][lane].y;
            }
            const int u = (int)(st / nsx), v = (int)(st % nsx) * kGrStrip + warp;
            if (v < hv && lane < nviews) grids[(size_t)lane * grid_stride + (size_t)u * hv + v] = t;
        }
        return;
    }
    const int u = item / ngrp, g = item % ngrp;
    const int sx = g * 8 + warp;
    if (sx < nsx) {
        const int64_t st = (int64_t)u * nsx + sx;
        if (!heavy[st])
            gr_strip_sum(sptr[st], sptr[st + 1], sid, sp, sq, tl, lane, s_id[warp], s_p[warp],
                         s_q[warp], acc);
    }
#pragma unroll
    for (int i = 0; i < kGrStrip; ++i) tile[warp * kGrStrip + i][lane] = acc[i];
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int v = e >> 5, cl = e & 31;
        const int cv = g * 32 + cl;                       // cell along v in the row
        const int csx = cv / kGrStrip;
        if (v < nviews && cv < hv && !heavy[(int64_t)u * nsx + csx])
            grids[(size_t)v * grid_stride + (size_t)u * hv + cv] = tile[cl][v];
    }
}

// node-scaled t-spectra: out[id][v] = fac_id * (conj?) in[v][src_id] for
// ids [0, n), views v < nb (views >= nb unwritten; the readers mask them)
__global__ void k_views_nodes(const float2* __restrict__ in, int nb, int64_t nspec,
                              const GrNode* __restrict__ tab, int64_t n,
                              float2* __restrict__ out);

// forward: out[v][col] = fac * sum_taps w * grid_v   for views [v0, v0 + nv).
// HALF: the grids are the [K0][K1/2+1] half spectra of real inputs (R2C);
// cells with k1 > K1/2 are read as conj(G[-k]) (copied from the mirror
// asynchronously, conjugated in place after the wait).
template <int J, int VG, bool HALF = false>
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
    const FastDiv dreg(nreg), dR1(R1);
    const int K0 = tg.K[0], K1 = tg.K[1];
    const int ld = HALF ? K1 / 2 + 1 : K1;
    for (int e = threadIdx.x; e < nv * nreg; e += blockDim.x) {
        const int v = dreg.div(e), c = e - v * nreg;
        const int r0 = dR1.div(c), r1 = c - r0 * R1;
        int g0 = wrapc(o[0] + r0, K0), g1 = wrapc(o[1] + r1, K1);
        if (HALF && g1 > K1 / 2) {
            g0 = g0 ? K0 - g0 : 0;
            g1 = K1 - g1;
        }
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(tile + e)),
                     "l"(grids + (size_t)(v0 + v) * grid_stride + (size_t)g0 * ld + g1));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if constexpr (HALF) {
        // conjugate the mirrored cells: those whose wrapped k1 exceeds K1/2
        for (int e = threadIdx.x; e < nv * nreg; e += blockDim.x) {
            const int c = e - dreg.div(e) * nreg;
            const int r1 = c - dR1.div(c) * R1;
            if (wrapc(o[1] + r1, K1) > K1 / 2) tile[e].y = -tile[e].y;
        }
    }
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
