// Views-in-lanes resampling records shared by the forward gather
// (cbn_projector.cu) and the backprojector's transposed spread
// (cbn_backproject.cu).
#pragma once

#include "cbn_kernels.cuh"
#include "cbn_projector.h"
#include "cbn_sources.cuh"

namespace cbn {

// Taps of one base-view (view 0) umbrella target in grid order (rho, theta,
// phi): view v's phi taps are these shifted by v * (2 n_phi / V) cells with the
// same weights (u_phi(v) = u_phi(0) - 2 v n_phi / V exactly), so the per-view
// kernel does no index math at all.
template <int J>
struct RsTap {
    int f[3];       // first tap per axis, wrapped into [0, K)
    int valid;
    float w[3][J];
};

template <int J>
__global__ void k_rs_taps(UmbrellaSrc src, KBSet kb, int64_t n, RsTap<J>* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double wd[3];
    UmbrellaSrc::Aux aux;
    src.node(i, wd, aux);                               // device order (phi, theta, rho)
    const double w[3] = {wd[2], wd[1], wd[0]};          // grid order (rho, theta, phi)
    int first[3];
    float wt[3][J];
    tap_setup<3, J>(kb, w, first, wt);
    RsTap<J> t;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        t.f[d] = wrapc(first[d], kb.ax[d].K);
#pragma unroll
        for (int p = 0; p < J; ++p) t.w[d][p] = wt[d][p];
    }
    t.valid = aux.valid ? 1 : 0;
    out[i] = t;
}

// ----------------------------------------------------------------------
// Transposed resample (resample_transpose, pipeline.py:183-184) as a gather.
// With views in lanes the transpose is a scatter of 283 M targets x 27 taps
// of fp32 REDs per step at config 2, bound by L2 atomic element throughput
// (consecutive-address REDs from views-in-lanes measured slower still).  The
// targets of view v are view 0's shifted by v * shift phi cells, so a grid
// column (rho, theta) of the phi-fast grid receives exactly the view-0
// targets whose rho/theta taps cover it, each at every view: a per-plan CSR
// of (target, rho/theta weight) entries per column turns the transpose into
// a gather with one thread per phi cell, register accumulation, and one
// plain store of every grid cell (no atomics, no memset).
struct RsColEntry {
    int t;          // view-0 target (row of the transposed values)
    int f2;         // first phi tap of view 0
    float wab;      // rho x theta weight of this column
    float w2[3];    // phi weights (J = 3)
};

template <int J>
__global__ void k_rs_col_count(const RsTap<J>* __restrict__ taps, int64_t n, int K0, int K1,
                               int* __restrict__ counts) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const RsTap<J> tp = taps[t];
    if (!tp.valid) return;
#pragma unroll
    for (int a = 0; a < J; ++a)
#pragma unroll
        for (int b = 0; b < J; ++b)
            atomicAdd(counts + (size_t)wrapc(tp.f[0] + a, K0) * K1 + wrapc(tp.f[1] + b, K1), 1);
}

template <int J>
__global__ void k_rs_col_fill(const RsTap<J>* __restrict__ taps, int64_t n, int K0, int K1,
                              int* __restrict__ cursor, RsColEntry* __restrict__ out) {
    static_assert(J == 3, "column entries hold three phi weights");
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const RsTap<J> tp = taps[t];
    if (!tp.valid) return;
#pragma unroll
    for (int a = 0; a < J; ++a)
#pragma unroll
        for (int b = 0; b < J; ++b) {
            const size_t col = (size_t)wrapc(tp.f[0] + a, K0) * K1 + wrapc(tp.f[1] + b, K1);
            RsColEntry e;
            e.t = (int)t;
            e.f2 = tp.f[2];
            e.wab = tp.w[0][a] * tp.w[1][b];
#pragma unroll
            for (int c = 0; c < 3; ++c) e.w2[c] = tp.w[2][c];
            out[atomicAdd(cursor + col, 1)] = e;
        }
}

// the fill's atomic cursors leave each column's entries in arrival order;
// sorting them by target makes every column sum (and so the transposed
// resample, den included) independent of the plan build: one thread per
// column, insertion sort (a few to a few hundred entries per column)
static __global__ void k_rs_col_sort(const int* __restrict__ col_ptr, int64_t ncol,
                                     RsColEntry* __restrict__ ent) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    const int lo = col_ptr[c], hi = col_ptr[c + 1];
    for (int i = lo + 1; i < hi; ++i) {
        const RsColEntry e = ent[i];
        int j = i - 1;
        while (j >= lo && ent[j].t > e.t) {
            ent[j + 1] = ent[j];
            --j;
        }
        ent[j + 1] = e;
    }
}

// acc[e] += gain * prod_d scale_d[e_d] * IFFT(g)[k], k_d = idx_d[e_d], from
// F = the forward 3D FFT of the real grid g kept as the half spectrum along
// axis 0 (phi; [rho][theta][phi/2+1], strides a_d.sstride): IFFT(g)[k] is
// conj(F[k]) for k_0 <= K_0/2 and F[-k] otherwise.
// Through 32 x 32 (axis 0 x axis 2) shared-memory tiles per axis-1 cell:
// F's contiguous axis is 0 (phi), acc's is 2 (rho).  Grid
// (ceil(a2.n / 32), ceil(a0.n / 32), a1.n), block (32, 8).
static __global__ void k_remap_half_acc_tile(const float2* __restrict__ F, float2* __restrict__ acc,
                                             RemapAxis a0, RemapAxis a1, RemapAxis a2, int K0,
                                             int K1, int K2) {
    __shared__ float2 tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int e00 = blockIdx.y * 32, e20 = blockIdx.x * 32, e1 = blockIdx.z;
    const int k1c = a1.idx[e1];
    const float s1 = a1.scale[e1];
    const int e0 = e00 + tx;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int e2 = e20 + r;
        if (e0 >= a0.n || e2 >= a2.n) continue;
        int k0 = a0.idx[e0], k1 = k1c, k2 = a2.idx[e2];
        float2 v = make_float2(0.f, 0.f);
        if (k0 >= 0 && k1 >= 0 && k2 >= 0) {
            const float sc = a0.scale[e0] * s1 * a2.scale[e2];
            float sg = -1.f;
            if (k0 > K0 / 2) {
                k0 = K0 - k0;
                k1 = k1 ? K1 - k1 : 0;
                k2 = k2 ? K2 - k2 : 0;
                sg = 1.f;
            }
            const float2 f = F[k0 * a0.sstride + k1 * a1.sstride + k2 * a2.sstride];
            v = make_float2(sc * f.x, sg * sc * f.y);
        }
        tile[r][tx] = v;
    }
    __syncthreads();
    const int e2 = e20 + tx;
    if (e2 >= a2.n) return;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int ee0 = e00 + r;
        if (ee0 >= a0.n) break;
        float2* d = acc + ((size_t)ee0 * a1.n + e1) * a2.n + e2;
        const float2 o = *d, v = tile[tx][r];
        *d = make_float2(o.x + v.x, o.y + v.y);
    }
}

// rho lines from the half spectrum G [K_rho][K_theta][K_phi/2+1] of the used
// rho planes (others read as zero): lines[(iph * nth + ith) * K_rho + x] =
// G[x][lth[ith]][lph[iph]], through 32 x 32 tiles per ith.  Grid
// (ceil(K_rho / 32), ceil(nph / 32), nth), block (32, 8).
static __global__ void k_lines_from_half(const float2* __restrict__ G,
                                         const unsigned char* __restrict__ used,
                                         const int* __restrict__ lth, const int* __restrict__ lph,
                                         int nth, int nph, int Kr, int Kt, int hp,
                                         float2* __restrict__ lines) {
    __shared__ float2 tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x0 = blockIdx.x * 32, ip0 = blockIdx.y * 32, it = blockIdx.z;
    const int kt = lth[it];
    const int ip = ip0 + tx;
    const int kp = ip < nph ? lph[ip] : 0;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int x = x0 + r;
        if (x >= Kr || ip >= nph) continue;
        tile[r][tx] = used[x] ? G[((size_t)x * Kt + kt) * hp + kp] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    const int x = x0 + tx;
    if (x >= Kr) return;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int q = ip0 + r;
        if (q >= nph) break;
        lines[((size_t)q * nth + it) * Kr + x] = tile[tx][r];
    }
}

// the transposed-resample crop from the rho lines F (forward FFT along rho):
// acc[e0][e1][e2] += s0 s1 s2 * IFFT(g)[k] with k_d = idx_d[e_d] (phi, theta,
// rho), IFFT(g)[k] = conj F(k0, k1; k2) for k0 <= K0/2, else F(-k0, -k1; -k2).
// Grid (ceil(a2.n / 256), a1.n, a0.n).
static __global__ void k_crop_from_lines(const float2* __restrict__ F, RemapAxis a0, RemapAxis a1,
                                         RemapAxis a2, const int* __restrict__ thmap,
                                         const int* __restrict__ phmap, int nth, int K0, int K1,
                                         int K2, float2* __restrict__ acc) {
    const int e2 = blockIdx.x * blockDim.x + threadIdx.x;
    if (e2 >= a2.n) return;
    const int e0 = blockIdx.z, e1 = blockIdx.y;
    int k0 = a0.idx[e0], k1 = a1.idx[e1], k2 = a2.idx[e2];
    if (k0 < 0 || k1 < 0 || k2 < 0) return;
    const float sc = a0.scale[e0] * a1.scale[e1] * a2.scale[e2];
    float sg = -1.f;
    if (k0 > K0 / 2) {
        k0 = K0 - k0;
        k1 = k1 ? K1 - k1 : 0;
        k2 = k2 ? K2 - k2 : 0;
        sg = 1.f;
    }
    const float2 f = F[((size_t)phmap[k0] * nth + thmap[k1]) * K2 + k2];
    float2* d = acc + ((size_t)e0 * a1.n + e1) * a2.n + e2;
    const float2 o = *d;
    *d = make_float2(o.x + sc * f.x, o.y + sg * sc * f.y);
}

// ----------------------------------------------------------------------
// Pole targets (theta == 0; see UmbrellaSrc): the reference sets their phi
// per view from signed zeros, so view 0's taps shifted by whole phi cells do
// not apply.  They are listed once per plan, dropped from the view-0 tap
// records (valid = 0, after the rho-plane scan), and handled per view by
// k_rs_pole_gather (forward) / k_rs_pole_spread (transpose) -- one or two
// targets per view.
constexpr int kMaxPoles = 4096;

template <int J>
__global__ void k_rs_poles(UmbrellaSrc src0, int64_t n, RsTap<J>* __restrict__ taps,
                           int* __restrict__ list, int* __restrict__ count) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double wd[3];
    UmbrellaSrc::Aux aux;
    src0.node(t, wd, aux);
    if (!aux.pole) return;
    taps[t].valid = 0;
    const int k = atomicAdd(count, 1);
    if (k < kMaxPoles) list[k] = (int)t;
}

// lists the poles into u.poles / u.n_poles and clears their tap records
template <int J>
void build_poles(UmbrellaTables& u, const UmbrellaSrc& src0, int64_t n, RsTap<J>* taps,
                 cudaStream_t s) {
    DevBuf<int> cnt(1);
    CBN_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), s));
    u.poles.alloc(kMaxPoles);
    k_rs_poles<J><<<blocks_for(n, 256), 256, 0, s>>>(src0, n, taps, u.poles.p, cnt.p);
    CBN_LAUNCH_CHECK();
    int h = 0;
    CBN_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    CBN_REQUIRE(h <= kMaxPoles, "too many pole targets");
    u.n_poles = h;
}

// Re(resample_apply) at the pole targets of views [v0, v0 + nb): the grid is
// phi-fast [rho][theta][phi] (ES floats per cell, the real part read); kb in
// grid order (rho, theta, phi); src.view0 = v0
template <int J, int ES>
__global__ void k_rs_pole_gather(const float* __restrict__ G, KBSet kb, UmbrellaSrc src,
                                 const int* __restrict__ poles, int npoles, int64_t per_view, int nb,
                                 float* __restrict__ vals, const float* __restrict__ tscale,
                                 int n_t) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= npoles * nb) return;
    const int v = q / npoles;
    const int64_t t = poles[q % npoles];
    double wd[3];
    UmbrellaSrc::Aux aux;
    src.node((int64_t)v * per_view + t, wd, aux);
    const double w[3] = {wd[2], wd[1], wd[0]};
    int first[3];
    float wt[3][J];
    tap_setup<3, J>(kb, w, first, wt);
    const int K0 = kb.ax[0].K, K1 = kb.ax[1].K, K2 = kb.ax[2].K;
    float acc = 0.f;
    for (int a = 0; a < J; ++a)
        for (int b = 0; b < J; ++b) {
            const size_t row = ((size_t)wrapc(first[0] + a, K0) * K1 + wrapc(first[1] + b, K1)) * K2;
            float r = 0.f;
            for (int c = 0; c < J; ++c)
                r = fmaf(wt[2][c], __ldg(G + ES * (row + wrapc(first[2] + c, K2))), r);
            acc = fmaf(wt[0][a] * wt[1][b], r, acc);
        }
    if (!aux.valid) acc = 0.f;
    vals[(size_t)v * per_view + t] = tscale ? acc * tscale[t % n_t] : acc;
}

// transposed resample at the pole targets of views [v0, v0 + nb) into the
// real phi-fast grid G (after the column gather wrote it): values from valsT
// [target][nb] (null: the validity mask, den)
template <int J>
__global__ void k_rs_pole_spread(float* __restrict__ G, KBSet kb, UmbrellaSrc src,
                                 const int* __restrict__ poles, int npoles, int64_t per_view, int nb,
                                 const float* __restrict__ valsT) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= npoles * nb) return;
    const int v = q / npoles;
    const int64_t t = poles[q % npoles];
    double wd[3];
    UmbrellaSrc::Aux aux;
    src.node((int64_t)v * per_view + t, wd, aux);
    if (!aux.valid) return;
    const double w[3] = {wd[2], wd[1], wd[0]};
    int first[3];
    float wt[3][J];
    tap_setup<3, J>(kb, w, first, wt);
    const float x = valsT ? valsT[(size_t)t * nb + v] : 1.f;
    const int K0 = kb.ax[0].K, K1 = kb.ax[1].K, K2 = kb.ax[2].K;
    for (int a = 0; a < J; ++a)
        for (int b = 0; b < J; ++b) {
            const size_t row = ((size_t)wrapc(first[0] + a, K0) * K1 + wrapc(first[1] + b, K1)) * K2;
            const float wab = wt[0][a] * wt[1][b] * x;
            for (int c = 0; c < J; ++c) atomicAdd(G + row + wrapc(first[2] + c, K2), wab * wt[2][c]);
        }
}

// used[k] = 1 for every axis-0 (rho) plane a valid target's taps touch
template <int J>
__global__ void k_rs_rho_used(const RsTap<J>* __restrict__ taps, int64_t n, int K0,
                              int* __restrict__ used) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n || !taps[t].valid) return;
    const int f = taps[t].f[0];
#pragma unroll
    for (int a = 0; a < J; ++a) {
        const int k = f + a >= K0 ? f + a - K0 : f + a;
        if (!used[k]) used[k] = 1;
    }
}

// vals [nv][n] -> valsT [n][nv]
static __global__ void k_transpose_vals(const float* __restrict__ in, int nv, int64_t n,
                                 float* __restrict__ out) {
    __shared__ float tile[32][33];
    const int64_t t0 = (int64_t)blockIdx.x * 32;
    const int v0 = blockIdx.y * 32;
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
        const int v = e >> 5, tt = e & 31;
        if (v0 + v < nv && t0 + tt < n) tile[v][tt] = in[(size_t)(v0 + v) * n + t0 + tt];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
        const int tt = e >> 5, v = e & 31;
        if (v0 + v < nv && t0 + tt < n) out[(size_t)(t0 + tt) * nv + v0 + v] = tile[v][tt];
    }
}

// One CTA per grid column (rho, theta); threads over phi.  Views [vlo, vlo+nv)
// of valsT [target][nv]; writes num if gnum -- and den if gden -- to every
// cell of the column of the real grid (den-only passes: gnum and valsT null).
constexpr int kRsColThreads = 256;

static __global__ void __launch_bounds__(kRsColThreads)
k_rs_gather_cols(float* __restrict__ gnum, float* __restrict__ gden, int K2,
                 const int* __restrict__ col_ptr, const RsColEntry* __restrict__ ent,
                 const float* __restrict__ valsT, int vlo, int nv, int shift) {
    const size_t col = blockIdx.x;
    const int beg = col_ptr[col], end = col_ptr[col + 1];
    for (int phi = threadIdx.x; phi < K2; phi += kRsColThreads) {
        float num = 0.f, den = 0.f;
        for (int k = beg; k < end; ++k) {
            const RsColEntry e = ent[k];
            const float* vt = valsT + (size_t)e.t * nv;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                // view v covers phi = f2 - v shift + c  (mod K2)
                int d = e.f2 + c - phi;
                d = d < 0 ? d + K2 : (d >= K2 ? d - K2 : d);
                const int v = d / shift;
                const int rel = v - vlo;
                if (v * shift == d && rel >= 0 && rel < nv) {
                    const float wk = e.wab * e.w2[c];
                    if (valsT) num = fmaf(wk, __ldg(vt + rel), num);
                    den += wk;
                }
            }
        }
        if (gnum) gnum[col * K2 + phi] = num;
        if (gden) gden[col * K2 + phi] = den;
    }
}

// shift = 2 (K2 = 2 V, configs 2 and 3): thread i owns the cell pair
// (2i, 2i+1).  With d = f2 - 2i and base = floor(d / 2), the three phi taps of
// an entry land as
//   d even: cell 2i   <- w0 val[base] + w2 val[base+1],  cell 2i+1 <- w1 val[base]
//   d odd:  cell 2i+1 <- w0 val[base] + w2 val[base+1],  cell 2i   <- w1 val[base+1]
// so every entry costs two value loads and three FMAs per thread, no search.
constexpr int kRsPairThreads = 384;

template <bool DEN>   // false: values into gnum; true: validity mask into gden
static __global__ void __launch_bounds__(kRsPairThreads)
k_rs_gather_cols2(float* __restrict__ gnum, float* __restrict__ gden, int V,
                  const int* __restrict__ col_ptr, const RsColEntry* __restrict__ ent,
                  const float* __restrict__ valsT, int vlo, int nv,
                  const unsigned char* __restrict__ plane_used, int K1) {
    const size_t col = blockIdx.x;
    if (!plane_used[col / K1]) return;   // rho plane never transformed
    const int beg = col_ptr[col], end = col_ptr[col + 1];
    for (int i = threadIdx.x; i < V; i += kRsPairThreads) {
        float ne = 0.f, no = 0.f, de = 0.f, dn = 0.f;
#pragma unroll 4
        for (int k = beg; k < end; ++k) {
            const RsColEntry e = ent[k];
            const int d = e.f2 - 2 * i;
            int b0 = d >> 1;                       // floor(d / 2)
            b0 += b0 < 0 ? V : 0;
            int b1 = b0 + 1;
            b1 -= b1 >= V ? V : 0;
            int r0 = b0 - vlo, r1 = b1 - vlo;
            r0 += r0 < 0 ? V : 0;
            r1 += r1 < 0 ? V : 0;
            const bool ok0 = r0 < nv, ok1 = r1 < nv;
            const float* vt = valsT + (size_t)e.t * nv;
            const float x0 = (ok0 && !DEN) ? __ldg(vt + r0) : 0.f;
            const float x1 = (ok1 && !DEN) ? __ldg(vt + r1) : 0.f;
            const float u0 = ok0 ? 1.f : 0.f, u1 = ok1 ? 1.f : 0.f;
            const float w0 = e.wab * e.w2[0], w1 = e.wab * e.w2[1], w2 = e.wab * e.w2[2];
            if ((d & 1) == 0) {
                ne = fmaf(w0, x0, fmaf(w2, x1, ne));
                no = fmaf(w1, x0, no);
                de = fmaf(w0, u0, fmaf(w2, u1, de));
                dn = fmaf(w1, u0, dn);
            } else {
                no = fmaf(w0, x0, fmaf(w2, x1, no));
                ne = fmaf(w1, x1, ne);
                dn = fmaf(w0, u0, fmaf(w2, u1, dn));
                de = fmaf(w1, u1, de);
            }
        }
        if (!DEN) *(reinterpret_cast<float2*>(gnum + col * 2 * V) + i) = make_float2(ne, no);
        else *(reinterpret_cast<float2*>(gden + col * 2 * V) + i) = make_float2(de, dn);
    }
}

// Strip form of the column gather: a target's 3 x 3 (rho, theta) taps put
// the same 2 value loads and phi weights into 9 columns; strips of kRsStrip
// consecutive theta columns of one rho plane, with a strip's column lists
// merged by target at plan time (host, sorted by target), load each value
// pair once per strip and apply it to every column the target reaches there
// (per-column rho-theta weight wab[c], zero elsewhere).
constexpr int kRsStrip = 4;

struct RsStripEnt {
    int t;          // view-0 target
    int f2;         // first phi tap of view 0
};

template <bool DEN>
static __global__ void __launch_bounds__(kRsPairThreads)
k_rs_gather_strips(float* __restrict__ gnum, float* __restrict__ gden, int V,
                   const int* __restrict__ sptr, const RsStripEnt* __restrict__ ent,
                   const float4* __restrict__ w2s, const float4* __restrict__ wabs,
                   const float* __restrict__ valsT, int vlo, int nv,
                   const unsigned char* __restrict__ plane_used, int K1, int nsx) {
    const int strip = blockIdx.x;
    const int rho = strip / nsx, c0 = (strip - rho * nsx) * kRsStrip;
    if (!plane_used[rho]) return;   // rho plane never transformed
    const int beg = sptr[strip], end = sptr[strip + 1];
    for (int i = threadIdx.x; i < V; i += kRsPairThreads) {
        float ev[kRsStrip], od[kRsStrip];
#pragma unroll
        for (int c = 0; c < kRsStrip; ++c) ev[c] = od[c] = 0.f;
#pragma unroll 2
        for (int k = beg; k < end; ++k) {
            const RsStripEnt e = ent[k];
            const float4 w2 = w2s[k], wab = wabs[k];
            const int d = e.f2 - 2 * i;
            int b0 = d >> 1;                       // floor(d / 2)
            b0 += b0 < 0 ? V : 0;
            int b1 = b0 + 1;
            b1 -= b1 >= V ? V : 0;
            int r0 = b0 - vlo, r1 = b1 - vlo;
            r0 += r0 < 0 ? V : 0;
            r1 += r1 < 0 ? V : 0;
            const bool ok0 = r0 < nv, ok1 = r1 < nv;
            float x0, x1;
            if constexpr (DEN) {
                x0 = ok0 ? 1.f : 0.f;
                x1 = ok1 ? 1.f : 0.f;
            } else {
                const float* vt = valsT + (size_t)e.t * nv;
                x0 = ok0 ? __ldg(vt + r0) : 0.f;
                x1 = ok1 ? __ldg(vt + r1) : 0.f;
            }
            // the target's contribution to the even / odd phi cell of the pair
            const float a = fmaf(w2.x, x0, w2.z * x1);
            const float b = (d & 1) == 0 ? w2.y * x0 : w2.y * x1;
            const float ae = (d & 1) == 0 ? a : b, ao = (d & 1) == 0 ? b : a;
            const float wc[4] = {wab.x, wab.y, wab.z, wab.w};
#pragma unroll
            for (int c = 0; c < kRsStrip; ++c) {
                ev[c] = fmaf(wc[c], ae, ev[c]);
                od[c] = fmaf(wc[c], ao, od[c]);
            }
        }
        float* g = DEN ? gden : gnum;
#pragma unroll
        for (int c = 0; c < kRsStrip; ++c)
            if (c0 + c < K1)
                *(reinterpret_cast<float2*>(g + ((size_t)rho * K1 + c0 + c) * 2 * V) + i) =
                    make_float2(ev[c], od[c]);
    }
}

}  // namespace cbn
