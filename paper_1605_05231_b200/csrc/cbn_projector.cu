// NUFFT cone-beam forward projector and direct backprojector on the B200.
//
// Forward  (pipeline.py:122-147):
//   volume --[deapod/pad, cuFFT (2N)^3, KB J gather at radial nodes, phase *
//   trilinear * i omega]--> radial lines --[cuFFT along rho]--> derivative
//   Radon lattice --[origin average, rho pad, cuFFT]--> lattice spectrum;
//   per reference view batch: [LS fit, deapod/pad, cuFFT 2x, KB J=3 gather at
//   umbrella targets] --> umbrella values; per view: [t cuFFT, filter, 2D KB
//   spread, cuFFT, crop/deapod/w1, ring mean] --> detector frames.
// Backprojector (pipeline.py:150-212): the transposed chain.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "cbn_projector.h"
#include "cbn_resample_views.cuh"
#include "cbn_dirichlet.cuh"
#include "cbn_specgather.cuh"

using namespace cbn;

namespace cbn {

// ----------------------------------------------------------------- tables
void RadialTables::build(int nr, int nt, int np_, double rmax, double vox, cudaStream_t s) {
    n_rho = nr;
    n_theta = nt;
    n_phi = np_;
    rho_max = rmax;
    d_rho = 2.0 * rmax / nr;                  // RadialGridSpec.delta_rho
    std::vector<double> h_om(nr), h_cp(np_), h_sp(np_), h_ct(nt), h_st(nt);
    std::vector<float> h_omp(nr), h_stf(nt);
    for (int k = 0; k < nr; ++k) {
        // radial_omega (radon_fourier.py:46-49), then * voxel (radon_fourier.py:61)
        double omega = (kTwoPi * (double)(k - nr / 2)) / ((double)nr * d_rho);
        h_om[k] = omega * vox;
        h_omp[k] = (float)omega;
    }
    for (int j = 0; j < nt; ++j) {
        double th = ((double)j * kPi) / (double)nt;
        h_ct[j] = std::cos(th);
        h_st[j] = std::sin(th);
        h_stf[j] = (float)h_st[j];
    }
    for (int k = 0; k < np_; ++k) {
        double ph = (((double)k * 2.0) * kPi) / (double)np_;
        h_cp[k] = std::cos(ph);
        h_sp[k] = std::sin(ph);
    }
    om.upload(h_om.data(), nr, s);
    cphi.upload(h_cp.data(), np_, s);
    sphi.upload(h_sp.data(), np_, s);
    cth.upload(h_ct.data(), nt, s);
    sth.upload(h_st.data(), nt, s);
    om_phys.upload(h_omp.data(), nr, s);
    sin_theta.upload(h_stf.data(), nt, s);
    CBN_CUDA(cudaStreamSynchronize(s));
}

void UmbrellaTables::build(const cbn_geometry& g, int nmu, int nt, double pitch, cudaStream_t s) {
    n_mu = nmu;
    n_t = nt;
    dt = pitch;
    std::vector<double> ca(g.n_views), sa(g.n_views), cm(nmu), sm(nmu), om(nt);
    for (int k = 0; k < g.n_views; ++k) {
        double a = (kTwoPi * (double)k) / (double)g.n_views;   // ConeGeometry.view_angle
        ca[k] = std::cos(a);
        sa[k] = std::sin(a);
    }
    for (int i = 0; i < nmu; ++i) {
        double mu = ((double)i * kPi) / (double)nmu;             // umbrella_line_grid
        cm[i] = std::cos(mu);
        sm[i] = std::sin(mu);
    }
    for (int j = 0; j < nt; ++j)
        om[j] = (kTwoPi * (double)(j - nt / 2)) / ((double)nt * pitch);   // grangeat.py:109
    cos_a.upload(ca.data(), ca.size(), s);
    sin_a.upload(sa.data(), sa.size(), s);
    cos_mu.upload(cm.data(), cm.size(), s);
    sin_mu.upload(sm.data(), sm.size(), s);
    omega_t.upload(om.data(), om.size(), s);
    CBN_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------- epilogues

// radial spectrum -> i omega * trilinear * phase, written at the ifftshifted
// rho position of its line (image_to_radial_spectrum + trilinear_transfer +
// spectral_rho_derivative + the input shift of _centered_ifft).
__global__ void k_radial_pairs(RadialSrc r, KBSet kb, int J, int64_t lines, int* __restrict__ idx,
                               int* __restrict__ extra, int64_t base_count, int64_t line0) {
    const int n = r.n_rho, nh = n / 2 + 1;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= lines * nh) return;
    const int k = (int)(e % nh);
    const int64_t line = line0 + e / nh;
    const int64_t f = line * n + k;
    if (k == 0 || k == n / 2) {
        idx[e] = ~(int)f;
        return;
    }
    double w[3], wm[3];
    RadialSrc::Aux a, am;
    r.node(f, w, a);
    r.node(line * n + (n - k), wm, am);
    bool exact = true;
#pragma unroll
    for (int d = 0; d < 3; ++d)
        // mirrored up to rounding (no 2 pi jump at a wrap tie), same tap structure
        exact = exact && fabs(w[d] + wm[d]) < 1e-12 && fabs(a.wc[d] + am.wc[d]) < 1e-12 &&
                mirror_taps_match(kb.ax[d].K, J, w[d], wm[d]);
    if (exact) {
        idx[e] = (int)f;
    } else {
        idx[e] = ~(int)f;
        idx[base_count + atomicAdd(extra, 1)] = ~(int)(line * n + (n - k));
    }
}

// perm[k] = idx[perm[k]] (in place)
__global__ void k_gather_index(const int* __restrict__ idx, int64_t n, int* __restrict__ perm) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) perm[k] = idx[perm[k]];
}

struct SpecOut {
    float2* out;
    const float* om_phys;
    int N[3];              // volume dims (centre phase * plan phase, per node representative)
    int n_rho;
    int tri;
    int spectrum_only;     // 1: image_to_radial_spectrum values in node order
    int packed = 0;   // 1: i is a RadialPackedSrc entry (f: mirror too, ~f: node alone)
    CBN_D void put(int64_t i, float2 v, const double (&w)[3], const RadialSrc::Aux& a) const {
        double ang = centre_plan_angle<3>(a.wc, w, N);
        double sn, cs;
        sincos(ang, &sn, &cs);
        float2 r = cmul(v, make_float2((float)cs, (float)sn));
        const int64_t line = (i >= 0 ? i : ~i) / n_rho;
        const bool mirror = packed && i >= 0;   // the conjugate goes to rho index n_rho - ir
        if (spectrum_only) {
            out[line * n_rho + a.ir] = r;
            if (mirror) out[line * n_rho + (n_rho - a.ir)] = make_float2(r.x, -r.y);
            return;
        }
        if (tri) {
            float t = 1.f;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                float x = (float)(a.raw[d] * (1.0 / kTwoPi));
                float sc = x == 0.f ? 1.f : sinpif(x) / (3.14159265358979f * x);
                t *= sc * sc;
            }
            r = cscale(r, t);
        }
        const float o = om_phys[a.ir];
        const int k = (a.ir + n_rho - n_rho / 2) % n_rho;
        const float2 val = make_float2(-r.y * o, r.x * o);
        out[line * n_rho + k] = val;
        if (mirror)   // the derivative spectrum of a real volume is Hermitian along the line
            out[line * n_rho + (n_rho - a.ir + n_rho - n_rho / 2) % n_rho] = make_float2(val.x, -val.y);
    }
};

// per-plan records of k_spec_gather (cbn_specgather.cuh), one per sorted
// primary node: the KB argument y and edge-tap decision per axis exactly as
// kb_weights forms them from tap_setup, the tap origin in its bin tile, the
// SpecOut epilogue factor in float64 and the lattice indices
template <int J>
__global__ void k_spec_records(RadialSrc src, KBSet kb, TileGeom<3> tg,
                               const int* __restrict__ perm, int64_t m,
                               const float* __restrict__ om_phys, int n_vol, int tri,
                               float4* __restrict__ rec, float2* __restrict__ fac,
                               int2* __restrict__ out) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= m) return;
    const int f = perm[pos];
    double w[3];
    RadialSrc::Aux a;
    src.node(f >= 0 ? f : ~f, w, a);
    unsigned bits = 0;
    float y[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        int first;
        const double u = axis_coord(w[d], kb.ax[d].K, 0.5 * (double)J, first);
        const double fr = dsub(u, (double)first);
        y[d] = (float)(2.0 * (fr - (0.5 * J - 1.0)) - 1.0);
        const bool drop = fr >= 0.5 * J * (1.0 - 1e-12) && !kb_inside(fr, J);
        bits |= (unsigned)(wrapc(first, kb.ax[d].K) % tg.T[d]) << (5 * d);
        if (drop) bits |= 1u << (15 + d);
    }
    rec[pos] = make_float4(y[0], y[1], y[2], __uint_as_float(bits));
    const int N3[3] = {n_vol, n_vol, n_vol};
    double sn, cs;
    sincos(centre_plan_angle<3>(a.wc, w, N3), &sn, &cs);
    double t = 1.0;
    if (tri) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double x = a.raw[d] * (1.0 / kTwoPi);
            const double sc = x == 0.0 ? 1.0 : sinpi(x) / (kPi * x);
            t *= sc * sc;
        }
    }
    // val = i * omega * t * e^{i ang} * v
    const double g = t * (double)om_phys[a.ir];
    fac[pos] = make_float2((float)(-sn * g), (float)(cs * g));
    const int n_rho = src.n_rho;
    const int line = (f >= 0 ? f : ~f) / n_rho;
    out[pos] = make_int2(line * n_rho + (a.ir + n_rho - n_rho / 2) % n_rho,
                         f >= 0 ? line * n_rho + (n_rho - a.ir + n_rho - n_rho / 2) % n_rho : -1);
}

struct UmbOut {
    float* vals;
    const float* tscale = nullptr;   // optional per-t factor (1 / w2 of the Grangeat step)
    int n_t = 1;
    CBN_D void put(int64_t i, float2 v, const double (&)[3], const UmbrellaSrc::Aux& a) const {
        float x = a.valid ? v.x : 0.f;   // Re(resample_apply), invalid -> 0 (pipeline.py:136-137)
        if (tscale) x *= tscale[i % n_t];
        vals[i] = x;
    }
};

// Resample gather with views in lanes, for geometries where consecutive views'
// targets differ by a whole number of oversampled phi cells (2 n_phi / V
// integer) and share one resample grid.  The grid is stored phi-fastest
// [rho][theta][phi]; a warp takes one base target and lanes take 32 views, so
// the rho/theta taps and index math are warp-uniform and the phi taps of
// the lanes are consecutive cells.  32 base targets per CTA; values are
// transposed through shared memory so each view's row is stored coalesced.
template <int J>
__global__ void __launch_bounds__(256)
k_resample_views(const float2* __restrict__ G, int K0, int K1, int K2,
                 const RsTap<J>* __restrict__ taps, int64_t per_view, int v0, int nviews,
                 int shift, float* __restrict__ vals, const float* __restrict__ tscale, int n_t) {
    __shared__ float tile[32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t0 = (int64_t)blockIdx.x * 32;
    const int v = v0 + lane;
    const int pshift = (int)(((int64_t)v * shift) % K2);
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
        const int tl = warp * 4 + q;
        const int64_t t = t0 + tl;
        float out = 0.f;
        if (t < per_view) {
            const RsTap<J> tp = taps[t];
            if (tp.valid && lane < nviews) {
                const int fp = tp.f[2] - pshift;
                int c2[J];
#pragma unroll
                for (int c = 0; c < J; ++c) {
                    int x = fp + c;
                    x = x < 0 ? x + K2 : x;
                    c2[c] = x >= K2 ? x - K2 : x;
                }
                float acc = 0.f;
#pragma unroll
                for (int a = 0; a < J; ++a) {
                    const float2* plane = G + (size_t)wrapc(tp.f[0] + a, K0) * K1 * K2;
                    float pa = 0.f;
#pragma unroll
                    for (int b = 0; b < J; ++b) {
                        const float2* row = plane + (size_t)wrapc(tp.f[1] + b, K1) * K2;
                        float r = 0.f;
#pragma unroll
                        for (int c = 0; c < J; ++c) r = fmaf(tp.w[2][c], __ldg(row + c2[c]).x, r);
                        pa = fmaf(tp.w[1][b], r, pa);
                    }
                    acc = fmaf(tp.w[0][a], pa, acc);
                }
                out = acc;   // Re(resample_apply): only the real part is kept
            }
        }
        tile[lane][tl] = out;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int v = e >> 5, tt = e & 31;
        if (v < nviews && t0 + tt < per_view) {
            const float x = tile[v][tt];
            vals[(size_t)v * per_view + t0 + tt] = tscale ? x * tscale[(t0 + tt) % n_t] : x;
        }
    }
}

// J = 3 (the reference default) view-lane gather on precomputed rows: the nine
// (rho, theta) tap rows of a view-0 target as 32-bit cell offsets of the
// phi-fast grid and the nine rho x theta weight products, so a lane's work is
// nine row bases, 27 loads of real parts and 36 FMAs -- the warp-uniform
// index math of k_resample_views is done once per plan instead of per lane.
struct alignas(16) RsRow3 {
    unsigned int row[9];   // (wrap(f0 + a) K1 + wrap(f1 + b)) K2, a major
    int f2;                // first phi tap of view 0
    int valid;
    float w2[3];
    float wab[9];          // w0[a] w1[b]
    int pad;               // 96 bytes: six 16-byte loads per record
};

__global__ void k_rs_rows3(const RsTap<3>* __restrict__ taps, int64_t n, int K0, int K1, int K2,
                           RsRow3* __restrict__ out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const RsTap<3> tp = taps[t];
    RsRow3 r;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            r.row[a * 3 + b] = (unsigned)(((int64_t)wrapc(tp.f[0] + a, K0) * K1 +
                                           wrapc(tp.f[1] + b, K1)) * K2);
            r.wab[a * 3 + b] = tp.w[0][a] * tp.w[1][b];
        }
    r.f2 = tp.f[2];
    r.valid = tp.valid;
    r.pad = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) r.w2[c] = tp.w[2][c];
    out[t] = r;
}

template <int ES>   // floats per grid cell: 1 real grid, 2 complex (real part read)
__global__ void __launch_bounds__(256)
k_resample_rows3(const float* __restrict__ G, int K2, const RsRow3* __restrict__ rows,
                 int64_t per_view, int v0, int nviews, int shift, float* __restrict__ vals,
                 const float* __restrict__ tscale, int n_t) {
    __shared__ float tile[32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t0 = (int64_t)blockIdx.x * 32;
    const int pshift = (int)(((int64_t)(v0 + lane) * shift) % K2);
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
        const int tl = warp * 4 + q;
        const int64_t t = t0 + tl;
        float out = 0.f;
        if (t < per_view) {
            // the whole record through six 16-byte loads (same address in all lanes)
            RsRow3 rr;
            const uint4* src = reinterpret_cast<const uint4*>(rows + t);
            uint4* dst = reinterpret_cast<uint4*>(&rr);
#pragma unroll
            for (int k = 0; k < 6; ++k) dst[k] = __ldg(src + k);
            if (rr.valid == 1 && lane < nviews) {
                int c0 = rr.f2 - pshift;
                c0 += c0 < 0 ? K2 : 0;
                int c1 = c0 + 1, c2 = c0 + 2;
                c1 -= c1 >= K2 ? K2 : 0;
                c2 -= c2 >= K2 ? K2 : 0;
                const float w0 = rr.w2[0], w1 = rr.w2[1], w2 = rr.w2[2];
                float acc = 0.f;
                if constexpr (ES == 1) {
                    // 32-bit cell index (grid < 2^32 cells).  The three phi taps
                    // c0..c0+2 lie in two aligned cell pairs (K2 even, so pairs
                    // never straddle the row end): two 8-byte loads per row
                    // instead of three 4-byte ones, and with the view shift of
                    // 2 cells the warp's pairs are one contiguous 256-byte span
                    (void)c1;
                    (void)c2;
                    const unsigned p0 = (unsigned)c0 & ~1u;
                    const unsigned p1 = p0 + 2 == (unsigned)K2 ? 0u : p0 + 2;
                    const bool odd = c0 & 1;
#pragma unroll
                    for (int ab = 0; ab < 9; ++ab) {
                        const unsigned b = rr.row[ab];
                        const float2 q0 = __ldg(reinterpret_cast<const float2*>(G + (b + p0)));
                        const float2 q1 = __ldg(reinterpret_cast<const float2*>(G + (b + p1)));
                        const float t0 = odd ? q0.y : q0.x;
                        const float t1 = odd ? q1.x : q0.y;
                        const float t2 = odd ? q1.y : q1.x;
                        float r = w0 * t0;
                        r = fmaf(w1, t1, r);
                        r = fmaf(w2, t2, r);
                        acc = fmaf(rr.wab[ab], r, acc);
                    }
                } else {
                    const float* g0 = G + (size_t)ES * c0;
                    const float* g1 = G + (size_t)ES * c1;
                    const float* g2 = G + (size_t)ES * c2;
#pragma unroll
                    for (int ab = 0; ab < 9; ++ab) {
                        const size_t o = (size_t)ES * rr.row[ab];
                        float r = w0 * __ldg(g0 + o);
                        r = fmaf(w1, __ldg(g1 + o), r);
                        r = fmaf(w2, __ldg(g2 + o), r);
                        acc = fmaf(rr.wab[ab], r, acc);
                    }
                }
                out = acc;   // Re(resample_apply): the real part of each cell
            }
        }
        tile[lane][tl] = out;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int v = e >> 5, tt = e & 31;
        if (v < nviews && t0 + tt < per_view) {
            const float x = tile[v][tt];
            vals[(size_t)v * per_view + t0 + tt] = tscale ? x * tscale[(t0 + tt) % n_t] : x;
        }
    }
}

// Windowed view-chunk gather (J = 3, real phi-fast grid).  View v of a target
// reads the three phi cells c0(v) = f2 - shift v (+0, 1, 2) of each of its nine
// (rho, theta) rows, and c0 does not depend on the row.  So per target the
// row-weighted sum R(c) = sum_ab wab[ab] G_ab[c] is formed once over the phi
// window the chunk's views reach (length shift (nv - 1) + 3, in aligned float4
// slots, coalesced 16-byte loads), kept in shared memory, and every view is
// then three shared-memory reads and three FMAs: 9 x 4 B per window cell
// instead of 27 x 4 B per view (views overlap 1-2 cells at shift 2), and the
// row reads are contiguous spans instead of 64-lane scatters.
//   CTA = 8 warps x 4 targets = 32 consecutive targets; each warp owns a
//   window buffer (K2 + 4 floats); the [view][32 targets] output tile goes out
//   in 128-byte rows.  Pole targets (valid == 2) read their per-view phi cell
//   from `pole_f2` ([pole][V]); invalid targets (valid == 0) are zero.
// chunk of 120 views: at shift 2 the window is <= 61 float4 slots, two passes of
// the warp (360 = 3 x 120 at config 2)
constexpr int kWinWarps = 8, kWinTargets = 4, kWinChunk = 120;

__host__ __device__ constexpr int win_buf_floats(int K2) { return ((K2 + 4 + 3) / 4) * 4; }

__global__ void __launch_bounds__(kWinWarps * 32)
k_resample_window(const float* __restrict__ G, int K2, const RsRow3* __restrict__ rows,
                  int64_t per_view, int v0, int nv, int shift, const int* __restrict__ pole_f2,
                  int n_views, float* __restrict__ vals, const float* __restrict__ tscale, int n_t) {
    extern __shared__ float4 smem4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bufn = win_buf_floats(K2);
    float* buf = reinterpret_cast<float*>(smem4) + warp * bufn;
    float* tile = reinterpret_cast<float*>(smem4) + kWinWarps * bufn;   // [nv][33] (padded)
    const int64_t t0 = (int64_t)blockIdx.x * (kWinWarps * kWinTargets);
    const int K4 = K2 >> 2;
    const float4* G4 = reinterpret_cast<const float4*>(G);
    const int L = shift * (nv - 1) + 3;           // window cells the chunk's views reach
    const bool full = L > K2 - 4;
    // shift * view offsets mod K2 (32-bit: shift * n_views < 2^31)
    const int sh_last = (int)(((int64_t)shift * (v0 + nv - 1)) % K2);
    const int sh_lane = (int)(((int64_t)shift * (v0 + lane)) % K2);
    const int step32 = (32 * shift) % K2;
#pragma unroll 1
    for (int q = 0; q < kWinTargets; ++q) {
        const int tl = warp * kWinTargets + q;
        const int64_t t = t0 + tl;
        if (t >= per_view) break;
        RsRow3 rr;
        {
            const uint4* src = reinterpret_cast<const uint4*>(rows + t);
            uint4* dst = reinterpret_cast<uint4*>(&rr);
#pragma unroll
            for (int k = 0; k < 6; ++k) dst[k] = __ldg(src + k);
        }
        if (rr.valid == 0) {
            for (int v = lane; v < nv; v += 32) tile[v * 33 + tl] = 0.f;
            continue;
        }
        if (rr.valid == 2) {
            // pole target: its phi cell follows each view's own geometry
            for (int v = lane; v < nv; v += 32) {
                const int c0 = pole_f2[(int64_t)rr.pad * n_views + v0 + v];
                CBN_DCHECK(c0 >= 0 && c0 < K2, "window gather: pole cell out of range");
                const int c1 = c0 + 1 >= K2 ? c0 + 1 - K2 : c0 + 1;
                const int c2 = c0 + 2 >= K2 ? c0 + 2 - K2 : c0 + 2;
                float acc = 0.f;
#pragma unroll
                for (int ab = 0; ab < 9; ++ab) {
                    const float* g = G + rr.row[ab];
                    float r = rr.w2[0] * __ldg(g + c0);
                    r = fmaf(rr.w2[1], __ldg(g + c1), r);
                    r = fmaf(rr.w2[2], __ldg(g + c2), r);
                    acc = fmaf(rr.wab[ab], r, acc);
                }
                tile[v * 33 + tl] = acc;
            }
            continue;
        }
        // window start cell (the last view's c0) and its float4 slots
        int cs = rr.f2 - sh_last;
        cs += cs < 0 ? K2 : 0;
        const int s4 = full ? 0 : (cs >> 2);
        const int n4 = full ? K4 : (((cs & 3) + L + 3) >> 2);
        for (int j = lane; j < n4; j += 32) {
            int g4 = s4 + j;
            g4 -= g4 >= K4 ? K4 : 0;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            float4 x[9];
#pragma unroll
            for (int ab = 0; ab < 9; ++ab) x[ab] = __ldg(G4 + (rr.row[ab] >> 2) + g4);
#pragma unroll
            for (int ab = 0; ab < 9; ++ab) {
                const float w = rr.wab[ab];
                a.x = fmaf(w, x[ab].x, a.x);
                a.y = fmaf(w, x[ab].y, a.y);
                a.z = fmaf(w, x[ab].z, a.z);
                a.w = fmaf(w, x[ab].w, a.w);
            }
            reinterpret_cast<float4*>(buf)[j] = a;
        }
        __syncwarp();
        if (full && lane < 2) buf[K2 + lane] = buf[lane];   // circular tail
        __syncwarp();
        const int base = full ? 0 : 4 * s4;
        // o(v) = f2 - shift (v0 + v) - base (mod K2), stepped by 32 views
        int o = rr.f2 - sh_lane - base;
        o += o < 0 ? K2 : 0;
        o += o < 0 ? K2 : 0;
        for (int v = lane; v < nv; v += 32, o -= step32, o += o < 0 ? K2 : 0) {
            // the three cells as one aligned pair + one cell (an even shift keeps
            // the lanes' pairs on distinct banks: 2 wavefronts per read)
            CBN_DCHECK(o >= 0 && o + 2 < (full ? K2 + 2 : 4 * n4), "window gather: cell outside window");
            float b0, b1, b2;
            if (o & 1) {
                b0 = buf[o];
                const float2 q = *reinterpret_cast<const float2*>(buf + o + 1);
                b1 = q.x;
                b2 = q.y;
            } else {
                const float2 q = *reinterpret_cast<const float2*>(buf + o);
                b0 = q.x;
                b1 = q.y;
                b2 = buf[o + 2];
            }
            float r = rr.w2[0] * b0;
            r = fmaf(rr.w2[1], b1, r);
            r = fmaf(rr.w2[2], b2, r);
            tile[v * 33 + tl] = r;
        }
        __syncwarp();
    }
    __syncthreads();
    // [view][32 targets] tile -> vals[v][t0 + tt] (128-byte rows)
    {
        // each thread keeps one target column (256 threads = 8 view rows x 32)
        const int tt = threadIdx.x & 31;
        const int64_t t = t0 + tt;
        if (t < per_view) {
            const float sc = tscale ? tscale[(int)(t % n_t)] : 1.f;
            float* dst = vals + t;
            for (int v = threadIdx.x >> 5; v < nv; v += kWinWarps)
                dst[(size_t)v * per_view] = tile[v * 33 + tt] * sc;
        }
    }
}

inline size_t win_smem_bytes(int K2, int nv) {
    return sizeof(float) * ((size_t)kWinWarps * win_buf_floats(K2) + (size_t)nv * 33);
}

// pole rows: valid = 2, pad = pole index; per-view phi cells of every pole
__global__ void k_pole_rows(const int* __restrict__ poles, int npoles, RsRow3* __restrict__ rows) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= npoles) return;
    rows[poles[q]].valid = 2;
    rows[poles[q]].pad = q;
}

__global__ void k_pole_table(UmbrellaSrc src0, KBSet kb, const int* __restrict__ poles, int npoles,
                             int n_views, int f0_ref_check, int* __restrict__ table,
                             int* __restrict__ mismatch) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= npoles * n_views) return;
    const int q = e / n_views, v = e % n_views;
    UmbrellaSrc sv = src0;
    sv.view0 = v;
    double wd[3];
    UmbrellaSrc::Aux aux;
    sv.node(poles[q], wd, aux);
    const double w[3] = {wd[2], wd[1], wd[0]};
    int first[3];
    float wt[3][3];
    tap_setup<3, 3>(kb, w, first, wt);
    table[e] = wrapc(first[2], kb.ax[2].K);
    // the pole's rho / theta taps must be view 0's (theta == 0, rho snapped)
    if (f0_ref_check) {
        UmbrellaSrc s0 = src0;
        s0.view0 = 0;
        double w0d[3];
        s0.node(poles[q], w0d, aux);
        const double ww[3] = {w0d[2], w0d[1], w0d[0]};
        int f0[3];
        float wt0[3][3];
        tap_setup<3, 3>(kb, ww, f0, wt0);
        if (f0[0] != first[0] || f0[1] != first[1]) atomicAdd(mismatch, 1);
    }
}

// ----------------------------------------------------------------- kernels

// lattice[line][j] = raw[line][(j - n//2) mod n] * scale   (fftshift of the IFFT)
__global__ void k_lattice_final(const float2* __restrict__ raw, float2* __restrict__ out, int n,
                                int64_t total, float scale) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    int j = (int)(e % n);
    int64_t line = e / n;
    float2 v = raw[line * n + (j - n / 2 + n) % n];
    out[e] = make_float2(v.x * scale, v.y * scale);
}

// partial sums of src[line][col] over lines (complex, float64)
__global__ void k_col_partial(const float2* __restrict__ src, int64_t lines, int64_t ld, int col,
                              double* __restrict__ partial) {
    double re = 0.0, im = 0.0;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < lines;
         l += (int64_t)gridDim.x * blockDim.x) {
        float2 v = src[l * ld + col];
        re += v.x;
        im += v.y;
    }
    __shared__ double sr[32], si[32];
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sr[threadIdx.x >> 5] = re;
        si[threadIdx.x >> 5] = im;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += sr[w];
            b += si[w];
        }
        partial[2 * blockIdx.x] = a;
        partial[2 * blockIdx.x + 1] = b;
    }
}

__global__ void k_partial_final(const double* __restrict__ partial, int nblk, double mul,
                                double* __restrict__ out) {
    if (threadIdx.x != 0) return;
    double a = 0, b = 0;
    for (int i = 0; i < nblk; ++i) {
        a += partial[2 * i];
        b += partial[2 * i + 1];
    }
    out[0] = a * mul;
    out[1] = b * mul;
}

constexpr int kRedBlocks = 296;

// mean over lines of src[line][col] * scale -> out[0..1]
static void column_mean(const float2* src, int64_t lines, int64_t ld, int col, double scale,
                        double* partial, double* out, cudaStream_t s) {
    k_col_partial<<<kRedBlocks, 256, 0, s>>>(src, lines, ld, col, partial);
    CBN_LAUNCH_CHECK();
    k_partial_final<<<1, 32, 0, s>>>(partial, kRedBlocks, scale / (double)lines, out);
    CBN_LAUNCH_CHECK();
}

// x = pad_rho(origin_average(lattice)) (resampling.py:106-117, 144-145) in the
// device layout [line][rho_padded]; src[line][(j + shift) % n] * scale is the
// lattice value at rho index j.
__global__ void k_pad_lattice(const float2* __restrict__ src, int shift, float scale, int n,
                              int pad, int dr, int64_t total, const double* __restrict__ mean,
                              float2* __restrict__ out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    int r = (int)(e % dr);
    int64_t line = e / dr;
    int j = r - pad;
    float2 v = make_float2(0.f, 0.f);
    if (j >= 0 && j < n) {
        if (j == n / 2) {
            v = make_float2((float)mean[0], (float)mean[1]);
        } else {
            float2 g = src[line * n + (j + shift) % n];
            v = make_float2(g.x * scale, g.y * scale);
        }
    }
    out[e] = v;
}

// ---- reverse Grangeat (grangeat.py:149-170)
// k_views_nodes fused with the real-to-complex split: `z` holds the length-M
// complex FFTs (M = n_t / 2) of the real t lines read as complex pairs
// (z[n] = x[2n] + i x[2n+1]), [view][mu][M]; bin k of the real FFT is
// E[k] + W^k O[k], W = exp(-2 pi i / n_t), with E / O the even / odd-sample
// spectra (Z[k] +- conj Z[-k]) / (2, 2i).  Rows as k_views_nodes.
__global__ void k_views_nodes_z(const float2* __restrict__ z, int nb, int n_mu, int M,
                                const GrNode* __restrict__ tab, int64_t n,
                                float2* __restrict__ out) {
    __shared__ float2 tile[32][33];
    __shared__ GrNode nd[32];
    __shared__ int zk[32], zm[32];
    __shared__ float2 tw[32];
    const int64_t e0 = (int64_t)blockIdx.x * 32;
    const int nh = M + 1;
    if (threadIdx.x < 32 && e0 + threadIdx.x < n) {
        const GrNode g = tab[e0 + threadIdx.x];
        nd[threadIdx.x] = g;
        const int mu = g.src / nh, k = g.src - mu * nh;
        zk[threadIdx.x] = mu * M + (k == M ? 0 : k);
        zm[threadIdx.x] = mu * M + (k == 0 ? 0 : M - k);
        float sn, cs;
        sincospif((float)k / (float)M, &sn, &cs);     // 2 pi k / n_t
        tw[threadIdx.x] = make_float2(cs, -sn);
    }
    __syncthreads();
    const int64_t per = (int64_t)n_mu * M;
    // 256 threads: thread = (view row q / 32, node e), four view rows each; the
    // eight loads of a thread are issued before the first is used
    const int e = threadIdx.x & 31, v0 = threadIdx.x >> 5;
    const bool live = e0 + e < n;
    float2 za[4], zb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int v = v0 + 8 * i;
        if (live && v < nb) {
            za[i] = z[(size_t)v * per + zk[e]];
            zb[i] = z[(size_t)v * per + zm[e]];   // conj taken below
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int v = v0 + 8 * i;
        if (live && v < nb) {
            const GrNode g = nd[e];
            const float2 a = za[i], b = zb[i];
            // E = (a + conj b) / 2, O = (a - conj b) / (2i)
            const float2 E = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
            const float2 O = make_float2(0.5f * (a.y + b.y), -0.5f * (a.x - b.x));
            const float2 w = tw[e];
            float2 x = make_float2(E.x + w.x * O.x - w.y * O.y, E.y + w.x * O.y + w.y * O.x);
            if (g.conj) x.y = -x.y;
            tile[v][e] = make_float2(g.fac.x * x.x - g.fac.y * x.y, g.fac.x * x.y + g.fac.y * x.x);
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int eo = v0 + 8 * i, v = e;
        if (v < nb && e0 + eo < n) out[(size_t)(e0 + eo) * 32 + v] = tile[v][eo];
    }
}

__global__ void k_views_nodes(const float2* __restrict__ in, int nb, int64_t nspec,
                              const GrNode* __restrict__ tab, int64_t n,
                              float2* __restrict__ out) {
    __shared__ float2 tile[32][33];
    __shared__ GrNode nd[32];
    const int64_t e0 = (int64_t)blockIdx.x * 32;
    if (threadIdx.x < 32 && e0 + threadIdx.x < n) nd[threadIdx.x] = tab[e0 + threadIdx.x];
    __syncthreads();
    for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) {
        const int v = q >> 5, e = q & 31;
        if (v < nb && e0 + e < n) {
            const GrNode g = nd[e];
            float2 x = in[(size_t)v * nspec + g.src];
            if (g.conj) x.y = -x.y;
            tile[v][e] = make_float2(g.fac.x * x.x - g.fac.y * x.y, g.fac.x * x.y + g.fac.y * x.x);
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) {
        const int e = q >> 5, v = q & 31;
        if (v < nb && e0 + e < n) out[(size_t)(e0 + e) * 32 + v] = tile[v][e];
    }
}

// rows of vals * (1 / w2[t]) (grangeat.py:152) for callers passing raw values
__global__ void k_gr_scale(const float* __restrict__ vals, const float* __restrict__ w2inv, int n_t,
                           int64_t total, float* __restrict__ out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    out[e] = vals[e] * w2inv[e % n_t];
}

CBN_D double w1_at(int u, int v, int nu, int nv, double pu, double pv, double so) {
    double uc = (((double)u - (double)nu / 2.0) + 0.5) * pu;
    double vc = (((double)v - (double)nv / 2.0) + 0.5) * pv;
    return so / sqrt(so * so + uc * uc + vc * vc);
}

struct GrPost {
    int nu, nv, Ku, Kv;
    const float* pix;   // [nu][nv] s_u s_v / w1
};

CBN_D float gr_re(const float2* g, size_t i) { return g[i].x; }
CBN_D float gr_re(const float* g, size_t i) { return g[i]; }

// detector pixel (u, v) of one view's inverse-transformed grid (complex: Re;
// real: the complex-to-real output), [Ku][Kv]
template <class T>
CBN_D float gr_value(const T* grid, const GrPost& p, int u, int v) {
    int gu = (u - p.nu / 2 + p.Ku) % p.Ku;
    int gv = (v - p.nv / 2 + p.Kv) % p.Kv;
    return gr_re(grid, (size_t)gu * p.Kv + gv) * p.pix[(size_t)u * p.nv + v];
}

// per-pixel factor of the Grangeat post / pre step, once per plan in float64:
// reverse: s_u s_v / w1 (grangeat.py:166, nufft.py:247); forward: w1 s_u s_v
// (grangeat.py:139, nufft.py:226)
__global__ void k_gr_pix(const float* __restrict__ s32, int smax, int nu, int nv, double pu,
                         double pv, double so, int reverse, float* __restrict__ pix) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nu * nv) return;
    const int u = e / nv, v = e % nv;
    const double w1 = w1_at(u, v, nu, nv, pu, pv, so);
    const double sc = (double)s32[u] * (double)s32[smax + v];
    pix[e] = (float)(reverse ? sc / w1 : sc * w1);
}

void ensure_gr_pix(const cbn_projector_s* p, GrangeatPlan& gp, bool reverse, cudaStream_t s) {
    if (gp.pix.p) return;
    const int nu = p->g.nu, nv = p->g.nv;
    gp.pix.alloc((size_t)nu * nv);
    k_gr_pix<<<blocks_for((int64_t)nu * nv, 256), 256, 0, s>>>(gp.s32.p, gp.smax, nu, nv, gp.pu,
                                                              gp.pv, p->g.so_mm, reverse ? 1 : 0,
                                                              gp.pix.p);
    CBN_LAUNCH_CHECK();
}

// mean of the outermost detector ring per view (grangeat.py:167-169)
template <class T>
__global__ void k_gr_ring(const T* __restrict__ grids, GrPost p, double* __restrict__ mean) {
    const int v = blockIdx.x;
    const T* grid = grids + (size_t)v * p.Ku * p.Kv;
    const int nring = p.nu == 1 || p.nv == 1 ? p.nu * p.nv : 2 * p.nu + 2 * p.nv - 4;
    double acc = 0.0;
    for (int r = threadIdx.x; r < nring; r += blockDim.x) {
        int u, w;
        if (p.nu == 1 || p.nv == 1) {
            u = r / p.nv;
            w = r % p.nv;
        } else if (r < p.nv) {
            u = 0;
            w = r;
        } else if (r < 2 * p.nv) {
            u = p.nu - 1;
            w = r - p.nv;
        } else {
            int k = r - 2 * p.nv;   // columns 0 and nv-1 of rows 1..nu-2
            u = 1 + k / 2;
            w = (k & 1) ? p.nv - 1 : 0;
        }
        acc += gr_value(grid, p, u, w);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        mean[v] = t / nring;
    }
}

template <class T>
__global__ void k_gr_frame(const T* __restrict__ grids, GrPost p,
                           const double* __restrict__ mean, float norm, float* __restrict__ frames,
                           int* __restrict__ flag) {
    // grid (nv / 256, nu, views): one detector row per (blockIdx.y, blockIdx.z)
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= p.nv) return;
    const int u = blockIdx.y, v = blockIdx.z;
    float g = gr_value(grids + (size_t)v * p.Ku * p.Kv, p, u, w);
    float out = (float)((double)g - mean[v]) * norm;
    if (!isfinite(out)) atomicOr(flag, 1);
    frames[((size_t)v * p.nu + u) * p.nv + w] = out;
}

}  // namespace cbn

// =================================================================== plan

namespace {

using P = cbn_projector_s;

int64_t spectrum_chunk(const P* p, int64_t m) {
    int64_t ch = p->c.plan_chunk > 0 ? p->c.plan_chunk : (int64_t)1 << 21;
    return std::min(m, ch);
}

std::vector<std::pair<int, int>> view_batches(int n_views, int64_t per_view, int64_t target) {
    int64_t step = std::max<int64_t>(1, target / per_view);
    std::vector<std::pair<int, int>> out;
    for (int64_t lo = 0; lo < n_views; lo += step)
        out.emplace_back((int)lo, (int)std::min<int64_t>(lo + step, n_views));
    return out;
}

int64_t target_batch(const P* p) { return p->c.target_batch > 0 ? p->c.target_batch : (int64_t)1 << 20; }

const int64_t* rows_for(P* p, int64_t m, int& n) {
    auto it = p->ls_rows.find(m);
    if (it == p->ls_rows.end())
        throw Error(CBN_EINVAL, "scaling-fit rows for a " + std::to_string(m) +
                                    "-node plan were not supplied (cbn_projector_set_ls_rows)");
    n = (int)it->second->n;
    return it->second->p;
}

void add_needed(P* p, int64_t m) {
    if (std::find(p->ls_needed.begin(), p->ls_needed.end(), m) == p->ls_needed.end())
        p->ls_needed.push_back(m);
}

int rho_pad_of(int cfg_pad, int n_rho) { return cfg_pad < 0 ? n_rho / 2 : cfg_pad; }

// resample_j may differ per axis (ProjectorConfig, resampling.py:79): the
// generic resample kernels loop the largest count (shorter axes carry zero
// weights, kb_weights); the views-in-lanes kernels need J = 3 on every axis
}  // namespace
int cbn::res_jmax(const AxisPlan* ax) { return std::max(ax[0].J, std::max(ax[1].J, ax[2].J)); }
bool cbn::res_j3(const AxisPlan* ax) { return ax[0].J == 3 && ax[1].J == 3 && ax[2].J == 3; }
namespace {

UmbrellaGeom umb_geom(const P* p, const UmbrellaTables& u, const RadialTables& r, int pad) {
    UmbrellaGeom g;
    g.cos_a = u.cos_a.p;
    g.sin_a = u.sin_a.p;
    g.cos_mu = u.cos_mu.p;
    g.sin_mu = u.sin_mu.p;
    g.so = p->g.so_mm;
    g.dt = u.dt;
    g.n_mu = u.n_mu;
    g.n_t = u.n_t;
    g.rho_max = r.rho_max;
    g.d_rho = r.d_rho;
    g.n_rho = r.n_rho;
    g.n_theta = r.n_theta;
    g.n_phi = r.n_phi;
    g.pad = pad;
    g.padded[0] = (double)(r.n_rho + 2 * pad);
    g.padded[1] = (double)r.n_theta;
    g.padded[2] = (double)r.n_phi;
    g.n_views = p->g.n_views;
    return g;
}

__global__ void k_umb_cache(UmbrellaSrc src, int64_t n, double4* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double pos[3];
    bool valid;
    src.position(i, pos, valid);
    out[i] = make_double4(pos[0], pos[1], pos[2], valid ? 1.0 : 0.0);
}

// umbrella source for the gathers / spreads: base-view cache + phi rotation
UmbrellaSrc cached_umbrella(P* p, UmbrellaTables& u, const RadialTables& r, int pad, int view0,
                            cudaStream_t s) {
    UmbrellaSrc src{umb_geom(p, u, r, pad), 0};
    if (!u.base_ready) {
        const int64_t per_view = (int64_t)u.n_mu * u.n_t;
        u.base.alloc((size_t)per_view);
        k_umb_cache<<<blocks_for(per_view, 256), 256, 0, s>>>(src, per_view, u.base.p);
        CBN_LAUNCH_CHECK();
        u.base_ready = true;
    }
    src.view0 = view0;
    const char* off = std::getenv("CBN_NO_UMB_CACHE");
    src.cache = (off && off[0] == '1') ? nullptr : u.base.p;
    return src;
}

void build_grangeat(P* p, GrangeatPlan& gp, const UmbrellaTables& u, int taper, cudaStream_t s) {
    gp.ax[0] = make_axis(p->g.nu, 5, 2.0);    // plan_grangeat j=(5,5), oversample 2 (grangeat.py:93-118)
    gp.ax[1] = make_axis(p->g.nv, 5, 2.0);
    gp.kb.ax[0] = gp.ax[0].kb;
    gp.kb.ax[1] = gp.ax[1].kb;
    gp.smax = std::max(p->g.nu, p->g.nv);
    gp.pu = p->pu;
    gp.pv = p->pv;
    gp.m = (int64_t)u.n_mu * u.n_t;
    gp.s32.alloc(2 * (size_t)gp.smax);
    std::vector<double> om(u.n_t);
    CBN_CUDA(cudaMemcpy(om.data(), u.omega_t.p, sizeof(double) * u.n_t, cudaMemcpyDeviceToHost));
    double amax = 0;
    for (double o : om) amax = std::max(amax, std::fabs(o));
    const double c2 = 1.0 / (2.0 * u.n_mu * u.n_t * u.dt);
    std::vector<float> w2(u.n_t), w2inv(u.n_t), q(u.n_t);
    const double so = p->g.so_mm;
    for (int j = 0; j < u.n_t; ++j) {
        double t = (double)(j - u.n_t / 2) * u.dt;
        w2[j] = (float)((so * so + t * t) / (so * so));
        w2inv[j] = (float)((so * so) / (so * so + t * t));
        double tp = 1.0;
        if (taper == 1) {
            double cv = std::cos(kPi * om[j] / (2.0 * amax));
            tp = cv * cv;
        }
        double sg = om[j] > 0 ? 1.0 : (om[j] < 0 ? -1.0 : 0.0);
        q[j] = (float)(-sg * tp * u.dt * c2);
    }
    gp.w2.upload(w2.data(), w2.size(), s);
    gp.w2inv.upload(w2inv.data(), w2inv.size(), s);
    gp.fac_im.upload(q.data(), q.size(), s);
    CBN_CUDA(cudaStreamSynchronize(s));
}

void fit_grangeat(P* p, GrangeatPlan& gp, const UmbrellaTables& u, cudaStream_t s) {
    int n;
    const int64_t* rows = rows_for(p, gp.m, n);
    PolarSrc src{u.omega_t.p, u.cos_mu.p, u.sin_mu.p, gp.pu, gp.pv, u.n_t};
    ls_fit<2>(src, rows, n, gp.ax, p->ls, gp.s32.p, gp.smax, s);
    gp.built = true;
}

void build_forward(P* p, cudaStream_t s) {
    if (p->fw_built) return;
    const cbn_projector_config& c = p->c;
    CBN_REQUIRE(c.method == 0 || c.method == 1, "method must be 0 ('a') or 1 ('b')");
    CBN_REQUIRE(c.method == 0 || (c.side_lobes >= 0 && c.side_lobes + 1 <= kMaxDirTaps),
                "side_lobes must be 0..7");
    CBN_REQUIRE(c.spectrum_j >= 2 && c.spectrum_j <= 8, "spectrum_j must be 2..8");
    p->frad.build(c.spec.n_rho, c.spec.n_theta, c.spec.n_phi, c.spec.rho_max, p->voxel, s);
    const double dt = c.t_pitch_mm > 0 ? c.t_pitch_mm : p->pu;
    p->fumb.build(p->g, c.n_mu, c.n_t, dt, s);
    for (int d = 0; d < 3; ++d) p->fspec[d] = make_axis(p->n_vol, c.spectrum_j, c.oversample_factor);
    p->fpad = rho_pad_of(c.rho_pad, c.spec.n_rho);
    const int dr = c.spec.n_rho + 2 * p->fpad;
    p->fres[0] = make_axis(c.spec.n_phi, c.resample_j[2], c.oversample_factor);
    p->fres[1] = make_axis(c.spec.n_theta, c.resample_j[1], c.oversample_factor);
    p->fres[2] = make_axis(dr, c.resample_j[0], c.oversample_factor);
    build_grangeat(p, p->fgr, p->fumb, c.t_taper, s);
    p->fw_built = true;
}

void build_backward(P* p, cudaStream_t s) {
    if (p->bw_built) return;
    const cbn_projector_config& c = p->c;
    CBN_REQUIRE(c.method == 0 || c.method == 1, "method must be 0 ('a') or 1 ('b')");
    CBN_REQUIRE(c.method == 0 || (c.side_lobes >= 0 && c.side_lobes + 1 <= kMaxDirTaps),
                "side_lobes must be 0..7");
    const int out = p->n_vol;
    const double extent = out * p->voxel;
    const int n_rho = 2 * (int)std::ceil(1.5 * out / 2.0);                 // pipeline.py:165
    p->brad.build(n_rho, c.spec.n_theta, c.spec.n_phi, extent * std::sqrt(3.0) / 2.0, p->voxel, s);
    p->bumb.build(p->g, c.n_mu, c.bp_n_t > 0 ? c.bp_n_t : 2 * p->g.nu,     // pipeline.py:168
                  c.bp_t_pitch_mm > 0 ? c.bp_t_pitch_mm : p->pu, s);
    for (int d = 0; d < 3; ++d) p->bspec[d] = make_axis(out, c.spectrum_j, c.oversample_factor);
    p->bpad = std::min(n_rho / 8, 32);                                       // pipeline.py:169
    const int dr = n_rho + 2 * p->bpad;
    p->bres[0] = make_axis(c.spec.n_phi, c.resample_j[2], c.oversample_factor);
    p->bres[1] = make_axis(c.spec.n_theta, c.resample_j[1], c.oversample_factor);
    p->bres[2] = make_axis(dr, c.resample_j[0], c.oversample_factor);
    build_grangeat(p, p->bgr, p->bumb, 0, s);
    p->bw_built = true;
}

void compute_needed(P* p) {
    const cbn_projector_config& c = p->c;
    p->ls_needed.clear();
    if (p->direction & 1) {
        int64_t M = (int64_t)c.spec.n_rho * c.spec.n_theta * c.spec.n_phi;
        add_needed(p, spectrum_chunk(p, M));
        int64_t per_view = (int64_t)c.n_mu * c.n_t;
        for (auto& b : view_batches(p->g.n_views, per_view, target_batch(p)))
            add_needed(p, per_view * (b.second - b.first));
        add_needed(p, per_view);
    }
    if (p->direction & 2) {
        const int n_rho = 2 * (int)std::ceil(1.5 * p->n_vol / 2.0);
        int64_t M = (int64_t)n_rho * c.spec.n_theta * c.spec.n_phi;
        add_needed(p, spectrum_chunk(p, M));
        int64_t per_view = (int64_t)c.n_mu * (c.bp_n_t > 0 ? c.bp_n_t : 2 * p->g.nu);
        for (auto& b : view_batches(p->g.n_views, per_view, target_batch(p)))
            add_needed(p, per_view * (b.second - b.first));
        add_needed(p, per_view);
    }
}

// per-axis tables from the scalings in p->s32 (stride smax) for one mode
void build_tables(P* p, int mode, const AxisPlan* ax, int smax, cudaStream_t s, RemapAxis* out,
                  const int64_t* sstride) {
    size_t need = 0;
    for (int d = 0; d < 3; ++d) need += (mode == kTabPad || mode == kTabPadShift) ? ax[d].K : ax[d].N;
    p->tab_idx.ensure(need);
    p->tab_sc.ensure(need);
    size_t off = 0;
    for (int d = 0; d < 3; ++d) {
        int n = (mode == kTabPad || mode == kTabPadShift) ? ax[d].K : ax[d].N;
        build_table(mode, ax[d].N, ax[d].K, p->s32.p + (size_t)d * smax, p->tab_idx.p + off,
                    p->tab_sc.p + off, s);
        out[d].idx = p->tab_idx.p + off;
        out[d].scale = p->tab_sc.p + off;
        out[d].n = n;
        out[d].sstride = sstride[d];
        off += n;
    }
}

int smax_of(const AxisPlan* ax) { return std::max(ax[0].N, std::max(ax[1].N, ax[2].N)); }

int64_t ktot(const AxisPlan* ax) { return (int64_t)ax[0].K * ax[1].K * ax[2].K; }

// ---------------------------------------------------------------- forward

// radial lattice in raw layout (IFFT output, ifftshifted rho) into p->lattice;
// with `spectrum` the image_to_radial_spectrum values go there instead (node
// order, no basis transfer / derivative / IFFT)
// spectrum gather at the radial nodes: `spectrum` set -> image_to_radial_spectrum
// values in node order; else the pre-IFFT lattice into `lat` (default
// p->lattice) followed by the radial IFFT.  nparts > 1: only the nodes of
// bin-subproblem share `part` (lat zeroed first); raw_only: stop before the
// IFFT (the sharded caller sums the shares, then fwd_views runs it)
bool spec_records_off() {   // CBN_SPEC_RECORDS=0: node generation per step (A/B)
    const char* e = std::getenv("CBN_SPEC_RECORDS");
    return e && e[0] == '0';
}

// buffers, cached scaling, pad tables and the compact pad lists of the spectrum
// NUFFT's input side (everything ahead of the pad kernel)
void spectrum_setup(P* p, cudaStream_t s, RemapAxis (&rax)[3]) {
    const RadialTables& r = p->frad;
    const AxisPlan* ax = p->fspec;
    const int64_t M = r.nodes();
    const int n = p->n_vol;
    const int64_t K3 = ktot(ax);
    p->big.ensure((size_t)K3);
    p->lattice.ensure((size_t)M);
    const int smax = n;
    p->s32.ensure(3 * (size_t)smax);
    {
        StageScope st(p->timer, "spectrum_fit", s);
        if (!p->fspec_fit) {
            // scaling of the first sub-plan of nufft_forward_chunked (nufft.py:250-265), cached
            int nrows;
            const int64_t* rows = rows_for(p, spectrum_chunk(p, M), nrows);
            p->fspec_s32.alloc(3 * (size_t)smax);
            ls_fit<3>(r.src(), rows, nrows, ax, p->ls, p->fspec_s32.p, smax, s);
            p->fspec_fit = true;
        }
        CBN_CUDA(cudaMemcpyAsync(p->s32.p, p->fspec_s32.p, sizeof(float) * 3 * smax,
                                 cudaMemcpyDeviceToDevice, s));
        const int64_t sstr[3] = {(int64_t)n * n, n, 1};
        build_tables(p, kTabPad, ax, smax, s, rax, sstr);
    }
    // the deapodised, padded volume is real: R2C to the half spectrum (the
    // gather reads k2 > K2/2 as conj(G[-k])); real grid at the front of `big`,
    // half spectrum behind it
    const long long kd[3] = {ax[0].K, ax[1].K, ax[2].K};
    const int64_t real_cells = (int64_t)kd[0] * kd[1] * kd[2];
    const int64_t half_off = (real_cells + 1) / 2;                // float2 units
    const int64_t half_cells = (int64_t)kd[0] * kd[1] * (kd[2] / 2 + 1);
    p->big.ensure((size_t)(half_off + half_cells));
    if (!p->fspec_list.p) {
        std::vector<int> all;
        for (int d = 0; d < 3; ++d) {
            const std::vector<int> l = pad_positions(ax[d].N, ax[d].K, false, false);
            p->fspec_nl[d] = (int)l.size();
            all.insert(all.end(), l.begin(), l.end());
        }
        p->fspec_list.upload(all.data(), all.size(), s);
        CBN_CUDA(cudaStreamSynchronize(s));
    }
}

// Staged input of the drop-in forward call (cbn_forward_stage_volume): the
// host converts and uploads the volume in chunks of its slowest axis, and each
// chunk's rows are deapodised, padded and 2D-transformed as soon as they are
// on the device, so only the last chunk's share of that work (and the pass
// along the slowest axis) is left when the upload ends.  Rows map to grid
// planes k = (n - N/2) mod K (pad_positions): rows >= N/2 to planes from 0,
// rows < N/2 to the planes below K; the compact list is sorted by plane.
void spectrum_stage_rows(P* p, const float* vol, int n_lo, int n_hi, cudaStream_t s) {
    const AxisPlan* ax = p->fspec;
    const int N = ax[0].N, K = ax[0].K, h = N / 2;
    CBN_REQUIRE(K >= N && p->fspec_nl[0] == N, "staged input needs one grid plane per volume row");
    const long long kd[3] = {ax[0].K, ax[1].K, ax[2].K};
    const int64_t real_cells = (int64_t)kd[0] * kd[1] * kd[2];
    const int64_t half_off = (real_cells + 1) / 2;
    const long long hz = kd[2] / 2 + 1, hplane = kd[1] * hz, rplane = kd[1] * kd[2];
    const long long k2[2] = {kd[1], kd[2]};
    float2* half = p->big.p + half_off;
    const float* real = reinterpret_cast<const float*>(p->big.p);
    const int* l = p->fspec_list.p;
    // (list index, first plane, count) of the rows below and from N/2
    const int part[2][2] = {{std::max(n_lo, h), std::max(n_hi, h)}, {std::min(n_lo, h), std::min(n_hi, h)}};
    for (int q = 0; q < 2; ++q) {
        const int a = part[q][0], b = part[q][1];
        if (b <= a) continue;
        const int li = q == 0 ? a - h : (N - h) + a;
        const int k0 = q == 0 ? a - h : K - h + a;
        k_remap_list3<float, kStoreRe><<<dim3((unsigned)((p->fspec_nl[2] + 255) / 256),
                                              p->fspec_nl[1], b - a), 256, 0, s>>>(
            vol, p->big.p, p->fspec_rax[0], p->fspec_rax[1], p->fspec_rax[2], l + li,
            l + p->fspec_nl[0], l + p->fspec_nl[0] + p->fspec_nl[1], p->fspec_nl[2], 1.0f);
        CBN_LAUNCH_CHECK();
        p->fft.exec_r2c3(p->fft.get_r2c2(k2, b - a), real + (long long)k0 * rplane,
                         half + (long long)k0 * hplane, s);
    }
}

void spectrum_stage_begin(P* p, cudaStream_t s) {
    spectrum_setup(p, s, p->fspec_rax);
    const AxisPlan* ax = p->fspec;
    const long long kd[3] = {ax[0].K, ax[1].K, ax[2].K};
    const int64_t real_cells = (int64_t)kd[0] * kd[1] * kd[2];
    const int64_t half_off = (real_cells + 1) / 2;
    const long long hplane = kd[1] * (kd[2] / 2 + 1);
    float2* half = p->big.p + half_off;
    // only the x planes the pad reaches are transformed: zero those
    for (const auto& rn : pad_runs(ax[0].N, ax[0].K, false))
        CBN_CUDA(cudaMemsetAsync(reinterpret_cast<float*>(p->big.p) + rn.first * kd[1] * kd[2], 0,
                                 sizeof(float) * kd[1] * kd[2] * (rn.second - rn.first), s));
    int lo = 0;
    for (const auto& rn : pad_runs(ax[0].N, ax[0].K, false)) {
        if (rn.first > lo)
            CBN_CUDA(cudaMemsetAsync(half + lo * hplane, 0, sizeof(float2) * hplane * (rn.first - lo), s));
        lo = rn.second;
    }
    if (lo < kd[0])
        CBN_CUDA(cudaMemsetAsync(half + lo * hplane, 0, sizeof(float2) * hplane * (kd[0] - lo), s));
}

void radial_lattice_raw(P* p, const float* vol, cudaStream_t s, float2* spectrum = nullptr,
                        int part = 0, int nparts = 1, float2* lat = nullptr,
                        bool raw_only = false, bool staged = false) {
    const RadialTables& r = p->frad;
    const AxisPlan* ax = p->fspec;
    const int64_t M = r.nodes();
    const int n = p->n_vol;
    RemapAxis rax[3];
    if (!staged) spectrum_setup(p, s, rax);
    p->fspec_staged = 0;            // staged rows are consumed (or discarded) here
    p->fspec_staged_vol = nullptr;
    long long kd[3] = {ax[0].K, ax[1].K, ax[2].K};
    const int64_t real_cells = (int64_t)kd[0] * kd[1] * kd[2];
    const int64_t half_off = (real_cells + 1) / 2;                // float2 units
    const int64_t half_cells = (int64_t)kd[0] * kd[1] * (kd[2] / 2 + 1);
    if (!staged)
    {
        // zero the grid, then fill only the cells the pad reaches (1/8 of them)
        StageScope st(p->timer, "spectrum_pad", s);
        // only the x planes the pad reaches are transformed: zero those
        double zeroed = 0.0;
        for (const auto& rn : pad_runs(ax[0].N, ax[0].K, false)) {
            CBN_CUDA(cudaMemsetAsync(reinterpret_cast<float*>(p->big.p) + rn.first * kd[1] * kd[2], 0,
                                     sizeof(float) * kd[1] * kd[2] * (rn.second - rn.first), s));
            zeroed += (double)kd[1] * kd[2] * (rn.second - rn.first);
        }
        // zero those planes, read the volume, write its N^3 cells
        p->timer.add_bytes("spectrum_pad", 4.0 * zeroed + 8.0 * (double)n * n * n, 0.0);
        const int* l = p->fspec_list.p;
        k_remap_list3<float, kStoreRe><<<dim3((unsigned)((p->fspec_nl[2] + 255) / 256),
                                              p->fspec_nl[1], p->fspec_nl[0]), 256, 0, s>>>(
            vol, p->big.p, rax[0], rax[1], rax[2], l, l + p->fspec_nl[0],
            l + p->fspec_nl[0] + p->fspec_nl[1], p->fspec_nl[2], 1.0f);
        CBN_LAUNCH_CHECK();
    }
    {
        // pruned 3D R2C: only the x planes the pad fills are non-zero, so the
        // batched 2D R2C over (y, z) runs on those planes (the others' half
        // planes are zeroed), then the C2C along x over every column
        StageScope st(p->timer, "spectrum_fft", s);
        const long long hz = kd[2] / 2 + 1, hplane = kd[1] * hz, rplane = kd[1] * kd[2];
        const long long k2[2] = {kd[1], kd[2]};
        float2* half = p->big.p + half_off;
        const float* real = reinterpret_cast<const float*>(p->big.p);
        int lo = 0;
        for (const auto& rn : staged ? std::vector<std::pair<int, int>>() : pad_runs(ax[0].N, ax[0].K, false)) {
            if (rn.first > lo)
                CBN_CUDA(cudaMemsetAsync(half + lo * hplane, 0,
                                         sizeof(float2) * hplane * (rn.first - lo), s));
            p->fft.exec_r2c3(p->fft.get_r2c2(k2, rn.second - rn.first), real + rn.first * rplane,
                             half + rn.first * hplane, s);
            lo = rn.second;
        }
        if (!staged && lo < kd[0])
            CBN_CUDA(cudaMemsetAsync(half + lo * hplane, 0, sizeof(float2) * hplane * (kd[0] - lo),
                                     s));
        p->fft.exec(p->fft.get_strided(kd[0], hplane, hplane, 1), half, half, CUFFT_FORWARD, s);
    }
    const float2* spec_half = p->big.p + half_off;
    if (!lat) lat = p->lattice.p;
    // a node-sharded plan (cbn_projector_set_node_shard) holds only its own
    // lines and writes only their lattice entries (gathered across ranks);
    // otherwise a share of the bin subproblems over all lines, summed across ranks
    const bool compact = p->fshard_nparts > 1;
    CBN_REQUIRE(!compact || (spectrum == nullptr && raw_only && part == p->fshard_part &&
                             nparts == p->fshard_nparts),
                "node-sharded plan: only its own cbn_forward_lattice share can run");
    const int64_t line_lo = compact ? r.lines() * part / nparts : 0;
    const int64_t line_hi = compact ? r.lines() * (part + 1) / nparts : r.lines();
    if (nparts > 1 && !compact) CBN_CUDA(cudaMemsetAsync(lat, 0, sizeof(float2) * M, s));
    SpecOut epi;
    epi.out = spectrum ? spectrum : lat;
    epi.om_phys = r.om_phys.p;
    for (int d = 0; d < 3; ++d) epi.N[d] = n;
    epi.n_rho = r.n_rho;
    epi.tri = p->c.basis == 0;
    epi.spectrum_only = spectrum != nullptr;
    // half the nodes: rho indices 0..n_rho/2 of every line, mirrors by conjugation
    if (!p->fpairs_n) {
        // plan step: the primary nodes (about half: conjugate pairs along each line)
        const int64_t nl = line_hi - line_lo;
        const int64_t base_n = nl * (r.n_rho / 2 + 1);
        p->fpairs.alloc((size_t)base_n + (size_t)nl * (r.n_rho / 2));
        DevBuf<int> extra(1);
        CBN_CUDA(cudaMemsetAsync(extra.p, 0, sizeof(int), s));
        KBSet kbp;
        for (int d = 0; d < 3; ++d) kbp.ax[d] = ax[d].kb;
        k_radial_pairs<<<blocks_for(base_n, 256), 256, 0, s>>>(r.src(), kbp, ax[0].J, nl,
                                                               p->fpairs.p, extra.p, base_n,
                                                               line_lo);
        CBN_LAUNCH_CHECK();
        int h_extra = 0;
        CBN_CUDA(cudaMemcpyAsync(&h_extra, extra.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CBN_CUDA(cudaStreamSynchronize(s));
        p->fpairs_n = base_n + h_extra;
    }
    const RadialPairSrc hsrc{r.src(), p->fpairs.p};
    const int64_t Mh = p->fpairs_n;
    epi.packed = 1;
    KBSet kb;
    for (int d = 0; d < 3; ++d) kb.ax[d] = ax[d].kb;
    if (!p->fspec_bins.ready) {
        StageScope st(p->timer, "spectrum_bins", s);
        // gather-only plan (no staging): 8 x 16 x 16 while the region stays under 48 KB
        const int tile[3] = {kTile3, ax[0].J <= 6 ? 2 * kTile3 : kTile3, kTile3Fast};
        dispatch_j(ax[0].J, [&](auto jc) {
            build_bins<3, decltype(jc)::value>(p->fspec_bins, hsrc, kb, Mh, tile, 4 * kMaxSub, s);   // gather only: larger subproblems, fewer region loads
            return 0;
        });
        // the sorted order stores the packed node entries themselves
        k_gather_index<<<blocks_for(Mh, 256), 256, 0, s>>>(p->fpairs.p, Mh, p->fspec_bins.perm.p);
        CBN_LAUNCH_CHECK();
    }
    {
        StageScope st(p->timer, "spectrum_gather", s);
        const BinPlan& bp = p->fspec_bins;
        const int s0 = compact ? 0 : (int)((int64_t)bp.nsubs * part / nparts);
        const int s1 = compact ? bp.nsubs : (int)((int64_t)bp.nsubs * (part + 1) / nparts);
        CBN_REQUIRE(bp.tg.R[2] <= 32, "half-spectrum gather: region rows above 32 cells");
        {
            // half spectrum read once, every lattice node written (mirrors by
            // conjugation), J^3 shared-memory tap reads per primary node
            const double f = bp.nsubs ? (double)(s1 - s0) / bp.nsubs : 0.0;
            const double J = ax[0].J;
            // + the 32-byte point records of the record-driven gather
            const double rec = (!epi.spectrum_only && !spec_records_off()) ? 32.0 * Mh : 0.0;
            p->timer.add_bytes("spectrum_gather", f * (8.0 * half_cells + 8.0 * M + rec),
                               f * 8.0 * J * J * J * (double)Mh);
        }
        // lattice values (not the API spectrum): the record-driven gather
        const bool recs = !epi.spectrum_only && !spec_records_off() &&
                          bp.tg.R[0] * bp.tg.R[1] <= kSpecMaxRows;
        if (recs && !p->fspec_rec.p) {
            p->fspec_rec.alloc((size_t)Mh);
            p->fspec_fac.alloc((size_t)Mh);
            p->fspec_out.alloc((size_t)Mh);
            dispatch_j(ax[0].J, [&](auto jc) {
                k_spec_records<decltype(jc)::value><<<blocks_for(Mh, 256), 256, 0, s>>>(
                    r.src(), kb, bp.geom<3>(), bp.perm.p, Mh, r.om_phys.p, n, epi.tri,
                    p->fspec_rec.p, p->fspec_fac.p, p->fspec_out.p);
                return 0;
            });
            CBN_LAUNCH_CHECK();
        }
        dispatch_j(ax[0].J, [&](auto jc) {
            constexpr int J = decltype(jc)::value;
            if (s1 <= s0) return 0;
            if (recs) {
                CBN_CUDA(cudaFuncSetAttribute(k_spec_gather<J>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)(sizeof(float2) * bp.nreg)));
                k_spec_gather<J><<<s1 - s0, 256, sizeof(float2) * bp.nreg, s>>>(
                    spec_half, kb, bp.geom<3>(),
                    SpecRec{p->fspec_rec.p, p->fspec_fac.p, p->fspec_out.p}, epi.out,
                    bp.subs.p + s0);
            } else
                k_gather_binned<3, J, RadialPackedSrc, SpecOut, true><<<s1 - s0, 256, sizeof(float2) * bp.nreg, s>>>(
                    spec_half, kb, bp.geom<3>(), RadialPackedSrc{r.src()}, epi, bp.perm.p,
                    bp.subs.p + s0);
            return 0;
        });
        CBN_LAUNCH_CHECK();
    }
    if (spectrum || raw_only) return;
    // centred IFFT along rho (radon_fourier.py:122-124,133-135); 1/(n d_rho) applied by consumers
    long long nr1[1] = {r.n_rho};
    StageScope st(p->timer, "radial_ifft", s);
    p->fft.exec(p->fft.get(1, nr1, r.lines()), lat, lat, CUFFT_INVERSE, s);
}

// lattice spectrum for resampling: fftn(pad(origin_avg(lattice))) into p->padded
// (src/shift/scale describe how to read the lattice value at rho index j)
void lattice_spectrum(P* p, const float2* src, int shift, float scale, cudaStream_t s) {
    const RadialTables& r = p->frad;
    const int dr = r.n_rho + 2 * p->fpad;
    const int64_t total = r.lines() * dr;
    p->padded.ensure((size_t)total);
    StageScope st(p->timer, "lattice_spectrum", s);
    p->red.ensure(2 * kRedBlocks + 64);
    double* mean = p->red.p + 2 * kRedBlocks;
    column_mean(src, r.lines(), r.n_rho, (r.n_rho / 2 + shift) % r.n_rho, scale, p->red.p, mean, s);
    k_pad_lattice<<<blocks_for(total, 256), 256, 0, s>>>(src, shift, scale, r.n_rho, p->fpad, dr,
                                                         total, mean, p->padded.p);
    CBN_LAUNCH_CHECK();
    if (p->c.method == 1) return;   // method B interpolates the padded lattice itself
    long long dims[3] = {r.n_phi, r.n_theta, dr};
    p->fft.exec(p->fft.get(3, dims, 1), p->padded.p, p->padded.p, CUFFT_FORWARD, s);
}

// method B (resampling.py:149-161): Re(periodic-sinc gather) at the umbrella
// targets of views [v0, v0 + nb) straight from the padded lattice
void gather_views_b(P* p, int v0, int nb, float* vals, cudaStream_t s, const float* tscale) {
    const RadialTables& r = p->frad;
    const int dr = r.n_rho + 2 * p->fpad;
    const int64_t per_view = (int64_t)p->fumb.n_mu * p->fumb.n_t;
    const int64_t m = per_view * nb;
    UmbrellaSrc src = cached_umbrella(p, p->fumb, r, p->fpad, v0, s);
    const DirGrid g{{dr, r.n_theta, r.n_phi}, {1, (int64_t)dr, (int64_t)r.n_theta * dr}};
    StageScope st(p->timer, "resample_gather", s);
    dispatch_taps(p->c.side_lobes + 1, [&](auto tc) {
        k_dir_gather<decltype(tc)::value><<<blocks_for(m, 256), 256, 0, s>>>(
            p->padded.p, g, src, m, nullptr, vals, tscale, p->fumb.n_t);
        return 0;
    });
    CBN_LAUNCH_CHECK();
}

// Fit the resample scalings of every view batch once (plan_resample's
// plan_nufft, resampling.py:102) and group batches with equal scalings.
void ensure_batch_plan(P* p, BatchPlan& bp, const UmbrellaTables& u, const RadialTables& r,
                       int pad, const AxisPlan* ax, cudaStream_t s) {
    if (bp.ready) return;
    StageScope st(p->timer, "batch_scalings", s);
    const int64_t per_view = (int64_t)u.n_mu * u.n_t;
    bp.batches = view_batches(p->g.n_views, per_view, target_batch(p));
    const int B = (int)bp.batches.size();
    bp.smax = smax_of(ax);
    const size_t per = 3 * (size_t)bp.smax;
    bp.s32.alloc(per * B);
    DevBuf<double> s64((size_t)per * B);
    CBN_CUDA(cudaMemsetAsync(s64.p, 0, sizeof(double) * per * B, s));
    for (int b = 0; b < B; ++b) {
        UmbrellaSrc src{umb_geom(p, u, r, pad), bp.batches[b].first};
        int nrows;
        const int64_t* rows =
            rows_for(p, per_view * (bp.batches[b].second - bp.batches[b].first), nrows);
        ls_fit<3>(src, rows, nrows, ax, p->ls, bp.s32.p + per * b, bp.smax, s);
        CBN_CUDA(cudaMemcpyAsync(s64.p + per * b, p->ls.s64.p, sizeof(double) * per,
                                 cudaMemcpyDeviceToDevice, s));
    }
    std::vector<double> h(per * B);
    CBN_CUDA(cudaMemcpyAsync(h.data(), s64.p, sizeof(double) * per * B, cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    bp.group.assign(B, -1);
    std::vector<int> reps;
    for (int b = 0; b < B; ++b) {
        for (int rep : reps) {
            double worst = 0.0;
            for (int d = 0; d < 3; ++d)
                for (int k = 0; k < ax[d].N; ++k) {
                    double x = h[per * b + (size_t)d * bp.smax + k];
                    double y = h[per * rep + (size_t)d * bp.smax + k];
                    worst = std::max(worst, std::fabs(x - y) / std::fabs(y));
                }
            if (worst <= 1e-9) {
                bp.group[b] = rep;
                break;
            }
        }
        if (bp.group[b] < 0) {
            bp.group[b] = b;
            reps.push_back(b);
        }
    }
    bp.ready = true;
}

// G = FFT_2x(pad(fftshift(F) / size * scaling)) for a batch's scalings
// (resample_apply + nufft_forward, resampling.py:146-147, nufft.py:226-231)
// phi_fast: grid stored [rho][theta][phi] for k_resample_views, else [phi][theta][rho]
bool views_in_lanes(const P* p);

// the resample grid is kept as Re(G) only (C2R) on the views-in-lanes J = 3 path
bool rho_lines_off() {   // CBN_RHO_LINES=0: the strided rho pass on the half spectrum (A/B)
    const char* e = std::getenv("CBN_RHO_LINES");
    return e && e[0] == '0';
}

bool real_grid(const P* p) {
    const char* off = std::getenv("CBN_COMPLEX_GRID");
    if (off && off[0] == '1') return false;
    return views_in_lanes(p) && res_j3(p->fres) && p->c.method == 0;
}

// the windowed view-chunk gather (k_resample_window) on the real grid; off
// with CBN_WINDOW_GATHER=0 (A/B against the 32-view k_resample_rows3)
bool window_gather(const P* p) {
    const char* e = std::getenv("CBN_WINDOW_GATHER");
    if (e && e[0] == '0') return false;
    return real_grid(p) && p->fres[0].K % 4 == 0;
}

void ensure_lane_taps(P* p, cudaStream_t s);

// Resample grid, rho lines first (phi-fast real grid): the padded, scaled
// lattice spectrum v on the (theta, phi) pad positions with their mirrors as
// contiguous rho lines [phi_i][theta_i][K_rho] (zero outside the rho pad) ...
__global__ void k_rho_lines_pad(const float2* __restrict__ src, RemapAxis ar, RemapAxis at,
                                RemapAxis ap, const int* __restrict__ lth,
                                const int* __restrict__ lph, int nth, float gain,
                                float2* __restrict__ lines) {
    const int kr = blockIdx.x * blockDim.x + threadIdx.x;
    if (kr >= ar.n) return;
    const int it = blockIdx.y, ip = blockIdx.z;
    const int kt = lth[it], kp = lph[ip];
    const int i0 = ar.idx[kr], i1 = at.idx[kt], i2 = ap.idx[kp];
    float2 v = make_float2(0.f, 0.f);
    if (i0 >= 0 && i1 >= 0 && i2 >= 0) {
        const float sc = gain * ar.scale[kr] * at.scale[kt] * ap.scale[kp];
        const float2 g = src[(int64_t)i0 * ar.sstride + (int64_t)i1 * at.sstride +
                             (int64_t)i2 * ap.sstride];
        v = make_float2(g.x * sc, g.y * sc);
    }
    lines[((size_t)ip * nth + it) * ar.n + kr] = v;
}

// ... forward FFT F along rho, then the half spectrum of the used rho planes x:
// H[x][kt][kp] = (conj F(x, kt, kp) + F(x, -kt, -kp)) / 2, kp <= K_phi / 2
// (= the inverse rho FFT of the Hermitian part), through 32 x 32 tiles per kt.
// Grid (ceil(H / 32), ceil(nx / 32), K_theta), block (32, 8).
__global__ void k_rho_lines_herm(const float2* __restrict__ F, const int* __restrict__ xs, int nx,
                                 const int* __restrict__ thmap, const int* __restrict__ phmap,
                                 int nth, int Kr, int Kt, int Kp, float2* __restrict__ dst) {
    __shared__ float2 tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int qx0 = blockIdx.y * 32, kp0 = blockIdx.x * 32, kt = blockIdx.z;
    const int hp = Kp / 2 + 1;
    const int ktm = kt ? Kt - kt : 0;
    const int ith = thmap[kt], ithm = thmap[ktm];
    const int qx = qx0 + tx;
    const int x = qx < nx ? xs[qx] : 0;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int kp = kp0 + r;
        if (qx >= nx || kp >= hp) continue;
        const int kpm = kp ? Kp - kp : 0;
        const int iph = phmap[kp], iphm = phmap[kpm];
        float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
        if (ith >= 0 && iph >= 0) a = F[((size_t)iph * nth + ith) * Kr + x];
        if (ithm >= 0 && iphm >= 0) b = F[((size_t)iphm * nth + ithm) * Kr + x];
        tile[r][tx] = make_float2(0.5f * (a.x + b.x), 0.5f * (b.y - a.y));
    }
    __syncthreads();
    const int kp = kp0 + tx;
    if (kp >= hp) return;
    for (int r = ty; r < 32; r += blockDim.y) {
        const int q = qx0 + r;
        if (q >= nx) break;
        dst[((size_t)xs[q] * Kt + kt) * hp + kp] = tile[tx][r];
    }
}

void build_resample_grid(P* p, const float* s32b, int smax, cudaStream_t s, bool phi_fast = false) {
    const RadialTables& r = p->frad;
    const AxisPlan* ax = p->fres;   // (phi, theta, rho)
    const int dr = r.n_rho + 2 * p->fpad;
    RemapAxis rax[3];
    const int64_t sstr[3] = {(int64_t)r.n_theta * dr, dr, 1};
    size_t need = (size_t)ax[0].K + ax[1].K + ax[2].K;
    p->tab_idx.ensure(need);
    p->tab_sc.ensure(need);
    size_t off = 0;
    for (int d = 0; d < 3; ++d) {
        build_table(kTabPadShift, ax[d].N, ax[d].K, s32b + (size_t)d * smax, p->tab_idx.p + off,
                    p->tab_sc.p + off, s);
        rax[d] = RemapAxis{p->tab_idx.p + off, p->tab_sc.p + off, ax[d].K, sstr[d]};
        off += ax[d].K;
    }
    if (phi_fast) std::swap(rax[0], rax[2]);
    const double size = (double)dr * r.n_theta * r.n_phi;
    if (real_grid(p)) {
        ensure_lane_taps(p, s);   // the rho planes the gather reads
        // only Re(G) is read (real weights, Re of the result): pad straight to
        // the conjugated Hermitian half spectrum and complex-to-real FFT it,
        // into a float grid behind the half spectrum in `big`
        const long long kd3[3] = {rax[0].n, rax[1].n, rax[2].n};
        const int64_t half = (int64_t)kd3[0] * kd3[1] * (kd3[2] / 2 + 1);
        p->big.ensure((size_t)half + (size_t)(kd3[0] * kd3[1] * kd3[2] + 1) / 2);
        if (!p->fres_list.p) {
            // per grid axis (after the phi-fast swap): the pad positions and their mirrors
            const AxisPlan* ga[3] = {&ax[0], &ax[1], &ax[2]};
            if (phi_fast) std::swap(ga[0], ga[2]);
            std::vector<int> all;
            for (int d = 0; d < 3; ++d) {
                const std::vector<int> l = pad_positions(ga[d]->N, ga[d]->K, true, d == 2);
                p->fres_nl[d] = (int)l.size();
                all.insert(all.end(), l.begin(), l.end());
            }
            p->fres_list.upload(all.data(), all.size(), s);
            CBN_CUDA(cudaStreamSynchronize(s));
        }
        if (rax[0].sstride == 1 && !rho_lines_off()) {
            // rho lines first: contiguous forward FFTs along rho on the (theta,
            // phi) pad positions, then the half spectrum of the used rho planes
            if (!p->fres_lth.p) {
                const std::vector<int> lth = pad_positions(ax[1].N, ax[1].K, true, false);
                const AxisPlan& aph = phi_fast ? ax[0] : ax[2];
                const std::vector<int> lph = pad_positions(aph.N, aph.K, true, false);
                std::vector<int> thmap((size_t)ax[1].K, -1), phmap((size_t)aph.K, -1), xs;
                for (size_t q = 0; q < lth.size(); ++q) thmap[(size_t)lth[q]] = (int)q;
                for (size_t q = 0; q < lph.size(); ++q) phmap[(size_t)lph[q]] = (int)q;
                for (const auto& rn : p->fres_rho_runs)
                    for (int x = rn.first; x < rn.second; ++x) xs.push_back(x);
                p->fres_nth = (int)lth.size();
                p->fres_nph = (int)lph.size();
                p->fres_nx = (int)xs.size();
                p->fres_lth.upload(lth.data(), lth.size(), s);
                p->fres_lph.upload(lph.data(), lph.size(), s);
                p->fres_thmap.upload(thmap.data(), thmap.size(), s);
                p->fres_phmap.upload(phmap.data(), phmap.size(), s);
                p->fres_xs.upload(xs.data(), std::max<size_t>(xs.size(), 1), s);
                CBN_CUDA(cudaStreamSynchronize(s));
            }
            const int Kr = (int)kd3[0], Kt = (int)kd3[1], Kp = (int)kd3[2];
            const int64_t nlines = (int64_t)p->fres_nth * p->fres_nph;
            p->rlines.ensure((size_t)nlines * Kr);
            {
                StageScope st(p->timer, "resample_pad", s);
                k_rho_lines_pad<<<dim3((unsigned)((Kr + 255) / 256), p->fres_nth, p->fres_nph), 256,
                                  0, s>>>(p->padded.p, rax[0], rax[1], rax[2], p->fres_lth.p,
                                          p->fres_lph.p, p->fres_nth, (float)(1.0 / size),
                                          p->rlines.p);
                CBN_LAUNCH_CHECK();
            }
            StageScope st(p->timer, "resample_fft", s);
            long long kr1[1] = {Kr};
            p->fft.exec(p->fft.get(1, kr1, nlines), p->rlines.p, p->rlines.p, CUFFT_FORWARD, s);
            const int hp = Kp / 2 + 1;
            if (p->fres_nx > 0) {
                k_rho_lines_herm<<<dim3((unsigned)((hp + 31) / 32),
                                        (unsigned)((p->fres_nx + 31) / 32), Kt),
                                   dim3(32, 8), 0, s>>>(p->rlines.p, p->fres_xs.p, p->fres_nx,
                                                        p->fres_thmap.p, p->fres_phmap.p,
                                                        p->fres_nth, Kr, Kt, Kp, p->big.p);
                CBN_LAUNCH_CHECK();
            }
            const long long k2[2] = {Kt, Kp};
            const long long plane = (long long)Kt * hp, rplane = (long long)Kt * Kp;
            float* re = reinterpret_cast<float*>(p->big.p + half);
            for (const auto& rn : p->fres_rho_runs)
                p->fft.exec_c2r(p->fft.get_c2r2(k2, rn.second - rn.first),
                                p->big.p + (size_t)rn.first * plane, re + rn.first * rplane, s);
            p->grid_re = re;
            return;
        }
        {
            // zero the half spectrum, then fill only the cells P or its mirror reaches
            StageScope st(p->timer, "resample_pad", s);
            CBN_CUDA(cudaMemsetAsync(p->big.p, 0, sizeof(float2) * half, s));
            const int* l = p->fres_list.p;
            if (rax[0].sstride == 1)   // phi-fast grid from the rho-fast padded lattice
                k_remap_herm3_tile<<<dim3((unsigned)((p->fres_nl[2] + 31) / 32),
                                          (unsigned)((p->fres_nl[0] + 31) / 32), p->fres_nl[1]),
                                     dim3(32, 8), 0, s>>>(
                    p->padded.p, p->big.p, rax[0], rax[1], rax[2], l, l + p->fres_nl[0],
                    l + p->fres_nl[0] + p->fres_nl[1], p->fres_nl[0], p->fres_nl[2],
                    (float)(1.0 / size));
            else
                k_remap_herm3_list<<<dim3((unsigned)((p->fres_nl[2] + 255) / 256), p->fres_nl[1],
                                      p->fres_nl[0]), 256, 0, s>>>(
                p->padded.p, p->big.p, rax[0], rax[1], rax[2], l, l + p->fres_nl[0],
                l + p->fres_nl[0] + p->fres_nl[1], p->fres_nl[2], (float)(1.0 / size));
            CBN_LAUNCH_CHECK();
        }
        StageScope st(p->timer, "resample_fft", s);
        // pruned 3D C2R: the pad fills only the theta planes in pad_positions
        // (and their mirrors), so the inverse C2C along rho (slowest axis,
        // strided columns) runs on those theta ranges only; then a batched 2D
        // C2R over the (theta, phi) planes
        {
            const long long hz = kd3[2] / 2 + 1, plane = kd3[1] * hz;
            for (const auto& rn : pad_runs(ax[1].N, ax[1].K, true)) {
                float2* at = p->big.p + (size_t)rn.first * hz;
                p->fft.exec(p->fft.get_strided(kd3[0], (long long)(rn.second - rn.first) * hz,
                                               plane, 1),
                            at, at, CUFFT_INVERSE, s);
            }
            // then the 2D C2R only on the rho planes the umbrella taps read
            const long long k2[2] = {kd3[1], kd3[2]};
            float* re = reinterpret_cast<float*>(p->big.p + half);
            const long long rplane = kd3[1] * kd3[2];
            for (const auto& rn : p->fres_rho_runs)
                p->fft.exec_c2r(p->fft.get_c2r2(k2, rn.second - rn.first),
                                p->big.p + (size_t)rn.first * plane, re + rn.first * rplane, s);
        }
        p->grid_re = reinterpret_cast<float*>(p->big.p + half);
        return;
    }
    p->big.ensure((size_t)ktot(ax));
    {
        StageScope st(p->timer, "resample_pad", s);
        launch_remap<float2, kStoreC>(3, p->padded.p, p->big.p, rax, (float)(1.0 / size), s);
        CBN_LAUNCH_CHECK();
    }
    long long kd[3] = {ax[0].K, ax[1].K, ax[2].K};
    if (phi_fast) std::swap(kd[0], kd[2]);
    // the zero padding leaves whole slowest-axis planes empty: skip their 2D FFTs
    const int slow = phi_fast ? 2 : 0;
    if (p->fres_planes.empty() || p->fres_planes_slow != slow) {
        size_t o = 0;
        for (int d = 0; d < slow; ++d) o += ax[d].K;
        p->fres_planes = index_runs(p->tab_idx.p + o, ax[slow].K, true, s);
        p->fres_planes_slow = slow;
    }
    StageScope st(p->timer, "resample_fft", s);
    fft3_pruned(p->fft, p->big.p, kd, 1, p->fres_planes, CUFFT_FORWARD, s);
}

// views-in-lanes path applies when every view's targets are view 0's shifted by
// a whole number of oversampled phi cells: 2 n_phi k / V integer for all k
bool views_in_lanes(const P* p) {
    const char* off = std::getenv("CBN_NO_VIEW_LANES");
    if (off && off[0] == '1') return false;
    const int V = p->g.n_views;
    return (2LL * p->frad.n_phi) % V == 0 && p->fres[0].K == 2 * p->frad.n_phi;
}

// per-target resample taps of the views-in-lanes gather (built once)
void ensure_lane_taps(P* p, cudaStream_t s) {
    UmbrellaTables& u = p->fumb;
    if (u.taps_ready) return;
    const AxisPlan* ax = p->fres;
    const int64_t per_view = (int64_t)u.n_mu * u.n_t;
    dispatch_j(res_jmax(ax), [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        UmbrellaSrc src = cached_umbrella(p, u, p->frad, p->fpad, 0, s);
        KBSet kb;
        kb.ax[0] = ax[2].kb;
        kb.ax[1] = ax[1].kb;
        kb.ax[2] = ax[0].kb;
        u.taps.alloc((size_t)per_view * sizeof(RsTap<J>));
        k_rs_taps<J><<<blocks_for(per_view, 256), 256, 0, s>>>(
            src, kb, per_view, reinterpret_cast<RsTap<J>*>(u.taps.p));
        CBN_LAUNCH_CHECK();
        {
            // rho planes the taps read: the grid's other planes are never
            // inverse-transformed (build_resample_grid)
            const int K0 = ax[2].K;
            DevBuf<int> used((size_t)K0);
            CBN_CUDA(cudaMemsetAsync(used.p, 0, sizeof(int) * K0, s));
            k_rs_rho_used<J><<<blocks_for(per_view, 256), 256, 0, s>>>(
                reinterpret_cast<const RsTap<J>*>(u.taps.p), per_view, K0, used.p);
            CBN_LAUNCH_CHECK();
            std::vector<int> h((size_t)K0);
            CBN_CUDA(cudaMemcpyAsync(h.data(), used.p, sizeof(int) * K0, cudaMemcpyDeviceToHost, s));
            CBN_CUDA(cudaStreamSynchronize(s));
            p->fres_rho_runs.clear();
            for (int k = 0; k < K0; ++k) {
                if (!h[(size_t)k]) continue;
                if (!p->fres_rho_runs.empty() && p->fres_rho_runs.back().second == k)
                    p->fres_rho_runs.back().second = k + 1;
                else
                    p->fres_rho_runs.emplace_back(k, k + 1);
            }
        }
        // pole targets leave the view-0 records (their planes are already counted)
        build_poles<J>(u, src, per_view, reinterpret_cast<RsTap<J>*>(u.taps.p), s);
        if constexpr (J == 3) {
            CBN_REQUIRE((int64_t)ax[2].K * ax[1].K * ax[0].K < (1LL << 32),
                        "resample grid above 2^32 cells");
            u.rows.alloc((size_t)per_view * sizeof(RsRow3));
            k_rs_rows3<<<blocks_for(per_view, 256), 256, 0, s>>>(
                reinterpret_cast<const RsTap<3>*>(u.taps.p), per_view, ax[2].K, ax[1].K,
                ax[0].K, reinterpret_cast<RsRow3*>(u.rows.p));
            CBN_LAUNCH_CHECK();
            if (u.n_poles) {
                // pole records (valid = 2) and their per-view phi taps
                k_pole_rows<<<blocks_for(u.n_poles, 128), 128, 0, s>>>(
                    u.poles.p, u.n_poles, reinterpret_cast<RsRow3*>(u.rows.p));
                CBN_LAUNCH_CHECK();
                const int V = p->g.n_views;
                u.pole_f2.alloc((size_t)u.n_poles * V);
                DevBuf<int> bad(1);
                CBN_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
                KBSet kbg;   // grid order (rho, theta, phi)
                kbg.ax[0] = ax[2].kb;
                kbg.ax[1] = ax[1].kb;
                kbg.ax[2] = ax[0].kb;
                k_pole_table<<<blocks_for((int64_t)u.n_poles * V, 128), 128, 0, s>>>(
                    src, kbg, u.poles.p, u.n_poles, V, 1, u.pole_f2.p, bad.p);
                CBN_LAUNCH_CHECK();
                int h_bad = 0;
                CBN_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
                CBN_CUDA(cudaStreamSynchronize(s));
                CBN_REQUIRE(h_bad == 0, "pole target with view-dependent rho/theta taps");
            }
        }
        return 0;
    });
    u.taps_ready = true;
}

// Re(resample_apply) for consecutive views [v0, v0 + nb) from a phi-fast grid:
// up to kWinChunk views per launch with the window gather, else 32 per launch
void gather_views_lanes(P* p, int v0, int nb, float* vals, cudaStream_t s,
                        const float* tscale = nullptr) {
    const AxisPlan* ax = p->fres;
    const int64_t per_view = (int64_t)p->fumb.n_mu * p->fumb.n_t;
    const int per_launch = res_j3(ax) && window_gather(p) ? kWinChunk : 32;
    if (nb > per_launch) {
        for (int k = 0; k < nb; k += per_launch)
            gather_views_lanes(p, v0 + k, std::min(per_launch, nb - k), vals + (size_t)k * per_view,
                               s, tscale);
        return;
    }
    const int shift = (int)(2LL * p->frad.n_phi / p->g.n_views);
    ensure_lane_taps(p, s);
    dispatch_j(res_jmax(ax), [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        UmbrellaTables& u = p->fumb;
        StageScope st(p->timer, "resample_gather", s);
        const bool re = J == 3 && real_grid(p);
        if (J == 3 && re && window_gather(p)) {
            // chunk of up to kWinChunk views: one window sum per target
            const RsRow3* rows = reinterpret_cast<const RsRow3*>(u.rows.p);
            const int K2 = ax[0].K;
            const size_t smem = win_smem_bytes(K2, nb);
            CBN_CUDA(cudaFuncSetAttribute(k_resample_window,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const unsigned nblk = (unsigned)((per_view + kWinWarps * kWinTargets - 1) /
                                             (kWinWarps * kWinTargets));
            k_resample_window<<<nblk, kWinWarps * 32, smem, s>>>(
                p->grid_re, K2, rows, per_view, v0, nb, shift, u.pole_f2.p, p->g.n_views, vals,
                tscale, u.n_t);
            CBN_LAUNCH_CHECK();
            // outputs + records once; on chip: 9 rows x the window's float4
            // slots per target, 3 reads per view
            const double win = std::min<double>(shift * (nb - 1) + 3 + 3, ax[0].K);
            p->timer.add_bytes("resample_gather", 4.0 * nb * per_view + 96.0 * per_view,
                               (double)per_view * (9.0 * 4.0 * win + 12.0 * nb));
            return 0;
        }
        if constexpr (J == 3) {
            const unsigned nblk = (unsigned)((per_view + 31) / 32);
            const RsRow3* rows = reinterpret_cast<const RsRow3*>(u.rows.p);
            if (re)
                k_resample_rows3<1><<<nblk, 256, 0, s>>>(p->grid_re, ax[0].K, rows, per_view, v0,
                                                         nb, shift, vals, tscale, p->fumb.n_t);
            else
                k_resample_rows3<2><<<nblk, 256, 0, s>>>(reinterpret_cast<const float*>(p->big.p),
                                                         ax[0].K, rows, per_view, v0, nb, shift,
                                                         vals, tscale, p->fumb.n_t);
        } else {
            k_resample_views<J><<<(unsigned)((per_view + 31) / 32), 256, 0, s>>>(
                p->big.p, ax[2].K, ax[1].K, ax[0].K, reinterpret_cast<const RsTap<J>*>(u.taps.p),
                per_view, v0, nb, shift, vals, tscale, p->fumb.n_t);
        }
        CBN_LAUNCH_CHECK();
        // outputs + one read of the tap records per launch; on chip: J^2 rows
        // per target and view (rows3: two 8-byte cell pairs per row)
        p->timer.add_bytes("resample_gather",
                           4.0 * nb * per_view + (J == 3 ? 96.0 : (double)sizeof(RsTap<J>)) * per_view,
                           (double)nb * per_view * (J == 3 ? 9.0 * 16.0 : 4.0 * (re ? 1 : 2) * J * J * J));
        if (u.n_poles) {
            // pole targets per view (their records are not in the view-0 taps)
            UmbrellaSrc src = cached_umbrella(p, u, p->frad, p->fpad, v0, s);
            KBSet kb;   // grid order (rho, theta, phi)
            kb.ax[0] = ax[2].kb;
            kb.ax[1] = ax[1].kb;
            kb.ax[2] = ax[0].kb;
            const int nq = u.n_poles * nb;
            if (re)
                k_rs_pole_gather<J, 1><<<blocks_for(nq, 128), 128, 0, s>>>(
                    p->grid_re, kb, src, u.poles.p, u.n_poles, per_view, nb, vals, tscale, u.n_t);
            else
                k_rs_pole_gather<J, 2><<<blocks_for(nq, 128), 128, 0, s>>>(
                    reinterpret_cast<const float*>(p->big.p), kb, src, u.poles.p, u.n_poles,
                    per_view, nb, vals, tscale, u.n_t);
            CBN_LAUNCH_CHECK();
        }
        return 0;
    });
}

// Re(resample_apply) at the umbrella targets of views [lo, hi) from the current grid
void gather_views(P* p, int lo, int hi, float* vals, cudaStream_t s,
                  const float* tscale = nullptr) {
    const RadialTables& r = p->frad;
    const AxisPlan* ax = p->fres;
    const int64_t per_view = (int64_t)p->fumb.n_mu * p->fumb.n_t;
    UmbrellaSrc src = cached_umbrella(p, p->fumb, r, p->fpad, lo, s);
    const int64_t m = per_view * (hi - lo);
    KBSet kb;
    for (int d = 0; d < 3; ++d) kb.ax[d] = ax[d].kb;
    StageScope st(p->timer, "resample_gather", s);
    p->timer.add_bytes("resample_gather", 4.0 * m,
                       8.0 * m * ax[0].J * ax[1].J * ax[2].J);
    dispatch_j(res_jmax(ax), [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        k_gather<3, J><<<blocks_for(m, 256), 256, 0, s>>>(p->big.p, kb, src,
                                                         UmbOut{vals, tscale, p->fumb.n_t}, m);
        return 0;
    });
    CBN_LAUNCH_CHECK();
}

// sorted polar nodes with their precomputed taps and factors (plan data)
void prepare_gr_points(P* p, GrangeatPlan& gp, const UmbrellaTables& u, bool reverse,
                       cudaStream_t s) {
    if (gp.pts_ready) return;
    PolarSrc src{u.omega_t.p, u.cos_mu.p, u.sin_mu.p, gp.pu, gp.pv, u.n_t};
    const int edge = reverse ? kGrTileRev : kGrTile;
    const int tile[2] = {edge, edge};
    build_bins<2, kGrJ>(gp.bins, src, gp.kb, gp.m, tile, kMaxSub, s);
    gp.pts.alloc((size_t)gp.m * sizeof(GrPoint<kGrJ>));
    GrFactor f;
    f.n_t = u.n_t;
    f.reverse = reverse ? 1 : 0;
    f.N[0] = p->g.nu;
    f.N[1] = p->g.nv;
    f.q = gp.fac_im.p;
    f.omega = u.omega_t.p;
    f.pupv = (float)(gp.pu * gp.pv);
    k_gr_points<kGrJ><<<gp.bins.nsubs, 256, 0, s>>>(gp.kb, gp.bins.geom<2>(), src, f,
                                                    gp.bins.perm.p, gp.bins.subs.p,
                                                    reinterpret_cast<GrPoint<kGrJ>*>(gp.pts.p));
    CBN_LAUNCH_CHECK();
    gp.pts_ready = true;
}

GrPost gr_post(const P* p, const GrangeatPlan& gp) {
    GrPost q;
    q.nu = p->g.nu;
    q.nv = p->g.nv;
    q.Ku = gp.ax[0].K;
    q.Kv = gp.ax[1].K;
    q.pix = gp.pix.p;
    return q;
}

// Work items of k_gr_gather_cells from the host copy of the cell CSR offsets
// h (full plane, Ku*Kv + 1): half-plane cells whose two entry lists exceed
// kGrHeavy entries get a CTA of their own (8 warps split the lists); the rest
// go in blocks of 32 cells.  Items are ordered by descending cost so the
// dense cells near the origin (polar nodes crowd there) start first instead
// of forming the tail.
constexpr int64_t kGrHeavy = 1024;

void gr_cell_schedule(GrangeatPlan& gp, const std::vector<int>& h, int Ku, int Kv,
                      cudaStream_t s) {
    const int hv = Kv / 2 + 1;
    const int64_t nhalf = (int64_t)Ku * hv;
    std::vector<unsigned char> heavy((size_t)nhalf, 0);
    std::vector<std::pair<int64_t, int>> items;   // (cost, item)
    const int64_t nblk = (nhalf + 31) / 32;
    std::vector<int64_t> bcost((size_t)nblk, 0);
    for (int64_t c = 0; c < nhalf; ++c) {
        const int u = (int)(c / hv), v = (int)(c % hv);
        const int64_t k = (int64_t)u * Kv + v;
        const int64_t km = (int64_t)(u ? Ku - u : 0) * Kv + (v ? Kv - v : 0);
        const int64_t cost = (int64_t)(h[k + 1] - h[k]) + (h[km + 1] - h[km]);
        if (cost > kGrHeavy) {
            heavy[(size_t)c] = 1;
            items.emplace_back((cost + 7) / 8, (int)(-c - 1));
        } else {
            bcost[(size_t)(c / 32)] += cost;
        }
    }
    // a block's 8 warps take 4 cells each: its time is about cost / 8
    for (int64_t b = 0; b < nblk; ++b) items.emplace_back((bcost[(size_t)b] + 7) / 8, (int)b);
    std::stable_sort(items.begin(), items.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<int> order(items.size());
    for (size_t i = 0; i < items.size(); ++i) order[i] = items[i].second;
    gp.n_items = (int)order.size();
    gp.cell_order.upload(order.data(), order.size(), s);
    gp.cell_heavy.upload(heavy.data(), heavy.size(), s);
    CBN_CUDA(cudaStreamSynchronize(s));
}

// Strip form of the cell CSR (k_gr_gather_strips), built once per plan on the
// host from the device cell CSR: per half-plane strip the entries of its
// kGrStrip direct cells and of their mirrors, merged by node row (sorted, so
// the strip sums are deterministic), and the work schedule.
static int64_t gr_heavy_strip() {   // strips above this many entries get a CTA of their own
    const char* e = std::getenv("CBN_GR_HEAVY_STRIP");
    return e ? std::atoll(e) : 640;
}

void gr_build_strips(GrangeatPlan& gp, int Ku, int Kv, cudaStream_t s) {
    const int hv = Kv / 2 + 1;
    const int nsx = (hv + kGrStrip - 1) / kGrStrip;
    const int ngrp = (nsx + 7) / 8;
    const int64_t ncell = (int64_t)Ku * Kv, nstrips = (int64_t)Ku * nsx;
    std::vector<int> ptr((size_t)ncell + 1);
    std::vector<GrEntry> ent((size_t)gp.n_entries);
    CBN_CUDA(cudaMemcpyAsync(ptr.data(), gp.cell_ptr.p, sizeof(int) * ptr.size(),
                             cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaMemcpyAsync(ent.data(), gp.cell_ent.p, sizeof(GrEntry) * ent.size(),
                             cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    struct Rec {
        int id;
        float p[kGrStrip], q[kGrStrip];
    };
    std::vector<std::vector<Rec>> rows((size_t)Ku);
#pragma omp parallel for schedule(dynamic, 4)
    for (int u = 0; u < Ku; ++u) {
        std::vector<std::pair<int, int>> items;   // (node, slot: cell i, mirror flag)
        std::vector<float> wts;
        std::vector<Rec>& out = rows[(size_t)u];
        for (int sx = 0; sx < nsx; ++sx) {
            items.clear();
            wts.clear();
            for (int i = 0; i < kGrStrip; ++i) {
                const int v = sx * kGrStrip + i;
                if (v >= hv) break;
                const int64_t k = (int64_t)u * Kv + v;
                const int64_t km = (int64_t)(u ? Ku - u : 0) * Kv + (v ? Kv - v : 0);
                for (int e = ptr[(size_t)k]; e < ptr[(size_t)k + 1]; ++e) {
                    items.emplace_back(ent[(size_t)e].id, 2 * i);
                    wts.push_back(ent[(size_t)e].w);
                }
                for (int e = ptr[(size_t)km]; e < ptr[(size_t)km + 1]; ++e) {
                    items.emplace_back(ent[(size_t)e].id, 2 * i + 1);
                    wts.push_back(ent[(size_t)e].w);
                }
            }
            std::vector<int> ord(items.size());
            for (size_t q = 0; q < ord.size(); ++q) ord[q] = (int)q;
            std::sort(ord.begin(), ord.end(), [&](int a, int b) {
                return items[(size_t)a] < items[(size_t)b];
            });
            // a strip record per node; double sums over the node's taps
            size_t q = 0;
            const size_t start = out.size();
            while (q < ord.size()) {
                const int id = items[(size_t)ord[q]].first;
                double w[kGrStrip] = {0}, m[kGrStrip] = {0};
                for (; q < ord.size() && items[(size_t)ord[q]].first == id; ++q) {
                    const int slot = items[(size_t)ord[q]].second;
                    (slot & 1 ? m : w)[slot >> 1] += wts[(size_t)ord[q]];
                }
                Rec r;
                r.id = id;
                for (int i = 0; i < kGrStrip; ++i) {
                    r.p[i] = (float)(0.5 * (w[i] + m[i]));
                    r.q[i] = (float)(0.5 * (w[i] - m[i]));
                }
                out.push_back(r);
            }
            // strip boundary marker: the count goes into a separate pass below
            out.push_back(Rec{-1 - (int)(out.size() - start), {0}, {0}});
        }
    }
    // flatten: strip_ptr, ids, p, q (the markers hold each strip's count)
    std::vector<int> sptr((size_t)nstrips + 1, 0), sid;
    std::vector<float4> sp, sq;
    std::vector<unsigned char> heavy((size_t)nstrips, 0);
    std::vector<std::pair<int64_t, int>> work;
    const int64_t heavy_at = gr_heavy_strip();
    int64_t st = 0;
    for (int u = 0; u < Ku; ++u) {
        const auto& out = rows[(size_t)u];
        size_t q = 0;
        std::vector<int64_t> gcost((size_t)ngrp, 0);
        for (int sx = 0; sx < nsx; ++sx, ++st) {
            for (; out[q].id >= 0; ++q) {
                sid.push_back(out[q].id);
                sp.push_back(make_float4(out[q].p[0], out[q].p[1], out[q].p[2], out[q].p[3]));
                sq.push_back(make_float4(out[q].q[0], out[q].q[1], out[q].q[2], out[q].q[3]));
            }
            const int cnt = -1 - out[q].id;
            ++q;
            sptr[(size_t)st + 1] = sptr[(size_t)st] + cnt;
            if (cnt > heavy_at) {
                heavy[(size_t)st] = 1;
                work.emplace_back((cnt + 7) / 8, (int)(-st - 1));
            } else {
                gcost[(size_t)(sx / 8)] += cnt;
            }
        }
        for (int g = 0; g < ngrp; ++g) work.emplace_back((gcost[(size_t)g] + 7) / 8, u * ngrp + g);
    }
    std::stable_sort(work.begin(), work.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<int> order(work.size());
    for (size_t i = 0; i < work.size(); ++i) order[i] = work[i].second;
    gp.n_strip_entries = (int64_t)sid.size();
    if (sid.empty()) {
        sid.push_back(0);
        sp.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
        sq.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
    }
    gp.n_strip_items = (int)order.size();
    gp.strip_ptr.upload(sptr.data(), sptr.size(), s);
    gp.strip_id.upload(sid.data(), sid.size(), s);
    gp.strip_p.upload(sp.data(), sp.size(), s);
    gp.strip_q.upload(sq.data(), sq.size(), s);
    gp.strip_order.upload(order.data(), order.size(), s);
    gp.strip_heavy.upload(heavy.data(), heavy.size(), s);
    CBN_CUDA(cudaStreamSynchronize(s));
}

bool gr_strips_on() {   // CBN_GR_STRIPS=0: the per-cell gather (A/B)
    const char* e = std::getenv("CBN_GR_STRIPS");
    return !(e && e[0] == '0');
}

bool cell_gather_on() {
    const char* spread_env = std::getenv("CBN_GR_SPREAD");
    return !(spread_env && spread_env[0] == '1');
}

// reverse_grangeat_view for nb views: vals (nb x n_mu x n_t) -> frames (nb x nu x nv)
void grangeat_reverse(P* p, const float* vals, float* frames, int nb, cudaStream_t s,
                      GrBufs B) {
    GrangeatPlan& gp = p->fgr;
    if (!gp.built) fit_grangeat(p, gp, p->fumb, s);
    const UmbrellaTables& u = p->fumb;
    const int Ku = gp.ax[0].K, Kv = gp.ax[1].K;
    const int64_t tl = (int64_t)nb * u.n_mu * u.n_t;
    const int nh = u.n_t / 2 + 1;
    B.t.ensure((size_t)nb * u.n_mu * nh);
    B.grid.ensure((size_t)nb * Ku * Kv);
    prepare_gr_points(p, gp, u, true, s);
    if (p->timer.on) p->timer.begin("grangeat_tfft", s);
    (void)tl;
    // vals arrive already divided by w2 (folded into the resample store), so
    // the t lines go straight through a real-to-complex FFT
    // even n_t: complex FFTs of half length on the lines read as complex pairs;
    // the real-to-complex split is fused into the node-row transpose below
    const bool zsplit = u.n_t % 2 == 0 && cell_gather_on();
    if (zsplit) {
        long long m1[1] = {u.n_t / 2};
        B.fft.exec(B.fft.get(1, m1, (long long)nb * u.n_mu), const_cast<float*>(vals), B.t.p,
                   CUFFT_FORWARD, s);
    } else {
        B.fft.exec_r2c(B.fft.get_r2c(u.n_t, (long long)nb * u.n_mu), vals, B.t.p, s);
    }
    const bool cell_gather = cell_gather_on();
    if (!cell_gather) CBN_CUDA(cudaMemsetAsync(B.grid.p, 0, sizeof(float2) * nb * Ku * Kv, s));
    if (p->timer.on) p->timer.end(s);
    if (cell_gather) {
        const int64_t ncell = (int64_t)Ku * Kv;
        if (!gp.cell_ptr.p) {
            // plan step: node rows (GrNode), then the per-cell CSR of (row, weight) entries
            const BinPlan& bb = gp.bins;
            const int64_t nspec = (int64_t)u.n_mu * nh;
            const GrPoint<kGrJ>* pts = reinterpret_cast<const GrPoint<kGrJ>*>(gp.pts.p);
            const PolarSrc psrc{u.omega_t.p, u.cos_mu.p, u.sin_mu.p, gp.pu, gp.pv, u.n_t};
            const int64_t m = gp.m;
            DevBuf<int> node_id((size_t)m), mult((size_t)m), nextra(1);
            DevBuf<GrNode> tab((size_t)(nspec + m));
            CBN_CUDA(cudaMemsetAsync(tab.p, 0, sizeof(GrNode) * (nspec + m), s));
            CBN_CUDA(cudaMemsetAsync(nextra.p, 0, sizeof(int), s));
            k_gr_node_ids<kGrJ><<<blocks_for(m, 256), 256, 0, s>>>(
                pts, bb.perm.p, m, psrc, gp.kb, (int)nspec, node_id.p, mult.p, tab.p, nextra.p);
            CBN_LAUNCH_CHECK();
            int h_extra = 0;
            CBN_CUDA(cudaMemcpyAsync(&h_extra, nextra.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            DevBuf<int> counts((size_t)ncell);
            CBN_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int) * ncell, s));
            k_gr_csr_count<kGrJ><<<bb.nsubs, 256, 0, s>>>(bb.geom<2>(), pts, bb.subs.p, node_id.p,
                                                         counts.p);
            CBN_LAUNCH_CHECK();
            std::vector<int> h((size_t)ncell + 1, 0);
            CBN_CUDA(cudaMemcpyAsync(h.data() + 1, counts.p, sizeof(int) * ncell,
                                     cudaMemcpyDeviceToHost, s));
            CBN_CUDA(cudaStreamSynchronize(s));
            gp.n_rows = nspec + h_extra;
            gp.node_tab.alloc((size_t)gp.n_rows);
            CBN_CUDA(cudaMemcpyAsync(gp.node_tab.p, tab.p, sizeof(GrNode) * gp.n_rows,
                                     cudaMemcpyDeviceToDevice, s));
            for (size_t q = 1; q < h.size(); ++q) h[q] += h[q - 1];
            gp.cell_ptr.upload(h.data(), h.size(), s);
            gp.cell_ent.alloc(sizeof(GrEntry) * (size_t)std::max(h.back(), 1));
            gp.n_entries = h.back();
            CBN_CUDA(cudaMemcpyAsync(counts.p, h.data(), sizeof(int) * ncell, cudaMemcpyHostToDevice,
                                     s));
            k_gr_csr_fill<kGrJ><<<bb.nsubs, 256, 0, s>>>(bb.geom<2>(), pts, bb.subs.p, node_id.p,
                                                         mult.p, counts.p,
                                                         reinterpret_cast<GrEntry*>(gp.cell_ent.p));
            CBN_LAUNCH_CHECK();
            gr_cell_schedule(gp, h, Ku, Kv, s);
            CBN_CUDA(cudaStreamSynchronize(s));
            if (gr_strips_on()) gr_build_strips(gp, Ku, Kv, s);
        }
        const int64_t nspec = (int64_t)u.n_mu * nh;
        B.tv.ensure(std::max((size_t)gp.n_rows * 32, ((size_t)nb * Ku * Kv + 1) / 2));
        {
            // t-spectra of the block read once, view-fastest node rows written once
            StageScope st(p->timer, "grangeat_rows", s);
            p->timer.add_bytes("grangeat_rows",
                               8.0 * nb * (double)u.n_mu * (zsplit ? u.n_t / 2 : nh) +
                                   8.0 * nb * gp.n_rows,
                               0.0);
            if (zsplit)
                k_views_nodes_z<<<(unsigned)((gp.n_rows + 31) / 32), 256, 0, s>>>(
                    B.t.p, nb, u.n_mu, u.n_t / 2, gp.node_tab.p, gp.n_rows, B.tv.p);
            else
                k_views_nodes<<<(unsigned)((gp.n_rows + 31) / 32), 256, 0, s>>>(
                    B.t.p, nb, nspec, gp.node_tab.p, gp.n_rows, B.tv.p);
            CBN_LAUNCH_CHECK();
        }
        StageScope st(p->timer, "grangeat_spread", s);
        // Hermitian half plane [Ku][Kv/2+1] of the grid (only Re of its
        // inverse FFT is used), then a complex-to-real 2D FFT into tv
        const int64_t nhalf = (int64_t)Ku * (Kv / 2 + 1);
        // node rows of the block once, CSR entries once, the half-plane grids
        // written once; on chip: one row value per entry and view
        if (gr_strips_on() && gp.strip_ptr.p) {
            // node rows once, strip records (4 + 32 B) once, the half planes
            // written once; on chip: one row value per strip entry and view
            const int hv = Kv / 2 + 1;
            const int nsx = (hv + kGrStrip - 1) / kGrStrip;
            p->timer.add_bytes("grangeat_spread",
                               8.0 * nb * gp.n_rows + 36.0 * gp.n_strip_entries +
                                   8.0 * nb * nhalf,
                               8.0 * nb * (double)gp.n_strip_entries);
            k_gr_gather_strips<<<(unsigned)gp.n_strip_items, 256, 0, s>>>(
                B.grid.p, (size_t)nhalf, hv, nsx, (nsx + 7) / 8, gp.strip_ptr.p, gp.strip_id.p,
                gp.strip_p.p, gp.strip_q.p, B.tv.p, nb, gp.strip_order.p, gp.strip_heavy.p);
        } else {
            p->timer.add_bytes("grangeat_spread",
                               8.0 * nb * gp.n_rows + (double)sizeof(GrEntry) * gp.n_entries +
                                   8.0 * nb * nhalf,
                               8.0 * nb * (double)gp.n_entries);
            k_gr_gather_cells<<<(unsigned)gp.n_items, 256, 0, s>>>(
                B.grid.p, (size_t)nhalf, nhalf, gp.cell_ptr.p,
                reinterpret_cast<const GrEntry*>(gp.cell_ent.p), B.tv.p, nb, Ku, Kv,
                gp.cell_order.p, gp.cell_heavy.p);
        }
        CBN_LAUNCH_CHECK();
    } else {
        StageScope st(p->timer, "grangeat_spread", s);
        const BinPlan& bb = gp.bins;
        constexpr size_t smem = gr_spread_owned_smem<kGrJ, kGrTileRev>();
        CBN_CUDA(cudaFuncSetAttribute(k_gr_spread_owned<kGrJ, kGrTileRev>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_gr_spread_owned<kGrJ, kGrTileRev><<<bb.nsubs, kGrJ * 32, smem, s>>>(
            B.grid.p, (size_t)Ku * Kv, bb.geom<2>(),
            reinterpret_cast<const GrPoint<kGrJ>*>(gp.pts.p), bb.subs.p, B.t.p,
            (size_t)u.n_mu * nh, nb);
        CBN_LAUNCH_CHECK();
    }
    long long kd[2] = {Ku, Kv};
    StageScope st(p->timer, "grangeat_ifft_post", s);
    ensure_gr_pix(p, gp, true, s);
    GrPost q = gr_post(p, gp);
    B.red.ensure(2 * kRedBlocks + 64 + (size_t)nb);
    double* mean = B.red.p + 2 * kRedBlocks + 64;
    auto post = [&](const auto* g) {
        k_gr_ring<<<nb, 256, 0, s>>>(g, q, mean);
        CBN_LAUNCH_CHECK();
        k_gr_frame<<<dim3((unsigned)((p->g.nv + 255) / 256), p->g.nu, nb), 256, 0, s>>>(
            g, q, mean, (float)p->c.normalization, frames, p->flag.p);
        CBN_LAUNCH_CHECK();
    };
    if (cell_gather) {
        float* re = reinterpret_cast<float*>(B.tv.p);
        B.fft.exec_c2r(B.fft.get_c2r2(kd, nb), B.grid.p, re, s);
        post(static_cast<const float*>(re));
    } else {
        B.fft.exec(B.fft.get(2, kd, nb), B.grid.p, B.grid.p, CUFFT_INVERSE, s);
        post(static_cast<const float2*>(B.grid.p));
    }
}

void grangeat_reverse(P* p, const float* vals, float* frames, int nb, cudaStream_t s) {
    grangeat_reverse(p, vals, frames, nb, s, main_bufs(p));
}

constexpr int kViewBlock = 32;   // views per reverse-Grangeat block

// views per resample-gather chunk of the forward view loop
int gather_chunk(const P* p) {
    return views_in_lanes(p) && res_j3(p->fres) && window_gather(p) ? kWinChunk : kViewBlock;
}

// Views [lo, hi): one resample grid per run of batches with equal scalings,
// gather at the umbrella targets, then reverse Grangeat in blocks of up to
// kViewBlock consecutive views.  With `values_out` only the umbrella values
// are produced (stage API).
void resample_and_reverse(P* p, int lo, int hi, float* frames, cudaStream_t s,
                          float* values_out = nullptr) {
    if (p->c.method == 1) {
        const int64_t pv = (int64_t)p->fumb.n_mu * p->fumb.n_t;
        if (!values_out) p->values.ensure((size_t)pv * kViewBlock);
        for (int v = lo; v < hi; v += kViewBlock) {
            const int nb = std::min(kViewBlock, hi - v);
            if (values_out) {
                gather_views_b(p, v, nb, values_out + (size_t)(v - lo) * pv, s, nullptr);
                continue;
            }
            gather_views_b(p, v, nb, p->values.p, s, p->fgr.w2inv.p);
            grangeat_reverse(p, p->values.p, frames + (size_t)(v - lo) * p->g.nu * p->g.nv, nb, s);
            p->block_done(v - lo, v - lo + nb, s);
        }
        return;
    }
    BatchPlan& bp = p->fbatch;
    ensure_batch_plan(p, bp, p->fumb, p->frad, p->fpad, p->fres, s);
    const int64_t per_view = (int64_t)p->fumb.n_mu * p->fumb.n_t;
    const size_t frame_sz = (size_t)p->g.nu * p->g.nv;
    const bool lanes = views_in_lanes(p);
    // views per gather chunk (the window gather takes up to kWinChunk at once);
    // the reverse Grangeat runs on 32-view blocks of each chunk
    const int chunk = lanes ? gather_chunk(p) : kViewBlock;
    if (!values_out) p->values.ensure((size_t)per_view * chunk);
    // two lanes (the caller's stream and s1) alternate over view blocks so one
    // block's Grangeat FFTs overlap the next block's resample gather
    const bool dual = lanes && !values_out && lanes_allowed() && !p->timer.on;
    if (dual) ensure_lane1(p);
    if (dual) {
        p->lane1.values.ensure((size_t)per_view * chunk);
        // everything s1 reads besides the grid exists before the first grid event
        ensure_lane_taps(p, s);
        if (!p->fgr.built) fit_grangeat(p, p->fgr, p->fumb, s);
        prepare_gr_points(p, p->fgr, p->fumb, true, s);
        // the per-pixel factors lane 1's k_gr_frame reads (built lazily on
        // first use): build them on s, before the first ev_s0 the lane waits on
        ensure_gr_pix(p, p->fgr, true, s);
    }
    int lane = 0;
    bool s1_used = false, s1_stale = true;   // s1 has not yet waited for the current grid
    auto lane_stream = [&]() -> cudaStream_t {
        if (!lane) return s;
        if (s1_stale) {
            CBN_CUDA(cudaStreamWaitEvent(p->s1, p->ev_s0, 0));
            s1_stale = false;
        }
        s1_used = true;
        return p->s1;
    };
    auto lane_done = [&]() {
        if (lane) CBN_CUDA(cudaEventRecord(p->ev_s1, p->s1));
    };
    int cur = -1, blk_lo = lo, blk_n = 0;
    auto flush = [&]() {
        if (!blk_n) return;
        const cudaStream_t ls = lane_stream();
        const float* vb = lane ? p->lane1.values.p : p->values.p;
        for (int k = 0; k < blk_n; k += kViewBlock) {
            const int nk = std::min(kViewBlock, blk_n - k);
            grangeat_reverse(p, vb + (size_t)k * per_view,
                             frames + (size_t)(blk_lo + k - lo) * frame_sz, nk, ls,
                             lane ? lane_bufs(p) : main_bufs(p));
            p->block_done(blk_lo + k - lo, blk_lo + k - lo + nk, ls);
        }
        lane_done();
        blk_lo += blk_n;
        blk_n = 0;
        if (dual) lane ^= 1;
    };
    // internal values feed the Grangeat step directly: store them divided by w2
    const float* tscale = values_out ? nullptr : p->fgr.w2inv.p;
    auto gather = [&](int v, int n, float* out) {
        if (!lanes) {
            gather_views(p, v, v + n, out, s, tscale);
            return;
        }
        const cudaStream_t ls = values_out ? s : lane_stream();
        gather_views_lanes(p, v, n, out, ls, tscale);
        if (!values_out) lane_done();
    };
    // runs of consecutive batches (clipped to [lo, hi)) sharing one scaling group
    const size_t nbat = bp.batches.size();
    size_t b = 0;
    while (b < nbat) {
        const int vlo = std::max(lo, bp.batches[b].first);
        int vhi = std::min(hi, bp.batches[b].second);
        if (vlo >= vhi) {
            ++b;
            continue;
        }
        const int g = bp.group[b];
        size_t e = b + 1;
        while (e < nbat && bp.group[e] == g && bp.batches[e].first < hi) {
            vhi = std::min(hi, bp.batches[e].second);
            ++e;
        }
        if (g != cur) {
            // the previous grid may still be read on s1
            if (s1_used) CBN_CUDA(cudaStreamWaitEvent(s, p->ev_s1, 0));
            build_resample_grid(p, bp.s32.p + (size_t)g * 3 * bp.smax, bp.smax, s, lanes);
            {
                // the gathers read the built grid once: the rho planes the
                // taps reach (views-in-lanes: real grid of those planes only)
                const AxisPlan* ax = p->fres;
                const double plane = (double)ax[0].K * ax[1].K;
                double planes = ax[2].K;
                if (lanes && !p->fres_rho_runs.empty()) {
                    planes = 0;
                    for (const auto& rn : p->fres_rho_runs) planes += rn.second - rn.first;
                }
                const double es = lanes && real_grid(p) ? 4.0 : 8.0;
                p->timer.add_bytes("resample_gather", es * plane * planes, 0.0);
            }
            if (dual) {
                CBN_CUDA(cudaEventRecord(p->ev_s0, s));
                s1_stale = true;
            }
            cur = g;
        }
        for (int v = vlo; v < vhi;) {
            if (values_out) {
                const int take = std::min(vhi - v, chunk);
                gather(v, take, values_out + (size_t)(v - lo) * per_view);
                v += take;
                continue;
            }
            const int take = std::min(vhi - v, chunk - blk_n);
            gather(v, take, (lane ? p->lane1.values.p : p->values.p) + (size_t)blk_n * per_view);
            blk_n += take;
            v += take;
            if (blk_n == chunk) flush();
        }
        b = e;
    }
    flush();
    if (s1_used) CBN_CUDA(cudaStreamWaitEvent(s, p->ev_s1, 0));
}

// views [lo, hi) from a radial lattice (after the radial IFFT) -> frames
// raises CBN_ENONFINITE if any projection of the call was non-finite (syncs s)
void check_flag(P* p, cudaStream_t s) {
    int flag = 0;
    CBN_CUDA(cudaMemcpyAsync(&flag, p->flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    if (flag) throw Error(CBN_ENONFINITE, "non-finite projection values");
}

void project_views(P* p, const float2* lat, float* frames, int lo, int hi, cudaStream_t s,
                   bool check = true) {
    p->flag.ensure(1);
    CBN_CUDA(cudaMemsetAsync(p->flag.p, 0, sizeof(int), s));
    const RadialTables& r = p->frad;
    lattice_spectrum(p, lat, r.n_rho - r.n_rho / 2, (float)(1.0 / (r.n_rho * r.d_rho)), s);
    resample_and_reverse(p, lo, hi, frames, s);
    if (check) check_flag(p, s);
}

// sharded forward, phase 2: the summed pre-IFFT lattice (consumed) -> views
void fwd_views(P* p, float2* lat, float* frames, int lo, int hi, cudaStream_t s) {
    build_forward(p, s);
    const RadialTables& r = p->frad;
    long long nr1[1] = {r.n_rho};
    {
        StageScope st(p->timer, "radial_ifft", s);
        p->fft.exec(p->fft.get(1, nr1, r.lines()), lat, lat, CUFFT_INVERSE, s);
    }
    project_views(p, lat, frames, lo, hi, s);
}

void forward_project(P* p, const float* vol, float* frames, int lo, int hi, cudaStream_t s,
                     bool check = true, bool staged = false) {
    build_forward(p, s);
    radial_lattice_raw(p, vol, s, nullptr, 0, 1, nullptr, false, staged);
    project_views(p, p->lattice.p, frames, lo, hi, s, check);
}

}  // namespace

// backprojector lives in cbn_backproject.cu
namespace cbn {
void backproject_impl(cbn_projector_s* p, const float* frames, float* vol, cudaStream_t s);
void bp_views(cbn_projector_s* p, const float* frames, int lo, int hi, float2* acc, cudaStream_t s);
void bp_finish(cbn_projector_s* p, float2* acc, int part, int nparts, float2* grid, cudaStream_t s);
void bp_crop(cbn_projector_s* p, float2* grid, float* vol, cudaStream_t s);
void bp_crop_slab(cbn_projector_s* p, float2* slab, int x_lo, int x_hi, int nparts, float2* send,
                  cudaStream_t s);
void bp_crop_cols(cbn_projector_s* p, float2* cols, int y_lo, int y_hi, float* vol_part,
                  cudaStream_t s);
void bp_sizes(cbn_projector_s* p, int64_t* lattice, int64_t* grid, cudaStream_t s);
void build_backward_plan(cbn_projector_s* p, cudaStream_t s) { build_backward(p, s); }
void build_forward_plan(cbn_projector_s* p, cudaStream_t s) { build_forward(p, s); }
bool projector_views_in_lanes(const cbn_projector_s* p) { return views_in_lanes(p); }
bool projector_real_grid(const cbn_projector_s* p) { return real_grid(p); }
void projector_prepare_gr_points(cbn_projector_s* p, GrangeatPlan& gp, const UmbrellaTables& u,
                                 bool reverse, cudaStream_t s) {
    prepare_gr_points(p, gp, u, reverse, s);
}
UmbrellaSrc projector_cached_umbrella(cbn_projector_s* p, UmbrellaTables& u, const RadialTables& r,
                                      int pad, int view0, cudaStream_t s) {
    return cached_umbrella(p, u, r, pad, view0, s);
}
void projector_batch_plan(cbn_projector_s* p, BatchPlan& bp, const UmbrellaTables& u,
                          const RadialTables& r, int pad, const AxisPlan* ax, cudaStream_t s) {
    ensure_batch_plan(p, bp, u, r, pad, ax, s);
}
const int64_t* projector_rows(cbn_projector_s* p, int64_t m, int& n) { return rows_for(p, m, n); }
std::vector<std::pair<int, int>> projector_batches(int n_views, int64_t per_view, int64_t target) {
    return view_batches(n_views, per_view, target);
}
int64_t projector_chunk(const cbn_projector_s* p, int64_t m) { return spectrum_chunk(p, m); }
int64_t projector_target_batch(const cbn_projector_s* p) { return target_batch(p); }
UmbrellaGeom projector_umb_geom(const cbn_projector_s* p, const UmbrellaTables& u,
                                const RadialTables& r, int pad) {
    return umb_geom(p, u, r, pad);
}
void projector_build_tables(cbn_projector_s* p, int mode, const AxisPlan* ax, int smax,
                            cudaStream_t s, RemapAxis* out, const int64_t* sstride) {
    build_tables(p, mode, ax, smax, s, out, sstride);
}
void projector_fit_grangeat(cbn_projector_s* p, GrangeatPlan& gp, const UmbrellaTables& u,
                            cudaStream_t s) {
    fit_grangeat(p, gp, u, s);
}
void projector_gr_pix(const cbn_projector_s* p, GrangeatPlan& gp, bool reverse, cudaStream_t s) {
    ensure_gr_pix(p, gp, reverse, s);
}
void projector_column_mean(const float2* src, int64_t lines, int64_t ld, int col, double scale,
                           double* partial, double* out, cudaStream_t s) {
    column_mean(src, lines, ld, col, scale, partial, out, s);
}
}  // namespace cbn

// =================================================================== C ABI
extern "C" {

int cbn_projector_create(cbn_projector** out, const cbn_geometry* geom,
                         const cbn_projector_config* cfg, int32_t n_vol, double voxel_mm,
                         int32_t direction) {
    try {
        CBN_REQUIRE(out && geom && cfg, "null argument");
        CBN_REQUIRE(geom->so_mm > 0 && geom->sd_mm > geom->so_mm, "invalid geometry");
        CBN_REQUIRE(geom->nu >= 1 && geom->nv >= 1 && geom->n_views >= 1, "invalid detector");
        CBN_REQUIRE(cfg->spec.n_rho >= 2 && cfg->spec.n_rho % 2 == 0, "n_rho must be even and >= 2");
        CBN_REQUIRE(cfg->spec.n_theta >= 1 && cfg->spec.n_phi >= 1, "n_theta, n_phi must be >= 1");
        CBN_REQUIRE(cfg->spec.rho_max > 0, "rho_max must be positive");
        CBN_REQUIRE(cfg->n_mu >= 1 && cfg->n_t >= 1, "n_mu and n_t must be >= 1");
        CBN_REQUIRE(n_vol >= 1 && voxel_mm > 0, "invalid volume size");
        CBN_REQUIRE(direction >= 1 && direction <= 3, "direction must be 1..3");
        CBN_REQUIRE(cfg->oversample_factor >= 1.0, "oversample_factor must be >= 1");
        auto p = std::make_unique<cbn_projector_s>();
        p->g = *geom;
        p->c = *cfg;
        p->n_vol = n_vol;
        p->voxel = voxel_mm;
        p->direction = direction;
        const double mag = geom->sd_mm / geom->so_mm;
        p->pu = (geom->det_width_mm / geom->nu) / mag;
        p->pv = (geom->det_height_mm / geom->nv) / mag;
        compute_needed(p.get());
        *out = p.release();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_destroy(cbn_projector* proj) {
    delete proj;
    return CBN_OK;
}

int cbn_projector_ls_sizes(const cbn_projector* p, int64_t* sizes, int32_t* count) {
    try {
        CBN_REQUIRE(p && count, "null argument");
        int cap = *count;
        *count = (int32_t)p->ls_needed.size();
        if (sizes)
            for (int i = 0; i < std::min<int>(cap, *count); ++i) sizes[i] = p->ls_needed[i];
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_set_ls_rows(cbn_projector* p, int64_t m, const int64_t* rows, int64_t n) {
    try {
        CBN_REQUIRE(p && rows, "null argument");
        CBN_REQUIRE(n >= 1 && n <= kMaxLS && n <= m, "row count must be 1..min(m, 8192)");
        for (int64_t i = 0; i < n; ++i) CBN_REQUIRE(rows[i] >= 0 && rows[i] < m, "row out of range");
        auto* buf = new DevBuf<int64_t>();
        buf->alloc((size_t)n);
        CBN_CUDA(cudaMemcpy(buf->p, rows, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
        auto it = p->ls_rows.find(m);
        if (it != p->ls_rows.end()) delete it->second;
        p->ls_rows[m] = buf;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_info(const cbn_projector* p, int32_t* n_vol, int32_t* n_views, int32_t* nu,
                       int32_t* nv) {
    try {
        CBN_REQUIRE(p, "null argument");
        if (n_vol) *n_vol = p->n_vol;
        if (n_views) *n_views = p->g.n_views;
        if (nu) *nu = p->g.nu;
        if (nv) *nv = p->g.nv;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_scratch_bytes(const cbn_projector* p, int64_t* bytes) {
    try {
        CBN_REQUIRE(p && bytes, "null argument");
        *bytes = (int64_t)(p->big.bytes() + p->lattice.bytes() + p->padded.bytes() +
                           p->gr_t.bytes() + p->gr_grid.bytes() + p->values.bytes());
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_project(cbn_projector* p, const float* vol, float* frames, int32_t lo, int32_t hi,
                        void* stream) {
    try {
        CBN_REQUIRE(p && vol && frames, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        forward_project(p, vol, frames, lo, hi, static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_project_async(cbn_projector* p, const float* vol, float* frames, int32_t lo,
                              int32_t hi, void* stream) {
    try {
        CBN_REQUIRE(p && vol && frames, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        p->track_blocks = true;
        p->blk_count = 0;
        try {
            forward_project(p, vol, frames, lo, hi, static_cast<cudaStream_t>(stream), false);
        } catch (...) {
            p->track_blocks = false;
            throw;
        }
        p->track_blocks = false;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_stage_volume(cbn_projector* p, const float* vol, int32_t row_lo, int32_t row_hi,
                             void* stream) {
    try {
        CBN_REQUIRE(p && vol, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(0 <= row_lo && row_lo < row_hi && row_hi <= p->n_vol, "row range out of bounds");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        if (p->fshard_nparts > 1 || p->fspec[0].K < p->fspec[0].N)
            throw Error(CBN_EUNSUPPORTED, "staged volume input: plan shape not supported");
        if (row_lo == 0) {
            spectrum_stage_begin(p, s);
            p->fspec_staged = 0;
            p->fspec_staged_vol = vol;
        }
        CBN_REQUIRE(row_lo == p->fspec_staged && vol == p->fspec_staged_vol,
                    "volume rows must be staged in ascending contiguous chunks from row 0");
        spectrum_stage_rows(p, vol, row_lo, row_hi, s);
        p->fspec_staged = row_hi;
        return CBN_OK;
    } catch (const std::exception& e) {
        if (p) p->fspec_staged = 0;
        return fail(e);
    }
}

int cbn_forward_project_staged_async(cbn_projector* p, float* frames, int32_t lo, int32_t hi,
                                     void* stream) {
    try {
        CBN_REQUIRE(p && frames, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        CBN_REQUIRE(p->fspec_staged == p->n_vol && p->fspec_staged_vol,
                    "the whole volume must be staged first (cbn_forward_stage_volume)");
        p->track_blocks = true;
        p->blk_count = 0;
        try {
            forward_project(p, p->fspec_staged_vol, frames, lo, hi, static_cast<cudaStream_t>(stream),
                            false, true);
        } catch (...) {
            p->track_blocks = false;
            p->fspec_staged = 0;
            throw;
        }
        p->track_blocks = false;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_blocks(cbn_projector* p, int32_t* view_lo, int32_t* view_hi, int32_t* count) {
    try {
        CBN_REQUIRE(p && count, "null argument");
        const int cap = *count;
        *count = p->blk_count;
        for (int k = 0; k < std::min(cap, p->blk_count); ++k) {
            if (view_lo) view_lo[k] = p->blk_lo[(size_t)k];
            if (view_hi) view_hi[k] = p->blk_hi[(size_t)k];
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_block_sync(cbn_projector* p, int32_t k) {
    try {
        CBN_REQUIRE(p && k >= 0 && k < p->blk_count, "block out of range");
        CBN_CUDA(cudaEventSynchronize(p->blk_ev[(size_t)k]));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_finish(cbn_projector* p, void* stream) {
    try {
        CBN_REQUIRE(p, "null argument");
        check_flag(p, static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject(cbn_projector* p, const float* frames, float* vol, void* stream) {
    try {
        CBN_REQUIRE(p && vol && frames, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        backproject_impl(p, frames, vol, static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_lattice_size(cbn_projector* p, int64_t* lattice_elems, void* stream) {
    try {
        CBN_REQUIRE(p && lattice_elems, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        build_forward(p, static_cast<cudaStream_t>(stream));
        *lattice_elems = p->frad.nodes();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_set_node_shard(cbn_projector* p, int32_t part, int32_t nparts, int64_t* node_lo,
                                 int64_t* node_hi, void* stream) {
    try {
        CBN_REQUIRE(p, "null argument");
        CBN_REQUIRE(p->direction == 1, "node shards need a forward-only projector");
        CBN_REQUIRE(nparts >= 1 && 0 <= part && part < nparts, "bad part");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        const int64_t lines = p->frad.lines(), n_rho = p->frad.n_rho;
        if (nparts > 1 && lines % nparts != 0)
            throw Error(CBN_EUNSUPPORTED, "radial lines do not split evenly over the parts");
        if (p->fshard_part != part || p->fshard_nparts != nparts) {
            // the spectrum plan (pairs, bins, records) is rebuilt for the new share
            CBN_CUDA(cudaStreamSynchronize(s));
            p->fpairs_n = 0;
            p->fspec_bins.ready = false;
            p->fspec_bins.perm.release();
            p->fspec_bins.subs.release();
            p->fspec_bins.nsubs = 0;
            p->fspec_rec.release();
            p->fspec_fac.release();
            p->fspec_out.release();
            p->fshard_part = nparts > 1 ? part : 0;
            p->fshard_nparts = nparts;
        }
        if (node_lo) *node_lo = lines * part / nparts * n_rho;
        if (node_hi) *node_hi = lines * (part + 1) / nparts * n_rho;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_lattice(cbn_projector* p, const float* vol, int32_t part, int32_t nparts,
                        void* lattice, void* stream) {
    try {
        CBN_REQUIRE(p && vol && lattice, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(nparts >= 1 && 0 <= part && part < nparts, "bad part");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        // the pre-IFFT lattice values of this share (fwd_views runs the IFFT)
        radial_lattice_raw(p, vol, s, nullptr, part, nparts, static_cast<float2*>(lattice), true);
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_forward_views(cbn_projector* p, void* lattice, float* frames, int32_t lo, int32_t hi,
                      void* stream) {
    try {
        CBN_REQUIRE(p && lattice && frames, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        fwd_views(p, static_cast<float2*>(lattice), frames, lo, hi, static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_sizes(cbn_projector* p, int64_t* lattice_elems, int64_t* grid_elems,
                          void* stream) {
    try {
        CBN_REQUIRE(p && lattice_elems && grid_elems, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        bp_sizes(p, lattice_elems, grid_elems, static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_views(cbn_projector* p, const float* frames, int32_t lo, int32_t hi,
                          void* lattice, void* stream) {
    try {
        CBN_REQUIRE(p && frames && lattice, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        bp_views(p, frames, lo, hi, static_cast<float2*>(lattice), static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_finish(cbn_projector* p, void* lattice, int32_t part, int32_t nparts, void* grid,
                           void* stream) {
    try {
        CBN_REQUIRE(p && lattice && grid, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        CBN_REQUIRE(nparts >= 1 && 0 <= part && part < nparts, "bad part");
        bp_finish(p, static_cast<float2*>(lattice), part, nparts, static_cast<float2*>(grid),
                  static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_crop(cbn_projector* p, void* grid, float* vol, void* stream) {
    try {
        CBN_REQUIRE(p && grid && vol, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        bp_crop(p, static_cast<float2*>(grid), vol, static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_crop_slab(cbn_projector* p, void* slab, int32_t x_lo, int32_t x_hi,
                              int32_t nparts, void* send, void* stream) {
    try {
        CBN_REQUIRE(p && slab && send, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        bp_crop_slab(p, static_cast<float2*>(slab), x_lo, x_hi, nparts, static_cast<float2*>(send),
                     static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_crop_cols(cbn_projector* p, void* cols, int32_t y_lo, int32_t y_hi,
                              float* vol_part, void* stream) {
    try {
        CBN_REQUIRE(p && cols && vol_part, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        bp_crop_cols(p, static_cast<float2*>(cols), y_lo, y_hi, vol_part,
                     static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_radial_lattice(cbn_projector* p, const float* vol, void* lattice, void* stream) {
    try {
        CBN_REQUIRE(p && vol && lattice, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        radial_lattice_raw(p, vol, s);
        const RadialTables& r = p->frad;
        const int64_t M = r.nodes();
        k_lattice_final<<<blocks_for(M, 256), 256, 0, s>>>(p->lattice.p, static_cast<float2*>(lattice),
                                                           r.n_rho, M,
                                                           (float)(1.0 / (r.n_rho * r.d_rho)));
        CBN_LAUNCH_CHECK();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// diagnostics: the forward plan's sorted polar-node records (GrPoint<5>, 56 B
// each, sorted order) and the sorted node ids; sizes via *m
int cbn_projector_grangeat_records(cbn_projector* p, void* records, int32_t* perm, int64_t* m,
                                   void* stream) {
    try {
        CBN_REQUIRE(p && m, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        GrangeatPlan& gp = p->fgr;
        if (!gp.built) fit_grangeat(p, gp, p->fumb, s);
        prepare_gr_points(p, gp, p->fumb, true, s);
        const int64_t cap = *m;
        *m = gp.m;
        if (records && cap >= gp.m) {
            CBN_CUDA(cudaMemcpy(records, gp.pts.p, sizeof(GrPoint<kGrJ>) * gp.m, cudaMemcpyDeviceToHost));
            CBN_CUDA(cudaMemcpy(perm, gp.bins.perm.p, sizeof(int) * gp.m, cudaMemcpyDeviceToHost));
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_radial_spectrum(cbn_projector* p, const float* vol, void* spectrum, void* stream) {
    try {
        CBN_REQUIRE(p && vol && spectrum, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        radial_lattice_raw(p, vol, s, static_cast<float2*>(spectrum));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_resample_views(cbn_projector* p, const void* lattice, float* values, int32_t lo,
                                 int32_t hi, void* stream) {
    try {
        CBN_REQUIRE(p && lattice && values, "null argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        lattice_spectrum(p, static_cast<const float2*>(lattice), 0, 1.0f, s);
        resample_and_reverse(p, lo, hi, nullptr, s, values);
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_grangeat_reverse(cbn_projector* p, const float* values, float* frames,
                                   int32_t nb, void* stream) {
    try {
        CBN_REQUIRE(p && values && frames && nb >= 1, "bad argument");
        CBN_REQUIRE(p->direction & 1, "projector was not created for the forward direction");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_forward(p, s);
        p->flag.ensure(1);
        CBN_CUDA(cudaMemsetAsync(p->flag.p, 0, sizeof(int), s));
        const size_t per_view = (size_t)p->fumb.n_mu * p->fumb.n_t;
        const size_t fsz = (size_t)p->g.nu * p->g.nv;
        p->values.ensure(per_view * 32);
        for (int v = 0; v < nb; v += 32) {
            int k = std::min(32, nb - v);
            const int64_t tot = (int64_t)k * per_view;
            k_gr_scale<<<blocks_for(tot, 256), 256, 0, s>>>(values + v * per_view, p->fgr.w2inv.p,
                                                            p->fumb.n_t, tot, p->values.p);
            CBN_LAUNCH_CHECK();
            grangeat_reverse(p, p->values.p, frames + v * fsz, k, s);
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_set_timing(cbn_projector* p, int32_t on) {
    try {
        CBN_REQUIRE(p, "null argument");
        p->timer.reset();
        p->timer.on = on != 0;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_stage_bytes(cbn_projector* p, double* hbm, double* chip, int32_t* count,
                              char* names, int32_t names_len, int32_t reset) {
    try {
        CBN_REQUIRE(p && count, "null argument");
        const int cap = *count;
        *count = (int32_t)p->timer.bytes.size();
        std::string joined;
        for (int i = 0; i < *count; ++i) {
            if (i < cap) {
                if (hbm) hbm[i] = p->timer.bytes[i].second.hbm;
                if (chip) chip[i] = p->timer.bytes[i].second.chip;
            }
            if (i) joined += ";";
            joined += p->timer.bytes[i].first;
        }
        if (names && names_len > 0) {
            std::strncpy(names, joined.c_str(), (size_t)names_len - 1);
            names[names_len - 1] = 0;
        }
        if (reset) p->timer.bytes.clear();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_stage_times(cbn_projector* p, double* ms, int32_t* count, char* names,
                              int32_t names_len, int32_t reset) {
    try {
        CBN_REQUIRE(p && count, "null argument");
        p->timer.collect();
        const int cap = *count;
        *count = (int32_t)p->timer.totals.size();
        std::string joined;
        for (int i = 0; i < *count; ++i) {
            if (ms && i < cap) ms[i] = p->timer.totals[i].second;
            if (i) joined += ";";
            joined += p->timer.totals[i].first;
        }
        if (names && names_len > 0) {
            std::strncpy(names, joined.c_str(), (size_t)names_len - 1);
            names[names_len - 1] = 0;
        }
        if (reset) p->timer.totals.clear();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
