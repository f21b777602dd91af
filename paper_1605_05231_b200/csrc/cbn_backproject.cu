// Direct NUFFT backprojector (pipeline.py:150-212) on the B200:
//   per reference view batch:
//     forward Grangeat (grangeat.py:131-146): w1, deapod/pad, cuFFT 2D,
//       KB J=5 gather at polar nodes, i omega, centred t IFFT, w2
//     resample transpose (resampling.py:164-196): KB J=3 spread of the values
//       and of the validity mask (num/den) at umbrella targets, cuFFT^-1,
//       crop + per-batch deapodisation, accumulated over batches
//   then: ifftshift + cuFFT^-1 of the accumulators, rho crop, origin average,
//   num/den with the vacancy threshold, centred radial FFT, ramp * sin(theta)
//   * trilinear, KB J spread onto (2N)^3, cuFFT^-1, crop + deapodisation.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <numeric>

#include "cbn_projector.h"
#include "cbn_resample_views.cuh"
#include "cbn_dirichlet.cuh"

namespace cbn {

const int64_t* projector_rows(cbn_projector_s* p, int64_t m, int& n);
std::vector<std::pair<int, int>> projector_batches(int n_views, int64_t per_view, int64_t target);
int64_t projector_chunk(const cbn_projector_s* p, int64_t m);
int64_t projector_target_batch(const cbn_projector_s* p);
UmbrellaGeom projector_umb_geom(const cbn_projector_s* p, const UmbrellaTables& u,
                                const RadialTables& r, int pad);
void projector_build_tables(cbn_projector_s* p, int mode, const AxisPlan* ax, int smax,
                            cudaStream_t s, RemapAxis* out, const int64_t* sstride);
void projector_fit_grangeat(cbn_projector_s* p, GrangeatPlan& gp, const UmbrellaTables& u,
                            cudaStream_t s);
void projector_gr_pix(const cbn_projector_s* p, GrangeatPlan& gp, bool reverse, cudaStream_t s);
void projector_column_mean(const float2* src, int64_t lines, int64_t ld, int col, double scale,
                           double* partial, double* out, cudaStream_t s);
void build_backward_plan(cbn_projector_s* p, cudaStream_t s);
UmbrellaSrc projector_cached_umbrella(cbn_projector_s* p, UmbrellaTables& u, const RadialTables& r,
                                      int pad, int view0, cudaStream_t s);
void projector_batch_plan(cbn_projector_s* p, BatchPlan& bp, const UmbrellaTables& u,
                          const RadialTables& r, int pad, const AxisPlan* ax, cudaStream_t s);

namespace {

constexpr int kRed = 296;

CBN_D int pad_src(int g, int N, int K) {
    const int h = N / 2;
    if (g < N - h) return g + h;
    if (g >= K - h) return g - K + h;
    return -1;
}

// h = frame * w1 ; y = h * scaling placed at rolled positions (nufft.py:226-230)
template <int V>   // cells per thread: 4 (Kv % 4 == 0, one 16-byte store) or 1
__global__ void k_grf_pad(const float* __restrict__ frames, int nu, int nv, int Ku, int Kv,
                          const float* __restrict__ pix, float* __restrict__ grids) {
    // grid (Kv / (256 V), Ku, views): one padded row per (blockIdx.y, blockIdx.z)
    const int gv = V * (blockIdx.x * blockDim.x + threadIdx.x);
    if (gv >= Kv) return;
    const int gu = blockIdx.y, v = blockIdx.z;
    const int nu_i = pad_src(gu, nu, Ku);
    float o[V];
#pragma unroll
    for (int q = 0; q < V; ++q) o[q] = 0.f;
    if (nu_i >= 0) {
        const float* fr = frames + ((size_t)v * nu + nu_i) * nv;
        const float* px = pix + (size_t)nu_i * nv;
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const int nv_i = pad_src(gv + q, nv, Kv);
            if (nv_i >= 0) o[q] = fr[nv_i] * px[nv_i];
        }
    }
    float* dst = grids + ((size_t)v * Ku + gu) * Kv + gv;
    if constexpr (V == 4) *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
    else dst[0] = o[0];
}

// values = Re(fftshift(ifft)) / dt * w2   (grangeat.py:144-145)
__global__ void k_grf_post(const float2* __restrict__ t, const float* __restrict__ w2, int n_t,
                           double inv, int64_t total, float* __restrict__ vals) {
    // two outputs (j, j + 1) per thread, j even; n_t % 4 == 0 so the two
    // source bins (j - n_t/2 mod n_t) are one aligned 16-byte pair
    const int64_t e = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (e >= total) return;
    const int64_t row = e / n_t;
    const int j = (int)(e - row * n_t);
    const int src = j < n_t / 2 ? j + n_t / 2 : j - n_t / 2;
    const float4 q = *reinterpret_cast<const float4*>(t + row * n_t + src);
    *reinterpret_cast<float2*>(vals + e) =
        make_float2((float)(q.x * inv) * w2[j], (float)(q.z * inv) * w2[j + 1]);
}

// k_grf_post writing target-major: valsT[target * ldT + voff + v] for the
// block's views v < nb (<= 32); 32 targets x 32 views per CTA through shared
// memory, so both the reads (along t) and the writes (along views) coalesce
__global__ void k_grf_post_t(const float2* __restrict__ t, const float* __restrict__ w2, int n_t,
                             double inv, int64_t per_view, int nb, float* __restrict__ valsT,
                             int64_t ldT, int voff) {
    __shared__ float tile[32][33];
    const int64_t t0 = (int64_t)blockIdx.x * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tt = t0 + lane;
    if (tt < per_view) {
        const int64_t line = tt / n_t;
        const int j = (int)(tt - line * n_t);
        const int src = j < n_t / 2 ? j + (n_t - n_t / 2) : j - n_t / 2;
        const float w = w2[j];
        for (int v = warp; v < nb; v += 8) {
            const float re = t[((int64_t)v * (per_view / n_t) + line) * n_t + src].x;
            tile[v][lane] = (float)(re * inv) * w;
        }
    }
    __syncthreads();
    for (int q = warp; q < 32; q += 8) {
        const int64_t tq = t0 + q;
        if (tq < per_view && lane < nb) valsT[tq * ldT + voff + lane] = tile[lane][q];
    }
}

__global__ void k_grf_post1(const float2* __restrict__ t, const float* __restrict__ w2, int n_t,
                            double inv, int64_t total, float* __restrict__ vals) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int64_t row = e / n_t;
    const int j = (int)(e - row * n_t);
    const float re = t[row * n_t + (j - n_t / 2 + n_t) % n_t].x;
    vals[e] = (float)(re * inv) * w2[j];
}

// num / den spreads of one resample batch (resample_transpose, called with the
// values and with the validity mask, pipeline.py:183-184); real inputs, the
// phases cancel, so only the real part of each grid receives data
template <int J>
__global__ void __launch_bounds__(256)
k_rs_spread2(float* __restrict__ gnum, float* __restrict__ gden, KBSet kb, UmbrellaSrc src,
             const float* __restrict__ vals, int64_t m) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double w[3];
    UmbrellaSrc::Aux aux;
    src.node(i, w, aux);
    if (!aux.valid) return;
    const float vn = (vals && gnum) ? vals[i] : 0.f;   // den-only passes: no values
    if (vn == 0.f && !gden) return;
    int first[3];
    float wt[3][J];
    tap_setup<3, J>(kb, w, first, wt);
    const int K0 = kb.ax[0].K, K1 = kb.ax[1].K, K2 = kb.ax[2].K;
    int c2[J];
#pragma unroll
    for (int c = 0; c < J; ++c) c2[c] = wrapc(first[2] + c, K2);
#pragma unroll
    for (int a = 0; a < J; ++a) {
        const size_t pa = (size_t)wrapc(first[0] + a, K0) * K1;
#pragma unroll
        for (int b = 0; b < J; ++b) {
            const size_t row = (pa + (size_t)wrapc(first[1] + b, K1)) * K2;
            const float wab = wt[0][a] * wt[1][b];
#pragma unroll
            for (int c = 0; c < J; ++c) {
                const float wk = wab * wt[2][c];
                const size_t idx = 2 * (row + c2[c]);
                if (vn != 0.f) atomicAdd(gnum + idx, wk * vn);
                if (gden) atomicAdd(gden + idx, wk);
            }
        }
    }
}

// final den lattice (origin average and 1/size applied), node order
__global__ void k_den_final(const float2* __restrict__ acc_den, int64_t lines, int dr, int pad,
                            int n, double inv, const double* __restrict__ means,
                            float* __restrict__ den) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= lines * n) return;
    const int j = (int)(e % n);
    const int64_t line = e / n;
    den[e] = (j == n / 2) ? (float)means[0] : (float)((double)acc_den[line * dr + pad + j].x * inv);
}

// keep = den > tol * max(den) (pipeline.py:187-188) decided per phi orbit
// {c, c + s, ...} from the orbit's float64 mean, for rotation-aligned views:
// each view's targets are view 0's rotated by s whole lattice phi cells, so
// the transposed resample is phi-shift equivariant and the reference's den is
// uniform over an orbit (to ~1e-8 of the threshold away from the poles, whose
// targets take per-view phi).  The float32 den of one orbit scatters by ~1e-5
// of the threshold, enough to split an orbit that sits that close to it, which
// the reference never does; the mean decides for the whole orbit, while every
// entry is still divided by its own den.  Node order [phi][theta][rho].
__global__ void k_den_keep_orbit(const float* __restrict__ den, int n_rho, int n_theta, int n_phi,
                                 int sft, const double* __restrict__ dmax, double tol,
                                 unsigned char* __restrict__ keep) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t plane = (int64_t)n_rho * n_theta;
    if (e >= plane * sft) return;
    const int c = (int)(e / plane);
    const int64_t rt = e - (int64_t)c * plane;
    double sum = 0.0;
    int cnt = 0;
    for (int f = c; f < n_phi; f += sft, ++cnt) sum += (double)den[(int64_t)f * plane + rt];
    const unsigned char k = sum / cnt > tol * dmax[0] ? 1 : 0;
    for (int f = c; f < n_phi; f += sft) keep[(int64_t)f * plane + rt] = k;
}

bool den_orbit_off() {   // CBN_DEN_ORBIT=0: per-entry keep decision (A/B)
    const char* e = std::getenv("CBN_DEN_ORBIT");
    return e && e[0] == '0';
}

__global__ void k_max_partial(const float* __restrict__ x, int64_t total, double* __restrict__ partial) {
    double mx = -1e308;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x)
        mx = fmax(mx, (double)x[e]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = sh[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
        partial[blockIdx.x] = m;
    }
}

__global__ void k_max_final(const double* __restrict__ partial, int n, double* __restrict__ out) {
    if (threadIdx.x) return;
    double m = -1e308;
    for (int i = 0; i < n; ++i) m = fmax(m, partial[i]);
    out[0] = m;
}

// lattice = num / den where den > tol * max (pipeline.py:187-188), written at
// the ifftshifted rho position for the centred radial FFT (radon_fourier.py:117-130)
__global__ void k_bp_div(const float2* __restrict__ acc_num, const float* __restrict__ den,
                         int64_t lines, int dr, int pad, int n, double inv,
                         const double* __restrict__ means, const double* __restrict__ dmax,
                         double tol, const unsigned char* __restrict__ keep,
                         float2* __restrict__ out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= lines * n) return;
    const int j = (int)(e % n);
    const int64_t line = e / n;
    double nr, ni;
    if (j == n / 2) {
        nr = means[0];
        ni = means[1];
    } else {
        float2 a = acc_num[line * dr + pad + j];
        nr = a.x * inv;
        ni = a.y * inv;
    }
    const double d = den[e];
    float2 v = make_float2(0.f, 0.f);
    if (keep ? keep[e] != 0 : d > tol * dmax[0]) v = make_float2((float)(nr / d), (float)(ni / d));
    out[line * n + (j - n / 2 + n) % n] = v;
}

// y for the 3D adjoint: fftshift(FFT) * d_rho * (-i omega apod c3) * sin(theta)
// * trilinear * conj(centre phase) * conj(plan phase)   (pipeline.py:189-210)
struct BpSrc : RadialSrc {
    const float2* X;
    const float* q;        // per rho bin: omega * apod * c3 * d_rho
    const float* sin_th;
    int N[3];              // output dims (centre / plan phases per node representative)
    int tri;
    CBN_D float2 value(int64_t i, const double (&w)[3], const RadialSrc::Aux& a) const {
        const int64_t line = i / n_rho;
        float2 x = X[line * n_rho + (a.ir - n_rho / 2 + n_rho) % n_rho];
        const float qq = q[a.ir] * sin_th[a.it];
        float2 v = make_float2(x.y * qq, -x.x * qq);
        if (tri) {
            float t = 1.f;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                float xx = (float)(a.raw[d] * (1.0 / kTwoPi));
                float sc = xx == 0.f ? 1.f : sinpif(xx) / (3.14159265358979f * xx);
                t *= sc * sc;
            }
            v = cscale(v, t);
        }
        double sn, cs;
        sincos(-centre_plan_angle<3>(a.wc, w, N), &sn, &cs);   // conj(centre) * conj(plan)
        return cmul(v, make_float2((float)cs, (float)sn));
    }
};

// BpSrc over packed conjugate-pair entries: for a pair entry f the adjoint
// only needs Re(IFFT) of the spread, so node f carries v(f) + conj(v(mirror))
// and the mirror is not spread (the Hermitian part of the grid is unchanged)
struct BpPairSrc : BpSrc {
    CBN_D void node(int64_t i, double (&w)[3], Aux& a) const {
        RadialSrc::node(i >= 0 ? i : ~i, w, a);
    }
    CBN_D float2 value(int64_t i, const double (&w)[3], const RadialSrc::Aux& a) const {
        const int64_t f = i >= 0 ? i : ~i;
        float2 v = BpSrc::value(f, w, a);
        if (i >= 0) {
            const int64_t fm = f / n_rho * n_rho + (n_rho - a.ir);
            double wm[3];
            RadialSrc::Aux am;
            RadialSrc::node(fm, wm, am);
            const float2 vm = BpSrc::value(fm, wm, am);
            v.x += vm.x;
            v.y -= vm.y;
        }
        return v;
    }
};

// BpPairSrc from per-plan records (sorted order): KB arguments and bin-local
// first taps as k_spec_records forms them, the two lattice samples a primary
// node reads (its own and, for a pair, its mirror's) and their factors
// -i * q * sin(theta) * sinc^2 transfer * conj(centre * plan phase), so the
// spread's staging reads 40 bytes and two lattice values per point
struct BpRecSrc {
    using is_record_src = void;
    using Aux = RadialSrc::Aux;
    const float4* rec;    // y0, y1, y2, bits (l0 | l1 << 5 | l2 << 10 | edge drops << 15)
    const float4* g;      // factor of X[i1] (x, y), factor of X[i2] (z, w)
    const int2* idx;      // i1, i2 (-1: no mirror)
    const float2* X;      // ramp-filtered lattice, node order
    const float2* vals;   // or: the values already formed in sorted order (k_bp_values)
    template <int J>
    CBN_D void stage(const KBSet& kb, int64_t pos, float2& v, int (&l)[3], float (&wt)[3][J]) const {
        const float4 q = rec[pos];
        const unsigned bits = __float_as_uint(q.w);
        l[0] = bits & 31;
        l[1] = (bits >> 5) & 31;
        l[2] = (bits >> 10) & 31;
        kb_weights_y<J>(kb.ax[0], q.x, (bits >> 15) & 1, wt[0]);
        kb_weights_y<J>(kb.ax[1], q.y, (bits >> 16) & 1, wt[1]);
        kb_weights_y<J>(kb.ax[2], q.z, (bits >> 17) & 1, wt[2]);
        if (vals) {
            v = vals[pos];
            return;
        }
        const float4 f = g[pos];
        const int2 ix = idx[pos];
        v = cmul(X[ix.x], make_float2(f.x, f.y));
        if (ix.y >= 0) {
            const float2 m = cmul(X[ix.y], make_float2(f.z, f.w));
            v.x += m.x;
            v.y -= m.y;
        }
    }
};

// the spread's point values in sorted order, one streaming pass ahead of the
// spread so its staging reads them sequentially instead of gathering two
// lattice samples per point behind each round's barrier
__global__ void k_bp_values(const float4* __restrict__ g, const int2* __restrict__ idx,
                            const float2* __restrict__ X, int64_t m, float2* __restrict__ vals) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= m) return;
    const float4 f = g[pos];
    const int2 ix = idx[pos];
    float2 v = cmul(X[ix.x], make_float2(f.x, f.y));
    if (ix.y >= 0) {
        const float2 q = cmul(X[ix.y], make_float2(f.z, f.w));
        v.x += q.x;
        v.y -= q.y;
    }
    vals[pos] = v;
}

bool bp_values_pass_on() {   // CBN_BP_VALUES=0: values gathered inside the spread (A/B)
    const char* e = std::getenv("CBN_BP_VALUES");
    return !(e && e[0] == '0');
}

template <int J>
__global__ void k_bp_records(BpSrc src, KBSet kb, TileGeom<3> tg, const int* __restrict__ perm,
                             int64_t m, float4* __restrict__ rec, float4* __restrict__ g,
                             int2* __restrict__ idx) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= m) return;
    const int e = perm[pos];
    const int f = e >= 0 ? e : ~e;
    double w[3];
    RadialSrc::Aux a;
    src.RadialSrc::node(f, w, a);
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
    const int n_rho = src.n_rho;
    // factor of BpSrc::value at node f: x * (-i qq t) * e^{-i ang}
    auto factor = [&](const double (&wn)[3], const RadialSrc::Aux& an) {
        double t = 1.0;
        if (src.tri) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double x = an.raw[d] * (1.0 / kTwoPi);
                const double sc = x == 0.0 ? 1.0 : sinpi(x) / (kPi * x);
                t *= sc * sc;
            }
        }
        const double gq = (double)src.q[an.ir] * (double)src.sin_th[an.it] * t;
        double sn, cs;
        sincos(-centre_plan_angle<3>(an.wc, wn, src.N), &sn, &cs);
        return make_float2((float)(sn * gq), (float)(-cs * gq));
    };
    const int line = f / n_rho;
    const float2 g1 = factor(w, a);
    const int i1 = line * n_rho + (a.ir - n_rho / 2 + n_rho) % n_rho;
    float2 g2 = make_float2(0.f, 0.f);
    int i2 = -1;
    if (e >= 0) {
        const int fm = line * n_rho + (n_rho - a.ir);
        double wm[3];
        RadialSrc::Aux am;
        src.RadialSrc::node(fm, wm, am);
        g2 = factor(wm, am);
        i2 = line * n_rho + (am.ir - n_rho / 2 + n_rho) % n_rho;
    }
    g[pos] = make_float4(g1.x, g1.y, g2.x, g2.y);
    idx[pos] = make_int2(i1, i2);
}

bool bp_records_off() {   // CBN_BP_RECORDS=0: node generation per step (A/B)
    const char* e = std::getenv("CBN_BP_RECORDS");
    return e && e[0] == '0';
}

}  // namespace

void projector_prepare_gr_points(cbn_projector_s* p, GrangeatPlan& gp, const UmbrellaTables& u,
                                 bool reverse, cudaStream_t s);

// forward_grangeat_view for nb (<= 32) views: frames (nb x nu x nv) -> values
// (nb x n_mu x n_t), grangeat.py:131-146
// values: [nb][n_mu][n_t]; or, with valsT, target-major valsT[target * ldT + voff + v]
void grangeat_forward_block(cbn_projector_s* p, const float* frames, int nb, float* values,
                            cudaStream_t s, GrBufs B, float* valsT = nullptr, int64_t ldT = 0,
                            int voff = 0) {
    GrangeatPlan& gp = p->bgr;
    if (!gp.built) projector_fit_grangeat(p, gp, p->bumb, s);
    projector_prepare_gr_points(p, gp, p->bumb, false, s);
    const UmbrellaTables& u = p->bumb;
    const int Ku = gp.ax[0].K, Kv = gp.ax[1].K;
    const int nu = p->g.nu, nv = p->g.nv;
    const int64_t per_view = (int64_t)u.n_mu * u.n_t;
    // the padded frame is real: real-to-complex 2D FFT to the half spectrum
    // [Ku][Kv/2+1]; the gather reads the other half as conjugate mirrors
    const int64_t hk = (int64_t)Ku * (Kv / 2 + 1);
    B.grid.ensure((size_t)nb * hk);
    B.tv.ensure(((size_t)nb * Ku * Kv + 1) / 2);
    B.t.ensure((size_t)nb * per_view);
    float* padded = reinterpret_cast<float*>(B.tv.p);
    const int64_t gtot = (int64_t)nb * Ku * Kv;
    projector_gr_pix(p, gp, false, s);
    if (Kv % 4 == 0)
        k_grf_pad<4><<<dim3((unsigned)((Kv / 4 + 255) / 256), Ku, nb), 256, 0, s>>>(
            frames, nu, nv, Ku, Kv, gp.pix.p, padded);
    else
        k_grf_pad<1><<<dim3((unsigned)((Kv + 255) / 256), Ku, nb), 256, 0, s>>>(
            frames, nu, nv, Ku, Kv, gp.pix.p, padded);
    (void)gtot;
    CBN_LAUNCH_CHECK();
    long long kd[2] = {Ku, Kv};
    B.fft.exec_r2c3(B.fft.get_r2c2(kd, nb), padded, B.grid.p, s);
    const BinPlan& bb = gp.bins;
    dim3 grid(bb.nsubs, (nb + kGrVG - 1) / kGrVG);
    k_gr_gather_binned<kGrJ, kGrVG, true><<<grid, 256, sizeof(float2) * kGrVG * bb.nreg, s>>>(
        B.grid.p, (size_t)hk, bb.geom<2>(), reinterpret_cast<const GrPoint<kGrJ>*>(gp.pts.p),
        bb.subs.p, B.t.p, (size_t)per_view, nb);
    CBN_LAUNCH_CHECK();
    long long nt[1] = {u.n_t};
    B.fft.exec(B.fft.get(1, nt, (long long)nb * u.n_mu), B.t.p, B.t.p, CUFFT_INVERSE, s);
    const int64_t vt = (int64_t)nb * per_view;
    const double inv = 1.0 / ((double)u.n_t * u.dt);
    if (valsT) {
        k_grf_post_t<<<blocks_for(per_view, 32), 256, 0, s>>>(B.t.p, gp.w2.p, u.n_t, inv, per_view,
                                                            nb, valsT, ldT, voff);
        CBN_LAUNCH_CHECK();
        return;
    }
    if (u.n_t % 4 == 0)
        k_grf_post<<<blocks_for(vt / 2, 256), 256, 0, s>>>(B.t.p, gp.w2.p, u.n_t, inv, vt, values);
    else
        k_grf_post1<<<blocks_for(vt, 256), 256, 0, s>>>(B.t.p, gp.w2.p, u.n_t, inv, vt, values);
    CBN_LAUNCH_CHECK();
}

void grangeat_forward_block(cbn_projector_s* p, const float* frames, int nb, float* values,
                            cudaStream_t s) {
    grangeat_forward_block(p, frames, nb, values, s, main_bufs(p));
}

// ------------------------------------------------------------------ phases
// The backprojector runs in three phases so that views and nodes can be
// sharded across ranks:
//   1. bp_views:  transposed resample of a view range into a padded-lattice
//                 accumulator (ranks' accumulators are summed);
//   2. bp_finish: lattice division by the cached den, ramp, and the 3D spread
//                 of a share of the bin subproblems into a K^3 grid (summed);
//   3. bp_crop:   inverse FFT, crop, deapodisation and Re * bp_normalization.
// cbn_backproject runs all three on one device.
struct BpCtx {
    int dr = 0;
    int64_t dsize = 0, kres = 0, k3 = 0, per_view = 0;
    bool method_b = false, lanes = false;
    int shift = 0, slow_axis = 0;
    long long kd3[3] = {0, 0, 0};
    int64_t sstr[3] = {0, 0, 0};
    KBSet kbr{};
};

bool rs_strips_on() {   // CBN_RS_STRIPS=0: the per-column transposed gather (A/B)
    const char* e = std::getenv("CBN_RS_STRIPS");
    return !(e && e[0] == '0');
}

// Strip form of the transposed-resample column CSR (k_rs_gather_strips):
// per rho plane, strips of kRsStrip theta columns, their (sorted) column lists
// merged by target on the host once per plan.
void bp_build_col_strips(cbn_projector_s* p, int64_t K0, int64_t K1, cudaStream_t s) {
    const int64_t ncol = K0 * K1;
    const int nsx = (int)((K1 + kRsStrip - 1) / kRsStrip);
    const int64_t nstrips = K0 * nsx;
    std::vector<int> ptr((size_t)ncol + 1);
    std::vector<RsColEntry> ent((size_t)p->bcol_n);
    CBN_CUDA(cudaMemcpyAsync(ptr.data(), p->bcol_ptr.p, sizeof(int) * ptr.size(),
                             cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaMemcpyAsync(ent.data(), p->bcol_ent.p, sizeof(RsColEntry) * ent.size(),
                             cudaMemcpyDeviceToHost, s));
    CBN_CUDA(cudaStreamSynchronize(s));
    struct Rec {
        int t, f2;
        float w2[3];
        float wab[kRsStrip];
    };
    std::vector<std::vector<Rec>> planes((size_t)K0);
    std::vector<std::vector<int>> counts((size_t)K0, std::vector<int>((size_t)nsx, 0));
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t r = 0; r < K0; ++r) {
        std::vector<std::pair<int, int>> items;   // (target, entry index)
        auto& out = planes[(size_t)r];
        for (int sx = 0; sx < nsx; ++sx) {
            items.clear();
            for (int c = 0; c < kRsStrip; ++c) {
                const int64_t th = (int64_t)sx * kRsStrip + c;
                if (th >= K1) break;
                const int64_t col = r * K1 + th;
                for (int e = ptr[(size_t)col]; e < ptr[(size_t)col + 1]; ++e)
                    items.emplace_back(ent[(size_t)e].t, e);
            }
            std::sort(items.begin(), items.end());
            size_t q = 0;
            int cnt = 0;
            while (q < items.size()) {
                const int t = items[q].first;
                Rec rec{};
                const RsColEntry& e0 = ent[(size_t)items[q].second];
                rec.t = t;
                rec.f2 = e0.f2;
                for (int k = 0; k < 3; ++k) rec.w2[k] = e0.w2[k];
                for (; q < items.size() && items[q].first == t; ++q) {
                    const int e = items[q].second;
                    int col_in = 0;   // which of the strip's columns holds entry e
                    for (int c = 0; c < kRsStrip; ++c) {
                        const int64_t col = r * K1 + (int64_t)sx * kRsStrip + c;
                        if ((int64_t)sx * kRsStrip + c < K1 && e >= ptr[(size_t)col] &&
                            e < ptr[(size_t)col + 1])
                            col_in = c;
                    }
                    rec.wab[col_in] += ent[(size_t)e].wab;
                }
                out.push_back(rec);
                ++cnt;
            }
            counts[(size_t)r][(size_t)sx] = cnt;
        }
    }
    std::vector<int> sptr((size_t)nstrips + 1, 0);
    std::vector<RsStripEnt> se;
    std::vector<float4> w2, wab;
    int64_t st = 0;
    for (int64_t r = 0; r < K0; ++r) {
        const auto& out = planes[(size_t)r];
        size_t q = 0;
        for (int sx = 0; sx < nsx; ++sx, ++st) {
            const int cnt = counts[(size_t)r][(size_t)sx];
            for (int k = 0; k < cnt; ++k, ++q) {
                const Rec& rc = out[q];
                se.push_back(RsStripEnt{rc.t, rc.f2});
                w2.push_back(make_float4(rc.w2[0], rc.w2[1], rc.w2[2], 0.f));
                wab.push_back(make_float4(rc.wab[0], rc.wab[1], rc.wab[2], rc.wab[3]));
            }
            sptr[(size_t)st + 1] = sptr[(size_t)st] + cnt;
        }
    }
    p->bstrip_n = (int64_t)se.size();
    if (se.empty()) {
        se.push_back(RsStripEnt{0, 0});
        w2.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
        wab.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
    }
    p->bstrip_nsx = nsx;
    p->bstrip_ptr.upload(sptr.data(), sptr.size(), s);
    p->bstrip_ent.alloc(sizeof(RsStripEnt) * se.size());
    CBN_CUDA(cudaMemcpyAsync(p->bstrip_ent.p, se.data(), sizeof(RsStripEnt) * se.size(),
                             cudaMemcpyHostToDevice, s));
    p->bstrip_w2.upload(w2.data(), w2.size(), s);
    p->bstrip_wab.upload(wab.data(), wab.size(), s);
    CBN_CUDA(cudaStreamSynchronize(s));
}

BpCtx bp_context(cbn_projector_s* p, cudaStream_t s) {
    build_backward_plan(p, s);
    const cbn_projector_config& c = p->c;
    const RadialTables& r = p->brad;
    const UmbrellaTables& u = p->bumb;
    GrangeatPlan& gp = p->bgr;
    if (!gp.built) projector_fit_grangeat(p, gp, u, s);
    const AxisPlan* rax = p->bres;
    BatchPlan& bp = p->bbatch;
    if (c.method == 0) projector_batch_plan(p, bp, u, r, p->bpad, rax, s);   // method A scalings
    BpCtx x;
    x.dr = r.n_rho + 2 * p->bpad;
    x.dsize = (int64_t)x.dr * r.n_theta * r.n_phi;
    x.kres = (int64_t)rax[0].K * rax[1].K * rax[2].K;
    x.k3 = (int64_t)p->bspec[0].K * p->bspec[1].K * p->bspec[2].K;
    x.per_view = (int64_t)u.n_mu * u.n_t;
    for (int d = 0; d < 3; ++d) x.kbr.ax[d] = rax[d].kb;
    // views in lanes (as the forward gather): when view k's targets are view 0's
    // shifted by whole oversampled phi cells, the transposed grid is stored
    // phi-fastest [rho][theta][phi] and built by the column gather
    // (k_rs_gather_cols) instead of the atomic scatter
    const char* no_lanes = std::getenv("CBN_NO_VIEW_LANES");
    x.method_b = c.method == 1;
    x.lanes = !x.method_b && !(no_lanes && no_lanes[0] == '1') && res_j3(rax) &&
              (2LL * r.n_phi) % p->g.n_views == 0 && rax[0].K == 2 * r.n_phi;
    x.shift = (int)(2LL * r.n_phi / p->g.n_views);
    x.kd3[0] = rax[0].K;
    x.kd3[1] = rax[1].K;
    x.kd3[2] = rax[2].K;
    x.sstr[0] = (int64_t)rax[1].K * rax[2].K;
    x.sstr[1] = rax[2].K;
    x.sstr[2] = 1;
    if (x.lanes) {
        x.kd3[0] = rax[2].K;
        x.kd3[2] = rax[0].K;
        x.sstr[0] = 1;
        x.sstr[1] = rax[0].K;
        x.sstr[2] = (int64_t)rax[1].K * rax[0].K;
        if (!p->bcol_ptr.p) {
            // plan step: view-0 taps, then the per-column CSR of (target, tap) entries
            UmbrellaSrc src0 = projector_cached_umbrella(p, p->bumb, r, p->bpad, 0, s);
            KBSet kb;
            kb.ax[0] = rax[2].kb;
            kb.ax[1] = rax[1].kb;
            kb.ax[2] = rax[0].kb;
            const int64_t n = x.per_view;
            DevBuf<RsTap<3>> taps((size_t)n);
            k_rs_taps<3><<<blocks_for(n, 256), 256, 0, s>>>(src0, kb, n, taps.p);
            CBN_LAUNCH_CHECK();
            // pole targets are spread per view (k_rs_pole_spread), not from the CSR
            std::vector<int> pole_f0;
            build_poles<3>(p->bumb, src0, n, taps.p, s);
            for (int q = 0; q < p->bumb.n_poles; ++q) {
                int t = 0;
                RsTap<3> tp;
                CBN_CUDA(cudaMemcpy(&t, p->bumb.poles.p + q, sizeof(int), cudaMemcpyDeviceToHost));
                CBN_CUDA(cudaMemcpy(&tp, taps.p + t, sizeof(tp), cudaMemcpyDeviceToHost));
                pole_f0.push_back(tp.f[0]);
            }
            const int64_t ncol = x.kd3[0] * x.kd3[1];
            DevBuf<int> counts((size_t)ncol);
            CBN_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int) * ncol, s));
            k_rs_col_count<3><<<blocks_for(n, 256), 256, 0, s>>>(taps.p, n, (int)x.kd3[0],
                                                                (int)x.kd3[1], counts.p);
            CBN_LAUNCH_CHECK();
            std::vector<int> h((size_t)ncol + 1, 0);
            CBN_CUDA(cudaMemcpyAsync(h.data() + 1, counts.p, sizeof(int) * ncol,
                                     cudaMemcpyDeviceToHost, s));
            CBN_CUDA(cudaStreamSynchronize(s));
            {
                // rho planes (cols rho * K_theta + theta) that hold any entry
                const int64_t kt = x.kd3[1];
                std::vector<unsigned char> used((size_t)x.kd3[0], 0);
                for (int f0 : pole_f0)    // the pole targets' rho planes
                    for (int a = 0; a < 3; ++a) used[(size_t)((f0 + a) % x.kd3[0])] = 1;
                p->bres_rho_runs.clear();
                for (int64_t rr = 0; rr < x.kd3[0]; ++rr) {
                    for (int64_t t = 0; t < kt && !used[(size_t)rr]; ++t)
                        used[(size_t)rr] = h[(size_t)(rr * kt + t) + 1] > 0;
                    if (!used[(size_t)rr]) continue;
                    if (!p->bres_rho_runs.empty() && p->bres_rho_runs.back().second == rr)
                        p->bres_rho_runs.back().second = (int)rr + 1;
                    else
                        p->bres_rho_runs.emplace_back((int)rr, (int)rr + 1);
                }
                p->bres_rho_used.upload(used.data(), used.size(), s);
            }
            std::partial_sum(h.begin(), h.end(), h.begin());
            p->bcol_ptr.upload(h.data(), h.size(), s);
            p->bcol_ent.alloc(sizeof(RsColEntry) * (size_t)std::max(h.back(), 1));
            p->bcol_n = h.back();
            CBN_CUDA(cudaMemcpyAsync(counts.p, h.data(), sizeof(int) * ncol, cudaMemcpyHostToDevice,
                                     s));
            k_rs_col_fill<3><<<blocks_for(n, 256), 256, 0, s>>>(
                taps.p, n, (int)x.kd3[0], (int)x.kd3[1], counts.p,
                reinterpret_cast<RsColEntry*>(p->bcol_ent.p));
            CBN_LAUNCH_CHECK();
            k_rs_col_sort<<<blocks_for(ncol, 128), 128, 0, s>>>(
                p->bcol_ptr.p, ncol, reinterpret_cast<RsColEntry*>(p->bcol_ent.p));
            CBN_LAUNCH_CHECK();
            if (rs_strips_on() && res_j3(rax)) bp_build_col_strips(p, x.kd3[0], x.kd3[1], s);
            CBN_CUDA(cudaStreamSynchronize(s));
        }
    }
    x.slow_axis = x.lanes ? 2 : 0;
    p->big.ensure((size_t)std::max(x.kres, x.k3));
    p->padded.ensure((size_t)2 * x.dsize);
    return x;
}

bool rho_lines_off_bp() {   // CBN_RHO_LINES=0: the strided rho pass (A/B)
    const char* e = std::getenv("CBN_RHO_LINES");
    return e && e[0] == '0';
}

// forward Grangeat of n views (frames: the first of them) into values
// ([view][n_mu][n_t]) or target-major outT columns k0 .. k0 + n - 1 of row
// length nb_total; blocks of 32 views alternate between the caller's stream
// and s1 when there are more than 32
void bp_grangeat_views(cbn_projector_s* p, const float* frames, int n, float* out, float* outT,
                       int nb_total, int k0, cudaStream_t s) {
    const int nu = p->g.nu, nv = p->g.nv;
    const int64_t per_view = (int64_t)p->bumb.n_mu * p->bumb.n_t;
    const bool dual = n > 32 && lanes_allowed() && !p->timer.on;
    if (dual) {
        // plan state both lanes read, then fork
        GrangeatPlan& gp = p->bgr;
        if (!gp.built) projector_fit_grangeat(p, gp, p->bumb, s);
        projector_prepare_gr_points(p, gp, p->bumb, false, s);
        // gp.pix is built lazily by the first block; build it before the
        // fork so lane 1's first pad kernel is ordered after it
        projector_gr_pix(p, gp, false, s);
        ensure_lane1(p);
        CBN_CUDA(cudaEventRecord(p->ev_s0, s));
        CBN_CUDA(cudaStreamWaitEvent(p->s1, p->ev_s0, 0));
    }
    for (int k = 0; k < n; k += 32) {
        const bool l1 = dual && ((k / 32) & 1);
        const cudaStream_t ls = l1 ? p->s1 : s;
        StageScope st(p->timer, "grangeat_forward", ls);
        const int m = std::min(32, n - k);
        grangeat_forward_block(p, frames + (size_t)k * nu * nv, m,
                               outT ? nullptr : out + (size_t)k * per_view, ls,
                               l1 ? lane_bufs(p) : main_bufs(p), outT, nb_total, k0 + k);
    }
    if (dual) {
        CBN_CUDA(cudaEventRecord(p->ev_s1, p->s1));
        CBN_CUDA(cudaStreamWaitEvent(s, p->ev_s1, 0));
    }
}

// transposed resample of views [lo, hi) accumulated into acc (dsize complex,
// zeroed here): the values of `frames` (views lo..hi-1), or -- den_only -- the
// validity mask of the same views (resample_transpose(valid), pipeline.py:184)
void bp_transpose(cbn_projector_s* p, const BpCtx& x, const float* frames, int lo, int hi,
                  float2* acc, bool den_only, cudaStream_t s) {
    const cbn_projector_config& c = p->c;
    const RadialTables& r = p->brad;
    const AxisPlan* rax = p->bres;
    BatchPlan& bp = p->bbatch;
    const int64_t per_view = x.per_view;
    const int nu = p->g.nu, nv = p->g.nv;
    CBN_CUDA(cudaMemsetAsync(acc, 0, sizeof(float2) * x.dsize, s));
    p->s32.ensure(3 * (size_t)std::max(bp.smax, p->n_vol));
    // out: [view][n_mu][n_t] values; or (outT) target-major [target][nb]
    auto forward_grangeat = [&](int v0, int nb, float* out, float* outT = nullptr) {
        bp_grangeat_views(p, frames + (size_t)(v0 - lo) * nu * nv, nb, out, outT, nb, 0, s);
    };
    // views-in-lanes: the transposed grid is real, [rho][theta][phi] (phi =
    // rax[0]), stored after its half spectrum [rho][theta][phi/2+1]
    const int64_t hphi = rax[0].K / 2 + 1;
    const int64_t half_sz = (int64_t)rax[2].K * rax[1].K * hphi;
    if (x.lanes) p->big.ensure((size_t)(half_sz + (x.kres + 1) / 2));
    float* greal = x.lanes ? reinterpret_cast<float*>(p->big.p + half_sz) : nullptr;
    float* gn = reinterpret_cast<float*>(p->big.p);    // the transposed grid (real parts)
    // one group of batches sharing a scaling: inverse FFT of the summed
    // spreads, crop * scaling, accumulate into acc
    auto flush = [&](int g) {
        size_t need = (size_t)rax[0].N + rax[1].N + rax[2].N;
        p->tab_idx.ensure(need);
        p->tab_sc.ensure(need);
        RemapAxis ax[3];
        size_t off = 0;
        for (int d = 0; d < 3; ++d) {
            build_table(kTabCropShift, rax[d].N, rax[d].K, bp.s32.p + ((size_t)g * 3 + d) * bp.smax,
                        p->tab_idx.p + off, p->tab_sc.p + off, s);
            ax[d] = RemapAxis{p->tab_idx.p + off, p->tab_sc.p + off, rax[d].N, x.sstr[d]};
            off += rax[d].N;
        }
        // theta cells the crop reads -- directly or as the mirror of a cell
        // past the phi half -- in runs, for the real-grid path's rho pass
        std::vector<std::pair<int, int>> bres_theta_runs;
        if (x.lanes) bres_theta_runs = pad_runs(rax[1].N, rax[1].K, true);
        // the crop reads only some slowest-axis planes: inverse-FFT just those in 2D
        if (p->bres_planes.empty() || p->bres_planes_slow != x.slow_axis) {
            size_t o = 0;
            for (int d = 0; d < x.slow_axis; ++d) o += rax[d].N;
            p->bres_planes = index_runs(p->tab_idx.p + o, rax[x.slow_axis].N, false, s);
            p->bres_planes_slow = x.slow_axis;
        }
        if (x.lanes) {
            // real grid: 2D R2C over the (theta, phi) planes, C2C along rho,
            // then the crop reads IFFT = conj(FFT) from the half spectrum
            {
                StageScope st(p->timer, "transpose_ifft", s);
                // 2D R2C only on the rho planes holding entries (the others'
                // half planes are zeroed)
                const long long k2[2] = {rax[1].K, rax[0].K};
                const long long hplane = (long long)rax[1].K * hphi;
                const long long rplane = (long long)rax[1].K * rax[0].K;
                // (the rho-lines extract reads unused planes as zero; the strided
                // pass needs them zeroed)
                const bool zero_unused = rho_lines_off_bp();
                int lo = 0;
                for (const auto& rn : p->bres_rho_runs) {
                    if (rn.first > lo && zero_unused)
                        CBN_CUDA(cudaMemsetAsync(p->big.p + lo * hplane, 0,
                                                 sizeof(float2) * hplane * (rn.first - lo), s));
                    p->fft.exec_r2c3(p->fft.get_r2c2(k2, rn.second - rn.first),
                                     greal + rn.first * rplane, p->big.p + rn.first * hplane, s);
                    lo = rn.second;
                }
                if (lo < rax[2].K && zero_unused)
                    CBN_CUDA(cudaMemsetAsync(p->big.p + lo * hplane, 0,
                                             sizeof(float2) * hplane * (rax[2].K - lo), s));
                if (!rho_lines_off_bp()) {
                    // the (theta, phi-half) columns the crop reads, as contiguous
                    // rho lines; forward FFT along rho; the crop reads the lines
                    if (!p->bres_lth.p) {
                        const std::vector<int> lth = pad_positions(rax[1].N, rax[1].K, true, false);
                        std::vector<char> onp((size_t)hphi, 0);
                        for (int k : pad_positions(rax[0].N, rax[0].K, false, false))
                            onp[(size_t)(k <= rax[0].K / 2 ? k : rax[0].K - k)] = 1;
                        std::vector<int> lph, thmap((size_t)rax[1].K, 0), phmap((size_t)hphi, 0);
                        for (int k = 0; k < (int)hphi; ++k)
                            if (onp[(size_t)k]) {
                                phmap[(size_t)k] = (int)lph.size();
                                lph.push_back(k);
                            }
                        for (size_t q = 0; q < lth.size(); ++q) thmap[(size_t)lth[q]] = (int)q;
                        p->bres_nth = (int)lth.size();
                        p->bres_nph = (int)lph.size();
                        p->bres_lth.upload(lth.data(), lth.size(), s);
                        p->bres_lph.upload(lph.data(), lph.size(), s);
                        p->bres_thmap.upload(thmap.data(), thmap.size(), s);
                        p->bres_phmap.upload(phmap.data(), phmap.size(), s);
                        CBN_CUDA(cudaStreamSynchronize(s));
                    }
                    const int Kr = rax[2].K;
                    const int64_t nlines = (int64_t)p->bres_nth * p->bres_nph;
                    p->brlines.ensure((size_t)nlines * Kr);
                    k_lines_from_half<<<dim3((unsigned)((Kr + 31) / 32),
                                             (unsigned)((p->bres_nph + 31) / 32), p->bres_nth),
                                        dim3(32, 8), 0, s>>>(
                        p->big.p, p->bres_rho_used.p, p->bres_lth.p, p->bres_lph.p, p->bres_nth,
                        p->bres_nph, Kr, rax[1].K, (int)hphi, p->brlines.p);
                    CBN_LAUNCH_CHECK();
                    long long kr1[1] = {Kr};
                    p->fft.exec(p->fft.get(1, kr1, nlines), p->brlines.p, p->brlines.p,
                                CUFFT_FORWARD, s);
                } else {
                    // along rho only the theta columns the crop reads (the crop
                    // table's distinct theta cells, in runs)
                    const long long plane = (long long)rax[1].K * hphi;
                    for (const auto& rn : bres_theta_runs) {
                        float2* at = p->big.p + (size_t)rn.first * hphi;
                        p->fft.exec(p->fft.get_strided(rax[2].K,
                                                       (long long)(rn.second - rn.first) * hphi,
                                                       plane, 1),
                                    at, at, CUFFT_FORWARD, s);
                    }
                }
            }
            StageScope st(p->timer, "transpose_crop", s);
            if (!rho_lines_off_bp()) {
                k_crop_from_lines<<<dim3((unsigned)((ax[2].n + 255) / 256), ax[1].n, ax[0].n), 256, 0,
                                    s>>>(p->brlines.p, ax[0], ax[1], ax[2], p->bres_thmap.p,
                                         p->bres_phmap.p, p->bres_nth, rax[0].K, rax[1].K,
                                         rax[2].K, acc);
                CBN_LAUNCH_CHECK();
                return;
            }
            ax[0].sstride = 1;
            ax[1].sstride = hphi;
            ax[2].sstride = (int64_t)rax[1].K * hphi;
            dim3 grid((ax[2].n + 31) / 32, (ax[0].n + 31) / 32, ax[1].n);
            k_remap_half_acc_tile<<<grid, dim3(32, 8), 0, s>>>(p->big.p, acc, ax[0], ax[1], ax[2],
                                                             rax[0].K, rax[1].K, rax[2].K);
            CBN_LAUNCH_CHECK();
            return;
        }
        {
            StageScope st(p->timer, "transpose_ifft", s);
            fft3_pruned(p->fft, p->big.p, x.kd3, 1, p->bres_planes, CUFFT_INVERSE, s);
        }
        StageScope st(p->timer, "transpose_crop", s);
        launch_remap<float2, kAccumC>(3, p->big.p, acc, ax, 1.0f, s);
        CBN_LAUNCH_CHECK();
        if (!x.lanes) CBN_CUDA(cudaMemsetAsync(p->big.p, 0, sizeof(float2) * x.kres, s));
    };

    if (x.method_b) {
        // method B (resampling.py:176-189): views in blocks of 32, forward
        // Grangeat, then the conjugate periodic-sinc spread straight into acc
        p->values.ensure((size_t)per_view * 32);
        const DirGrid dg{{x.dr, r.n_theta, r.n_phi}, {1, (int64_t)x.dr, (int64_t)r.n_theta * x.dr}};
        for (int v0 = lo; v0 < hi; v0 += 32) {
            const int nb = std::min(32, hi - v0);
            if (!den_only) forward_grangeat(v0, nb, p->values.p);
            UmbrellaSrc src = projector_cached_umbrella(p, p->bumb, r, p->bpad, v0, s);
            StageScope st(p->timer, "transpose_spread", s);
            const int64_t mb = per_view * nb;
            dispatch_taps(c.side_lobes + 1, [&](auto tc) {
                k_dir_spread<decltype(tc)::value><<<blocks_for(mb, 256), 256, 0, s>>>(
                    den_only ? nullptr : acc, den_only ? acc : nullptr, dg, src, mb, nullptr,
                    den_only ? nullptr : p->values.p);
                return 0;
            });
            CBN_LAUNCH_CHECK();
        }
        return;
    }
    if (x.lanes) {
        // runs of consecutive batches sharing a scaling group, clipped to
        // [lo, hi): forward Grangeat, target-major transpose, column gather
        const size_t nbat = bp.batches.size();
        size_t bi = 0;
        while (bi < nbat) {
            const int g = bp.group[bi];
            size_t e = bi + 1;
            while (e < nbat && bp.group[e] == g) ++e;
            const int vlo = std::max(lo, bp.batches[bi].first);
            const int vhi = std::min(hi, bp.batches[e - 1].second);
            bi = e;
            if (vlo >= vhi) continue;
            const int nvr = vhi - vlo;
            if (!den_only) {
                // the Grangeat post writes the values target-major for the
                // column gather (no separate transpose); a staged call
                // (cbn_backproject_stage_views) has done it view block by
                // view block while the frames were still being uploaded
                if (!(p->bp_staged == p->g.n_views && vlo == 0 && vhi == p->g.n_views)) {
                    p->values_t.ensure((size_t)per_view * nvr);
                    forward_grangeat(vlo, nvr, nullptr, p->values_t.p);
                }
            }
            {
                StageScope st(p->timer, "transpose_spread", s);
                const unsigned ncol = (unsigned)(x.kd3[0] * x.kd3[1]);
                {
                    // values (once), column entries (once), the real grid of
                    // the used rho planes written once; on chip: entries x
                    // views (two value loads + weights per entry per cell pair)
                    double planes = 0;
                    for (const auto& rn : p->bres_rho_runs) planes += rn.second - rn.first;
                    const bool strips = x.shift == 2 && rs_strips_on() && p->bstrip_ptr.p;
                    const double ents = strips ? 40.0 * p->bstrip_n
                                               : (double)sizeof(RsColEntry) * p->bcol_n;
                    p->timer.add_bytes("transpose_spread",
                                       (den_only ? 0.0 : 4.0 * per_view * nvr) + ents +
                                           4.0 * planes * x.kd3[1] * x.kd3[2],
                                       ents * (x.kd3[2] / 2));
                }
                const RsColEntry* ent = reinterpret_cast<const RsColEntry*>(p->bcol_ent.p);
                float* gnum = den_only ? nullptr : greal;
                float* gden = den_only ? greal : nullptr;
                const float* vt = den_only ? nullptr : p->values_t.p;
                if (x.shift == 2 && rs_strips_on() && p->bstrip_ptr.p) {
                    const unsigned char* used = p->bres_rho_used.p;
                    const int kt = (int)x.kd3[1];
                    const unsigned nst = (unsigned)(x.kd3[0] * p->bstrip_nsx);
                    const RsStripEnt* se = reinterpret_cast<const RsStripEnt*>(p->bstrip_ent.p);
                    if (den_only)
                        k_rs_gather_strips<true><<<nst, kRsPairThreads, 0, s>>>(
                            gnum, gden, p->g.n_views, p->bstrip_ptr.p, se, p->bstrip_w2.p,
                            p->bstrip_wab.p, vt, vlo, nvr, used, kt, p->bstrip_nsx);
                    else
                        k_rs_gather_strips<false><<<nst, kRsPairThreads, 0, s>>>(
                            gnum, gden, p->g.n_views, p->bstrip_ptr.p, se, p->bstrip_w2.p,
                            p->bstrip_wab.p, vt, vlo, nvr, used, kt, p->bstrip_nsx);
                } else if (x.shift == 2) {
                    const unsigned char* used = p->bres_rho_used.p;
                    const int kt = (int)x.kd3[1];
                    if (den_only)
                        k_rs_gather_cols2<true><<<ncol, kRsPairThreads, 0, s>>>(
                            gnum, gden, p->g.n_views, p->bcol_ptr.p, ent, vt, vlo, nvr, used, kt);
                    else
                        k_rs_gather_cols2<false><<<ncol, kRsPairThreads, 0, s>>>(
                            gnum, gden, p->g.n_views, p->bcol_ptr.p, ent, vt, vlo, nvr, used, kt);
                } else {
                    k_rs_gather_cols<<<ncol, kRsColThreads, 0, s>>>(
                        gnum, gden, (int)x.kd3[2], p->bcol_ptr.p, ent, vt, vlo, nvr, x.shift);
                }
                CBN_LAUNCH_CHECK();
                if (p->bumb.n_poles) {
                    // pole targets per view, after the column gather's stores
                    UmbrellaSrc src = projector_cached_umbrella(p, p->bumb, r, p->bpad, vlo, s);
                    KBSet kb;   // grid order (rho, theta, phi)
                    kb.ax[0] = rax[2].kb;
                    kb.ax[1] = rax[1].kb;
                    kb.ax[2] = rax[0].kb;
                    const int nq = p->bumb.n_poles * nvr;
                    k_rs_pole_spread<3><<<blocks_for(nq, 128), 128, 0, s>>>(
                        greal, kb, src, p->bumb.poles.p, p->bumb.n_poles, per_view, nvr, vt);
                    CBN_LAUNCH_CHECK();
                }
            }
            flush(g);
        }
        return;
    }
    // atomic scatter per batch (clipped to [lo, hi)), flushed per scaling group
    CBN_CUDA(cudaMemsetAsync(p->big.p, 0, sizeof(float2) * x.kres, s));
    int cur = -1;
    for (size_t bi = 0; bi < bp.batches.size(); ++bi) {
        const int bl = std::max(lo, bp.batches[bi].first);
        const int bh = std::min(hi, bp.batches[bi].second);
        if (bl >= bh) continue;
        const int g = bp.group[bi];
        if (cur >= 0 && g != cur) flush(cur);
        cur = g;
        const int nbv = bh - bl;
        const int64_t mb = per_view * nbv;
        if (!den_only) {
            p->values.ensure((size_t)mb);
            forward_grangeat(bl, nbv, p->values.p);
        }
        UmbrellaSrc src = projector_cached_umbrella(p, p->bumb, r, p->bpad, bl, s);
        StageScope st_sp(p->timer, "transpose_spread", s);
        dispatch_j(res_jmax(rax), [&](auto jc) {
            constexpr int J = decltype(jc)::value;
            k_rs_spread2<J><<<blocks_for(mb, 256), 256, 0, s>>>(
                den_only ? nullptr : gn, den_only ? gn : nullptr, x.kbr, src,
                den_only ? nullptr : p->values.p, mb);
            return 0;
        });
        CBN_LAUNCH_CHECK();
    }
    if (cur >= 0) flush(cur);
}

// lattice-domain inverse of a transposed accumulator: ifftn (method A, incl.
// 1/size) in place; returns the scale the origin mean / division use
double bp_lattice_ifft(cbn_projector_s* p, const BpCtx& x, float2* acc, cudaStream_t s) {
    const RadialTables& r = p->brad;
    long long dd[3] = {r.n_phi, r.n_theta, x.dr};
    // method A ends in ifftn (incl. 1 / size); method B's spread is the result
    if (!x.method_b) p->fft.exec(p->fft.get(3, dd, 1), acc, acc, CUFFT_INVERSE, s);
    return x.method_b ? 1.0 : 1.0 / (double)x.dsize;
}

// den (the transposed validity mask over every view) depends on the geometry
// only: computed once per plan and cached in lattice node order
void bp_den(cbn_projector_s* p, const BpCtx& x, cudaStream_t s) {
    if (p->den_cached) return;
    const RadialTables& r = p->brad;
    float2* acc_den = p->padded.p + x.dsize;
    bp_transpose(p, x, nullptr, 0, p->g.n_views, acc_den, true, s);
    const double inv = bp_lattice_ifft(p, x, acc_den, s);
    p->red.ensure(2 * kRed + 64);
    double* means = p->red.p + 2 * kRed;
    projector_column_mean(acc_den, r.lines(), x.dr, p->bpad + r.n_rho / 2, inv, p->red.p,
                          means + 2, s);
    const int64_t M = r.nodes();
    p->den_cache.alloc((size_t)M);
    p->den_max.alloc(1);
    k_den_final<<<blocks_for(M, 256), 256, 0, s>>>(acc_den, r.lines(), x.dr, p->bpad, r.n_rho, inv,
                                                    means + 2, p->den_cache.p);
    CBN_LAUNCH_CHECK();
    k_max_partial<<<kRed, 256, 0, s>>>(p->den_cache.p, M, p->red.p);
    CBN_LAUNCH_CHECK();
    k_max_final<<<1, 32, 0, s>>>(p->red.p, kRed, p->den_max.p);
    CBN_LAUNCH_CHECK();
    p->den_keep.release();
    if (x.lanes && p->bbatch.groups() == 1 && r.n_phi % p->g.n_views == 0 && !den_orbit_off()) {
        const int sft = r.n_phi / p->g.n_views;
        const int64_t orbits = (int64_t)r.n_rho * r.n_theta * sft;
        p->den_keep.alloc((size_t)M);
        k_den_keep_orbit<<<blocks_for(orbits, 256), 256, 0, s>>>(p->den_cache.p, r.n_rho, r.n_theta,
                                                                 r.n_phi, sft, p->den_max.p,
                                                                 p->c.den_tol, p->den_keep.p);
        CBN_LAUNCH_CHECK();
    }
    p->den_cached = true;
}

// num (values) / den (mask) of nufft_backproject for a view range, after the
// lattice-domain inverse FFT, rho crop and origin average: the sum over the
// range's batches of resample_transpose (resampling.py:164-196,
// pipeline.py:183-184), complex64 / float32 in node order [phi][theta][rho]
__global__ void k_num_final(const float2* __restrict__ acc, int64_t lines, int dr, int pad, int n,
                            double inv, const double* __restrict__ means, float2* __restrict__ num,
                            float* __restrict__ re) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= lines * n) return;
    const int j = (int)(e % n);
    const int64_t line = e / n;
    float2 v;
    if (j == n / 2) {
        v = make_float2((float)means[0], (float)means[1]);
    } else {
        const float2 a = acc[line * dr + pad + j];
        v = make_float2((float)((double)a.x * inv), (float)((double)a.y * inv));
    }
    if (num) num[e] = v;
    if (re) re[e] = v.x;
}

void bp_stage_transpose(cbn_projector_s* p, const float* frames, int lo, int hi, float2* num,
                        float* den, cudaStream_t s) {
    BpCtx x = bp_context(p, s);
    const RadialTables& r = p->brad;
    DevBuf<float2> acc((size_t)x.dsize);
    p->red.ensure(2 * kRed + 64);
    double* means = p->red.p + 2 * kRed;
    const int64_t M = r.nodes();
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 0 && !num) continue;
        if (pass == 1 && !den) continue;
        bp_transpose(p, x, frames, lo, hi, acc.p, pass == 1, s);
        const double inv = bp_lattice_ifft(p, x, acc.p, s);
        projector_column_mean(acc.p, r.lines(), x.dr, p->bpad + r.n_rho / 2, inv, p->red.p, means,
                              s);
        k_num_final<<<blocks_for(M, 256), 256, 0, s>>>(acc.p, r.lines(), x.dr, p->bpad, r.n_rho,
                                                        inv, means, pass == 0 ? num : nullptr,
                                                        pass == 1 ? den : nullptr);
        CBN_LAUNCH_CHECK();
    }
    CBN_CUDA(cudaStreamSynchronize(s));
}

// phase 1
void bp_views(cbn_projector_s* p, const float* frames, int lo, int hi, float2* acc,
              cudaStream_t s) {
    BpCtx x = bp_context(p, s);
    bp_den(p, x, s);
    bp_transpose(p, x, frames, lo, hi, acc, false, s);
}

// phase 2: acc (the summed accumulator) is consumed in place
void bp_finish(cbn_projector_s* p, float2* acc, int part, int nparts, float2* grid,
               cudaStream_t s) {
    BpCtx x = bp_context(p, s);
    bp_den(p, x, s);
    const cbn_projector_config& c = p->c;
    const RadialTables& r = p->brad;
    if (p->timer.on) p->timer.begin("bp_lattice", s);
    const double inv = bp_lattice_ifft(p, x, acc, s);
    p->red.ensure(2 * kRed + 64);
    double* means = p->red.p + 2 * kRed;        // num re, num im
    projector_column_mean(acc, r.lines(), x.dr, p->bpad + r.n_rho / 2, inv, p->red.p, means, s);
    const int64_t M = r.nodes();
    p->lattice.ensure((size_t)M);
    k_bp_div<<<blocks_for(M, 256), 256, 0, s>>>(acc, p->den_cache.p, r.lines(), x.dr, p->bpad,
                                                 r.n_rho, inv, means, p->den_max.p, c.den_tol,
                                                 p->den_keep.p, p->lattice.p);
    CBN_LAUNCH_CHECK();
    long long nr1[1] = {r.n_rho};
    p->fft.exec(p->fft.get(1, nr1, r.lines()), p->lattice.p, p->lattice.p, CUFFT_FORWARD, s);
    if (p->timer.on) p->timer.end(s);
    // ---- 3D type-1 NUFFT onto (2N)^3 (nufft_adjoint_chunked, nufft.py:268-282)
    const AxisPlan* sax = p->bspec;
    const int n = p->n_vol;
    KBSet kbs;
    for (int d = 0; d < 3; ++d) kbs.ax[d] = sax[d].kb;
    if (!p->bspec_fit) {
        // scaling of the first sub-plan, cached with the sorted node order
        int nrows;
        const int64_t* rows = projector_rows(p, projector_chunk(p, M), nrows);
        p->bspec_s32.alloc(3 * (size_t)n);
        ls_fit<3>(r.src(), rows, nrows, sax, p->ls, p->bspec_s32.p, n, s);
        // one node per +-rho pair (exact mirrors only), then bins over them
        const int64_t base_n = r.lines() * (r.n_rho / 2 + 1);
        p->bpairs.alloc((size_t)base_n + (size_t)r.lines() * (r.n_rho / 2));
        DevBuf<int> extra(1);
        CBN_CUDA(cudaMemsetAsync(extra.p, 0, sizeof(int), s));
        k_radial_pairs<<<blocks_for(base_n, 256), 256, 0, s>>>(r.src(), kbs, sax[0].J, r.lines(),
                                                               p->bpairs.p, extra.p, base_n);
        CBN_LAUNCH_CHECK();
        int h_extra = 0;
        CBN_CUDA(cudaMemcpyAsync(&h_extra, extra.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CBN_CUDA(cudaStreamSynchronize(s));
        p->bpairs_n = base_n + h_extra;
        const RadialPairSrc psrc{r.src(), p->bpairs.p};
        // 8 x 4 x 16 tiles: a 13 x 9 x 22 region (25 KB) lets 8 CTAs share an
        // SM (8 x 8 x 16: 6); measured 3.25 -> 3.12 ms at config 2
        int tile[3] = {kTile3, kTile3 / 2, kTile3Fast};
        if (const char* e = std::getenv("CBN_BP_TILE"))   // "t0,t1,t2" (tuning A/B)
            std::sscanf(e, "%d,%d,%d", &tile[0], &tile[1], &tile[2]);
        dispatch_j(sax[0].J, [&](auto jc) {
            build_bins<3, decltype(jc)::value>(p->bspec_bins, psrc, kbs, p->bpairs_n, tile, kMaxSub,
                                               s, true);
            return 0;
        });
        k_gather_index<<<blocks_for(p->bpairs_n, 256), 256, 0, s>>>(p->bpairs.p, p->bpairs_n,
                                                                   p->bspec_bins.perm.p);
        CBN_LAUNCH_CHECK();
        p->bspec_fit = true;
    }
    if (!p->ramp_q.p) {
        // ramp filter weights (pipeline.py:190-200), per rho bin incl. d_rho
        std::vector<float> q(r.n_rho);
        const double c3 = 1.0 / (4.0 * r.n_theta * r.n_phi * r.n_rho * r.d_rho);
        const double corner = kPi * std::sqrt(3.0) / p->voxel;
        for (int k = 0; k < r.n_rho; ++k) {
            double om = (kTwoPi * (double)(k - r.n_rho / 2)) / ((double)r.n_rho * r.d_rho);
            double ap = std::cos(kPi * std::min(std::fabs(om) / corner, 1.0) / 2.0);
            q[k] = (float)(om * ap * ap * c3 * r.d_rho);
        }
        p->ramp_q.upload(q.data(), q.size(), s);
        CBN_CUDA(cudaStreamSynchronize(s));
    }
    BpPairSrc bsrc;
    static_cast<RadialSrc&>(bsrc) = r.src();
    bsrc.X = p->lattice.p;
    bsrc.q = p->ramp_q.p;
    bsrc.sin_th = r.sin_theta.p;
    for (int d = 0; d < 3; ++d) bsrc.N[d] = n;
    bsrc.tri = c.basis == 0;
    StageScope st_sp(p->timer, "bp_spread", s);
    CBN_CUDA(cudaMemsetAsync(grid, 0, sizeof(float2) * x.k3, s));
    {
        // lattice read once, the (2N)^3 grid written once (this part's share);
        // on chip: J^3 shared-memory read + write per primary node
        const double f = (double)1.0 / nparts;
        const double J = sax[0].J;
        // + the 40-byte point records of the record-driven spread
        const double rec = bp_records_off() ? 0.0 : 40.0 * p->bpairs_n;
        p->timer.add_bytes("bp_spread", f * (8.0 * M + rec) + 8.0 * x.k3,
                           f * 16.0 * J * J * J * p->bpairs_n);
    }
    // this part's share of the bin subproblems (each node belongs to one)
    const BinPlan& bb = p->bspec_bins;
    const int s0 = (int)((int64_t)bb.nsubs * part / nparts);
    const int s1 = (int)((int64_t)bb.nsubs * (part + 1) / nparts);
    if (!bp_records_off()) {
        if (!p->bspec_rec.p) {
            const int64_t m = p->bpairs_n;
            p->bspec_rec.alloc((size_t)m);
            p->bspec_g.alloc((size_t)m);
            p->bspec_idx.alloc((size_t)m);
            dispatch_j(sax[0].J, [&](auto jc) {
                k_bp_records<decltype(jc)::value><<<blocks_for(m, 256), 256, 0, s>>>(
                    bsrc, kbs, bb.geom<3>(), bb.perm.p, m, p->bspec_rec.p, p->bspec_g.p,
                    p->bspec_idx.p);
                return 0;
            });
            CBN_LAUNCH_CHECK();
        }
        const float2* vals = nullptr;
        if (bp_values_pass_on()) {
            // the part's subproblems cover sorted positions [sub s0 start, sub s1 end)
            p->bspec_vals.ensure((size_t)p->bpairs_n);
            k_bp_values<<<blocks_for(p->bpairs_n, 256), 256, 0, s>>>(
                p->bspec_g.p, p->bspec_idx.p, p->lattice.p, p->bpairs_n, p->bspec_vals.p);
            CBN_LAUNCH_CHECK();
            vals = p->bspec_vals.p;
        }
        const BpRecSrc rsrc{p->bspec_rec.p, p->bspec_g.p, p->bspec_idx.p, p->lattice.p, vals};
        dispatch_j(sax[0].J, [&](auto jc) {
            launch_spread3<decltype(jc)::value>(grid, kbs, bb, rsrc, s, s0, s1);
            return 0;
        });
        return;
    }
    dispatch_j(sax[0].J, [&](auto jc) {
        launch_spread3<decltype(jc)::value>(grid, kbs, bb, bsrc, s, s0, s1);
        return 0;
    });
}

namespace {

// y/z crop + deapodisation of the 2D-transformed slab planes, written in the
// all-to-all send layout [y block d][x][y - y0_d][z] (blocks: the balanced
// split y0_d = d * ny / nparts), so each destination's chunk is contiguous and
// the received chunks, concatenated in source-rank order, are [x][y][z].
__global__ void k_crop_slab_yz(const float2* __restrict__ src, float2* __restrict__ dst,
                               RemapAxis ay, RemapAxis az, int xc, int64_t plane, int nparts) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int ny = ay.n, nz = az.n;
    if (q >= (int64_t)xc * ny * nz) return;
    const int z = (int)(q % nz);
    const int y = (int)((q / nz) % ny);
    const int x = (int)(q / ((int64_t)nz * ny));
    const int d = (int)(((int64_t)(y + 1) * nparts - 1) / ny);
    const int y0 = (int)((int64_t)d * ny / nparts), y1 = (int)((int64_t)(d + 1) * ny / nparts);
    const float sc = ay.scale[y] * az.scale[z];
    const float2 g = src[(int64_t)x * plane + (int64_t)ay.idx[y] * ay.sstride + az.idx[z]];
    dst[(int64_t)xc * y0 * nz + ((int64_t)x * (y1 - y0) + (y - y0)) * nz + z] =
        make_float2(g.x * sc, g.y * sc);
}

// x crop + deapodisation + Re of the x-transformed columns [K0][yc][nz]
__global__ void k_crop_cols_x(const float2* __restrict__ src, float* __restrict__ dst,
                              RemapAxis ax, int64_t row, float gain) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (int64_t)ax.n * row) return;
    const int x = (int)(q / row);
    const int64_t r = q % row;
    dst[q] = gain * ax.scale[x] * src[(int64_t)ax.idx[x] * row + r].x;
}

// Hermitian part of the spread grid on the z half: H[k] = (G[k] + conj G[-k]) / 2
// over [K0][K1][K2/2+1].  Re(IFFT(G)) -- all the crop keeps (pipeline.py:212)
// -- is the complex-to-real inverse FFT of H.
__global__ void k_herm_half3(const float2* __restrict__ g, float2* __restrict__ h, int K0, int K1,
                             int K2) {
    const int hz = K2 / 2 + 1;
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= hz) return;
    const int y = blockIdx.y, x = blockIdx.z;
    const int xm = x ? K0 - x : 0, ym = y ? K1 - y : 0, zm = z ? K2 - z : 0;
    const float2 a = g[((size_t)x * K1 + y) * K2 + z];
    const float2 b = g[((size_t)xm * K1 + ym) * K2 + zm];
    h[((size_t)x * K1 + y) * hz + z] = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
}

void crop_tables(cbn_projector_s* p, RemapAxis* cax, cudaStream_t s) {
    const AxisPlan* sax = p->bspec;
    const int n = p->n_vol;
    const int64_t cstr[3] = {(int64_t)sax[1].K * sax[2].K, sax[2].K, 1};
    p->s32.ensure(3 * (size_t)n);
    CBN_CUDA(cudaMemcpyAsync(p->s32.p, p->bspec_s32.p, sizeof(float) * 3 * n,
                             cudaMemcpyDeviceToDevice, s));
    projector_build_tables(p, kTabCrop, sax, n, s, cax, cstr);
}

}  // namespace

// phase 3: grid (the summed spread) is consumed in place.  Inverse 3D FFT
// pruned to the x planes the crop reads (1D along x, then 2D on N of 2N planes).
void bp_crop(cbn_projector_s* p, float2* grid, float* vol, cudaStream_t s) {
    build_backward_plan(p, s);
    CBN_REQUIRE(p->bspec_fit, "bp_crop before bp_finish");
    const AxisPlan* sax = p->bspec;
    StageScope st_ff(p->timer, "bp_ifft_crop", s);
    // Hermitian half on z, inverse C2C along x, then batched 2D C2R of only
    // the x planes the crop reads, into the (consumed) grid's memory as floats
    const int K0 = sax[0].K, K1 = sax[1].K, K2 = sax[2].K;
    const long long hz = K2 / 2 + 1, hplane = (long long)K1 * hz, rplane = (long long)K1 * K2;
    p->bp_half.ensure((size_t)K0 * hplane);
    float2* h = p->bp_half.p;
    k_herm_half3<<<dim3((unsigned)((hz + 255) / 256), K1, K0), 256, 0, s>>>(grid, h, K0, K1, K2);
    CBN_LAUNCH_CHECK();
    p->fft.exec(p->fft.get_strided(K0, hplane, hplane, 1), h, h, CUFFT_INVERSE, s);
    float* re = reinterpret_cast<float*>(grid);
    const long long k2[2] = {K1, K2};
    for (const auto& rn : pad_runs(sax[0].N, K0, false))
        p->fft.exec_c2r(p->fft.get_c2r2(k2, rn.second - rn.first), h + rn.first * hplane,
                        re + rn.first * rplane, s);
    RemapAxis cax[3];
    crop_tables(p, cax, s);
    launch_remap<float, kStoreRe>(3, re, vol, cax, (float)p->c.bp_normalization, s);
    CBN_LAUNCH_CHECK();
}

// phase 3 distributed by slabs of the slowest grid axis (SURVEY.md 8(e),
// adjoint steps 4-6).  slab: planes [x_lo, x_hi) of the summed grid (consumed);
// send: (x_hi - x_lo) * N * N complex in the all-to-all layout above.
void bp_crop_slab(cbn_projector_s* p, float2* slab, int x_lo, int x_hi, int nparts, float2* send,
                  cudaStream_t s) {
    build_backward_plan(p, s);
    CBN_REQUIRE(p->bspec_fit, "bp_crop_slab before bp_finish");
    const AxisPlan* sax = p->bspec;
    CBN_REQUIRE(0 <= x_lo && x_lo < x_hi && x_hi <= sax[0].K, "slab out of range");
    CBN_REQUIRE(nparts >= 1 && nparts <= sax[1].N, "bad part count");
    StageScope st_ff(p->timer, "bp_ifft_crop", s);
    const int xc = x_hi - x_lo;
    const long long k2[2] = {sax[1].K, sax[2].K};
    p->fft.exec(p->fft.get(2, k2, xc), slab, slab, CUFFT_INVERSE, s);
    RemapAxis cax[3];
    crop_tables(p, cax, s);
    const int64_t cells = (int64_t)xc * cax[1].n * cax[2].n;
    k_crop_slab_yz<<<blocks_for(cells, 256), 256, 0, s>>>(slab, send, cax[1], cax[2], xc,
                                                         (int64_t)sax[1].K * sax[2].K, nparts);
    CBN_LAUNCH_CHECK();
}

// cols: [2N][y_hi - y_lo][N] complex (the chunks received from every slab,
// consumed); vol_part: [N][y_hi - y_lo][N] float32 (the volume's y range).
void bp_crop_cols(cbn_projector_s* p, float2* cols, int y_lo, int y_hi, float* vol_part,
                  cudaStream_t s) {
    build_backward_plan(p, s);
    CBN_REQUIRE(p->bspec_fit, "bp_crop_cols before bp_finish");
    const AxisPlan* sax = p->bspec;
    CBN_REQUIRE(0 <= y_lo && y_lo < y_hi && y_hi <= sax[1].N, "y range out of bounds");
    StageScope st_ff(p->timer, "bp_ifft_crop", s);
    const int64_t row = (int64_t)(y_hi - y_lo) * sax[2].N;
    p->fft.exec(p->fft.get_strided(sax[0].K, row, row, 1), cols, cols, CUFFT_INVERSE, s);
    RemapAxis cax[3];
    crop_tables(p, cax, s);
    k_crop_cols_x<<<blocks_for((int64_t)cax[0].n * row, 256), 256, 0, s>>>(
        cols, vol_part, cax[0], row, (float)p->c.bp_normalization);
    CBN_LAUNCH_CHECK();
}

// the backprojector's transposed-resample path: views in lanes (column gather)
bool bp_uses_lanes(cbn_projector_s* p, cudaStream_t s) { return bp_context(p, s).lanes; }

void backproject_impl(cbn_projector_s* p, const float* frames, float* vol, cudaStream_t s) {
    BpCtx x = bp_context(p, s);
    struct Reset {   // a staged run is consumed (or abandoned) by this call
        cbn_projector_s* p;
        ~Reset() { p->bp_staged = 0; }
    } reset{p};
    bp_views(p, frames, 0, p->g.n_views, p->padded.p, s);
    bp_finish(p, p->padded.p, 0, 1, p->big.p, s);
    bp_crop(p, p->big.p, vol, s);
    (void)x;
}

// forward Grangeat of views [lo, hi) ahead of cbn_backproject (views-in-lanes
// path with one scaling group: the target-major values of every view feed one
// column gather); views must arrive in order, lo = the views staged so far
int bp_stage_views(cbn_projector_s* p, const float* frames, int lo, int hi, cudaStream_t s) {
    BpCtx x = bp_context(p, s);
    const BatchPlan& bp = p->bbatch;
    const bool one_group = !bp.group.empty() && bp.groups() == 1 && bp.batches.front().first == 0 &&
                           bp.batches.back().second == p->g.n_views;
    if (!x.lanes || x.method_b || !one_group) return CBN_EUNSUPPORTED;
    CBN_REQUIRE(lo == p->bp_staged, "staged views must arrive in order");
    CBN_REQUIRE(lo % 32 == 0 || hi == p->g.n_views, "staged view blocks must start on 32-view bounds");
    bp_den(p, x, s);   // geometry only; computed before the first view
    const int64_t per_view = (int64_t)p->bumb.n_mu * p->bumb.n_t;
    p->values_t.ensure((size_t)per_view * p->g.n_views);
    bp_grangeat_views(p, frames, hi - lo, nullptr, p->values_t.p, p->g.n_views, lo, s);
    p->bp_staged = hi;
    return CBN_OK;
}

void bp_sizes(cbn_projector_s* p, int64_t* lattice, int64_t* grid, cudaStream_t s) {
    BpCtx x = bp_context(p, s);
    *lattice = x.dsize;
    *grid = x.k3;
}

}  // namespace cbn

extern "C" int cbn_backproject_stage_transpose(cbn_projector* p, const float* frames, int32_t lo,
                                               int32_t hi, void* num, float* den, void* stream) {
    try {
        CBN_REQUIRE(p && frames && (num || den), "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        cbn::bp_stage_transpose(p, frames, lo, hi, static_cast<float2*>(num), den,
                                static_cast<cudaStream_t>(stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return cbn::fail(e);
    }
}

extern "C" int cbn_backproject_stage_views(cbn_projector* p, const float* frames, int32_t lo,
                                           int32_t hi, void* stream) {
    try {
        CBN_REQUIRE(p && frames, "null argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        CBN_REQUIRE(0 <= lo && lo < hi && hi <= p->g.n_views, "view range out of bounds");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        cbn::build_backward_plan(p, s);
        return cbn::bp_stage_views(p, frames, lo, hi, s);
    } catch (const std::exception& e) {
        p->bp_staged = 0;
        return cbn::fail(e);
    }
}

extern "C" int cbn_projector_grangeat_forward(cbn_projector* p, const float* frames, float* values,
                                              int32_t nb, void* stream) {
    using namespace cbn;
    try {
        CBN_REQUIRE(p && frames && values && nb >= 1, "bad argument");
        CBN_REQUIRE(p->direction & 2, "projector was not created for the back direction");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        build_backward_plan(p, s);
        const int64_t per_view = (int64_t)p->bumb.n_mu * p->bumb.n_t;
        for (int v0 = 0; v0 < nb; v0 += 32) {
            const int k = std::min(32, nb - v0);
            grangeat_forward_block(p, frames + (size_t)v0 * p->g.nu * p->g.nv, k,
                                   values + (size_t)v0 * per_view, s);
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
