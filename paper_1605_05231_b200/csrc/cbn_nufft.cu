// Generic NUFFT plan over explicit nodes: the device replacement of
// plan_nufft / nufft_forward / nufft_adjoint (nufft.py:137-247).
//
// Plan state is O(m*d) nodes (wrapped float64, or the caller's float32 values
// wrapped on the fly in float64), per-axis scalings, remap tables and -- for
// 2D/3D -- the bin-sorted node order with its subproblem list; interpolation
// weights are recomputed inside the gather/spread kernels instead of being
// stored (the reference stores J^d per node).
#include <cstring>
#include <string>
#include <vector>

#include "cbn_binned.cuh"
#include "cbn_plan.h"

namespace cbn {

template <int D>
struct ExplicitSrc {
    const double* nodes64;  // wrapped, m x D (or null)
    const float* nodes32;   // caller's float32 values, m x D, wrapped here (or null)
    const float* sorted32 = nullptr;   // nodes32 in the plan's bin order (or null)
    struct Aux {};
    CBN_D void node(int64_t i, double (&w)[D], Aux&) const {
        if (nodes64) {
#pragma unroll
            for (int d = 0; d < D; ++d) w[d] = nodes64[i * D + d];
        } else {
#pragma unroll
            for (int d = 0; d < D; ++d) w[d] = wrap_pi((double)nodes32[i * D + d]);
        }
    }
    // binned kernels: sorted position pos of original node i
    CBN_D void node_at(int64_t pos, int64_t i, double (&w)[D], Aux& a) const {
        if (sorted32) {
#pragma unroll
            for (int d = 0; d < D; ++d) w[d] = wrap_pi((double)sorted32[pos * D + d]);
        } else {
            node(i, w, a);
        }
    }
};

// plan.phase = exp(-i w . (N//2))  (nufft.py:215-216), angle in float64
template <int D>
struct PhaseOut {
    float2* y;
    double c[kMaxDim];
    CBN_D void put(int64_t i, float2 v, const double (&w)[D], const typename ExplicitSrc<D>::Aux&) const {
        double a = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) a += w[d] * c[d];
        double sn, cs;
        sincos(-a, &sn, &cs);
        y[i] = cmul(v, make_float2((float)cs, (float)sn));
    }
};

template <int D>
struct PhaseIn : ExplicitSrc<D> {
    const float2* yin;
    double c[kMaxDim];
    CBN_D float2 value(int64_t i, const double (&w)[D], const typename ExplicitSrc<D>::Aux&) const {
        double a = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) a += w[d] * c[d];
        double sn, cs;
        sincos(a, &sn, &cs);   // conj(phase)
        return cmul(yin[i], make_float2((float)cs, (float)sn));
    }
};

__global__ void k_wrap_nodes(const double* __restrict__ in, double* __restrict__ out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = wrap_pi(in[i]);
}

template <int D>
__global__ void k_first(ExplicitSrc<D> src, KBSet kb, int64_t m, int32_t* out, double* wrapped) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double w[D];
    typename ExplicitSrc<D>::Aux aux;
    src.node(i, w, aux);
#pragma unroll
    for (int d = 0; d < D; ++d) {
        if (wrapped) wrapped[i * D + d] = w[d];
        if (out) {
            int f;
            axis_coord(w[d], kb.ax[d].K, 0.5 * (double)kb.ax[d].J, f);
            out[i * D + d] = wrapc(f, kb.ax[d].K);
        }
    }
}

constexpr int kSpreadWarps = 4;

}  // namespace cbn

using namespace cbn;

struct cbn_nufft_s {
    int D = 0;
    int J = 0;
    int64_t m = 0;
    AxisPlan ax[kMaxDim];
    KBSet kb{};
    DevBuf<double> nodes;      // wrapped float64 nodes, or
    DevBuf<float> nodes32;     // float32 nodes (wrapped on the fly)
    DevBuf<float> sorted32;    // float32 nodes in bin order (2D / 3D float32 plans)
    DevBuf<float> s32;         // D x smax
    DevBuf<int> pad_idx, crop_idx;
    DevBuf<float> pad_sc, crop_sc;
    DevBuf<float2> grid;
    BinPlan bins;              // 2D / 3D: bin-sorted order and subproblems
    DeviceSortScratch sort;    // device-only counting sort (plan and re-sorts)
    StageTimer timer;          // per-stage events + algorithmic bytes (bench)
    std::vector<double> s64_host;
    int smax = 0;
    int64_t ktot = 1, ntot = 1;
    FFTCache fft;
    double centre[kMaxDim] = {0, 0, 0};
    template <int D_>
    ExplicitSrc<D_> src() const {
        return ExplicitSrc<D_>{nodes.p, nodes.p ? nullptr : nodes32.p,
                               nodes.p ? nullptr : sorted32.p};
    }
};

namespace {

template <int D>
void run_type2(cbn_nufft* p, const float2* x, float2* y, cudaStream_t s) {
    RemapAxis ax[kMaxDim];
    int64_t stride = 1;
    int koff = 0;
    for (int d = D - 1; d >= 0; --d) {
        ax[d].n = p->ax[d].K;
        ax[d].sstride = stride;
        stride *= p->ax[d].N;
    }
    for (int d = 0; d < D; ++d) {
        ax[d].idx = p->pad_idx.p + koff;
        ax[d].scale = p->pad_sc.p + koff;
        koff += p->ax[d].K;
    }
    launch_remap<float2, kStoreC>(D, x, p->grid.p, ax, 1.0f, s);
    CBN_LAUNCH_CHECK();
    long long kd[3];
    for (int d = 0; d < D; ++d) kd[d] = p->ax[d].K;
    p->fft.exec(p->fft.get(D, kd, 1), p->grid.p, p->grid.p, CUFFT_FORWARD, s);
    PhaseOut<D> epi;
    epi.y = y;
    for (int d = 0; d < D; ++d) epi.c[d] = p->centre[d];
    ExplicitSrc<D> src = p->src<D>();
    // grid read once, coordinates (float32: 4 B, float64: 8 B per axis) and
    // values once; on chip: J^D tap reads of 8 B per node
    const double cb = (p->nodes.p ? 8.0 : 4.0) * D;
    double taps = 1;
    for (int d = 0; d < D; ++d) taps *= p->J;
    p->timer.add_bytes("gather", 8.0 * p->ktot + (cb + 8.0) * p->m, 8.0 * taps * p->m);
    StageScope st(p->timer, "gather", s);
    dispatch_j(p->J, [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        if constexpr (D >= 2) {
            const BinPlan& bb = p->bins;
            k_gather_binned<D, J><<<bb.nsubs, 256, sizeof(float2) * bb.nreg, s>>>(
                p->grid.p, p->kb, bb.geom<D>(), src, epi, bb.perm.p, bb.subs.p);
        } else {
            k_gather<D, J><<<blocks_for(p->m, 256), 256, 0, s>>>(p->grid.p, p->kb, src, epi, p->m);
        }
        return 0;
    });
    CBN_LAUNCH_CHECK();
}

template <int D>
void run_type1(cbn_nufft* p, const float2* y, float2* x, cudaStream_t s) {
    PhaseIn<D> src;
    static_cast<ExplicitSrc<D>&>(src) = p->src<D>();
    src.yin = y;
    for (int d = 0; d < D; ++d) src.c[d] = p->centre[d];
    {
        // the grid written once (memset + flushes), coordinates and values
        // read once; on chip: J^D shared-memory read + write of 8 B per node
        const double cb = (p->nodes.p ? 8.0 : 4.0) * D;
        double taps = 1;
        for (int d = 0; d < D; ++d) taps *= p->J;
        p->timer.add_bytes("spread", 8.0 * p->ktot + (cb + 8.0) * p->m, 16.0 * taps * p->m);
    }
    StageScope st_sp(p->timer, "spread", s);
    CBN_CUDA(cudaMemsetAsync(p->grid.p, 0, p->grid.bytes(), s));
    dispatch_j(p->J, [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        if constexpr (D == 3) {
            launch_spread3<J>(p->grid.p, p->kb, p->bins, src, s);
        } else if constexpr (D == 2) {
            const BinPlan& bb = p->bins;
            const size_t smem = spread_smem_bytes<D, J, kSpreadWarps>(bb.nreg);
            CBN_CUDA(cudaFuncSetAttribute(k_spread_binned<D, J, kSpreadWarps, PhaseIn<D>>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_spread_binned<D, J, kSpreadWarps><<<bb.nsubs, kSpreadWarps * 32, smem, s>>>(
                p->grid.p, p->kb, bb.geom<D>(), src, bb.perm.p, bb.subs.p);
        } else {
            k_spread<D, J><<<blocks_for(p->m, 256), 256, 0, s>>>(p->grid.p, p->kb, src, p->m);
        }
        return 0;
    });
    CBN_LAUNCH_CHECK();
    long long kd[3];
    for (int d = 0; d < D; ++d) kd[d] = p->ax[d].K;
    p->fft.exec(p->fft.get(D, kd, 1), p->grid.p, p->grid.p, CUFFT_INVERSE, s);
    RemapAxis ax[kMaxDim];
    int64_t stride = 1;
    int noff = 0;
    for (int d = D - 1; d >= 0; --d) {
        ax[d].n = p->ax[d].N;
        ax[d].sstride = stride;
        stride *= p->ax[d].K;
    }
    for (int d = 0; d < D; ++d) {
        ax[d].idx = p->crop_idx.p + noff;
        ax[d].scale = p->crop_sc.p + noff;
        noff += p->ax[d].N;
    }
    launch_remap<float2, kStoreC>(D, p->grid.p, x, ax, 1.0f, s);
    CBN_LAUNCH_CHECK();
}

// bin-sorted order for the shared-memory gather/spread, entirely on the
// device (build_bins with DeviceSortScratch): 3D tiles 8 x 8 x 16 cells (the
// pitch-padded region holds 16 + J - 1 along z at no extra shared memory for
// J = 6, 8), 2D 16 x 16.  float32 nodes also get a bin-ordered copy, so the
// gather / spread stream their coordinates.
template <int D>
void sort_plan(cbn_nufft* p, cudaStream_t s) {
    ExplicitSrc<D> src{p->nodes.p, p->nodes.p ? nullptr : p->nodes32.p, nullptr};
    int tile[3] = {D == 3 ? 8 : 16, D == 3 ? 8 : 16, 16};
    if (const char* e = std::getenv("CBN_NUFFT_TILE"); e && D == 3)   // "t0,t1,t2" (tuning A/B)
        std::sscanf(e, "%d,%d,%d", &tile[0], &tile[1], &tile[2]);
    {
        // coordinates read twice (keys, interleave), keys written + read,
        // the permutation written; float32: the sorted copy (read + write)
        const double cb = (p->nodes.p ? 8.0 : 4.0) * D;
        p->timer.add_bytes("sort", p->m * (2.0 * cb + 8.0 + 8.0 + (p->nodes.p ? 0.0 : 2.0 * cb)), 0.0);
    }
    StageScope st(p->timer, "sort", s);
    // float32 node sets: the interleave pass also writes the bin-ordered copy
    // of the coordinates (sorted32[pos] = nodes32[perm[pos]])
    if (!p->nodes.p) p->sorted32.ensure((size_t)p->m * D);
    dispatch_j(p->J, [&](auto jc) {
        build_bins<D, decltype(jc)::value>(p->bins, src, p->kb, p->m, tile, 1024, s, true, &p->sort,
                                           p->nodes.p ? nullptr : p->nodes32.p,
                                           p->nodes.p ? nullptr : p->sorted32.p);
        return 0;
    });
}

template <int D>
void fit_plan(cbn_nufft* p, const int64_t* rows_host, int64_t n_ls, cudaStream_t s) {
    DevBuf<int64_t> rows;
    rows.upload(rows_host, (size_t)n_ls, s);
    LSScratch sc;
    ExplicitSrc<D> src = p->src<D>();
    ls_fit<D>(src, rows.p, (int)n_ls, p->ax, sc, p->s32.p, p->smax, s);
    p->s64_host.assign((size_t)D * p->smax, 0.0);
    CBN_CUDA(cudaMemcpyAsync(p->s64_host.data(), sc.s64.p, sizeof(double) * D * p->smax,
                             cudaMemcpyDeviceToHost, s));
    int koff = 0, noff = 0;
    for (int d = 0; d < D; ++d) {
        build_table(kTabPad, p->ax[d].N, p->ax[d].K, p->s32.p + (size_t)d * p->smax,
                    p->pad_idx.p + koff, p->pad_sc.p + koff, s);
        build_table(kTabCrop, p->ax[d].N, p->ax[d].K, p->s32.p + (size_t)d * p->smax,
                    p->crop_idx.p + noff, p->crop_sc.p + noff, s);
        koff += p->ax[d].K;
        noff += p->ax[d].N;
    }
    if constexpr (D >= 2) {
        // bin-sorted order for the shared-memory gather/spread (one-time plan step)
        // 3D: 8 x 8 x 16 cells (the pitch-padded region holds 16 + J - 1 along z
        // at no extra shared memory for J = 6, 8); 2D: 16 x 16
        sort_plan<D>(p, s);
    }
    CBN_CUDA(cudaStreamSynchronize(s));   // rows / host scaling copy must outlive the launch
}

template <class F>
auto dispatch_d(int D, F&& f) {
    switch (D) {
        case 1: return f(std::integral_constant<int, 1>{});
        case 2: return f(std::integral_constant<int, 2>{});
        case 3: return f(std::integral_constant<int, 3>{});
        default: throw Error(CBN_EINVAL, "ndim must be 1..3");
    }
}

int create_plan(cbn_nufft** out, int ndim, const int64_t* dims, const int32_t* taps,
                double oversample_factor, const double* nodes64, const float* nodes32, int64_t m,
                const int64_t* ls_rows, int64_t n_ls, void* stream) {
    CBN_REQUIRE(out && dims && taps, "null argument");
    CBN_REQUIRE(ndim >= 1 && ndim <= 3, "ndim must be 1..3");
    CBN_REQUIRE(oversample_factor >= 1.0, "oversample_factor must be >= 1");
    CBN_REQUIRE(m >= 1 && (nodes64 || nodes32), "need at least one node");
    CBN_REQUIRE(m < ((int64_t)1 << 31), "at most 2^31 - 1 nodes per plan");
    CBN_REQUIRE(n_ls >= 1 && n_ls <= kMaxLS && ls_rows, "scaling-fit rows must number 1..8192");
    for (int d = 0; d < ndim; ++d) {
        CBN_REQUIRE(dims[d] >= 1, "dims must be >= 1");
        CBN_REQUIRE(taps[d] >= 1, "tap counts must be >= 1");
    }
    for (int64_t r = 0; r < n_ls; ++r) CBN_REQUIRE(ls_rows[r] >= 0 && ls_rows[r] < m, "bad scaling-fit row");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto p = std::make_unique<cbn_nufft_s>();
    p->D = ndim;
    p->J = taps[0];   // the largest per-axis tap count sizes the kernels' tap loops
    for (int d = 1; d < ndim; ++d) p->J = std::max(p->J, (int)taps[d]);
    p->m = m;
    for (int d = 0; d < ndim; ++d) {
        p->ax[d] = make_axis((int)dims[d], taps[d], oversample_factor);
        p->kb.ax[d] = p->ax[d].kb;
        p->smax = std::max(p->smax, p->ax[d].N);
        p->ktot *= p->ax[d].K;
        p->ntot *= p->ax[d].N;
        p->centre[d] = (double)(dims[d] / 2);
    }
    if (nodes64) {
        DevBuf<double> raw;
        raw.upload(nodes64, (size_t)m * ndim, s);
        p->nodes.alloc((size_t)m * ndim);
        k_wrap_nodes<<<blocks_for(m * ndim, 256), 256, 0, s>>>(raw.p, p->nodes.p, m * ndim);
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaStreamSynchronize(s));
    } else {
        p->nodes32.upload(nodes32, (size_t)m * ndim, s);
    }
    size_t ksum = 0, nsum = 0;
    for (int d = 0; d < ndim; ++d) {
        ksum += p->ax[d].K;
        nsum += p->ax[d].N;
    }
    p->s32.alloc((size_t)ndim * p->smax);
    p->pad_idx.alloc(ksum);
    p->pad_sc.alloc(ksum);
    p->crop_idx.alloc(nsum);
    p->crop_sc.alloc(nsum);
    p->grid.alloc((size_t)p->ktot);
    dispatch_d(ndim, [&](auto dc) {
        fit_plan<decltype(dc)::value>(p.get(), ls_rows, n_ls, s);
        return 0;
    });
    *out = p.release();
    return CBN_OK;
}

}  // namespace

extern "C" {

int cbn_version(void) { return 1; }

double cbn_beatty_beta(int j, double alpha) { return cbn::beatty_beta(j, alpha); }

int cbn_nufft_create(cbn_nufft** out, int ndim, const int64_t* dims, const int32_t* taps,
                     double oversample_factor, const double* nodes, int64_t m,
                     const int64_t* ls_rows, int64_t n_ls, void* stream) {
    try {
        return create_plan(out, ndim, dims, taps, oversample_factor, nodes, nullptr, m, ls_rows,
                           n_ls, stream);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_create_f32(cbn_nufft** out, int ndim, const int64_t* dims, const int32_t* taps,
                         double oversample_factor, const float* nodes, int64_t m,
                         const int64_t* ls_rows, int64_t n_ls, void* stream) {
    try {
        return create_plan(out, ndim, dims, taps, oversample_factor, nullptr, nodes, m, ls_rows,
                           n_ls, stream);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_destroy(cbn_nufft* plan) {
    delete plan;
    return CBN_OK;
}

int cbn_nufft_set_phase(cbn_nufft* p, int32_t on) {
    try {
        CBN_REQUIRE(p, "null argument");
        for (int d = 0; d < p->D; ++d) p->centre[d] = on ? (double)(p->ax[d].N / 2) : 0.0;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_scaling(const cbn_nufft* p, double* out) {
    try {
        CBN_REQUIRE(p && out, "null argument");
        size_t k = 0;
        for (int d = 0; d < p->D; ++d)
            for (int n = 0; n < p->ax[d].N; ++n) out[k++] = p->s64_host[(size_t)d * p->smax + n];
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_wrapped_nodes(const cbn_nufft* p, double* out) {
    try {
        CBN_REQUIRE(p && out, "null argument");
        DevBuf<double> dev((size_t)p->m * p->D);
        dispatch_d(p->D, [&](auto dc) {
            constexpr int D = decltype(dc)::value;
            k_first<D><<<blocks_for(p->m, 256), 256>>>(p->src<D>(), p->kb, p->m, nullptr, dev.p);
            return 0;
        });
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaMemcpy(out, dev.p, sizeof(double) * p->m * p->D, cudaMemcpyDeviceToHost));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_first_indices(const cbn_nufft* p, int32_t* out, void* stream) {
    try {
        CBN_REQUIRE(p && out, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<int32_t> dev((size_t)p->m * p->D);
        dispatch_d(p->D, [&](auto dc) {
            constexpr int D = decltype(dc)::value;
            k_first<D><<<blocks_for(p->m, 256), 256, 0, s>>>(p->src<D>(), p->kb, p->m, dev.p,
                                                             nullptr);
            return 0;
        });
        CBN_LAUNCH_CHECK();
        CBN_CUDA(cudaMemcpyAsync(out, dev.p, sizeof(int32_t) * p->m * p->D, cudaMemcpyDeviceToHost, s));
        CBN_CUDA(cudaStreamSynchronize(s));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_resort(cbn_nufft* p, void* stream) {
    try {
        CBN_REQUIRE(p, "null argument");
        CBN_REQUIRE(p->D >= 2, "1D plans are not bin-sorted");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        dispatch_d(p->D, [&](auto dc) {
            constexpr int D = decltype(dc)::value;
            if constexpr (D >= 2) sort_plan<D>(p, s);
            return 0;
        });
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_set_timing(cbn_nufft* p, int32_t on) {
    try {
        CBN_REQUIRE(p, "null argument");
        p->timer.reset();
        p->timer.on = on != 0;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_stage_times(cbn_nufft* p, double* ms, double* hbm, double* chip, int32_t* count,
                          char* names, int32_t names_len) {
    try {
        CBN_REQUIRE(p && count, "null argument");
        p->timer.collect();
        const int cap = *count;
        *count = (int32_t)p->timer.totals.size();
        std::string joined;
        for (int i = 0; i < *count; ++i) {
            const std::string& nm = p->timer.totals[i].first;
            if (i < cap) {
                if (ms) ms[i] = p->timer.totals[i].second;
                double h = 0, c = 0;
                for (const auto& kv : p->timer.bytes)
                    if (kv.first == nm) {
                        h = kv.second.hbm;
                        c = kv.second.chip;
                    }
                if (hbm) hbm[i] = h;
                if (chip) chip[i] = c;
            }
            if (i) joined += ";";
            joined += nm;
        }
        if (names && names_len > 0) {
            std::strncpy(names, joined.c_str(), (size_t)names_len - 1);
            names[names_len - 1] = 0;
        }
        p->timer.reset();
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_type2(cbn_nufft* p, const void* x, void* y, void* stream) {
    try {
        CBN_REQUIRE(p && x && y, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        dispatch_d(p->D, [&](auto dc) {
            run_type2<decltype(dc)::value>(p, static_cast<const float2*>(x), static_cast<float2*>(y), s);
            return 0;
        });
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_nufft_type1(cbn_nufft* p, const void* y, void* x, void* stream) {
    try {
        CBN_REQUIRE(p && x && y, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        dispatch_d(p->D, [&](auto dc) {
            run_type1<decltype(dc)::value>(p, static_cast<const float2*>(y), static_cast<float2*>(x), s);
            return 0;
        });
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
