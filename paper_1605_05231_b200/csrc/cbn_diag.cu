// Plan diagnostics of the projector (C ABI): the first-tap indices of every
// node set the projector plans, and plan statistics.  Test and bench support
// only -- nothing on the operator path calls these.
//
// cbn_projector_first_indices exports per-axis `first mod K`
// (nufft.py:171-179) exactly as the projector's kernels use it:
//   set 0 / 3  radial lattice nodes of the forward spectrum NUFFT /
//              the backprojector's 3D adjoint (RadialSrc, J = spectrum_j),
//              radon_fourier.py:89-108, pipeline.py:202-210;
//   set 1 / 4  umbrella targets of view batch `batch` (J = resample_j), in the
//              reference's (rho, theta, phi) order: on the views-in-lanes
//              path from view 0's taps plus the whole-cell phi shift of view
//              k (what k_resample_rows3 / k_rs_gather_cols* read), otherwise
//              from the cached umbrella source the gathers/spreads evaluate
//              (resampling.py:79-103, pipeline.py:130-137,174-182);
//   set 2 / 5  polar Grangeat nodes (J = 5), grangeat.py:93-128.
// Invalid umbrella targets are pinned to the origin node for every view
// (pipeline.py:100-101): their first indices carry no view shift.
#include <algorithm>
#include <cstring>
#include <string>

#include "cbn_projector.h"
#include "cbn_resample_views.cuh"

namespace cbn {

void build_forward_plan(cbn_projector_s* p, cudaStream_t s);
void build_backward_plan(cbn_projector_s* p, cudaStream_t s);
bool projector_views_in_lanes(const cbn_projector_s* p);
bool projector_real_grid(const cbn_projector_s* p);
bool bp_uses_lanes(cbn_projector_s* p, cudaStream_t s);
UmbrellaSrc projector_cached_umbrella(cbn_projector_s* p, UmbrellaTables& u, const RadialTables& r,
                                      int pad, int view0, cudaStream_t s);
std::vector<std::pair<int, int>> projector_batches(int n_views, int64_t per_view, int64_t target);
int64_t projector_target_batch(const cbn_projector_s* p);

namespace {

// first mod K of node i per axis; rev: write the axes in reverse order
template <class Src, int D, int J>
__global__ void k_first_src(Src src, KBSet kb, int64_t m, int rev, int* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double w[D];
    typename Src::Aux aux;
    src.node(i, w, aux);
    int first[D];
    float wt[D][J];
    tap_setup<D, J>(kb, w, first, wt);
#pragma unroll
    for (int d = 0; d < D; ++d) out[i * D + (rev ? D - 1 - d : d)] = wrapc(first[d], kb.ax[d].K);
}

// views-in-lanes umbrella bins: view 0's taps (grid order rho, theta, phi),
// view v's phi tap shifted by v * shift cells (k_resample_rows3:
// c0 = f2 - v shift mod K2; k_rs_gather_cols2: f2 - 2 v)
template <int J>
__global__ void k_first_lanes(UmbrellaSrc src0, KBSet kb, int64_t per_view, int v0, int nv,
                              int shift, int* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= per_view * nv) return;
    const int v = v0 + (int)(i / per_view);
    const int64_t t = i % per_view;
    double wd[3];
    UmbrellaSrc::Aux aux;
    src0.node(t, wd, aux);
    if (aux.pole) {   // pole targets: per view, like k_rs_pole_gather / k_rs_pole_spread
        UmbrellaSrc sv = src0;
        sv.view0 = v;
        sv.node(t, wd, aux);
        shift = 0;
    }
    const double w[3] = {wd[2], wd[1], wd[0]};
    int first[3];
    float wt[3][J];
    tap_setup<3, J>(kb, w, first, wt);
    const int K2 = kb.ax[2].K;
    int f2 = wrapc(first[2], K2);
    if (aux.valid && shift) {
        f2 -= (int)(((int64_t)v * shift) % K2);
        f2 += f2 < 0 ? K2 : 0;
    }
    out[i * 3 + 0] = wrapc(first[0], kb.ax[0].K);
    out[i * 3 + 1] = wrapc(first[1], kb.ax[1].K);
    out[i * 3 + 2] = f2;
}

template <class Src, int D>
void first_src(const Src& src, const AxisPlan* ax, int64_t m, int rev, int* out, cudaStream_t s) {
    KBSet kb;
    for (int d = 0; d < D; ++d) kb.ax[d] = ax[d].kb;
    dispatch_j(ax[0].J, [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        k_first_src<Src, D, J><<<blocks_for(m, 256), 256, 0, s>>>(src, kb, m, rev, out);
        return 0;
    });
    CBN_LAUNCH_CHECK();
}

void require_uniform_axes(const AxisPlan* ax, int d) {
    for (int k = 1; k < d; ++k)
        CBN_REQUIRE(ax[k].J == ax[0].J, "per-axis tap counts differ");
}

}  // namespace
}  // namespace cbn

using namespace cbn;

extern "C" {

int cbn_projector_first_indices(cbn_projector* p, int32_t set, int32_t batch, int32_t* out,
                                int64_t* m, void* stream) {
    try {
        CBN_REQUIRE(p && m, "null argument");
        CBN_REQUIRE(set >= 0 && set <= 5, "set must be 0..5");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const bool back = set >= 3;
        CBN_REQUIRE(p->direction & (back ? 2 : 1), "projector was not created for that direction");
        if (back)
            build_backward_plan(p, s);
        else
            build_forward_plan(p, s);
        const int kind = set % 3;
        const int64_t cap = *m;
        DevBuf<int> dev;
        int64_t count = 0, dims = 3;
        if (kind == 0) {
            const RadialTables& r = back ? p->brad : p->frad;
            const AxisPlan* ax = back ? p->bspec : p->fspec;
            require_uniform_axes(ax, 3);
            count = r.nodes();
            if (out && cap >= count) {
                dev.alloc((size_t)count * 3);
                first_src<RadialSrc, 3>(r.src(), ax, count, 0, dev.p, s);
            }
        } else if (kind == 1) {
            UmbrellaTables& u = back ? p->bumb : p->fumb;
            const RadialTables& r = back ? p->brad : p->frad;
            const AxisPlan* ax = back ? p->bres : p->fres;    // device order (phi, theta, rho)
            require_uniform_axes(ax, 3);
            const int pad = back ? p->bpad : p->fpad;
            const int64_t per_view = (int64_t)u.n_mu * u.n_t;
            const auto batches =
                projector_batches(p->g.n_views, per_view, projector_target_batch(p));
            CBN_REQUIRE(batch >= 0 && batch < (int)batches.size(), "batch out of range");
            const int v0 = batches[(size_t)batch].first, v1 = batches[(size_t)batch].second;
            count = per_view * (v1 - v0);
            if (out && cap >= count) {
                dev.alloc((size_t)count * 3);
                const bool lanes = back ? (p->c.method == 0 && bp_uses_lanes(p, s))
                                        : (p->c.method == 0 && projector_views_in_lanes(p));
                if (lanes) {
                    UmbrellaSrc src0 = projector_cached_umbrella(p, u, r, pad, 0, s);
                    KBSet kb;   // grid order (rho, theta, phi)
                    kb.ax[0] = ax[2].kb;
                    kb.ax[1] = ax[1].kb;
                    kb.ax[2] = ax[0].kb;
                    const int shift = (int)(2LL * r.n_phi / p->g.n_views);
                    dispatch_j(ax[0].J, [&](auto jc) {
                        constexpr int J = decltype(jc)::value;
                        k_first_lanes<J><<<blocks_for(count, 256), 256, 0, s>>>(
                            src0, kb, per_view, v0, v1 - v0, shift, dev.p);
                        return 0;
                    });
                    CBN_LAUNCH_CHECK();
                } else {
                    UmbrellaSrc src = projector_cached_umbrella(p, u, r, pad, v0, s);
                    first_src<UmbrellaSrc, 3>(src, ax, count, 1, dev.p, s);
                }
            }
        } else {
            UmbrellaTables& u = back ? p->bumb : p->fumb;
            GrangeatPlan& gp = back ? p->bgr : p->fgr;
            dims = 2;
            count = gp.m;
            if (out && cap >= count) {
                dev.alloc((size_t)count * 2);
                const PolarSrc src{u.omega_t.p, u.cos_mu.p, u.sin_mu.p, gp.pu, gp.pv, u.n_t};
                first_src<PolarSrc, 2>(src, gp.ax, count, 0, dev.p, s);
            }
        }
        *m = count;
        if (out && cap >= count) {
            CBN_CUDA(cudaMemcpyAsync(out, dev.p, sizeof(int) * (size_t)(count * dims),
                                     cudaMemcpyDeviceToHost, s));
            CBN_CUDA(cudaStreamSynchronize(s));
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Plan statistics as (name, value) pairs; -1 where that part of the plan has
// not been built yet (most are built by the first operator call).
// Diagnostics: copy a named plan buffer to the host (bytes = its size; out may
// be null to query it): den_cache, den_max, bspec_s32, ramp_q, bpairs, bspec_perm,
// bspec_subs, bbatch_s32, fspec_s32, values_t, lattice, den_keep.
int cbn_projector_debug_buffer(cbn_projector* p, const char* name, void* out, int64_t* bytes,
                               void* stream) {
    try {
        CBN_REQUIRE(p && name && bytes, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const std::string n(name);
        const void* src = nullptr;
        size_t len = 0;
        auto pick = [&](const auto& buf) {
            src = buf.p;
            len = buf.bytes();
        };
        if (n == "den_cache") pick(p->den_cache);
        else if (n == "den_max") pick(p->den_max);
        else if (n == "bspec_s32") pick(p->bspec_s32);
        else if (n == "ramp_q") pick(p->ramp_q);
        else if (n == "bpairs") pick(p->bpairs);
        else if (n == "bspec_perm") pick(p->bspec_bins.perm);
        else if (n == "bspec_subs") pick(p->bspec_bins.subs);
        else if (n == "bbatch_s32") pick(p->bbatch.s32);
        else if (n == "fspec_s32") pick(p->fspec_s32);
        else if (n == "values_t") pick(p->values_t);
        else if (n == "lattice") pick(p->lattice);
        else if (n == "den_keep") pick(p->den_keep);
        else throw Error(CBN_EINVAL, "unknown buffer " + n);
        *bytes = (int64_t)len;
        if (out && src && len) {
            CBN_CUDA(cudaMemcpyAsync(out, src, len, cudaMemcpyDeviceToHost, s));
            CBN_CUDA(cudaStreamSynchronize(s));
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_projector_plan_stats(cbn_projector* p, int64_t* vals, int32_t* count, char* names,
                             int32_t names_len, void* stream) {
    try {
        CBN_REQUIRE(p && count, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        std::vector<std::pair<std::string, int64_t>> st;
        auto runs_sum = [](const std::vector<std::pair<int, int>>& runs) -> int64_t {
            if (runs.empty()) return -1;
            int64_t n = 0;
            for (const auto& r : runs) n += r.second - r.first;
            return n;
        };
        auto invalid_per_view = [&](UmbrellaTables& u, const RadialTables& r, int pad) -> int64_t {
            UmbrellaSrc src = projector_cached_umbrella(p, u, r, pad, 0, s);
            (void)src;
            const int64_t per_view = (int64_t)u.n_mu * u.n_t;
            std::vector<double4> h((size_t)per_view);
            CBN_CUDA(cudaMemcpyAsync(h.data(), u.base.p, sizeof(double4) * per_view,
                                     cudaMemcpyDeviceToHost, s));
            CBN_CUDA(cudaStreamSynchronize(s));
            int64_t bad = 0;
            for (const auto& c : h) bad += c.w == 0.0;
            return bad;
        };
        auto heavy = [&](const GrangeatPlan& gp) -> int64_t {
            if (!gp.cell_order.p) return -1;
            std::vector<int> h((size_t)gp.n_items);
            CBN_CUDA(cudaMemcpy(h.data(), gp.cell_order.p, sizeof(int) * gp.n_items,
                                cudaMemcpyDeviceToHost));
            int64_t n = 0;
            for (int v : h) n += v < 0;
            return n;
        };
        if (p->direction & 1) {
            build_forward_plan(p, s);
            st.emplace_back("fwd_spectrum_nodes", p->frad.nodes());
            st.emplace_back("fwd_spectrum_primary_nodes", p->fpairs.p ? p->fpairs_n : -1);
            st.emplace_back("fwd_resample_rho_planes", p->fres[2].K);
            st.emplace_back("fwd_resample_rho_planes_used", runs_sum(p->fres_rho_runs));
            st.emplace_back("fwd_resample_cells", (int64_t)p->fres[0].K * p->fres[1].K * p->fres[2].K);
            st.emplace_back("fwd_views_in_lanes", projector_views_in_lanes(p) ? 1 : 0);
            st.emplace_back("fwd_real_grid", projector_real_grid(p) ? 1 : 0);
            st.emplace_back("fwd_umbrella_targets_per_view", (int64_t)p->fumb.n_mu * p->fumb.n_t);
            st.emplace_back("fwd_umbrella_invalid_per_view", invalid_per_view(p->fumb, p->frad, p->fpad));
            st.emplace_back("fwd_batches", p->fbatch.ready ? (int64_t)p->fbatch.batches.size() : -1);
            st.emplace_back("fwd_batch_groups", p->fbatch.ready ? p->fbatch.groups() : -1);
            st.emplace_back("fwd_gr_cell_items", p->fgr.cell_order.p ? p->fgr.n_items : -1);
            st.emplace_back("fwd_gr_heavy_cells", heavy(p->fgr));
            {
                const GrangeatPlan& gp = p->fgr;
                int64_t hs = -1;
                if (gp.strip_order.p) {
                    std::vector<int> h((size_t)gp.n_strip_items);
                    CBN_CUDA(cudaMemcpy(h.data(), gp.strip_order.p, sizeof(int) * h.size(),
                                        cudaMemcpyDeviceToHost));
                    hs = 0;
                    for (int v : h) hs += v < 0;
                }
                st.emplace_back("fwd_gr_strip_items", gp.strip_order.p ? gp.n_strip_items : -1);
                st.emplace_back("fwd_gr_heavy_strips", hs);
                st.emplace_back("fwd_gr_strip_entries", gp.strip_order.p ? gp.n_strip_entries : -1);
                st.emplace_back("fwd_gr_cell_entries", gp.cell_ptr.p ? gp.n_entries : -1);
            }
        }
        if (p->direction & 2) {
            build_backward_plan(p, s);
            st.emplace_back("bp_nodes", p->brad.nodes());
            st.emplace_back("bp_primary_nodes", p->bpairs.p ? p->bpairs_n : -1);
            st.emplace_back("bp_rho_planes", p->bres[2].K);
            st.emplace_back("bp_rho_planes_used", runs_sum(p->bres_rho_runs));
            st.emplace_back("bp_column_entries", p->bcol_ent.p ? p->bcol_n : -1);
            st.emplace_back("bp_strip_entries", p->bstrip_ptr.p ? p->bstrip_n : -1);
            st.emplace_back("bp_resample_cells", (int64_t)p->bres[0].K * p->bres[1].K * p->bres[2].K);
            st.emplace_back("bp_umbrella_targets_per_view", (int64_t)p->bumb.n_mu * p->bumb.n_t);
            st.emplace_back("bp_umbrella_invalid_per_view", invalid_per_view(p->bumb, p->brad, p->bpad));
            st.emplace_back("bp_batches", p->bbatch.ready ? (int64_t)p->bbatch.batches.size() : -1);
            st.emplace_back("bp_batch_groups", p->bbatch.ready ? p->bbatch.groups() : -1);
        }
        const int cap = *count;
        *count = (int32_t)st.size();
        std::string joined;
        for (int i = 0; i < *count; ++i) {
            if (vals && i < cap) vals[i] = st[(size_t)i].second;
            if (i) joined += ";";
            joined += st[(size_t)i].first;
        }
        if (names && names_len > 0) {
            std::strncpy(names, joined.c_str(), (size_t)names_len - 1);
            names[names_len - 1] = 0;
        }
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
