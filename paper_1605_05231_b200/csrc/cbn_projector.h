// Projector plan: device state of nufft_forward_project / nufft_backproject
// (pipeline.py:122-212).  See DESIGN.md for the data layout.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "cbn_binned.cuh"
#include "cbn_grangeat.cuh"
#include "cbn_plan.h"
#include "cbn_sources.cuh"

namespace cbn {

// Radial lattice spec + the node tables of its 3D NUFFT (radon_fourier.py:46-67).
struct RadialTables {
    int n_rho = 0, n_theta = 0, n_phi = 0;
    double rho_max = 0, d_rho = 0;
    DevBuf<double> om, cphi, sphi, cth, sth;   // float64 node tables
    DevBuf<float> om_phys;                      // radial_omega (rad / mm)
    DevBuf<float> sin_theta;                    // sin(theta) as float
    int64_t lines() const { return (int64_t)n_theta * n_phi; }
    int64_t nodes() const { return lines() * n_rho; }
    void build(int n_rho, int n_theta, int n_phi, double rho_max, double voxel, cudaStream_t s);
    RadialSrc src() const { return RadialSrc{om.p, cphi.p, sphi.p, cth.p, sth.p, n_rho, n_theta}; }
};

// Umbrella line grid of one direction (forward: cfg t grid; back: detector grid).
struct UmbrellaTables {
    int n_mu = 0, n_t = 0;
    double dt = 0;
    DevBuf<double> cos_a, sin_a, cos_mu, sin_mu, omega_t;
    DevBuf<double4> base;   // view-0 target positions (see UmbrellaSrc::cache)
    bool base_ready = false;
    DevBuf<char> taps;      // view-0 resample taps (RsTap) for the views-in-lanes gather
    bool taps_ready = false;
    DevBuf<char> rows;      // J = 3: the same taps as grid-row offsets + weight products (RsRow3)
    DevBuf<int> poles;      // pole targets (theta == 0), handled per view (cbn_resample_views.cuh)
    int n_poles = 0;
    DevBuf<int> pole_f2;    // [pole][view] first phi tap of each pole target (k_resample_window)
    void build(const cbn_geometry& g, int n_mu, int n_t, double dt, cudaStream_t s);
};

// 2D NUFFT of the per-view Grangeat step (grangeat.py:93-128).
struct GrangeatPlan {
    AxisPlan ax[2];
    KBSet kb{};
    DevBuf<float> s32;     // 2 x smax
    int smax = 0;
    double pu = 0, pv = 0;
    int64_t m = 0;
    DevBuf<float> w2, fac_re, fac_im;   // per t: post-weight, reverse filter (complex)
    DevBuf<float> w2inv;                // per t: 1 / w2, folded into the resample store
    DevBuf<float> pix;                  // per detector pixel [nu][nv]: reverse s_u s_v / w1,
                                        // forward w1 s_u s_v (computed in float64 once)
    bool built = false;
    BinPlan bins;                       // polar nodes sorted by 2D tile
    DevBuf<char> pts;                   // GrPoint<5> per sorted node
    bool pts_ready = false;
    DevBuf<int> cell_ptr;               // reverse: CSR of (node, weight) entries per grid cell
    DevBuf<char> cell_ent;              // GrEntry per (node, tap)
    DevBuf<int> cell_order;             // work items of the half-plane cell gather, costliest
                                        // first: >= 0 block of 32 cells, < 0 one heavy cell
    DevBuf<unsigned char> cell_heavy;   // 1: half-plane cell handled by its own CTA
    int n_items = 0;
    DevBuf<GrNode> node_tab;            // reverse: node-scaled t-spectrum rows
    int64_t n_rows = 0;                 // rows of node_tab (nspec + second nodes)
    int64_t n_entries = 0;              // reverse: CSR entries (node, tap) over all cells
    // reverse, strip form of the cell CSR (k_gr_gather_strips): per half-plane
    // strip of kGrStrip cells along v, one entry per node with the strip's
    // per-cell weights of the node value (p) and of its conjugate's sign (q)
    DevBuf<int> strip_ptr, strip_id, strip_order;
    DevBuf<float4> strip_p, strip_q;
    DevBuf<unsigned char> strip_heavy;
    int n_strip_items = 0;
    int64_t n_strip_entries = 0;
};

constexpr int kGrJ = 5;        // plan_grangeat j=(5, 5) (grangeat.py:94)
constexpr int kGrTile = 16;    // forward (gather) tile edge
constexpr int kGrTileRev = 8;  // reverse (owner-computes spread) tile edge (6: 10.6 ms, 12: 10.1 ms, 8: 9.6 ms at cfg 2)
constexpr int kGrVG = 8;       // views per CTA in the binned Grangeat gather

constexpr int kTile3 = 8;      // 3D bin edge (oversampled cells), axes 0 and 1
constexpr int kTile3Fast = 16; // 3D bin edge along the fastest axis: the region's pitch
                               // padding (P = J mod 16) already covers 16 + J - 1 cells
constexpr int kMaxSub = 1024;  // points per subproblem

// Per-batch resample scalings of one direction (plan data: they depend only on
// the geometry), fitted once on the device and cached.  Batches whose
// scalings agree to 1e-9 relative on every axis share a representative
// (`group`), so they can share one resample grid / one transpose FFT.
struct BatchPlan {
    bool ready = false;
    std::vector<std::pair<int, int>> batches;
    std::vector<int> group;
    int smax = 0;
    DevBuf<float> s32;     // batches x 3 x smax
    int groups() const {
        int g = 0;
        for (size_t b = 0; b < group.size(); ++b) g += group[b] == (int)b;
        return g;
    }
};

}  // namespace cbn

struct cbn_projector_s {
    cbn_geometry g{};
    cbn_projector_config c{};
    int n_vol = 0;
    double voxel = 0;
    int direction = 0;
    double pu = 0, pv = 0;   // virtual pixel pitch

    std::map<int64_t, cbn::DevBuf<int64_t>*> ls_rows;
    std::vector<int64_t> ls_needed;

    cbn::FFTCache fft;
    cbn::LSScratch ls;
    cbn::StageTimer timer;

    // ---- forward
    cbn::RadialTables frad;
    cbn::UmbrellaTables fumb;
    cbn::GrangeatPlan fgr;
    cbn::AxisPlan fspec[3];     // spectrum NUFFT axes (N = n_vol)
    cbn::AxisPlan fres[3];      // resample NUFFT axes, device order (phi, theta, rho_padded)
    int fpad = 0;
    bool fw_built = false;
    cbn::BatchPlan fbatch;
    std::vector<std::pair<int, int>> fres_planes;   // non-zero slowest-axis planes of the resample grid
    int fres_planes_slow = -1;
    cbn::BinPlan fspec_bins;     // radial nodes sorted by spectrum-grid tile
    cbn::DevBuf<int> fpairs;     // primary radial nodes (RadialPairSrc); mirrors by conjugation
    cbn::DevBuf<float4> fspec_rec;   // per sorted primary node: KB arguments + tile offsets
    cbn::DevBuf<float2> fspec_fac;   // ... epilogue factor (i omega transfer phase)
    cbn::DevBuf<int2> fspec_out;     // ... lattice index and its conjugate mirror's
    cbn::DevBuf<int> fspec_list, fres_list;   // compact pad positions per axis (see pad_positions)
    int fspec_nl[3] = {0, 0, 0}, fres_nl[3] = {0, 0, 0};
    // staged spectrum input (cbn_forward_stage_volume): rows [0, fspec_staged)
    // of fspec_staged_vol are padded and 2D-transformed already
    cbn::RemapAxis fspec_rax[3];
    int fspec_staged = 0;
    const float* fspec_staged_vol = nullptr;
    // rho planes of the (views-in-lanes) resample grid the umbrella taps read
    std::vector<std::pair<int, int>> fres_rho_runs;
    // resample grid built rho-lines first: (theta, phi) pad positions with
    // mirrors, their inverse maps, the used rho planes, the line buffer
    cbn::DevBuf<int> fres_lth, fres_lph, fres_thmap, fres_phmap, fres_xs;
    int fres_nth = 0, fres_nph = 0, fres_nx = 0;
    cbn::DevBuf<float2> rlines;
    // backprojector: rho planes of the transposed grid with column entries, and
    // a per-plane flag for the column gather
    std::vector<std::pair<int, int>> bres_rho_runs;
    cbn::DevBuf<unsigned char> bres_rho_used;
    // rho lines of the transposed grid's spectrum the crop reads: theta and
    // phi-half positions, their inverse maps, the line buffer
    cbn::DevBuf<int> bres_lth, bres_lph, bres_thmap, bres_phmap;
    int bres_nth = 0, bres_nph = 0;
    cbn::DevBuf<float2> brlines;
    int64_t fpairs_n = 0;
    int fshard_part = 0, fshard_nparts = 1;   // forward node shard (cbn_projector_set_node_shard):
                                              // the spectrum plan covers lines of this share only
    bool fspec_fit = false;
    cbn::DevBuf<float> fspec_s32;   // cached first-sub-plan scaling of the spectrum NUFFT

    // ---- back
    cbn::RadialTables brad;
    cbn::UmbrellaTables bumb;
    cbn::GrangeatPlan bgr;
    cbn::AxisPlan bspec[3];
    cbn::AxisPlan bres[3];
    int bpad = 0;
    bool bw_built = false;
    cbn::BatchPlan bbatch;
    std::vector<std::pair<int, int>> bres_planes;   // slowest-axis planes the transpose crop reads
    int bres_planes_slow = -1;
    cbn::DevBuf<int> bcol_ptr;      // transposed-resample CSR: column -> entries (views in lanes)
    cbn::DevBuf<char> bcol_ent;     // RsColEntry per (target, rho tap, theta tap)
    int64_t bcol_n = 0;             // entries of the column CSR
    cbn::DevBuf<int> bstrip_ptr;    // strip form of the column CSR (k_rs_gather_strips)
    cbn::DevBuf<char> bstrip_ent;   // RsStripEnt per (target, strip)
    cbn::DevBuf<float4> bstrip_w2, bstrip_wab;   // phi weights; per-column rho-theta weights
    int64_t bstrip_n = 0;
    int bstrip_nsx = 0;
    cbn::DevBuf<float> values_t;    // umbrella values of a view run, target-major
    int bp_staged = 0;              // views [0, bp_staged) of the next backprojection already
                                    // forward-Grangeat'ed into values_t (cbn_backproject_stage_views)
    cbn::BinPlan bspec_bins;     // backprojector radial nodes sorted by grid tile
    cbn::DevBuf<int> bpairs;     // primary radial nodes of the 3D adjoint (conjugate pairs)
    cbn::DevBuf<float4> bspec_rec;   // per sorted primary node: KB arguments + tile offsets
    cbn::DevBuf<float4> bspec_g;     // ... factors of its lattice sample and its mirror's
    cbn::DevBuf<int2> bspec_idx;     // ... those two lattice indices
    cbn::DevBuf<float2> bspec_vals;  // ... the values of a step (k_bp_values)
    int64_t bpairs_n = 0;
    bool bspec_fit = false;
    cbn::DevBuf<float> bspec_s32;   // cached first-sub-plan scaling of the 3D adjoint
    bool den_cached = false;
    cbn::DevBuf<float> den_cache;   // final den lattice (incl. origin average), node order
    cbn::DevBuf<double> den_max;
    cbn::DevBuf<unsigned char> den_keep;   // per-orbit keep decision (rotation-aligned views), or empty
    cbn::DevBuf<float> ramp_q;      // backprojector ramp per rho bin

    // ---- scratch (shared by both directions, sized on demand)
    cbn::DevBuf<float2> big;        // spectrum grid / resample grid(s)
    const float* grid_re = nullptr; // Re(resample grid) inside `big` (real_grid path)
    cbn::DevBuf<float2> lattice;    // radial lattice (raw IFFT layout)
    cbn::DevBuf<float2> padded;     // padded lattice and its FFT / transpose accumulators
    cbn::DevBuf<float2> bp_half;    // backprojector crop: Hermitian half of the (2N)^3 grid
    cbn::DevBuf<float2> gr_t;       // Grangeat t-line buffers
    cbn::DevBuf<float2> gr_tv;      // reverse Grangeat t-spectra, view-fastest [mu][k][32 views]
    cbn::DevBuf<float2> gr_grid;    // Grangeat 2D grids
    cbn::DevBuf<float> values;      // umbrella values of a view batch
    cbn::DevBuf<float> s32;         // per-plan float32 scalings (3 x smax)
    cbn::DevBuf<int> tab_idx;
    cbn::DevBuf<float> tab_sc;
    cbn::DevBuf<double> red;        // reductions
    cbn::DevBuf<int> flag;          // non-finite flag

    // second lane of the forward view-block loop: the resample gather and the
    // reverse Grangeat of block k+1 run on `s1` while block k finishes on the
    // caller's stream (own FFT plans/work area and per-block scratch)
    struct Lane {
        cbn::FFTCache fft;
        cbn::DevBuf<float2> gr_t, gr_tv, gr_grid;
        cbn::DevBuf<float> values;
        cbn::DevBuf<double> red;
    };
    Lane lane1;
    // progress of an asynchronous forward projection: one event per reverse-
    // Grangeat block, recorded on the stream that wrote the block's frames
    // (cbn_forward_project_async / cbn_projector_block_sync)
    bool track_blocks = false;
    std::vector<cudaEvent_t> blk_ev;
    std::vector<int> blk_lo, blk_hi;
    int blk_count = 0;
    void block_done(int v_lo, int v_hi, cudaStream_t s) {
        if (!track_blocks) return;
        if (blk_count == (int)blk_ev.size()) {
            cudaEvent_t e;
            CBN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            blk_ev.push_back(e);
        }
        CBN_CUDA(cudaEventRecord(blk_ev[(size_t)blk_count], s));
        if ((int)blk_lo.size() <= blk_count) {
            blk_lo.resize((size_t)blk_count + 1);
            blk_hi.resize((size_t)blk_count + 1);
        }
        blk_lo[(size_t)blk_count] = v_lo;
        blk_hi[(size_t)blk_count] = v_hi;
        ++blk_count;
    }
    cudaStream_t s1 = nullptr;
    cudaEvent_t ev_s0 = nullptr, ev_s1 = nullptr;

    ~cbn_projector_s() {
        for (auto& kv : ls_rows) delete kv.second;
        for (auto e : blk_ev) cudaEventDestroy(e);
        if (ev_s0) cudaEventDestroy(ev_s0);
        if (ev_s1) cudaEventDestroy(ev_s1);
        if (s1) cudaStreamDestroy(s1);
    }
};

namespace cbn {

// per-lane Grangeat scratch: the projector's own buffers (lane 0, caller's
// stream) or lane1's (stream s1)
int res_jmax(const AxisPlan* ax);
bool res_j3(const AxisPlan* ax);

struct GrBufs {
    FFTCache& fft;
    DevBuf<float2>& t;
    DevBuf<float2>& tv;
    DevBuf<float2>& grid;
    DevBuf<double>& red;
};
inline GrBufs main_bufs(cbn_projector_s* p) {
    return {p->fft, p->gr_t, p->gr_tv, p->gr_grid, p->red};
}
inline GrBufs lane_bufs(cbn_projector_s* p) {
    auto& l = p->lane1;
    return {l.fft, l.gr_t, l.gr_tv, l.gr_grid, l.red};
}
inline void ensure_lane1(cbn_projector_s* p) {
    if (p->s1) return;
    CBN_CUDA(cudaStreamCreateWithFlags(&p->s1, cudaStreamNonBlocking));
    CBN_CUDA(cudaEventCreateWithFlags(&p->ev_s0, cudaEventDisableTiming));
    CBN_CUDA(cudaEventCreateWithFlags(&p->ev_s1, cudaEventDisableTiming));
}
// CBN_ONE_STREAM=1 keeps every lane on the caller's stream (diagnostics)
inline bool lanes_allowed() {
    const char* one = std::getenv("CBN_ONE_STREAM");
    return !(one && one[0] == '1');
}

}  // namespace cbn
