/*
 * cbnufft_b200 -- C ABI of the B200-native NUFFT cone-beam projector.
 *
 * The reference (`cbnufft`, /root/reference/pkg/src/cbnufft) is a pure-Python
 * package with no FFI; its operator API is the set of module functions
 * listed in SURVEY.md 8(b).  Each entry point below replaces one of them and
 * cites the reference function it stands in for.  The Python package
 * `paper_1605_05231_b200` binds these with ctypes (`_lib.py`) and re-exports
 * the reference names and signatures; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Plain C types only.  Array arguments marked [device] are CUDA device
 *    pointers (the Python layer passes torch tensor storage); [host] are host
 *    pointers.  Complex arrays are interleaved float32 pairs (complex64).
 *  - `stream` is a cudaStream_t passed as void*; every compute call is
 *    stream-ordered and asynchronous unless documented otherwise.
 *  - Return value: CBN_OK or an error status; cbn_last_error() gives a
 *    thread-local message.  CBN_EINVAL maps to ValueError and CBN_ENONFINITE
 *    to FloatingPointError in the Python layer (pipeline.py:144-145).
 *  - Caller owns all input/output buffers; plan objects own their scratch
 *    (cuFFT plans + workspace, tables, grids).  A plan must not be used from
 *    two streams at once.
 */
#ifndef CBNUFFT_B200_H
#define CBNUFFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBN_OK 0
#define CBN_EINVAL 1
#define CBN_ECUDA 2
#define CBN_ENOMEM 3
#define CBN_ENONFINITE 4
#define CBN_ENCCL 5
#define CBN_EUNSUPPORTED 6

const char* cbn_last_error(void);
int cbn_version(void);

/* Kaiser-Bessel shape parameter of the reference (nufft.py:53-56). */
double cbn_beatty_beta(int j, double alpha);

/* ------------------------------------------------------------------ NUFFT
 * Replaces plan_nufft / nufft_forward / nufft_adjoint (nufft.py:137-247).
 */
typedef struct cbn_nufft_s cbn_nufft;

/* plan_nufft(dims, nodes, oversample_factor, j)  (nufft.py:137-218)
 * nodes [host] m x ndim float64 row-major, any range (wrapped here);
 * taps [host] ndim tap counts; ls_rows [host] the scaling-fit subsample rows
 * (numpy default_rng(0).choice(m, 8192, replace=False) sorted, or 0..m-1),
 * nufft.py:163-168. */
int cbn_nufft_create(cbn_nufft** plan, int ndim, const int64_t* dims, const int32_t* taps,
                     double oversample_factor, const double* nodes, int64_t m,
                     const int64_t* ls_rows, int64_t n_ls, void* stream);
/* Same plan over float32 nodes (m x ndim, [host]), kept in float32 on the
 * device and wrapped to [-pi, pi) in float64 inside the kernels -- the
 * large-m path (100M nodes, 256^3, J=8).  Matches
 * plan_nufft(dims, nodes.astype(float64), ...) exactly. */
int cbn_nufft_create_f32(cbn_nufft** plan, int ndim, const int64_t* dims, const int32_t* taps,
                         double oversample_factor, const float* nodes, int64_t m,
                         const int64_t* ls_rows, int64_t n_ls, void* stream);
int cbn_nufft_destroy(cbn_nufft* plan);
/* per-axis float64 LS scaling vectors, concatenated (sum(dims) values) [host] */
int cbn_nufft_scaling(const cbn_nufft* plan, double* out);
/* wrapped nodes (m x ndim float64) and first-tap indices mod K (m x ndim int32) [host] */
int cbn_nufft_wrapped_nodes(const cbn_nufft* plan, double* out);
int cbn_nufft_first_indices(const cbn_nufft* plan, int32_t* out, void* stream);
/* nufft_forward (nufft.py:221-233): x [device] complex64 dims -> y [device] complex64 m */
int cbn_nufft_type2(cbn_nufft* plan, const void* x, void* y, void* stream);
/* nufft_adjoint (nufft.py:236-247): y [device] complex64 m -> x [device] complex64 dims */
int cbn_nufft_type1(cbn_nufft* plan, const void* y, void* x, void* stream);
/* apply (1, default) or omit (0) the per-node centring phase exp(-i w.(N//2))
 * (nufft.py:215-216) -- omitted where the caller's own phase cancels it
 * exactly (resampling.py:147-148, SURVEY finding 9) */
int cbn_nufft_set_phase(cbn_nufft* plan, int32_t on);

/* Re-run the plan's bin sort of its nodes on the device (keys, CUB scans,
 * scatter, subproblem list, bank interleave; no host round trip) -- the
 * "sort" of SURVEY 8(d)'s Msamples/s, timed per step by the bench.  2D/3D. */
int cbn_nufft_resort(cbn_nufft* plan, void* stream);
/* Stage events + algorithmic bytes (bench): set_timing(1) resets and turns
 * them on; stage_times returns per-stage ms, compulsory HBM bytes and
 * on-chip tap bytes since then (names ';'-separated: sort, gather, spread),
 * synchronises, and resets. */
int cbn_nufft_set_timing(cbn_nufft* plan, int32_t on);
int cbn_nufft_stage_times(cbn_nufft* plan, double* ms, double* hbm, double* chip, int32_t* count,
                          char* names, int32_t names_len);

/* ------------------------------------------------------------ resampling
 * plan_resample / resample_apply / resample_transpose, methods A and B
 * (resampling.py:79-103,136-161,164-196).  targets [host] m x 3 float64
 * fractional lattice indices (rho, theta, phi); lattice arrays [device]
 * complex64 in the reference layout (n_rho, n_theta, n_phi).
 */
typedef struct cbn_resample_s cbn_resample;
int cbn_resample_create(cbn_resample** plan, int32_t n_rho, int32_t n_theta, int32_t n_phi,
                        int32_t rho_pad, const int32_t* taps, double oversample_factor,
                        const double* targets, int64_t m, const int64_t* ls_rows, int64_t n_ls,
                        void* stream);
/* method B (resampling.py:126-161,164-196): truncated centred periodic sinc,
 * side_lobes + 1 taps per axis on the rho-padded lattice itself; the plan
 * keeps only the targets */
int cbn_resample_create_b(cbn_resample** plan, int32_t n_rho, int32_t n_theta, int32_t n_phi,
                          int32_t rho_pad, int32_t side_lobes, const double* targets, int64_t m,
                          void* stream);
int cbn_resample_destroy(cbn_resample* plan);
int cbn_resample_apply(cbn_resample* plan, const void* lattice, void* values, void* stream);
int cbn_resample_transpose(cbn_resample* plan, const void* values, void* lattice, void* stream);

/* radial_fft / radial_ifft (radon_fourier.py:117-135): centred FFT (inverse=0)
 * or IFFT (inverse=1, includes 1/n) of `lines` contiguous complex64 lines of
 * length n [device], in place, times `scale` */
int cbn_radial_fft(void* data, int64_t n, int64_t lines, int32_t inverse, double scale,
                   void* stream);

/* per-rho complex weights (spectral_rho_derivative radon_fourier.py:111-114,
 * ramp_filter_radial 160-164, the fbp2d_nufft ramp 206-207): complex64 data
 * [device] viewed as [outer][n][inner], element (o, k, i) *= w[k]; w is host
 * float64 (re, im) pairs, n of them */
int cbn_line_weight(void* data, int64_t outer, int64_t n, int64_t inner, const double* w,
                    void* stream);

/* _center_phase (radon_fourier.py:52-56) applied in place: values[i] (complex64,
 * device) *= exp(+-i nodes[i] . shift) (minus when conj != 0), times w[i / w_inner]
 * when w (host float64) is given; nodes are host float64 m x d, d <= 3 */
int cbn_node_phase(void* values, const double* nodes, int64_t m, int32_t d, const double* shift,
                   int32_t conj, const double* w, int64_t w_inner, void* stream);

/* trilinear_transfer (radon_fourier.py:75-86): prod_d sinc^2(node_d / 2 pi) at the
 * unwrapped radial nodes, written float64 [phi][theta][rho] (node order) [device] */
int cbn_trilinear_transfer(int32_t n_rho, int32_t n_theta, int32_t n_phi, double delta_rho,
                           double voxel_mm, double* out, void* stream);

/* Host dtype conversion of the drop-in operators (float64 numpy <-> float32
 * staging), threaded outside the caller's interpreter lock; threads <= 0: all
 * cores.  gather: dst[k * elems + i] = (float)src[k][i] for n_src arrays. */
int cbn_host_gather_f64_to_f32(const double* const* src, int64_t n_src, int64_t elems, float* dst,
                               int32_t threads);
int cbn_host_f64_to_f32(const double* src, float* dst, int64_t n, int32_t threads);
int cbn_host_f32_to_f64(const float* src, double* dst, int64_t n, int32_t threads);

/* Elementwise pieces of the general Grangeat transforms (grangeat.py:131-170,
 * any plan_grangeat j / oversample): real lines in [outer][n] -> complex64
 * out = in * w[k] (w host float64, n of them); complex64 lines ->
 * float32 out = Re(in) * w[k]; and g -= mean of the frame's outermost ring
 * (grangeat.py:167-169), all on device buffers. */
int cbn_lines_real_in(const float* in, int64_t outer, int64_t n, const double* w, void* out,
                      void* stream);
int cbn_lines_real_out(const void* in, int64_t outer, int64_t n, const double* w, float* out,
                       void* stream);
int cbn_frame_ring_center(float* g, int32_t nu, int32_t nv, void* stream);

/* -------------------------------------------------------------- projector
 * Replaces ConeGeometry / ProjectorConfig / nufft_forward_project /
 * nufft_backproject (geometry.py:21-64, pipeline.py:31-212).
 */
typedef struct {
    double so_mm, sd_mm, det_width_mm, det_height_mm;
    int32_t nu, nv, n_views;
    double object_extent_mm;
} cbn_geometry;

typedef struct {
    int32_t n_rho, n_theta, n_phi;
    double rho_max;
} cbn_radial_spec;

typedef struct {
    int32_t method;            /* 0 = 'a' (NUFFT resample), 1 = 'b' (periodic sinc) */
    cbn_radial_spec spec;
    int32_t n_mu, n_t;
    double t_pitch_mm;         /* <= 0 : None (virtual pixel pitch) */
    int32_t t_taper;           /* 0 = none, 1 = hann */
    int32_t spectrum_j;
    int32_t resample_j[3];
    int32_t side_lobes;        /* method 'b': side_lobes + 1 taps per axis */
    double oversample_factor;
    int32_t rho_pad;           /* < 0 : None (n_rho / 2) */
    int32_t basis;             /* 0 = trilinear, 1 = dirac */
    double normalization, bp_normalization, den_tol;
    int64_t target_batch;      /* pipeline._TARGET_BATCH */
    int64_t plan_chunk;        /* nufft._PLAN_CHUNK */
    int32_t bp_n_t;            /* <= 0 : 2 nu (pipeline.py:168); else the t grid of */
    double bp_t_pitch_mm;      /* <= 0 : virtual pixel; the back-direction Grangeat */
} cbn_projector_config;

typedef struct cbn_projector_s cbn_projector;

/* direction: 1 = forward, 2 = backprojector, 3 = both.
 * n_vol / voxel_mm: volume edge and pitch (forward: the input volume; back:
 * out_size, voxel_mm of nufft_backproject). */
int cbn_projector_create(cbn_projector** proj, const cbn_geometry* geom,
                         const cbn_projector_config* cfg, int32_t n_vol, double voxel_mm,
                         int32_t direction);
int cbn_projector_destroy(cbn_projector* proj);
/* node-set sizes m whose scaling-fit rows the host must supply */
int cbn_projector_ls_sizes(const cbn_projector* proj, int64_t* sizes, int32_t* count);
int cbn_projector_set_ls_rows(cbn_projector* proj, int64_t m, const int64_t* rows, int64_t n);
/* bytes of device scratch the plan will hold once built */
/* volume edge N, view count and detector size of a plan (for hosts that
 * size buffers from the plan alone, e.g. cbnufft_b200_comm.h) */
int cbn_projector_info(const cbn_projector* proj, int32_t* n_vol, int32_t* n_views, int32_t* nu,
                       int32_t* nv);
int cbn_projector_scratch_bytes(const cbn_projector* proj, int64_t* bytes);

/* nufft_forward_project (pipeline.py:122-147): vol [device] float32 N^3 [ix,iy,iz]
 * -> frames [device] float32 (view_hi - view_lo) x nu x nv, views [view_lo, view_hi).
 * Batches keep the reference's boundaries.  Returns CBN_ENONFINITE if any
 * projection value is non-finite (checked on device, synchronises). */
int cbn_forward_project(cbn_projector* proj, const float* vol, float* frames,
                        int32_t view_lo, int32_t view_hi, void* stream);
/* cbn_forward_project without the final synchronisation, for a host that
 * copies frames out while later views are still computing: the call enqueues
 * every kernel and returns; the frames of each reverse-Grangeat block (views
 * [view_lo[k], view_hi[k]) relative to lo, from cbn_projector_blocks) are
 * complete once cbn_projector_block_sync(k) returns (host wait on that
 * block's event); cbn_forward_finish synchronises `stream` and returns
 * CBN_ENONFINITE if any projection value of the call was non-finite
 * (pipeline.py:144-145). */
int cbn_forward_project_async(cbn_projector* proj, const float* vol, float* frames, int32_t view_lo,
                              int32_t view_hi, void* stream);
/* Upload-overlapped input of nufft_forward_project (pipeline.py:122-147; the
 * spectrum NUFFT's input side, nufft.py:226-231): a host that converts and
 * copies the volume in chunks of its slowest axis calls cbn_forward_stage_volume
 * for rows [row_lo, row_hi) of `vol` (the full device volume; ascending
 * contiguous chunks starting at row 0, all on `stream`) as soon as the chunk
 * is enqueued: its rows are deapodised, padded and 2D-transformed while the
 * host converts the next chunk.  cbn_forward_project_staged_async then runs
 * the rest of the projection on the staged volume (CBN_EINVAL unless every
 * row has been staged; otherwise as cbn_forward_project_async).  Any other
 * forward call discards staged rows.  CBN_EUNSUPPORTED for node-sharded plans:
 * the caller falls back to cbn_forward_project_async. */
int cbn_forward_stage_volume(cbn_projector* proj, const float* vol, int32_t row_lo, int32_t row_hi,
                             void* stream);
int cbn_forward_project_staged_async(cbn_projector* proj, float* frames, int32_t view_lo,
                                     int32_t view_hi, void* stream);
int cbn_projector_blocks(cbn_projector* proj, int32_t* view_lo, int32_t* view_hi, int32_t* count);
int cbn_projector_block_sync(cbn_projector* proj, int32_t k);
int cbn_forward_finish(cbn_projector* proj, void* stream);

/* nufft_forward_project in two phases, for sharding the radial nodes and the
 * views across devices; cbn_forward_project == lattice(0 of 1)
 * + views.  lattice [device] complex64 x lattice_elems, caller-owned:
 * lattice: spectrum-gather values of node part `part` of `nparts` (zero at the
 *          other nodes, before the radial IFFT) -- sum the parts over ranks
 * views:   consumes the summed lattice; views [lo, hi) into frames [device]
 *          float32 (hi - lo) x nu x nv; CBN_ENONFINITE as cbn_forward_project */
int cbn_forward_lattice_size(cbn_projector* proj, int64_t* lattice_elems, void* stream);
/* Node-sharded forward plan: the spectrum plan (conjugate pairs, bins,
 * records) of a forward-only projector covers only the radial lines of share
 * `part` of `nparts` (contiguous in node order), and cbn_forward_lattice(part,
 * nparts) then writes only the lattice entries [*node_lo, *node_hi) -- equal
 * blocks in rank order, so the shares are assembled with an in-place
 * all-gather (SURVEY.md 8(e) forward step 4) instead of an all-reduce of the
 * whole zero-padded lattice.  CBN_EUNSUPPORTED when nparts does not divide the
 * line count; a sharded plan refuses every other forward entry point. */
int cbn_projector_set_node_shard(cbn_projector* proj, int32_t part, int32_t nparts,
                                 int64_t* node_lo, int64_t* node_hi, void* stream);
int cbn_forward_lattice(cbn_projector* proj, const float* vol, int32_t part, int32_t nparts,
                        void* lattice, void* stream);
int cbn_forward_views(cbn_projector* proj, void* lattice, float* frames, int32_t lo, int32_t hi,
                      void* stream);
/* nufft_backproject (pipeline.py:150-212): frames [device] float32 V x nu x nv
 * -> vol [device] float32 N^3 */
int cbn_backproject(cbn_projector* proj, const float* frames, float* vol, void* stream);

/* Upload-overlapped nufft_backproject: the forward Grangeat step of views
 * [lo, hi) runs as soon as their frames are on the device (frames [device]
 * float32 (hi - lo) x nu x nv, the views themselves), while the host still
 * converts and copies later views; the next cbn_backproject on the same
 * stream consumes the staged views once all n_views have been staged (and
 * drops a partial staging).  Views arrive in order, blocks start on 32-view
 * bounds.  CBN_EUNSUPPORTED (nothing staged) where the plan has more than one
 * resample scaling group or uses method B: call cbn_backproject alone. */
int cbn_backproject_stage_views(cbn_projector* proj, const float* frames, int32_t lo, int32_t hi,
                                void* stream);

/* nufft_backproject in three phases, for sharding views and nodes across
 * devices; cbn_backproject == views(all) + finish(0 of 1) +
 * crop.  Buffers [device] complex64, caller-owned:
 *   lattice: lattice_elems  (padded-lattice accumulator; sum it over ranks)
 *   grid:    grid_elems     ((2N)^3 adjoint grid; sum it over ranks)
 * views:  transposed resample of views [lo, hi) -- `frames` holds those views
 *         (hi - lo frames of nu x nv) -- into `lattice` (overwritten)
 * finish: consumes the summed `lattice`; spreads part `part` of `nparts`
 *         of the radial nodes into `grid` (overwritten)
 * crop:   consumes the summed `grid`; vol [device] float32 N^3 */
int cbn_backproject_sizes(cbn_projector* proj, int64_t* lattice_elems, int64_t* grid_elems,
                          void* stream);
int cbn_backproject_views(cbn_projector* proj, const float* frames, int32_t lo, int32_t hi,
                          void* lattice, void* stream);
int cbn_backproject_finish(cbn_projector* proj, void* lattice, int32_t part, int32_t nparts,
                           void* grid, void* stream);
int cbn_backproject_crop(cbn_projector* proj, void* grid, float* vol, void* stream);

/* Phase 3 distributed by slabs of the slowest grid axis (x planes; SURVEY.md
 * 8(e) adjoint steps 4-6: reduce-scatter of the grid by slab, slab IFFT,
 * all-to-all transpose, column IFFT, crop).  Replaces cbn_backproject_crop
 * when the summed grid is reduce-scattered instead of all-reduced.  With
 * K = 2N and the balanced split y0_d = d * N / nparts:
 * crop_slab: slab [device] = grid planes [x_lo, x_hi) (consumed): 2D inverse
 *            FFT per plane, y/z crop + deapodisation; send [device]
 *            (x_hi - x_lo) * N * N complex64 laid out [d][x][y - y0_d][z],
 *            chunk d (contiguous) goes to the rank owning y range d.
 * crop_cols: cols [device] [K][y_hi - y_lo][N] complex64 = the chunks
 *            received from every slab in x order (consumed): inverse FFT
 *            along x, x crop + deapodisation, Re, * bp_normalization;
 *            vol_part [device] float32 [N][y_hi - y_lo][N]. */
int cbn_backproject_crop_slab(cbn_projector* proj, void* slab, int32_t x_lo, int32_t x_hi,
                              int32_t nparts, void* send, void* stream);
int cbn_backproject_crop_cols(cbn_projector* proj, void* cols, int32_t y_lo, int32_t y_hi,
                              float* vol_part, void* stream);

/* Diagnostics: the forward plan's per-node Grangeat records in bin-sorted
 * order (56-byte records: int16 lu, lv; int32 col; float2 factor; float w[10])
 * and the sorted node ids [host]; *m in: capacity, out: node count. */
int cbn_projector_grangeat_records(cbn_projector* proj, void* records, int32_t* perm, int64_t* m,
                                   void* stream);

/* Stage entry points (for stage parity and the mirrored module API). */
/* image_to_radial_spectrum (radon_fourier.py:89-108): complex64 node-order
 * values (n_phi, n_theta, n_rho), centre phase applied, no basis transfer */
int cbn_projector_radial_spectrum(cbn_projector* proj, const float* vol, void* spectrum,
                                  void* stream);
/* _radial_lattice (pipeline.py:113-119): complex64 lattice, layout
 * (n_phi, n_theta, n_rho) -- rho fastest, i.e. node order. */
int cbn_projector_radial_lattice(cbn_projector* proj, const float* vol, void* lattice,
                                 void* stream);
/* resample_apply of method A for the umbrella targets of views [lo, hi) with the
 * reference's per-batch plans (resampling.py:136-148, pipeline.py:130-137):
 * lattice [device] as above -> values [device] float32 (hi-lo) x n_mu x n_t */
int cbn_projector_resample_views(cbn_projector* proj, const void* lattice, float* values,
                                 int32_t view_lo, int32_t view_hi, void* stream);
/* reverse_grangeat_view for a block of views (grangeat.py:149-170):
 * values float32 (nv_blk x n_mu x n_t) -> frames float32 (nv_blk x nu x nv) */
int cbn_projector_grangeat_reverse(cbn_projector* proj, const float* values, float* frames,
                                   int32_t n_views_blk, void* stream);
/* forward_grangeat_view for a block of views (grangeat.py:131-146) with the
 * backprojector's t grid: frames -> values float32 (nv_blk x n_mu x 2 nu) */
int cbn_projector_grangeat_forward(cbn_projector* proj, const float* frames, float* values,
                                   int32_t n_views_blk, void* stream);

/* Stage parity of the backprojector (pipeline.py:174-184): the forward
 * Grangeat step and the transposed resample of views [lo, hi) (frames [device]
 * float32 (hi - lo) x nu x nv), summed over the range's view batches, after
 * the lattice inverse FFT, the rho crop and the origin average
 * (resampling.py:164-196): num [device] complex64 = sum of
 * resample_transpose(values), den [device] float32 = sum of
 * Re resample_transpose(valid); both in node order (n_phi, n_theta, n_rho)
 * of the backprojector's radial spec.  Either output may be NULL.
 * Synchronises. */
int cbn_backproject_stage_transpose(cbn_projector* proj, const float* frames, int32_t lo,
                                    int32_t hi, void* num, float* den, void* stream);

/* Plan diagnostics (test/bench support; not on the operator path).
 * first_indices: per-axis first-tap index mod K (nufft.py:171-179) of a node
 * set exactly as the projector's kernels use it -- the reference's
 * plan_nufft(...).interp.indices[:, 0] decoded per axis.  set: 0 forward
 * radial lattice nodes (J = spectrum_j, radon_fourier.py:89-108); 1 forward
 * umbrella targets of view batch `batch` (J = resample_j, (rho, theta, phi)
 * order, resampling.py:79-103); 2 forward polar Grangeat nodes (J = 5,
 * grangeat.py:93-128); 3-5 the same sets of the backprojector
 * (pipeline.py:165-210).  out [host] int32 m x d, or NULL to query *m;
 * *m in: capacity (rows), out: node count.  Synchronises. */
int cbn_projector_first_indices(cbn_projector* proj, int32_t set, int32_t batch, int32_t* out,
                                int64_t* m, void* stream);
/* Plan statistics as ';'-separated names and int64 values (-1: that part of
 * the plan is not built yet): primary nodes of the conjugate-pair gathers,
 * resample rho planes used, invalid umbrella targets per view, batch scaling
 * groups, reverse-Grangeat heavy cells, ...  Synchronises. */
/* Diagnostics: copy the named plan buffer (den_cache, den_max, bspec_s32,
 * ramp_q, bpairs, bspec_perm, bspec_subs, bbatch_s32, fspec_s32, values_t, lattice,
 * den_keep) to
 * host memory `out` (null: only report its size in *bytes) */
int cbn_projector_debug_buffer(cbn_projector* proj, const char* name, void* out, int64_t* bytes,
                               void* stream);
int cbn_projector_plan_stats(cbn_projector* proj, int64_t* vals, int32_t* count, char* names,
                             int32_t names_len, void* stream);

/* Per-stage CUDA-event timing: enable (1) / disable (0); when enabled every
 * operator call records events per stage, and the operators run their view
 * blocks on the caller's stream only (no second overlapping stream), so each
 * stage's event time is its kernels' own time.  stage_times synchronises and
 * returns the accumulated milliseconds per stage since the last reset
 * (names: ';'-separated), then resets if `reset` is non-zero. */
int cbn_projector_set_timing(cbn_projector* proj, int32_t on);
int cbn_projector_stage_times(cbn_projector* proj, double* ms, int32_t* count,
                              char* names, int32_t names_len, int32_t reset);

/* Algorithmic bytes per stage accumulated while timing is on (the bench's
 * roofline): compulsory HBM bytes and on-chip tap bytes of the work each
 * stage's kernels did; names ';'-separated; clears the
 * totals if `reset` is non-zero. */
int cbn_projector_stage_bytes(cbn_projector* proj, double* hbm, double* chip, int32_t* count,
                              char* names, int32_t names_len, int32_t reset);

/* ------------------------------------------------------------ baseline
 * ct_project_linear (baseline.py:52-98): ray-driven cone-beam projection with
 * trilinear volume sampling, N midpoint samples per clipped chord -- the
 * projector calibrate_bp_normalization runs (pipeline.py:245-257).
 * vol [device] float32 n^3 [ix][iy][iz]; frames [device] float32
 * n_views x nu x nv. */
int cbn_ct_project_linear(const cbn_geometry* geom, const float* vol, int32_t n, double voxel_mm,
                          float* frames, void* stream);

/* Number of kernels this library has launched in the process (cuFFT's own
 * kernels are not counted). */
long long cbn_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* CBNUFFT_B200_H */
