/* cbnufft_b200_comm.h -- multi-GPU operators over NCCL behind the C ABI.
 *
 * A separate library (libcbnufft_b200_comm.so, linked against
 * libcbnufft_b200.so and NCCL) so that single-GPU hosts never load NCCL.
 * One process per GPU; every call is stream-ordered: the collectives are
 * enqueued on `stream` between the projector phases of cbnufft_b200.h
 * (SURVEY.md 8(e)).  The reference has no multi-device path; these replace
 * the per-rank orchestration a non-Python host would otherwise rebuild
 * around cbn_forward_lattice / cbn_forward_views / cbn_backproject_views /
 * cbn_backproject_finish / cbn_backproject_crop_slab / cbn_backproject_crop_cols.
 *
 * Status codes are those of cbnufft_b200.h; NCCL failures return CBN_ENCCL
 * (5), with the NCCL error string in cbn_comm_last_error().
 */
#ifndef CBNUFFT_B200_COMM_H
#define CBNUFFT_B200_COMM_H

#include <stdint.h>

#include "cbnufft_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define CBN_COMM_ID_BYTES 128 /* sizeof(ncclUniqueId) */

typedef struct cbn_comm_s cbn_comm;

const char* cbn_comm_last_error(void);

/* rank 0 creates the id and hands it to every rank (any out-of-band channel) */
int cbn_comm_unique_id(void* id_out);

/* collective over `nranks` processes, one GPU each (the current device) */
int cbn_comm_init(cbn_comm** comm, const void* id, int32_t nranks, int32_t rank);
int cbn_comm_destroy(cbn_comm* comm);
int cbn_comm_rank(const cbn_comm* comm, int32_t* rank, int32_t* nranks);

/* nufft_forward_project sharded over the communicator (pipeline.py:122-147):
 *  - vol [device] float32 N^3: rank 0's volume, broadcast into every rank's;
 *  - each rank gathers the spectrum at its 1/nranks share of the radial
 *    nodes, the shares are summed with one all-reduce of the lattice;
 *  - frames [device] float32 (hi - lo) x nu x nv: this rank's views [lo, hi).
 * CBN_ENONFINITE as cbn_forward_project. */
int cbn_forward_project_sharded(cbn_projector* proj, cbn_comm* comm, float* vol, float* frames,
                                int32_t view_lo, int32_t view_hi, void* stream);

/* nufft_backproject sharded over the communicator (pipeline.py:150-212):
 * frames [device] float32 (hi - lo) x nu x nv = this rank's views; the
 * padded-lattice accumulators are all-reduced, each rank spreads its share of
 * the radial nodes into a (2N)^3 grid, the grids are reduce-scattered by
 * x slabs, each slab is inverse-transformed and cropped in y/z, an all-to-all
 * (grouped send/recv) moves the chunks to y-range owners, the x transform and
 * crop finish each y range, and an all-gather assembles the volume:
 * vol [device] float32 N^3 on every rank. */
int cbn_backproject_sharded(cbn_projector* proj, cbn_comm* comm, const float* frames,
                            int32_t view_lo, int32_t view_hi, float* vol, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CBNUFFT_B200_COMM_H */
