// Multi-GPU operators over NCCL (include/cbnufft_b200_comm.h).
//
// Orchestration only: the projector phases are the C ABI of
// libcbnufft_b200.so; between them this library enqueues the NCCL
// collectives of SURVEY.md 8(e) on the caller's stream, so a whole sharded
// projection is one stream-ordered call (no host round trip except the
// phase functions' own one-time plan steps).  Scratch buffers are owned by the
// communicator and grow to the largest plan it has served.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/cbnufft_b200_comm.h"

namespace {

thread_local std::string g_err;

struct CommError : std::runtime_error {
    int code;
    CommError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int fail(const std::exception& e) {
    g_err = e.what();
    if (auto* c = dynamic_cast<const CommError*>(&e)) return c->code;
    return CBN_ECUDA;
}

#define COMM_NCCL(expr)                                                                   \
    do {                                                                                  \
        ncclResult_t r_ = (expr);                                                         \
        if (r_ != ncclSuccess)                                                            \
            throw CommError(CBN_ENCCL, std::string(#expr ": ") + ncclGetErrorString(r_)); \
    } while (0)

#define COMM_CUDA(expr)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw CommError(e_ == cudaErrorMemoryAllocation ? CBN_ENOMEM : CBN_ECUDA,     \
                            std::string(#expr ": ") + cudaGetErrorString(e_));            \
    } while (0)

// a projector phase: propagate its status and message
#define COMM_PHASE(expr)                                                                  \
    do {                                                                                  \
        int st_ = (expr);                                                                 \
        if (st_ != CBN_OK) throw CommError(st_, std::string(#expr ": ") + cbn_last_error()); \
    } while (0)

struct Buf {
    void* p = nullptr;
    size_t n = 0;
    ~Buf() {
        if (p) cudaFree(p);
    }
    void* get(size_t bytes) {
        if (bytes > n) {
            if (p) COMM_CUDA(cudaFree(p));
            p = nullptr;
            COMM_CUDA(cudaMalloc(&p, bytes));
            n = bytes;
        }
        return p;
    }
};

// parts[d] = [N][cap][N] (y rows beyond the part's own count unused) -> vol [N][N][N]
__global__ void k_assemble_y(const float* __restrict__ parts, int n, int cap, const int* __restrict__ y0,
                             int world, float* __restrict__ vol) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)n * n * n;
    if (e >= total) return;
    const int z = (int)(e % n);
    const int y = (int)((e / n) % n);
    const int x = (int)(e / ((int64_t)n * n));
    int d = 0;
    while (d + 1 < world && y >= y0[d + 1]) ++d;
    vol[e] = parts[(((int64_t)d * n + x) * cap + (y - y0[d])) * n + z];
}

}  // namespace

struct cbn_comm_s {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1;
    Buf lattice, grid, slab, send, cols, part, gathered, y0;
};

extern "C" {

const char* cbn_comm_last_error(void) { return g_err.c_str(); }

int cbn_comm_unique_id(void* id_out) {
    try {
        if (!id_out) throw CommError(CBN_EINVAL, "null argument");
        static_assert(sizeof(ncclUniqueId) == CBN_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        COMM_NCCL(ncclGetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_comm_init(cbn_comm** out, const void* id, int32_t nranks, int32_t rank) {
    try {
        if (!out || !id) throw CommError(CBN_EINVAL, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw CommError(CBN_EINVAL, "bad rank");
        auto* c = new cbn_comm_s();
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            throw CommError(CBN_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
        c->rank = rank;
        c->nranks = nranks;
        *out = c;
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_comm_destroy(cbn_comm* c) {
    if (!c) return CBN_OK;
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
    return CBN_OK;
}

int cbn_comm_rank(const cbn_comm* c, int32_t* rank, int32_t* nranks) {
    if (!c) {
        g_err = "null argument";
        return CBN_EINVAL;
    }
    if (rank) *rank = c->rank;
    if (nranks) *nranks = c->nranks;
    return CBN_OK;
}

int cbn_forward_project_sharded(cbn_projector* p, cbn_comm* c, float* vol, float* frames,
                                int32_t lo, int32_t hi, void* stream) {
    try {
        if (!p || !c || !vol || (!frames && hi > lo)) throw CommError(CBN_EINVAL, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        int32_t n = 0, views = 0;
        COMM_PHASE(cbn_projector_info(p, &n, &views, nullptr, nullptr));
        if (lo < 0 || hi > views || lo > hi) throw CommError(CBN_EINVAL, "view range out of bounds");
        const size_t nvox = (size_t)n * n * n;
        // 1. the volume from rank 0 (SURVEY.md 8(e) forward step 1)
        if (c->nranks > 1) COMM_NCCL(ncclBroadcast(vol, vol, nvox, ncclFloat, 0, c->nccl, s));
        // 2-4. this rank's share of the radial nodes: with a forward-only plan
        //      whose lines split evenly, a node-sharded plan writes just its
        //      lattice block and an in-place all-gather assembles the lattice;
        //      otherwise a share of the bin subproblems, summed by all-reduce
        int64_t m = 0;
        COMM_PHASE(cbn_forward_lattice_size(p, &m, stream));
        auto* lat = static_cast<float*>(c->lattice.get(sizeof(float) * 2 * (size_t)m));
        int64_t nlo = 0, nhi = 0;
        const int st = c->nranks > 1
                           ? cbn_projector_set_node_shard(p, c->rank, c->nranks, &nlo, &nhi, stream)
                           : CBN_EUNSUPPORTED;
        COMM_PHASE(cbn_forward_lattice(p, vol, c->rank, c->nranks, lat, stream));
        if (st == CBN_OK) {
            COMM_NCCL(ncclAllGather(lat + 2 * nlo, lat, 2 * (size_t)(nhi - nlo), ncclFloat, c->nccl, s));
        } else if (c->nranks > 1) {
            COMM_NCCL(ncclAllReduce(lat, lat, 2 * (size_t)m, ncclFloat, ncclSum, c->nccl, s));
        }
        // 5. this rank's views
        if (hi > lo) COMM_PHASE(cbn_forward_views(p, lat, frames, lo, hi, stream));
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int cbn_backproject_sharded(cbn_projector* p, cbn_comm* c, const float* frames, int32_t lo,
                            int32_t hi, float* vol, void* stream) {
    try {
        if (!p || !c || !vol || (!frames && hi > lo)) throw CommError(CBN_EINVAL, "null argument");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int world = c->nranks, rank = c->rank;
        int32_t n = 0, views = 0;
        COMM_PHASE(cbn_projector_info(p, &n, &views, nullptr, nullptr));
        if (lo < 0 || hi > views || lo > hi) throw CommError(CBN_EINVAL, "view range out of bounds");
        int64_t L = 0, G = 0;
        COMM_PHASE(cbn_backproject_sizes(p, &L, &G, stream));
        // 1-2. this rank's views into the accumulator, summed over ranks
        auto* acc = c->lattice.get(sizeof(float) * 2 * (size_t)L);
        if (hi > lo) {
            COMM_PHASE(cbn_backproject_views(p, frames, lo, hi, acc, stream));
        } else {
            COMM_CUDA(cudaMemsetAsync(acc, 0, sizeof(float) * 2 * (size_t)L, s));
        }
        if (world > 1) COMM_NCCL(ncclAllReduce(acc, acc, 2 * (size_t)L, ncclFloat, ncclSum, c->nccl, s));
        // 3. this rank's share of the radial nodes spread into its own grid
        auto* grid = static_cast<float*>(c->grid.get(sizeof(float) * 2 * (size_t)G));
        COMM_PHASE(cbn_backproject_finish(p, acc, rank, world, grid, stream));
        if (world == 1) {
            COMM_PHASE(cbn_backproject_crop(p, grid, vol, stream));
            return CBN_OK;
        }
        // 4. grids reduce-scattered by x slab (all-reduce + own slab when the
        //    rank count does not divide K)
        const int64_t K = std::llround(std::cbrt((double)G));
        if (K * K * K != G) throw CommError(CBN_EINVAL, "grid is not a cube");
        const int64_t plane = K * K;
        std::vector<int64_t> xs(world + 1), ys(world + 1);
        for (int r = 0; r <= world; ++r) {
            xs[r] = K * r / world;
            ys[r] = (int64_t)n * r / world;
        }
        const int64_t xc = xs[rank + 1] - xs[rank], yc = ys[rank + 1] - ys[rank];
        float* slab;
        if (K % world == 0) {
            slab = static_cast<float*>(c->slab.get(sizeof(float) * 2 * (size_t)(plane * xc)));
            COMM_NCCL(ncclReduceScatter(grid, slab, 2 * (size_t)(plane * xc), ncclFloat, ncclSum,
                                        c->nccl, s));
        } else {
            COMM_NCCL(ncclAllReduce(grid, grid, 2 * (size_t)G, ncclFloat, ncclSum, c->nccl, s));
            slab = grid + 2 * xs[rank] * plane;
        }
        // 5. slab IFFT + y/z crop, chunk d for the owner of y range d
        auto* send = static_cast<float*>(c->send.get(sizeof(float) * 2 * (size_t)(xc * n * n)));
        COMM_PHASE(cbn_backproject_crop_slab(p, slab, (int32_t)xs[rank], (int32_t)xs[rank + 1], world,
                                             send, stream));
        //    all-to-all as grouped send/recv: rank q's x slab of my y range
        auto* cols = static_cast<float*>(c->cols.get(sizeof(float) * 2 * (size_t)(K * yc * n)));
        COMM_NCCL(ncclGroupStart());
        int64_t soff = 0, roff = 0;
        for (int d = 0; d < world; ++d) {
            const int64_t sc = xc * (ys[d + 1] - ys[d]) * n;       // complex elements to d
            const int64_t rc = (xs[d + 1] - xs[d]) * yc * n;       // complex elements from d
            COMM_NCCL(ncclSend(send + 2 * soff, 2 * (size_t)sc, ncclFloat, d, c->nccl, s));
            COMM_NCCL(ncclRecv(cols + 2 * roff, 2 * (size_t)rc, ncclFloat, d, c->nccl, s));
            soff += sc;
            roff += rc;
        }
        COMM_NCCL(ncclGroupEnd());
        // 6. x IFFT + crop of my y range, then every rank gets the volume
        int64_t cap = 0;
        for (int d = 0; d < world; ++d) cap = std::max(cap, ys[d + 1] - ys[d]);
        const size_t part_elems = (size_t)n * cap * n;
        auto* part = static_cast<float*>(c->part.get(sizeof(float) * part_elems));
        COMM_PHASE(cbn_backproject_crop_cols(p, cols, (int32_t)ys[rank], (int32_t)ys[rank + 1], part,
                                             stream));
        if (yc < cap) {
            // crop_cols wrote [N][yc][N]; spread it to the [N][cap][N] gather layout
            auto* tmp = static_cast<float*>(c->slab.get(sizeof(float) * part_elems));
            COMM_CUDA(cudaMemcpy2DAsync(tmp, sizeof(float) * cap * n, part, sizeof(float) * yc * n,
                                        sizeof(float) * yc * n, n, cudaMemcpyDeviceToDevice, s));
            part = tmp;
        }
        auto* gathered = static_cast<float*>(c->gathered.get(sizeof(float) * part_elems * world));
        COMM_NCCL(ncclAllGather(part, gathered, part_elems, ncclFloat, c->nccl, s));
        std::vector<int> y0(world);
        for (int d = 0; d < world; ++d) y0[d] = (int)ys[d];
        auto* dy0 = static_cast<int*>(c->y0.get(sizeof(int) * world));
        COMM_CUDA(cudaMemcpyAsync(dy0, y0.data(), sizeof(int) * world, cudaMemcpyHostToDevice, s));
        const int64_t total = (int64_t)n * n * n;
        k_assemble_y<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gathered, n, (int)cap, dy0, world,
                                                                   vol);
        COMM_CUDA(cudaGetLastError());
        return CBN_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
