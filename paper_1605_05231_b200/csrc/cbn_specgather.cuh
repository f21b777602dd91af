// Spectrum gather of the forward projector from per-point records.
//
// The radial spectrum gather (nufft_forward onto the radial lattice,
// nufft.py:221-233 + radon_fourier.py:89-119) is the same binned J^3 KB
// gather as k_gather_binned<3, J, RadialPackedSrc, SpecOut, HALF>, with two
// changes that remove most of its non-tap instructions:
//  * everything a point needs that depends on geometry only is computed once
//    per plan (k_spec_records) and streamed in bin-sorted order: the tap
//    origin inside the tile, the per-axis KB polynomial argument y and the
//    reference's edge-tap support decision, the epilogue factor
//    i * omega * sinc^2 transfer * centre/plan phase (float64, rounded once),
//    and the lattice output index (plus the conjugate mirror's).  32 bytes
//    per primary node replace the float64 node generation, wrapping, index
//    math, sincos and sinc evaluation of every step;
//  * the half-spectrum tile is filled row by row: a warp owns a region row,
//    its lanes are the row's cells along the fastest axis, so a lane's wrapped
//    column (and whether it reads the conjugate mirror) is fixed for the whole
//    fill and each cell costs an address add and one cp.async.
#pragma once

#include "cbn_binned.cuh"

namespace cbn {

struct SpecRec {
    const float4* rec;   // y0, y1, y2, bits (l0 | l1 << 5 | l2 << 10 | edge-tap drops << 15)
    const float2* fac;   // epilogue factor
    const int2* out;     // lattice index, conjugate-mirror index (-1: none)
};

constexpr int kSpecMaxRows = 512;   // region rows R0 x R1 (13 x 21 at J = 6)

template <int J>
__global__ void __launch_bounds__(256, 3)
k_spec_gather(const float2* __restrict__ grid, KBSet kb, TileGeom<3> tg, SpecRec r,
              float2* __restrict__ lat, const SubProblem* __restrict__ subs) {
    extern __shared__ float2 tile[];
    // grid offsets of the region rows, direct and conjugate-mirrored
    __shared__ long long rowoff[2][kSpecMaxRows];
    const SubProblem sp = subs[blockIdx.x];
    if (sp.count == 0) return;
    int o[3];
    bin_origin<3>(tg, sp.bin, o);
    const int R1 = tg.R[1], R2 = tg.R[2], P2 = tg.P;
    const int rows = tg.R[0] * R1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int K0 = tg.K[0], K1 = tg.K[1], K2 = tg.K[2], h2 = K2 / 2 + 1;
    for (int row = threadIdx.x; row < rows; row += blockDim.x) {
        const int r0 = row / R1, r1 = row - r0 * R1;
        const int i0 = wrapc(o[0] + r0, K0), i1 = wrapc(o[1] + r1, K1);
        rowoff[0][row] = ((long long)i0 * K1 + i1) * h2;
        rowoff[1][row] = ((long long)(i0 ? K0 - i0 : 0) * K1 + (i1 ? K1 - i1 : 0)) * h2;
    }
    // this lane's column of every region row
    const bool col = lane < R2;
    int i2 = wrapc(o[2] + lane, K2);
    const bool mir = col && i2 >= h2;   // read as conj(G[-k])
    if (mir) i2 = K2 - i2;
    __syncthreads();
    if (col) {
        const long long* ro = rowoff[mir ? 1 : 0];
        const float2* src = grid + i2;
        unsigned dst = (unsigned)__cvta_generic_to_shared(tile + warp * P2 + lane);
        const unsigned dstep = 8u * (unsigned)P2 * sizeof(float2);
        for (int row = warp; row < rows; row += 8, dst += dstep) {
            CBN_DCHECK(ro[row] + i2 < (long long)K0 * K1 * h2, "spec fill: cell");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src + ro[row]));
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (mir)
        for (int row = warp; row < rows; row += 8) tile[row * P2 + lane].y = -tile[row * P2 + lane].y;
    __syncthreads();
    for (int k = threadIdx.x; k < sp.count; k += blockDim.x) {
        const int64_t pos = (int64_t)sp.start + k;
        const float4 q = r.rec[pos];
        const unsigned bits = __float_as_uint(q.w);
        const int l0 = bits & 31, l1 = (bits >> 5) & 31, l2 = (bits >> 10) & 31;
        CBN_DCHECK(l0 < tg.T[0] && l1 < tg.T[1] && l2 < tg.T[2], "spec gather: point outside tile");
        float wt[3][J];
        kb_weights_y<J>(kb.ax[0], q.x, (bits >> 15) & 1, wt[0]);
        kb_weights_y<J>(kb.ax[1], q.y, (bits >> 16) & 1, wt[1]);
        kb_weights_y<J>(kb.ax[2], q.z, (bits >> 17) & 1, wt[2]);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < J; ++a) {
            float2 pa = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < J; ++b) {
                const float2* row = tile + ((l0 + a) * R1 + l1 + b) * P2 + l2;
                float2 s = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < J; ++c) {
                    const float2 g = row[c];
                    s.x = fmaf(wt[2][c], g.x, s.x);
                    s.y = fmaf(wt[2][c], g.y, s.y);
                }
                pa.x = fmaf(wt[1][b], s.x, pa.x);
                pa.y = fmaf(wt[1][b], s.y, pa.y);
            }
            acc.x = fmaf(wt[0][a], pa.x, acc.x);
            acc.y = fmaf(wt[0][a], pa.y, acc.y);
        }
        const float2 v = cmul(acc, r.fac[pos]);
        const int2 oi = r.out[pos];
        lat[oi.x] = v;
        if (oi.y >= 0) lat[oi.y] = make_float2(v.x, -v.y);
    }
}

}  // namespace cbn
