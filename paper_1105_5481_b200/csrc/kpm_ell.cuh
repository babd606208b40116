// kpm_ell.cuh -- fused recursion step for a general sparse H~ in ELL form.
//
// Same arithmetic as kpm_step_kernel<EllOp, STEP> (Eq 18 + the doubling inner
// products) with the row entries staged through shared memory: the CTA walks tiles
// of TILE = TS * kEllSPW consecutive rows; while it computes tile i, one thread copies
// the column indices and values of tile i+gridDim.x into the other half of a double
// buffer with 2 K bulk copies (cp.async.bulk, completion on an mbarrier; the [K][ld]
// device layout makes every entry column's tile slice one aligned contiguous run), so
// the gathers of a row never wait behind the load of their index and no other thread
// spends instructions on the staging (ncu r02: the per-element cp.async staging with its
// index arithmetic was ~60 of 172 warp instructions per row).
// One warp row of threads owns the 16-byte vector lanes of a row (one matrix entry
// serves all R vectors, BJ north_star); each thread keeps 8 gathers in flight.
#pragma once
#include <type_traits>

#include "kpm_kernels.cuh"
#include "kpm_tma.cuh"

namespace kpm {

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int kEllKMax = 16;  // rows with more entries use the generic step kernel
constexpr int kEllSPW = 4;    // rows per thread row per tile

__device__ __forceinline__ void cp_async(void* dst, const void* src, int bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    if (bytes == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
    else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ inline size_t ell_smem_bytes(int nthr, int TS, int K, bool cplx) {
    const size_t tile = (size_t)TS * kEllSPW;
    return 3 * (size_t)nthr * 16 + 2 * (size_t)K * tile * 4 + 16 + 2 * (size_t)K * tile * (cplx ? 16 : 8);
}

// KMAX: compile-time bound on the entries per row (4, 8 or 16; the row's K <= KMAX entries are
// unrolled, entries k >= K skipped by a CTA-uniform branch).  U rows per thread are processed
// together -- all their gathers issued before any is consumed -- so a thread keeps up to
// U (KMAX + 2) 16-byte loads in flight (ncu r01: the one-row-at-a-time loop with 8-entry padded
// chunks issued 196 warp instructions per row and stalled on L1TEX latency at 39% DRAM).  One
// 512-thread CTA per SM (128 registers hold the loads in flight).
template <bool CPLX, int KMAX, bool WIDE>
__global__ void __launch_bounds__(512, 1) kpm_ell_step_kernel(const EllOp<CPLX> op, const VecArgs v, const int tail) {
    pdl_entry();
    constexpr int U = KMAX == 4 ? 4 : (KMAX == 8 ? 2 : 1);  // U (K + 2) double2 in flight: 24, 20, 18
    static_assert(kEllSPW % U == 0, "rows per thread");
    // element offsets j * RG + rg in 32 bits unless the extended block has 2^31 lanes or more (WIDE)
    using off_t = typename std::conditional<WIDE, long long, unsigned>::type;
    const int TR = blockDim.x, TS = blockDim.y;
    const int nthr = TR * TS, tid = threadIdx.y * TR + threadIdx.x;
    const int rg = blockIdx.y * TR + threadIdx.x;
    const bool active = rg < v.RG;
    const int K = op.K, D = op.D;
    const off_t RG = (off_t)v.RG;
    const int TILE = TS * kEllSPW;
    extern __shared__ double2 sred[];                                     // [3][nthr]
    int* scol = reinterpret_cast<int*>(sred + 3 * nthr);                 // [2][K][TILE]
    const size_t vofs = ((size_t)2 * K * TILE * 4 + 15) / 16 * 16;
    unsigned char* sval = reinterpret_cast<unsigned char*>(scol) + vofs; // [2][K][TILE] double or double2
    constexpr int vb = CPLX ? 16 : 8;
    const int ntiles = (D + TILE - 1) / TILE;
    const double2* __restrict__ Cl = v.C + rg;  // this thread's lane of row 0
    double2* __restrict__ Pl = v.P + rg;

    __shared__ uint64_t sbar[2];
    // thread 0: the tile's K column slices and K value slices (the pad rows past D included)
    auto prefetch = [&](int tile, int buf) {
        mbar_expect_tx(sbar + buf, (uint32_t)K * TILE * (4 + vb));
        for (int k = 0; k < K; ++k) {
            const size_t ge = (size_t)k * op.ld + (size_t)tile * TILE;
            bulk_g2s(scol + ((size_t)buf * K + k) * TILE, op.col + ge, TILE * 4, sbar + buf);
            bulk_g2s(sval + ((size_t)buf * K + k) * TILE * vb, reinterpret_cast<const unsigned char*>(op.val) + ge * vb,
                     TILE * vb, sbar + buf);
        }
    };

    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
    int tile = blockIdx.x;
    if (tid == 0) {
        mbar_init(sbar, 1);
        mbar_init(sbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (tile < ntiles) prefetch(tile, 0);
    }
    __syncthreads();
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        mbar_wait(sbar + buf, (uint32_t)((it >> 1) & 1));
        __syncthreads();  // this tile's entries are in smem; nobody reads the other buffer any more
        if (tid == 0 && tile + (int)gridDim.x < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
            prefetch(tile + gridDim.x, buf ^ 1);
        }
        if (!active) continue;
        const int* tc = scol + (size_t)buf * K * TILE;
        const unsigned char* tv = sval + (size_t)buf * K * TILE * vb;
        const int nrow = min(TILE, D - tile * TILE);
#pragma unroll 1
        for (int u0 = 0; u0 < kEllSPW; u0 += U) {
            int ii[U];
            double2 x[U], p[U], xj[U][KMAX];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int i = threadIdx.y + (u0 + q) * TS;
                ii[q] = i < nrow ? i : 0;  // (ragged last tile: row 0's loads, result unused)
                const off_t o = (off_t)(tile * TILE + ii[q]) * RG;
                x[q] = __ldg(Cl + o);
                p[q] = __ldcs(Pl + o);
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (k < K) xj[q][k] = __ldg(Cl + (off_t)tc[k * TILE + ii[q]] * RG);
            }
#pragma unroll
            for (int q = 0; q < U; ++q) {
                if (threadIdx.y + (u0 + q) * TS >= nrow) continue;
                double2 h = scale2(op.shift, x[q]);
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    if (k >= K) break;
                    if (CPLX) h = add2(h, cmul(reinterpret_cast<const double2*>(tv)[k * TILE + ii[q]], xj[q][k]));
                    else h = fma2(reinterpret_cast<const double*>(tv)[k * TILE + ii[q]], xj[q][k], h);
                }
                const double2 y = make_double2(fma(2.0, h.x, -p[q].x), fma(2.0, h.y, -p[q].y));  // Eq 18
                __stcs(Pl + (off_t)(tile * TILE + ii[q]) * RG, y);
                dot_acc<CPLX>(acc0, x[q], x[q]);
                dot_acc<CPLX>(acc1, x[q], y);
                if (tail) dot_acc<CPLX>(acc2, y, y);
            }
        }
    }
    __syncthreads();
    sred[tid] = acc0;
    sred[nthr + tid] = acc1;
    sred[2 * nthr + tid] = acc2;
    __syncthreads();
    if (threadIdx.y == 0 && active) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double* rowk = k == 0 ? v.red0 : (k == 1 ? v.red1 : (tail ? v.red2 : nullptr));
            if (rowk == nullptr) continue;
            double2 sum = make_double2(0.0, 0.0);
            for (int ty = 0; ty < TS; ++ty) sum = add2(sum, sred[k * nthr + ty * TR + threadIdx.x]);
            double* row = rowk + (size_t)blockIdx.x * v.RP;
            if (CPLX) {
                row[rg] = sum.x;
            } else {
                row[2 * rg] = sum.x;
                row[2 * rg + 1] = sum.y;
            }
        }
    }
}

}  // namespace kpm
