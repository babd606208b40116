// kpm_ell.cuh -- fused recursion step for a general sparse H~ in ELL form.
//
// Same arithmetic as kpm_step_kernel<EllOp, STEP> (Eq 18 + the doubling inner
// products) with the row entries staged through shared memory: the CTA walks tiles
// of TILE = TS * kEllSPW consecutive rows; while it computes tile i, one thread copies
// the column indices and values of tile i+gridDim.x into the other half of a double
// buffer with 2 bulk copies (cp.async.bulk, completion on an mbarrier; the row-major
// [rows][KP] device layout makes a tile one contiguous run of each array), so the
// gathers of a row never wait behind the load of their index and no other thread spends
// instructions on the staging.  A row's KP column indices come out of shared memory as
// KP/4 16-byte loads and its values as 16-byte pairs (ncu r02, [K][ld] layout: 255 warp
// instructions per row for K = 7, most of them per-entry index loads, address arithmetic and
// entry predicates; KP is now a template constant, padding entries are (row, 0)).
// One warp row of threads owns the 16-byte vector lanes of a row (one matrix entry
// serves all R vectors, BJ north_star); each thread keeps up to 24 gathers in flight.
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

// a_n gather with an L2 cache-eviction policy (evict-last keeps the rows a later row re-reads --
// e.g. the z-neighbours one lattice plane away -- in L2 behind the streamed a_{n-1} / a_{n+1})
__device__ __forceinline__ double2 ldg_hint(const double2* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

constexpr int kEllKMax = 16;  // rows with more entries use the generic step kernel
constexpr int kEllSPW = 4;    // rows per thread row per tile (KP = 8: kEllSPW8, when it fits)
constexpr int kEllSPW8 = 16;  // (c3 via CSR: 1683 -> 1556 ms per call -- a quarter of the tile barriers)

__host__ __device__ inline int ell_kp(int K) { return (K + 3) / 4 * 4; }  // stored entries per row

__host__ __device__ inline size_t ell_smem_bytes(int nthr, int TS, int K, bool cplx, int spw = kEllSPW) {
    const size_t tile = (size_t)TS * spw, KP = (size_t)ell_kp(K);
    return 3 * (size_t)nthr * 16 + (2 * KP * tile * 4 + 15) / 16 * 16 + 2 * KP * tile * (cplx ? 16 : 8);
}

// KP: stored entries per row (4, 8, 12 or 16).  U rows per thread are processed together -- all
// their gathers issued before any is consumed -- so a thread keeps U (KP + 2) 16-byte loads in
// flight.  One 512-thread CTA per SM (128 registers hold the loads in flight).
template <bool CPLX, int KP, bool WIDE, int SPW = kEllSPW>
__global__ void __launch_bounds__(512, 1) kpm_ell_step_kernel(const EllOp<CPLX> op, const VecArgs v, const int tail) {
    pdl_entry();
    constexpr int U = KP <= 4 ? 4 : (KP <= 8 ? 2 : 1);  // U (KP + 2) double2 in flight: 24, 20, 14-18
    static_assert(SPW % U == 0 && KP % 4 == 0, "rows per thread, 16-byte index groups");
    // element offsets j * RG + rg in 32 bits unless the extended block has 2^31 lanes or more (WIDE)
    using off_t = typename std::conditional<WIDE, long long, unsigned>::type;
    const int TR = blockDim.x, TS = blockDim.y;
    const int nthr = TR * TS, tid = threadIdx.y * TR + threadIdx.x;
    const int rg = blockIdx.y * TR + threadIdx.x;
    const bool active = rg < v.RG;
    const int D = op.D;
    const off_t RG = (off_t)v.RG;
    const int TILE = TS * SPW;
    extern __shared__ double2 sred[];                                     // [3][nthr]
    int* scol = reinterpret_cast<int*>(sred + 3 * nthr);                 // [2][TILE][KP]
    const size_t vofs = ((size_t)2 * KP * TILE * 4 + 15) / 16 * 16;
    unsigned char* sval = reinterpret_cast<unsigned char*>(scol) + vofs; // [2][TILE][KP] double or double2
    constexpr int vb = CPLX ? 16 : 8;
    const int ntiles = (D + TILE - 1) / TILE;
    const double2* __restrict__ Cl = v.C + rg;  // this thread's lane of row 0
    double2* __restrict__ Pl = v.P + rg;

    __shared__ uint64_t sbar[2];
    // thread 0: the tile's index and value panels (the pad rows past D included), one bulk copy each
    auto prefetch = [&](int tile, int buf) {
        const size_t ge = (size_t)tile * TILE * KP;
        mbar_expect_tx(sbar + buf, (uint32_t)(KP * TILE * (4 + vb)));
        bulk_g2s(scol + (size_t)buf * TILE * KP, op.col + ge, TILE * KP * 4, sbar + buf);
        bulk_g2s(sval + (size_t)buf * TILE * KP * vb, reinterpret_cast<const unsigned char*>(op.val) + ge * vb,
                 TILE * KP * vb, sbar + buf);
    };

    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
    const uint64_t pol_last = policy_evict_last();
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
        const int* tc = scol + (size_t)buf * TILE * KP;
        const unsigned char* tv = sval + (size_t)buf * TILE * KP * vb;
        const int nrow = min(TILE, D - tile * TILE);
        const off_t row0 = (off_t)tile * TILE;
#pragma unroll 1
        for (int u0 = 0; u0 < SPW; u0 += U) {
            int ii[U];
            double2 x[U], p[U], xj[U][KP];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int i = threadIdx.y + (u0 + q) * TS;
                ii[q] = i < nrow ? i : 0;  // (ragged last tile: row 0's loads, result unused)
                const off_t o = (row0 + ii[q]) * RG;
                x[q] = __ldg(Cl + o);
                p[q] = __ldcs(Pl + o);
                const int4* ci = reinterpret_cast<const int4*>(tc + ii[q] * KP);
#pragma unroll
                for (int k4 = 0; k4 < KP / 4; ++k4) {
                    const int4 c = ci[k4];
                    xj[q][4 * k4 + 0] = ldg_hint(Cl + (off_t)c.x * RG, pol_last);  // (A/B c2 via CSR: 46.3 -> 41.2 ms)
                    xj[q][4 * k4 + 1] = ldg_hint(Cl + (off_t)c.y * RG, pol_last);
                    xj[q][4 * k4 + 2] = ldg_hint(Cl + (off_t)c.z * RG, pol_last);
                    xj[q][4 * k4 + 3] = ldg_hint(Cl + (off_t)c.w * RG, pol_last);
                }
            }
#pragma unroll
            for (int q = 0; q < U; ++q) {
                if (threadIdx.y + (u0 + q) * TS >= nrow) continue;
                double2 h = scale2(op.shift, x[q]);
                const double2* vv = reinterpret_cast<const double2*>(tv + (size_t)ii[q] * KP * vb);
                if (CPLX) {
#pragma unroll
                    for (int k = 0; k < KP; ++k) h = add2(h, cmul(vv[k], xj[q][k]));
                } else {
#pragma unroll
                    for (int k2 = 0; k2 < KP / 2; ++k2) {
                        const double2 w = vv[k2];  // values of entries 2 k2, 2 k2 + 1
                        h = fma2(w.x, xj[q][2 * k2], h);
                        h = fma2(w.y, xj[q][2 * k2 + 1], h);
                    }
                }
                const double2 y = make_double2(fma(2.0, h.x, -p[q].x), fma(2.0, h.y, -p[q].y));  // Eq 18
                __stcs(Pl + (row0 + ii[q]) * RG, y);
                dot_acc<CPLX>(acc0, x[q], x[q]);
                dot_acc<CPLX>(acc1, x[q], y);
                if (tail) dot_acc<CPLX>(acc2, y, y);
            }
        }
    }
    __syncthreads();
    // fixed-order CTA finish per vector lane (TR lanes x TS rows, TR a power of two <= 32)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double* rowk = k == 0 ? v.red0 : (k == 1 ? v.red1 : (tail ? v.red2 : nullptr));
        if (rowk == nullptr) continue;  // (uniform over the CTA)
        const double2 sum = cta_lane_sum_rt<512>(k == 0 ? acc0 : (k == 1 ? acc1 : acc2), tid, TR, sred);
        if (threadIdx.y == 0 && active) {
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
