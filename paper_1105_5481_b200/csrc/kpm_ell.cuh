// kpm_ell.cuh -- fused recursion step for a general sparse H~ in ELL form.
//
// Same arithmetic as kpm_step_kernel<EllOp, STEP> (Eq 18 + the doubling inner
// products) with the row entries staged through shared memory: the CTA walks tiles
// of TILE = TS * kEllSPW consecutive rows; while it computes tile i, cp.async copies
// the column indices and values of tile i+gridDim.x into the other half of a
// double buffer, so the gathers of a row never wait behind the load of their index.
// One warp row of threads owns the 16-byte vector lanes of a row (one matrix entry
// serves all R vectors, BJ north_star); each thread keeps 8 gathers in flight.
#pragma once
#include "kpm_kernels.cuh"

namespace kpm {

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

template <bool CPLX>
__global__ void __launch_bounds__(512) kpm_ell_step_kernel(const EllOp<CPLX> op, const VecArgs v, const int tail) {
    pdl_entry();
    const int TR = blockDim.x, TS = blockDim.y;
    const int nthr = TR * TS, tid = threadIdx.y * TR + threadIdx.x;
    const int rg = blockIdx.y * TR + threadIdx.x;
    const bool active = rg < v.RG;
    const int K = op.K, D = op.D;
    const int TILE = TS * kEllSPW;
    extern __shared__ double2 sred[];                                     // [3][nthr]
    int* scol = reinterpret_cast<int*>(sred + 3 * nthr);                 // [2][K][TILE]
    const size_t vofs = ((size_t)2 * K * TILE * 4 + 15) / 16 * 16;
    unsigned char* sval = reinterpret_cast<unsigned char*>(scol) + vofs; // [2][K][TILE] double or double2
    const int vb = CPLX ? 16 : 8;
    const int ntiles = (D + TILE - 1) / TILE;

    auto prefetch = [&](int tile, int buf) {
        for (int e = tid; e < K * TILE; e += nthr) {
            const int k = e / TILE, i = e - k * TILE;
            const int s = tile * TILE + i;
            if (s < D) {
                const size_t ge = (size_t)k * D + s;
                cp_async(scol + ((size_t)buf * K + k) * TILE + i, op.col + ge, 4);
                cp_async(sval + (((size_t)buf * K + k) * TILE + i) * vb, reinterpret_cast<const unsigned char*>(op.val) + ge * vb,
                         vb);
            }
        }
        cp_async_commit();
    };

    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
    int tile = blockIdx.x;
    if (tile < ntiles) prefetch(tile, 0);
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        cp_async_wait_all();
        __syncthreads();  // this tile's entries are in smem; nobody reads the other buffer any more
        if (tile + (int)gridDim.x < ntiles) prefetch(tile + gridDim.x, buf ^ 1);
        if (!active) continue;
        const int* tc = scol + (size_t)buf * K * TILE;
        const unsigned char* tv = sval + (size_t)buf * K * TILE * vb;
#pragma unroll 1
        for (int u = 0; u < kEllSPW; ++u) {
            const int i = threadIdx.y + u * TS;
            const int s = tile * TILE + i;
            if (s >= D) break;
            const size_t idx = (size_t)s * v.RG + rg;
            const double2 x = __ldg(v.C + idx);
            const double2 p = __ldcs(v.P + idx);
            double2 h = scale2(op.shift, x);
            for (int k0 = 0; k0 < K; k0 += 8) {
                double2 xj[8], vv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k = k0 + q < K ? k0 + q : K - 1;
                    const int j = tc[k * TILE + i];
                    xj[q] = __ldg(v.C + (size_t)j * v.RG + rg);
                    vv[q] = CPLX ? reinterpret_cast<const double2*>(tv)[k * TILE + i]
                                 : make_double2(reinterpret_cast<const double*>(tv)[k * TILE + i], 0.0);
                    if (k0 + q >= K) vv[q] = make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) h = CPLX ? add2(h, cmul(vv[q], xj[q])) : fma2(vv[q].x, xj[q], h);
            }
            const double2 y = make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));  // Eq 18
            __stcs(v.P + idx, y);
            dot_acc<CPLX>(acc0, x, x);
            dot_acc<CPLX>(acc1, x, y);
            if (tail) dot_acc<CPLX>(acc2, y, y);
        }
    }
    cp_async_wait_all();
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
