// kpm_dense.cuh -- the paper's dense-H variant (PAPER.md:140
// "When the H is considered as a dense matrix, the complexity of the part becomes
// O(D^2)", and the H_SIZE experiments PAPER.md:241-253).
//
// One recursion step over the whole vector block is a dense GEMM
//     a_{n+1} = 2 (H/a) a_n + 2 (-b/a) a_n - a_{n-1}                     (Eq 18)
// with M = D (rows of H), N = R (vectors), K = D.  FP64 has no tcgen05 kind, so the
// tensor-core instruction for it on sm_100a is DMMA (mma.sync m8n8k4 .f64).  The epilogue
// is fused: shift term, recursion, in-place store over a_{n-1}, and the doubling inner
// products <a_n|a_n>, <a_n|a_{n+1}> (odd-N tail <a_{n+1}|a_{n+1}>) per vector, reduced in a
// fixed order into one partial row per M-tile (the [slot][row][RP] layout finish_kernel sums).
//
// Layouts: H~ is stored row-major Dp x Dp (Dp = D rounded up to 64, zero padding, pre-scaled
// by 1/a); the vector block is [site][vector] = Dp x RP doubles (the lane layout of the
// sparse path with RP padded to 64; padded sites/vectors are zero and stay zero).
// CTA tile 64 x 64 x 32, 4 warps (2 x 2, 32 x 32 each = 4 x 4 DMMA tiles), 3-stage cp.async
// pipeline; padded smem strides make the fragment loads bank-conflict free.  Grid: x = N
// tile (fastest), y = M tile, so the CTAs sharing an H row stripe run together (H leaves
// HBM about once per step; the vector block, D x R doubles, stays in L2).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kpm_kernels.cuh"

namespace kpm {

constexpr int kDBM = 64, kDBN = 64, kDBK = 32, kDStages = 3, kDThreads = 128;
constexpr int kDHS = kDBK + 4;  // smem row stride (doubles) of the H tile   [64][36]
constexpr int kDAS = kDBN + 4;  // smem row stride (doubles) of the a_n tile [32][68]
constexpr size_t kDenseSmem = (size_t)kDStages * (kDBM * kDHS + kDBK * kDAS) * sizeof(double);

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gmem_src)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct DenseArgs {
    const double* H;  // Dp x Dp, row-major, H / a
    const double* A;  // a_n: Dp x RP
    double* P;        // STEP: a_{n-1} in, a_{n+1} out (in place); FIRST: a_1 out
    int Dp, RP;
    double shift;     // -b / a
    double* red0;     // partial rows [gridDim.y][RP] of <a_n|a_n>
    double* red1;     // <a_n|a_{n+1}>
    double* red2;     // odd-N tail <a_{n+1}|a_{n+1}> (nullable)
};

// FIRST = true: a_1 = H~ a_0 written to P (no recursion term); else Eq (18) in place over P.
template <bool FIRST>
__global__ void __launch_bounds__(kDThreads) kpm_dense_step_kernel(const DenseArgs g, const int tail) {
    pdl_entry();
    extern __shared__ __align__(16) double dsm[];
    double* Hs = dsm;                                // [stage][64][36]
    double* As = dsm + kDStages * kDBM * kDHS;       // [stage][32][68]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = warp >> 1, wn = warp & 1;         // warp tile (32 x 32) position
    const int n0 = blockIdx.x * kDBN, m0 = blockIdx.y * kDBM;
    const int KT = g.Dp / kDBK;

    auto load_stage = [&](int stage, int kt) {
        const int k0 = kt * kDBK;
        double* hs = Hs + stage * kDBM * kDHS;
        double* as = As + stage * kDBK * kDAS;
#pragma unroll
        for (int i = 0; i < (kDBM * kDBK / 2) / kDThreads; ++i) {  // 8 chunks of 16 B
            const int c = t + i * kDThreads;
            const int r = c / (kDBK / 2), cc = (c % (kDBK / 2)) * 2;
            cp_async16(hs + r * kDHS + cc, g.H + (size_t)(m0 + r) * g.Dp + k0 + cc);
        }
#pragma unroll
        for (int i = 0; i < (kDBK * kDBN / 2) / kDThreads; ++i) {
            const int c = t + i * kDThreads;
            const int r = c / (kDBN / 2), cc = (c % (kDBN / 2)) * 2;
            cp_async16(as + r * kDAS + cc, g.A + (size_t)(k0 + r) * g.RP + n0 + cc);
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < kDStages - 1; ++s) {
        if (s < KT) load_stage(s, s);
        cp_async_commit();
    }
    const int fr = lane >> 2, fc = lane & 3;  // fragment row / column within an 8x4 (4x8) tile
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<kDStages - 2>();
        __syncthreads();
        // prefetch stage kt + STAGES - 1 (its buffer was last read in iteration kt - 1)
        if (kt + kDStages - 1 < KT) load_stage((kt + kDStages - 1) % kDStages, kt + kDStages - 1);
        cp_async_commit();
        const double* hs = Hs + (kt % kDStages) * kDBM * kDHS + (wm * 32) * kDHS;
        const double* as = As + (kt % kDStages) * kDBK * kDAS + wn * 32;
#pragma unroll
        for (int kk = 0; kk < kDBK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = hs[(i * 8 + fr) * kDHS + kk + fc];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = as[(kk + fc) * kDAS + j * 8 + fr];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- fused epilogue: H~ a_n = acc + shift a_n; recursion; store; per-vector sums
    double s0[4][2], s1[4][2], s2[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) s0[j][0] = s0[j][1] = s1[j][0] = s1[j][1] = s2[j][0] = s2[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + wm * 32 + i * 8 + fr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + wn * 32 + j * 8 + 2 * fc;
            const size_t e = (size_t)m * g.RP + n;
            const double2 x = *reinterpret_cast<const double2*>(g.A + e);
            double2 y;
            if (FIRST) {
                y = make_double2(fma(g.shift, x.x, acc[i][j][0]), fma(g.shift, x.y, acc[i][j][1]));
            } else {
                const double2 p = __ldcs(reinterpret_cast<const double2*>(g.P + e));
                y = make_double2(fma(2.0, fma(g.shift, x.x, acc[i][j][0]), -p.x),
                                 fma(2.0, fma(g.shift, x.y, acc[i][j][1]), -p.y));
            }
            __stcs(reinterpret_cast<double2*>(g.P + e), y);
            s0[j][0] = fma(x.x, x.x, s0[j][0]);
            s0[j][1] = fma(x.y, x.y, s0[j][1]);
            s1[j][0] = fma(x.x, y.x, s1[j][0]);
            s1[j][1] = fma(x.y, y.y, s1[j][1]);
            s2[j][0] = fma(y.x, y.x, s2[j][0]);
            s2[j][1] = fma(y.y, y.y, s2[j][1]);
        }
    }
    // reduce over the 8 fragment rows of the warp (lane bits 2..4), fixed butterfly order
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
                s0[j][h] += __shfl_xor_sync(0xffffffffu, s0[j][h], off);
                s1[j][h] += __shfl_xor_sync(0xffffffffu, s1[j][h], off);
                s2[j][h] += __shfl_xor_sync(0xffffffffu, s2[j][h], off);
            }
    // then over the two M-warps through shared memory: [wm][slot][64 columns]
    double* sred = dsm;  // the pipeline buffers are free now
    if (fr == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = wn * 32 + j * 8 + 2 * fc + h;
                sred[(wm * 3 + 0) * kDBN + col] = s0[j][h];
                sred[(wm * 3 + 1) * kDBN + col] = s1[j][h];
                sred[(wm * 3 + 2) * kDBN + col] = s2[j][h];
            }
    }
    __syncthreads();
    if (t < kDBN) {
        const size_t row = (size_t)blockIdx.y * g.RP + n0 + t;
        g.red0[row] = sred[0 * kDBN + t] + sred[3 * kDBN + t];
        g.red1[row] = sred[1 * kDBN + t] + sred[4 * kDBN + t];
        if (tail && g.red2) g.red2[row] = sred[2 * kDBN + t] + sred[5 * kDBN + t];
    }
}

// a_0 of the dense path: Dp x RP, generated (Rademacher / unit vectors) for sites < D and
// vectors < R_loc, zero elsewhere.  Uses gen_lane of kpm_kernels.cuh (VecArgs v with
// RG = RP / 2, D = real number of sites).
template <bool CPLX>
__global__ void dense_gen_kernel(const VecArgs v, int Dp, double2* __restrict__ out) {
    pdl_entry();
    const long long n = (long long)Dp * v.RG;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(e / v.RG), rg = (int)(e % v.RG);
        out[e] = s < v.D ? gen_lane<CPLX>(v, s, rg) : make_double2(0.0, 0.0);
    }
}

}  // namespace kpm
