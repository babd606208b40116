// kpm_small.cuh -- the whole recursion in one launch for small problems.
//
// When both vector blocks of a lane group fit in one SM's shared memory (c1: 1024
// sites x 8 vectors = 2 x 64 KB), the per-step launches of the large-problem path are
// pure latency (a few microseconds each for microseconds of work).  Here one CTA per
// lane group keeps a_n and a_{n-1} in shared memory and runs the first step and all
// floor(N/2)-1 fused steps (Eq 17-18) with one CTA barrier per step.  Each thread row
// writes its per-step partial sums of <a_n|a_n>, <a_n|a_{n+1}> (and the odd-N tail)
// to the usual [slot][row][R] buffer, finished by finish_kernel in fixed order.
#pragma once
#include "kpm_kernels.cuh"

namespace kpm {

constexpr int kSmallThreads = 1024;
constexpr size_t kSmallSmemMax = 200 * 1024;

template <class OP, bool CPLX>
__global__ void __launch_bounds__(kSmallThreads, 1)
    kpm_small_kernel(const OP op, const VecArgs v, const int first_from_buf, const int N, double* __restrict__ part) {
    pdl_entry();
    const int TR = blockDim.x, TS = blockDim.y;
    const int rg = blockIdx.y * TR + threadIdx.x;
    const bool active = rg < v.RG;
    extern __shared__ double2 sm[];
    double2* bufA = sm;                  // a_{n-1}, then a_{n+1} in place
    double2* bufB = sm + (size_t)v.D * TR;  // a_n
    const int l = threadIdx.x;
    const size_t slot = (size_t)TS * v.RP;  // doubles per moment slot
    auto put = [&](int m, double2 a) {      // partial sums of slot m from this thread row
        if (!active || m >= N) return;
        double* row = part + (size_t)m * slot + (size_t)threadIdx.y * v.RP;
        if (CPLX) {
            row[rg] = a.x;
        } else {
            row[2 * rg] = a.x;
            row[2 * rg + 1] = a.y;
        }
    };
    const int M = N / 2;
    // ---- first step: a_0 (generated or the caller's block), a_1 = H~ a_0  (Eq 17)
    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
    if (active) {
        for (int s = threadIdx.y; s < v.D; s += TS) {
            const double2 x = first_from_buf ? v.P[(size_t)v.mem(s) * v.RG + rg] : gen_lane<CPLX>(v, s, rg);
            bufA[(size_t)s * TR + l] = x;
        }
    }
    __syncthreads();
    if (active) {
        auto X = [&](int j) { return bufA[(size_t)j * TR + l]; };
        for (int s = threadIdx.y; s < v.D; s += TS) {
            const double2 x = X(s);
            const double2 y = op.apply(s, X, x);
            bufB[(size_t)s * TR + l] = y;
            dot_acc<CPLX>(acc0, x, x);
            dot_acc<CPLX>(acc1, x, y);
            dot_acc<CPLX>(acc2, y, y);
        }
    }
    put(0, acc0);
    put(1, acc1);
    if (N == 3) put(2, acc2);
    __syncthreads();
    // ---- steps n = 1 .. M-1: a_{n+1} = 2 H~ a_n - a_{n-1} over a_{n-1}  (Eq 18)
    double2* cur = bufB;
    double2* prev = bufA;
    for (int n = 1; n <= M - 1; ++n) {
        acc0 = acc1 = acc2 = make_double2(0.0, 0.0);
        if (active) {
            auto X = [&](int j) { return cur[(size_t)j * TR + l]; };
            for (int s = threadIdx.y; s < v.D; s += TS) {
                const double2 x = X(s);
                const double2 h = op.apply(s, X, x);
                const size_t e = (size_t)s * TR + l;
                const double2 p = prev[e];
                const double2 y = make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));
                prev[e] = y;
                dot_acc<CPLX>(acc0, x, x);
                dot_acc<CPLX>(acc1, x, y);
                dot_acc<CPLX>(acc2, y, y);
            }
        }
        put(2 * n, acc0);
        put(2 * n + 1, acc1);
        if ((N & 1) && n == M - 1) put(2 * n + 2, acc2);
        __syncthreads();
        double2* t = cur;
        cur = prev;
        prev = t;
    }
}

}  // namespace kpm
