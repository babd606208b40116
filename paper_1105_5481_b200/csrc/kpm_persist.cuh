// kpm_persist.cuh -- the whole recursion in ONE cooperative (persistent) launch for vector
// blocks that fit in L2 ("persistent L2-resident mode for small per-GPU
// blocks", e.g. c2's per-GPU share at 8 GPUs under strong scaling: R = 8, 2 x 16.8 MB).
//
// Same arithmetic and partial-sum layout as the per-step launches (kpm_step_kernel: the first
// step a_1 = H~ a_0 with <a_0|a_0>, <a_0|a_1> (Eq 17, 19), then Eq 18 with the doubling inner
// products, a_{n+1} written over a_{n-1} in place), but the steps are separated by a grid-wide
// barrier instead of a kernel boundary: no launch gap, no per-launch ramp, and the two vector
// blocks stay in L2 between steps.  The vector blocks are read with ld.global.cg (L2 only; they
// change during the kernel, so the L1 / read-only path is not coherent for them).
#pragma once
#include <cooperative_groups.h>

#include "kpm_kernels.cuh"

namespace kpm {

template <class OP, bool CPLX>
__global__ void __launch_bounds__(512)
    kpm_persist_kernel(const OP op, VecArgs v, const int N, const int M, const int first_buf, const long long slot,
                       double* part) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    // first step: slots 0, 1 (and the odd-N tail slot 2 when N == 3)
    v.red0 = part;
    v.red1 = N > 1 ? part + slot : nullptr;
    v.red2 = N == 3 ? part + 2 * slot : nullptr;
    if (first_buf) step_body<OP, FIRST_BUF, CPLX, true>(op, v, N == 3);
    else step_body<OP, FIRST_GEN, CPLX, true>(op, v, N == 3);
    double2* cur = v.C;   // a_n
    double2* prev = v.P;  // a_{n-1}, overwritten by a_{n+1}
    for (int n = 1; n < M; ++n) {
        grid.sync();  // a_n complete everywhere (its neighbours are read by other CTAs)
        VecArgs w = v;
        w.C = cur;
        w.P = prev;
        const int tail = (N & 1) && n == M - 1;
        w.red0 = part + (size_t)(2 * n) * slot;
        w.red1 = part + (size_t)(2 * n + 1) * slot;
        w.red2 = tail ? part + (size_t)(2 * n + 2) * slot : nullptr;
        step_body<OP, STEP, CPLX, true>(op, w, tail);
        double2* t = cur;
        cur = prev;
        prev = t;
    }
}

}  // namespace kpm
