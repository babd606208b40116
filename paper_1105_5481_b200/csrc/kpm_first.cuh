// kpm_first.cuh -- the first recursion step for 2D/3D lattice stencils:
//     a_0 = r (Rademacher, Eq 14-15, generated on the GPU as the paper does; or the
//           caller's start block, from_buf = 1, read from the buffer -- the same summation order),
//     a_1 = H~ a_0 (Eq 17),   S_0 = <a_0|a_0>,  S_1 = <a_0|a_1>  (+ the odd-N tail <a_1|a_1>).
//
// The generic grid-stride kernel regenerates the counter hash of a_0 for a site AND for each of
// its 2 ndim neighbours (7 hashes per element in 3D; c5's first step took 92 ms).  Here a CTA
// marches a tile column (TX x TY sites x TL lanes) along the slowest dimension and generates every
// plane of a_0 ONCE, with a one-site halo, into a 3-plane shared-memory ring; a_1 of plane m is
// computed from planes m-1, m, m+1 of the ring.  Hashes per element: (TX+2)(TY+2)/(TX TY)
// (1.27 for 16 x 16 tiles), so the kernel is bound by writing a_0 and a_1 (2 D R s bytes).
// Columns are cut into segments of SEG planes when there are too few columns for the grid.
// Reductions: per-lane registers, fixed-order CTA finish per work item, one partial row per CTA.
#pragma once
#include "kpm_kernels.cuh"

namespace kpm {

struct FirstGeom {
    int L0, L1;         // in-plane extents (L1 unused in 2D)
    int TX, TY, TL;     // tile sites (TY = 1 in 2D) and lanes
    int PX, PY, G_L;    // pencils along x, y (PY = 1 in 2D), lane groups
    int Lm, SEG, NSEG;  // march extent (local), planes per segment, segments per column
    long long items;    // G_L * PY * PX * NSEG
    int rows_total;     // partial-sum rows per slot (>= gridDim.x; extra rows are zeroed)
    int ghost;          // row partition: the march neighbours of the slab ends are ghost planes
    double t, shift;    // t / a, -b / a
    const double* eps;  // (eps_i - b) / a, or nullptr
    const double2* phase;
};

constexpr int kFirstThreads = 512;  // 16 warps: one CTA per SM holds the whole partial-row budget of the plan

// shared-memory carve-up: ring [3][PYs][PXs][TL] double2 | eps~ [3][TY][TX] | sacc [3][RP] | sred [3][threads]
// double2, each region 16-byte aligned
__host__ __device__ inline size_t first_a16(size_t x) { return (x + 15) / 16 * 16; }
__host__ __device__ inline size_t first_smem_bytes(int ndim, int TX, int TY, int TL, int RP) {
    const int PXs = TX + 2, PYs = ndim == 3 ? TY + 2 : 1;
    return 3 * (size_t)PXs * PYs * TL * 16 + first_a16(3 * (size_t)TX * TY * 8) + first_a16(3 * (size_t)RP * 8) +
           3 * (size_t)kFirstThreads * 16;
}

template <int NDIM, bool ONSITE, bool PEIERLS, bool CPLX>
__global__ void __launch_bounds__(kFirstThreads) kpm_first_tile_kernel(const VecArgs v, const FirstGeom g, const int tail,
                                                                         const int from_buf) {
    pdl_entry();
    extern __shared__ __align__(128) unsigned char smem[];  // (every extern smem declaration of the TU must agree: TMA destinations need 128)
    const int PXs = g.TX + 2, PYs = NDIM == 3 ? g.TY + 2 : 1;
    const int plane_el = PXs * PYs * g.TL;
    double2* ring = reinterpret_cast<double2*>(smem);                  // [3][PYs][PXs][TL]
    double* seps = reinterpret_cast<double*>(ring + 3 * plane_el);    // [3][TY][TX] eps~ of the planes
    double* sacc = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(seps) + first_a16(3 * (size_t)g.TX * g.TY * 8));
    double2* sred = reinterpret_cast<double2*>(reinterpret_cast<unsigned char*>(sacc) + first_a16(3 * (size_t)v.RP * 8));
    const int t = threadIdx.x, nthr = blockDim.x;
    for (int i = t; i < 3 * v.RP; i += nthr) sacc[i] = 0.0;
    const int l = t % g.TL, k0 = t / g.TL, kstep = nthr / g.TL;
    const int nsite = g.TX * g.TY;
    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;

    for (long long item = blockIdx.x; item < g.items; item += gridDim.x) {
        long long q = item;
        const int seg = (int)(q % g.NSEG);
        q /= g.NSEG;
        const int px = (int)(q % g.PX);
        q /= g.PX;
        const int py = (int)(q % g.PY);
        const int lg = (int)(q / g.PY);
        const int x0 = px * g.TX, y0 = py * g.TY;
        const int m0 = seg * g.SEG, m1 = min(g.Lm, m0 + g.SEG);
        const int rg0 = lg * g.TL;
        // a_0 of plane m (march coordinate; m = -1 / Lm are the periodic images, or the ghost
        // planes of a slab) with its one-site in-plane halo, into ring slot `slot`
        // (thread t always handles lane l of tile sites k0, k0 + kstep, ...: the site coordinates
        // advance incrementally, no per-element division)
        auto gen = [&](int m, int slot) {
            double2* dst = ring + slot * plane_el;
            int mm = m;
            if (!g.ghost) mm = mm < 0 ? mm + g.Lm : (mm >= g.Lm ? mm - g.Lm : mm);
            const int rg = rg0 + l;
            const int jm = NDIM == 3 ? g.L0 * g.L1 * mm : g.L0 * mm;  // first site of plane mm
            int tx = k0 % PXs, ty = k0 / PXs;
            const int dx = kstep % PXs, dy = kstep / PXs;
            for (int s = k0; s < PXs * PYs; s += kstep) {
                int x = x0 + tx - 1;
                x = x < 0 ? x + g.L0 : (x >= g.L0 ? x - g.L0 : x);
                int j = jm + x;
                if (NDIM == 3) {
                    int y = y0 + ty - 1;
                    y = y < 0 ? y + g.L1 : (y >= g.L1 ? y - g.L1 : y);
                    j += g.L0 * y;
                }
                double2 a0 = make_double2(0.0, 0.0);
                if (rg < v.RG) {
                    if (from_buf) {  // the caller's start block, already in lane layout in P
                        const int row = j >= 0 ? j / g.L0 : -((-j + g.L0 - 1) / g.L0);
                        a0 = v.P[((long long)row * (g.L0 + 2 * v.xpad) + x + v.xpad) * v.RG + rg];
                    } else {
                        a0 = gen_lane<CPLX>(v, j, rg);
                    }
                }
                dst[s * g.TL + l] = a0;
                // eps~ of the interior sites, staged with the plane (a dependent global load per
                // element stalled the compute loop: ncu long-scoreboard on the a_1 FMA)
                if (ONSITE && l == 0 && tx >= 1 && tx <= g.TX && ty >= (NDIM == 3 ? 1 : 0) &&
                    ty < (NDIM == 3 ? g.TY + 1 : 1) && mm >= 0 && mm < g.Lm)
                    seps[slot * g.TX * g.TY + (NDIM == 3 ? ty - 1 : 0) * g.TX + tx - 1] = __ldg(g.eps + j);
                tx += dx;
                ty += dy;
                if (tx >= PXs) {
                    tx -= PXs;
                    ++ty;
                }
            }
        };
        __syncthreads();  // the previous item is done with the ring
        gen(m0 - 1, 0);
        gen(m0, 1);
        int s0 = 0, s1 = 1, s2 = 2;
        for (int m = m0; m < m1; ++m) {
            gen(m + 1, s2);
            __syncthreads();
            const double2* P0 = ring + s0 * plane_el;  // plane m-1
            const double2* P1 = ring + s1 * plane_el;  // plane m
            const double2* P2 = ring + s2 * plane_el;  // plane m+1
            const int rg = rg0 + l;
            int lx = k0 % g.TX, ly = k0 / g.TX;
            const int ex = kstep % g.TX, ey = kstep / g.TX;
            for (int k = k0; k < nsite && rg < v.RG; k += kstep) {
                const int x = x0 + lx, y = y0 + ly;
                const int lx0 = lx, ly0 = ly;
                lx += ex;
                ly += ey;
                if (lx >= g.TX) {
                    lx -= g.TX;
                    ++ly;
                }
                if (x >= g.L0 || (NDIM == 3 && y >= g.L1)) continue;  // ragged last tile
                const int c = ((NDIM == 3 ? ly0 + 1 : 0) * PXs + lx0 + 1) * g.TL + l;
                const double2 xc = P1[c];
                double2 nb = add2(P1[c - g.TL], P1[c + g.TL]);
                if (NDIM == 3) nb = add2(nb, add2(P1[c - PXs * g.TL], P1[c + PXs * g.TL]));
                const double2 mprev = P0[c], mnext = P2[c];
                int s;
                if (NDIM == 2 && PEIERLS) {
                    // y is the march dim: H[s][s+e_y] = t e^{-i theta_x}, H[s][s-e_y] = t e^{+i theta_x}
                    const double2 ph = __ldg(g.phase + x);
                    nb = add2(nb, add2(cmulc(ph, mnext), cmul(ph, mprev)));
                } else {
                    nb = add2(nb, add2(mprev, mnext));
                }
                const int row = NDIM == 3 ? y + g.L1 * m : m;  // x-row of the site
                s = x + g.L0 * row;
                const double e = ONSITE ? seps[s1 * g.TX * g.TY + ly0 * g.TX + lx0] : g.shift;
                const double2 a1 = fma2(e, xc, scale2(g.t, nb));  // a_1 = H~ a_0 (Eq 17)
                // memory site: x-rows carry a frame of xpad periodic images per side (3D)
                const long long ms = (long long)row * (g.L0 + 2 * v.xpad) + x + v.xpad;
                double2* pa = v.P + ms * v.RG + rg;
                double2* pc = v.C + ms * v.RG + rg;
                if (!from_buf) *pa = xc;
                *pc = a1;
                if (x < v.xpad) {  // (both images when L0 < 2 xpad)
                    if (!from_buf) pa[(long long)g.L0 * v.RG] = xc;
                    pc[(long long)g.L0 * v.RG] = a1;
                }
                if (x >= g.L0 - v.xpad && v.xpad) {
                    if (!from_buf) pa[-(long long)g.L0 * v.RG] = xc;
                    pc[-(long long)g.L0 * v.RG] = a1;
                }
                dot_acc<CPLX>(acc0, xc, xc);
                dot_acc<CPLX>(acc1, xc, a1);
                if (tail) dot_acc<CPLX>(acc2, a1, a1);
            }
            __syncthreads();  // plane m-1's slot is free
            const int tmp = s0;
            s0 = s1;
            s1 = s2;
            s2 = tmp;
        }
        // fixed-order CTA finish of this item's lane group
        sred[t] = acc0;
        sred[nthr + t] = acc1;
        sred[2 * nthr + t] = acc2;
        __syncthreads();
        if (t < g.TL && rg0 + t < v.RG) {
            for (int k = 0; k < 3; ++k) {
                double2 sum = make_double2(0.0, 0.0);
                for (int j = t; j < nthr; j += g.TL) sum = add2(sum, sred[k * nthr + j]);
                const int vv = rg0 + t;
                if (CPLX) {
                    sacc[k * v.RP + vv] += sum.x;
                } else {
                    sacc[k * v.RP + 2 * vv] += sum.x;
                    sacc[k * v.RP + 2 * vv + 1] += sum.y;
                }
            }
        }
        acc0 = acc1 = acc2 = make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int k = 0; k < 3; ++k) {
        double* rowk = k == 0 ? v.red0 : (k == 1 ? v.red1 : (tail ? v.red2 : nullptr));
        if (rowk == nullptr) continue;
        for (int i = t; i < v.RP; i += nthr) rowk[(size_t)blockIdx.x * v.RP + i] = sacc[k * v.RP + i];
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int i = t; i < v.RP; i += nthr) rowk[(size_t)rr * v.RP + i] = 0.0;
    }
}

}  // namespace kpm
