// kpm_tri.cuh -- THREE recursion steps per HBM pass (temporal blocking), 2D lattices.
//
// One launch advances the recursion by three steps (Eq 18 three times):
//     a_{n+1} = 2 H~ a_n - a_{n-1},  a_{n+2} = 2 H~ a_{n+1} - a_n,  a_{n+3} = 2 H~ a_{n+2} - a_{n+1},
// reading a_n and a_{n-1} from HBM once and writing a_{n+2} and a_{n+3} once: 4 D R s bytes per
// three steps (the two-step kernel, kpm_tma2.cuh, moves 4 D R s per two; single steps 3 D R s per
// one).  a_{n+1} and a_{n+2} live in shared-memory row rings.
//
// Same march as kpm_tma2.cuh (pencil of TX sites x TL lanes, rows of y), one level deeper:
//   level 0  a_n      rows m0-3 .. m1+2, sites x0-3 .. x0+TX+2  (TMA: main box + two 3-site boxes)
//   level -1 a_{n-1}  rows m0-2 .. m1+1, sites x0-2 .. x0+TX+1  (TMA: main box + two 2-site boxes)
//   level 1  a_{n+1}  rows m0-2 .. m1+1, sites x0-2 .. x0+TX+1  (computed, 3-row ring B1)
//   level 2  a_{n+2}  rows m0-1 .. m1,   sites x0-1 .. x0+TX    (computed, 2-row ring B2; rows m0..m1-1
//                                                                of sites x0..x0+TX-1 stored)
//   level 3  a_{n+3}  rows m0 .. m1-1,   sites x0 .. x0+TX-1    (stored)
// Iteration q of a segment computes level 1 at row r1 = m0-2+q, level 2 at r1-1 and level 3 at
// r1-2.  Interior sites: 8 warps, each thread NPI sites of a row; its level-1 and level-2 values
// of the last rows roll in registers (the y-neighbours and the "- a_{n-1}" terms of the next
// levels), x-neighbours and level 0 come from shared memory.  The halo sites (level 1: x0-2,
// x0-1, x0+TX, x0+TX+1; level 2: x0-1, x0+TX) are spread over the first 4 TL threads: thread
// t < 2 TL computes level 1 and then level 2 at x0-1 or x0+TX (its own level-1 value is the
// level-2 y-neighbour, so no barrier between them), threads 2 TL .. 4 TL - 1 level 1 at x0-2 or
// x0+TX+1.  (A ninth warp for the halo would cap registers at 168 -- 3 warps on one SM
// sub-partition -- and spilled.)  The last thread issues the TMA refills.  One CTA barrier per row.
//
// Reductions: <a_n|a_n>, <a_n|a_{n+1}>, <a_{n+1}|a_{n+1}>, <a_{n+1}|a_{n+2}>, <a_{n+2}|a_{n+2}>,
// <a_{n+2}|a_{n+3}> (and the odd-N tail <a_{n+3}|a_{n+3}>) over owned sites, per lane, fixed order.
#pragma once
#include "kpm_tma2.cuh"

namespace kpm {

// 2 H~ x - p at one site of a 2D lattice (Eq 18), with the factor 2 folded into the coefficients:
// x-neighbours xm, xp with t2 = 2t; y-neighbours ym, yp with the Peierls phases in tph2 = 2t e^{i phi}
// (Landau gauge: conj(e^{i phi}) yp + e^{i phi} ym, expanded: 8 real operations instead of 12);
// e2 = 2 eps~ (or -2b/a).  Accumulated onto -p: 7 operations per component (real lattice: 5).
template <bool PEIERLS>
__device__ __forceinline__ double2 hop_step(double2 x, double2 xm, double2 xp, double2 ym, double2 yp, double e2,
                                           double t2, double2 tph2, double2 p) {
    double hx, hy;
    if (PEIERLS) {
        hx = fma(e2, x.x, fma(t2, xm.x + xp.x, fma(tph2.x, ym.x + yp.x, fma(tph2.y, yp.y - ym.y, -p.x))));
        hy = fma(e2, x.y, fma(t2, xm.y + xp.y, fma(tph2.x, ym.y + yp.y, fma(tph2.y, ym.x - yp.x, -p.y))));
    } else {
        hx = fma(e2, x.x, fma(t2, (xm.x + xp.x) + (ym.x + yp.x), -p.x));
        hy = fma(e2, x.y, fma(t2, (xm.y + xp.y) + (ym.y + yp.y), -p.y));
    }
    return make_double2(hx, hy);
}

struct TriGeom {
    int L0, L1;          // lattice extents
    int TX, TL, RG, G_L, PX;
    long long W;         // output rows = G_L * PX * L1
    int RP;
    int rows_total;      // partial-sum rows per slot (>= gridDim.x; extra rows are zeroed)
    double t, shift;
    const double2* phase;
    double* red[7];      // slots 2n .. 2n+5, (tail) 2n+6; red[6] nullable
    double2* outB;       // a_{n+2}
    double2* outC;       // a_{n+3}
};

constexpr int kThreadsTri = 256;       // 8 warps: two per SM sub-partition, up to 255 registers
constexpr int kSAT = 5;                // a_n ring (2 rows ahead of the rows in use)
constexpr int kSPT = 4;                // a_{n-1} ring (3 ahead: ncu showed 30% of warp samples waiting on a 3-deep ring)

// a_n slot: [3 halo sites][TX][3 halo sites], then eps~ as three 128-byte aligned pieces
// [4 left (x0-4 ..)][TX][4 right] (TMA boxes need 16-byte multiples); a_{n-1} slot
// [2][TX][2].  The level-1 and level-2 rows only ever need the ENDS of the threads' site runs and
// the halo sites (x-neighbours inside a run stay in registers), so B1 rows hold [2 halo][2 per run]
// [2 halo] and B2 rows [1][2 per run][1] sites: bix() maps a tile x index to its slot.
__host__ __device__ constexpr int tri_runs(int TL) { return 256 / TL; }  // runs (threads per lane) per row
struct TriLayout {
    int site, a_bytes, eps_l, eps_m, eps_r, p_bytes, b1_bytes, b2_bytes;
    __host__ __device__ constexpr TriLayout(int TX, int TL, bool onsite)
        : site(TL * 16),
          a_bytes(onsite ? (TX + 6) * TL * 16 + 128 + (TX * 8 + 127) / 128 * 128 + 128 : (TX + 6) * TL * 16),
          eps_l((TX + 6) * TL * 16),
          eps_m((TX + 6) * TL * 16 + 128),
          eps_r((TX + 6) * TL * 16 + 128 + (TX * 8 + 127) / 128 * 128),
          p_bytes(((TX + 4) * TL * 16 + 127) / 128 * 128),
          b1_bytes(((2 * tri_runs(TL) + 4) * TL * 16 + 127) / 128 * 128),
          b2_bytes(((2 * tri_runs(TL) + 2) * TL * 16 + 127) / 128 * 128) {}
    // eps~ at tile x index lx in [-4, TX+3]
    __device__ __forceinline__ double eps(const unsigned char* slot, int lx, int TX) const {
        return *reinterpret_cast<const double*>(
            slot + (lx < 0 ? eps_l + (lx + 4) * 8 : (lx < TX ? eps_m + lx * 8 : eps_r + (lx - TX) * 8)));
    }
};

__host__ __device__ inline size_t tri_smem_bytes(int TX, int TL, bool onsite, int RP) {
    const TriLayout S(TX, TL, onsite);
    return (size_t)kSAT * S.a_bytes + (size_t)kSPT * S.p_bytes + 3 * (size_t)S.b1_bytes + 2 * (size_t)S.b2_bytes +
           (size_t)kThreadsTri * 16 + (size_t)(TX + 6) * 16 + (kSAT + kSPT) * 8;
}

template <int TL, int TX, bool ONSITE, bool PEIERLS, int NT = kThreadsTri>
__global__ void __launch_bounds__(NT, 1)
    kpm_step_tri_kernel(const __grid_constant__ CUtensorMap mapA,    // a_n main box {2TL, TX, 1}
                        const __grid_constant__ CUtensorMap mapA3,   // a_n 3-site box {2TL, 3, 1}
                        const __grid_constant__ CUtensorMap mapP,    // a_{n-1} main box
                        const __grid_constant__ CUtensorMap mapP2,   // a_{n-1} 2-site box {2TL, 2, 1}
                        const __grid_constant__ CUtensorMap mapE,    // eps~ box {TX, 1}
                        const __grid_constant__ CUtensorMap mapE4,   // eps~ box {4, 1}
                        const TriGeom g, const int tail) {
    pdl_entry();
    constexpr int CONS = NT;
    constexpr int PRODUCER = CONS - 1;  // (no halo work: 4 TL <= 128 < CONS - 1)
    constexpr int KSTEP = CONS / TL;  // tile sites per pass
    constexpr int NPI = TX / KSTEP;   // interior sites per thread
    static_assert(TX % KSTEP == 0 && TL * 16 >= 128, "tile shape");
    constexpr int SITE = TL * 16;
    constexpr TriLayout SL(TX, TL, ONSITE);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + kSAT * SL.a_bytes;
    unsigned char* ringB1 = ringP + kSPT * SL.p_bytes;
    unsigned char* ringB2 = ringB1 + 3 * SL.b1_bytes;
    double2* sred = reinterpret_cast<double2*>(ringB2 + 2 * SL.b2_bytes);  // [CONS]
    double2* sphase = sred + CONS;                                         // [TX + 6]: x0-3 .. x0+TX+2
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sphase + TX + 6);
    uint64_t* fullP = fullA + kSAT;

    const int t = threadIdx.x;
    const long long w_begin = g.W * blockIdx.x / gridDim.x;
    const long long w_end = g.W * (blockIdx.x + 1) / gridDim.x;

    // ---- producer state (thread CONS only; in shared memory)
    __shared__ LoadCursor cur_smem[2];
    __shared__ uint64_t pol_smem;
    LoadCursor& ca = cur_smem[0];
    LoadCursor& cp = cur_smem[1];
    auto issueA = [&](int slot) {  // next a_n row (3-site halos) into `slot`
        if (!ca.valid) return;
        const int row = ca.row, c0 = ca.c0, x0 = ca.x0, xl = ca.xl, xr = ca.xr;
        unsigned char* dst = ringA + slot * SL.a_bytes;
        mbar_expect_tx(fullA + slot, (TX + 6) * SITE + (ONSITE ? (TX + 8) * 8 : 0));
        tma_load(dst, &mapA3, fullA + slot, c0, xl, row);
        tma_load(dst + 3 * SITE, &mapA, fullA + slot, c0, x0, row);
        tma_load(dst + (TX + 3) * SITE, &mapA3, fullA + slot, c0, xr, row);
        if (ONSITE) {
            int xe = x0 - 4;
            if (xe < 0) xe += g.L0;
            tma_load_2d(dst + SL.eps_l, &mapE4, fullA + slot, xe, row);
            tma_load_2d(dst + SL.eps_m, &mapE, fullA + slot, x0, row);
            tma_load_2d(dst + SL.eps_r, &mapE4, fullA + slot, xr, row);
        }
        ca.next(g, 6);
    };
    auto issueP = [&](int slot) {  // next a_{n-1} row (2-site halos) into `slot`
        if (!cp.valid) return;
        const int row = cp.row, c0 = cp.c0, x0 = cp.x0, xl = cp.xl, xr = cp.xr;
        unsigned char* dst = ringP + slot * SL.p_bytes;
        mbar_expect_tx(fullP + slot, (TX + 4) * SITE);
        const uint64_t pol = pol_smem;
        tma_load_hint(dst, &mapP2, fullP + slot, c0, xl, row, pol);
        tma_load_hint(dst + 2 * SITE, &mapP, fullP + slot, c0, x0, row, pol);
        tma_load_hint(dst + (TX + 2) * SITE, &mapP2, fullP + slot, c0, xr, row, pol);
        cp.next(g, 4);
    };
    if (t == PRODUCER) {
        for (int i = 0; i < kSAT; ++i) mbar_init(fullA + i, 1);
        for (int i = 0; i < kSPT; ++i) mbar_init(fullP + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&mapA);
        prefetch_tmap(&mapA3);
        prefetch_tmap(&mapP);
        prefetch_tmap(&mapP2);
        if (ONSITE) {
            prefetch_tmap(&mapE);
            prefetch_tmap(&mapE4);
        }
        pol_smem = policy_evict_first();
        ca.init(g, w_begin, w_end, 6);
        cp.init(g, w_begin, w_end, 4);
        for (int i = 0; i < kSAT; ++i) issueA(i);
        for (int i = 0; i < kSPT; ++i) issueP(i);
    }
    __syncthreads();

    const int l = t % TL;
    const int k0 = t / TL;
    const int lo = l * 16;
    double2 acc[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) acc[k] = make_double2(0.0, 0.0);
    auto ld = [](const unsigned char* p) { return *reinterpret_cast<const double2*>(p); };
    auto st = [](unsigned char* p, double2 v) { *reinterpret_cast<double2*>(p) = v; };
    // A CTA's rows cover its lane groups in increasing order, each in one contiguous stretch: the sum
    // of lane group lgf is final when the CTA leaves it and goes straight to the CTA's partial row
    // (fixed order over the CTA's threads); columns of lane groups the CTA never touched are zeroed
    // at the end.
    auto flush = [&](int lgf) {
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const double2 s = cta_lane_sum<TL, CONS>(acc[k], t, sred);  // (fixed-order shuffle tree)
            if (t < TL && g.red[k] != nullptr && (k < 6 || tail)) {
                const int v = lgf * TL + t;
                double* row = g.red[k] + (size_t)blockIdx.x * g.RP;
                if (PEIERLS) {
                    row[v] = s.x;
                } else {
                    row[2 * v] = s.x;
                    row[2 * v + 1] = s.y;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 7; ++k) acc[k] = make_double2(0.0, 0.0);
    };
    // 2 H~ x - p from the 4 neighbours (y neighbours carry the Peierls phase) and the site value
    auto step_val = [&](double2 x, double2 xm, double2 xp, double2 ym, double2 yp, double e, double2 ph, double2 p) {
        return hop_step<PEIERLS>(x, xm, xp, ym, yp, 2.0 * e, 2.0 * g.t, ph, p);
    };
    // slot byte offsets of tile x index lx (level 0: [-3, TX+2]; level -1 and 1: [-2, TX+1]; level 2: [-1, TX])
    auto oA = [&](int lx, int ll) { return (lx + 3) * SITE + ll * 16; };
    auto oP = [&](int lx, int ll) { return (lx + 2) * SITE + ll * 16; };
    // compressed level-1 / level-2 rows: halo sites, then the two ends of every run
    auto bix = [&](int lx) { return lx < 0 ? lx : (lx >= TX ? 2 * (TX / NPI) + (lx - TX) : 2 * (lx / NPI) + (lx % NPI != 0)); };
    auto oB1 = [&](int lx, int ll) { return (bix(lx) + 2) * SITE + ll * 16; };
    auto oB2 = [&](int lx, int ll) { return (bix(lx) + 1) * SITE + ll * 16; };

    LoadCursor cs;  // segment iterator of the consumers (same sequence)
    cs.init(g, w_begin, w_end, 0);
    int ia = 0, ip = 0, cur_lg = -1;
    while (cs.valid) {
        const int lg = cs.lg, m0 = cs.m0, H = cs.H, x0 = cs.px * TX;
        if (cur_lg != -1 && lg != cur_lg) flush(cur_lg);
        cur_lg = lg;
        // thread k0 owns the NPI CONSECUTIVE sites k0*NPI .. k0*NPI+NPI-1 of the row: x-neighbours
        // inside that run come from its registers, only the two ends from shared memory
        const long long g0 = (long long)(x0 + k0 * NPI) * g.RG + (long long)lg * TL + l;
        const long long gstep = (long long)g.RG;
        const long long growstep = (long long)g.L0 * g.RG;
        if (PEIERLS) {
            if (t < TX + 6) sphase[t] = scale2(2.0 * g.t, __ldg(g.phase + (x0 + t - 3 + 2 * g.L0) % g.L0));
            __syncthreads();
        }
        const int ia_seg = ia;
        int s0 = ia_seg % kSAT;        // ring slot of a_n row r1-1
        int ps = ip % kSPT;
        int r2 = (m0 - 3 + 2 * g.L1) % g.L1;  // level-2 row of iteration 0
        int r3 = (m0 - 4 + 2 * g.L1) % g.L1;  // level-3 row
        // per interior site: a_n rows r1-1, r1 (am, ac); level 1 rows r1-2, r1-1 (bm, bc); level 2
        // rows r2-2, r2-1 (cm, cc); eps~ at rows r1-1, r1-2 (e2, e3)
        // Register histories, 3 rows deep, with roles rotating every row: at iteration q the a_n rows
        // r1-1, r1, r1+1 of the run are XA[q%3], XA[(q+1)%3], XA[(q+2)%3] (the new row overwrites the
        // oldest), the same for level 1 (rows r1-2, r1-1, r1: XB), level 2 (rows r2-2, r2-1, r2: XC) and
        // eps~ (rows r1-2, r1-1, r1: XE).  The row loop is unrolled by 3 so the indices are compile-
        // time constants: no register moves for the rolling (ncu: ~20% of the instructions were moves).
        double2 XA[3][NPI], XB[3][NPI], XC[3][NPI];
        double XE[3][NPI];
        const int lx0 = k0 * NPI;  // first site of this thread
        double2 PH[NPI];  // 2t e^{i phi} of the run's sites (Landau gauge: a function of x only)
#pragma unroll
        for (int p = 0; p < NPI; ++p) PH[p] = PEIERLS ? sphase[lx0 + p + 3] : make_double2(0.0, 0.0);
        // S (steady): all three levels computed and owned (q in [4, H+2)) -- compile-time, so the
        // levels of a row form one basic block the scheduler can interleave
        auto row = [&](const int q, const int u, auto steady) {  // iteration q of the segment, u = q % 3
            constexpr bool S = decltype(steady)::value;
            const int i0 = ia_seg + q;
            const int s1 = s0 + 1 == kSAT ? 0 : s0 + 1;
            const int s2 = s1 + 1 == kSAT ? 0 : s1 + 1;
            if (!S && q == 0) {
                mbar_wait(fullA + s0, (uint32_t)((i0 / kSAT) & 1));
                mbar_wait(fullA + s1, (uint32_t)(((i0 + 1) / kSAT) & 1));
            }
            mbar_wait(fullA + s2, (uint32_t)(((i0 + 2) / kSAT) & 1));
            mbar_wait(fullP + ps, (uint32_t)((ip / kSPT) & 1));
            const unsigned char* A0 = ringA + s0 * SL.a_bytes;  // a_n row r1-1
            const unsigned char* A1 = ringA + s1 * SL.a_bytes;  // a_n row r1
            const unsigned char* A2 = ringA + s2 * SL.a_bytes;  // a_n row r1+1
            const unsigned char* Pq = ringP + ps * SL.p_bytes;  // a_{n-1} row r1
            unsigned char* B1n = ringB1 + u * SL.b1_bytes;                             // level 1 row r1 (written)
            const unsigned char* B1c = ringB1 + ((u + 2) % 3) * SL.b1_bytes;          // row r1-1
            const unsigned char* B1m = ringB1 + ((u + 1) % 3) * SL.b1_bytes;          // row r1-2
            unsigned char* B2n = ringB2 + (q & 1) * SL.b2_bytes;                      // level 2 row r2 (written)
            const unsigned char* B2c = ringB2 + ((q & 1) ^ 1) * SL.b2_bytes;          // level 2 row r2-1 = r3
            const bool do2 = S || q >= 2, do3 = S || q >= 4;
            const bool own1 = S || (q >= 2 && q < H + 2);  // r1 in [m0, m1)
            const bool own2 = S || (q >= 3 && q < H + 3);  // r2 in [m0, m1)
            double2* outB = g.outB + r2 * growstep + g0;
            double2* outC = g.outC + r3 * growstep + g0;
            double2(&am)[NPI] = XA[u];
            double2(&ac)[NPI] = XA[(u + 1) % 3];
            double2(&ap)[NPI] = XA[(u + 2) % 3];
            double2(&bm)[NPI] = XB[u];
            double2(&bc)[NPI] = XB[(u + 1) % 3];
            double2(&b)[NPI] = XB[(u + 2) % 3];
            double2(&cm)[NPI] = XC[u];
            double2(&cc)[NPI] = XC[(u + 1) % 3];
            double2(&c)[NPI] = XC[(u + 2) % 3];
            double(&e3)[NPI] = XE[u];
            double(&e2)[NPI] = XE[(u + 1) % 3];
            double(&en)[NPI] = XE[(u + 2) % 3];
            // halo sites of this thread (level 1 at hx1; level 2 at hx1 when hx1 is -1 or TX)
            if (t < 4 * TL) {
                const int hg = t / TL, hl = t % TL;  // 0: x0-1, 1: x0+TX, 2: x0-2, 3: x0+TX+1
                const int hx = hg == 0 ? -1 : (hg == 1 ? TX : (hg == 2 ? -2 : TX + 1));
                const double2 ph = PEIERLS ? sphase[hx + 3] : make_double2(0.0, 0.0);
                const double e1 = ONSITE ? SL.eps(A1, hx, TX) : g.shift;
                const double2 hb = step_val(ld(A1 + oA(hx, hl)), ld(A1 + oA(hx - 1, hl)), ld(A1 + oA(hx + 1, hl)),
                                            ld(A0 + oA(hx, hl)), ld(A2 + oA(hx, hl)), e1, ph, ld(Pq + oP(hx, hl)));
                st(B1n + oB1(hx, hl), hb);
                if (hg < 2 && do2) {
                    const double e = ONSITE ? SL.eps(A0, hx, TX) : g.shift;
                    const double2 hc = step_val(ld(B1c + oB1(hx, hl)), ld(B1c + oB1(hx - 1, hl)), ld(B1c + oB1(hx + 1, hl)),
                                                ld(B1m + oB1(hx, hl)), hb, e, ph, ld(A0 + oA(hx, hl)));
                    st(B2n + oB2(hx, hl), hc);
                }
            }
            if (!S && q == 0) {
#pragma unroll
                for (int p = 0; p < NPI; ++p) {
                    am[p] = ld(A0 + oA(lx0 + p, l));
                    ac[p] = ld(A1 + oA(lx0 + p, l));
                }
            }
            // level 1 at row r1 for the run: a_n row r1+1 of the run, the run's x-end neighbours
#pragma unroll
            for (int p = 0; p < NPI; ++p) ap[p] = ld(A2 + oA(lx0 + p, l));
            {
                const double2 xl = ld(A1 + oA(lx0 - 1, l)), xr = ld(A1 + oA(lx0 + NPI, l));
#pragma unroll
                for (int p = 0; p < NPI; ++p) {
                    const int lx = lx0 + p;
                    const double2 ph = PH[p];
                    const double e1 = ONSITE ? reinterpret_cast<const double*>(A1 + SL.eps_m)[lx] : g.shift;
                    b[p] = step_val(ac[p], p == 0 ? xl : ac[p - 1], p == NPI - 1 ? xr : ac[p + 1], am[p], ap[p], e1, ph,
                                    ld(Pq + oP(lx, l)));
                    if (own1) {
                        dot_acc<PEIERLS>(acc[0], ac[p], ac[p]);
                        dot_acc<PEIERLS>(acc[1], ac[p], b[p]);
                    }
                    if (ONSITE) en[p] = e1;
                }
                st(B1n + oB1(lx0, l), b[0]);  // the run's ends: the neighbouring runs' and the halo's x-neighbours
                st(B1n + oB1(lx0 + NPI - 1, l), b[NPI - 1]);
            }
            // level 2 at row r2 = r1-1: centre bc, x-neighbours bc (run) / B1c (ends), y-neighbours bm, b
            if (do2) {
                const double2 xl = ld(B1c + oB1(lx0 - 1, l)), xr = ld(B1c + oB1(lx0 + NPI, l));
#pragma unroll
                for (int p = 0; p < NPI; ++p) {
                    const double2 ph = PH[p];
                    c[p] = step_val(bc[p], p == 0 ? xl : bc[p - 1], p == NPI - 1 ? xr : bc[p + 1], bm[p], b[p],
                                    ONSITE ? e2[p] : g.shift, ph, am[p]);
                    if (own2) {
                        __stcs(outB + p * gstep, c[p]);
                        dot_acc<PEIERLS>(acc[2], bc[p], bc[p]);
                        dot_acc<PEIERLS>(acc[3], bc[p], c[p]);
                    }
                }
                st(B2n + oB2(lx0, l), c[0]);
                st(B2n + oB2(lx0 + NPI - 1, l), c[NPI - 1]);
            }
            // level 3 at row r3 = r1-2: centre cc, x-neighbours cc (run) / B2c (ends), y-neighbours cm, c;
            // "- a_{n+1}" at row r1-2 = bm
            if (do3) {
                const double2 xl = ld(B2c + oB2(lx0 - 1, l)), xr = ld(B2c + oB2(lx0 + NPI, l));
#pragma unroll
                for (int p = 0; p < NPI; ++p) {
                    const double2 ph = PH[p];
                    const double2 d = step_val(cc[p], p == 0 ? xl : cc[p - 1], p == NPI - 1 ? xr : cc[p + 1], cm[p], c[p],
                                               ONSITE ? e3[p] : g.shift, ph, bm[p]);
                    __stcs(outC + p * gstep, d);
                    dot_acc<PEIERLS>(acc[4], cc[p], cc[p]);
                    dot_acc<PEIERLS>(acc[5], cc[p], d);
                    dot_acc<PEIERLS>(acc[6], d, d);  // (kept only with the tail; no branch in the row)
                }
            }
            __syncthreads();  // row q done: a_n row r1-1 and a_{n-1} row r1 are free; B rings advance
            if (t == PRODUCER) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issueA(s0);
                issueP(ps);
            }
            ++ip;
            s0 = s1;
            ps = ps + 1 == kSPT ? 0 : ps + 1;
            r2 = r2 + 1 == g.L1 ? 0 : r2 + 1;
            r3 = r3 + 1 == g.L1 ? 0 : r3 + 1;
        };
        for (int q0 = 0; q0 < H + 4; q0 += 3) {
            if (q0 >= 4 && q0 + 2 < H + 2) {
                row(q0, 0, std::true_type{});
                row(q0 + 1, 1, std::true_type{});
                row(q0 + 2, 2, std::true_type{});
            } else {
                row(q0, 0, std::false_type{});
                if (q0 + 1 < H + 4) row(q0 + 1, 1, std::false_type{});
                if (q0 + 2 < H + 4) row(q0 + 2, 2, std::false_type{});
            }
        }
        if (t == PRODUCER) {  // the segment's last two a_n rows are free too
            issueA((ia_seg + H + 4) % kSAT);
            issueA((ia_seg + H + 5) % kSAT);
        }
        ia = ia_seg + H + 6;
        cs.seg(g, 0);
    }
    if (cur_lg != -1) flush(cur_lg);
    // zeros in this CTA's row for the lane groups it did not process, and in rows >= gridDim.x
    const int lg_lo = (int)(w_begin / ((long long)g.PX * g.L1));
    const int lg_hi = w_end > w_begin ? (int)((w_end - 1) / ((long long)g.PX * g.L1)) : -1;  // inclusive
    const int per_lg = PEIERLS ? TL : 2 * TL;  // partial-row columns of one lane group
    for (int k = 0; k < 7; ++k) {
        double* rowk = g.red[k];
        if (rowk == nullptr || (k == 6 && !tail)) continue;
        for (int v = t; v < g.RP; v += blockDim.x) {
            const int lgv = v / per_lg;
            if (lgv < lg_lo || lgv > lg_hi) rowk[(size_t)blockIdx.x * g.RP + v] = 0.0;
        }
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int v = t; v < g.RP; v += blockDim.x) rowk[(size_t)rr * g.RP + v] = 0.0;
    }
}

}  // namespace kpm
