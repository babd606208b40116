// kpm_quad.cuh -- FOUR recursion steps per HBM pass (temporal blocking), 2D lattices.
//
// One launch advances the recursion by four steps (Eq 18 four times), reading a_n and a_{n-1}
// from HBM once and writing a_{n+3} and a_{n+4} once: 4 D R s bytes per four steps (the
// three-step kernel, kpm_tri.cuh, moves the same per three).  a_{n+1} .. a_{n+3} live in
// shared-memory row rings and registers.
//
// The march of kpm_tri.cuh, one level deeper (pencil of TX sites x TL lanes, rows of y):
//   level 0  a_n      rows m0-4 .. m1+3, sites x0-4 .. x0+TX+3  (TMA: main box + two 4-site boxes)
//   level -1 a_{n-1}  rows m0-3 .. m1+2, sites x0-3 .. x0+TX+2  (TMA: main box + two 3-site boxes)
//   level j  a_{n+j}  computed at sites x0-(4-j) .. x0+TX+3-j, row r1-(j-1) of iteration q,
//                     r1 = m0-3+q (j = 1..4); levels 3 and 4 are stored for rows m0..m1-1
// Interior sites: 8 warps, each thread a run of NPI consecutive sites of one lane; the run's
// rows of levels 0-3 roll in registers (three rows per level, roles rotating with the row loop
// unrolled by 3 -- no register moves), x-neighbours inside the run from registers, the run ends
// through shared memory.  Halo sites: "chains" -- level 1, 2, 3 at the site x0-1 (or x0+TX),
// levels 1, 2 at x0-2 (x0+TX+1), level 1 at x0-3 (x0+TX+2) -- a chain's own lower level is its
// y-neighbour for the next level, so no barrier splits it.  The 2 TL chains of distance 1 run in
// warp 0, those of distances 2 and 3 in warp 1 (3 and 2 extra evaluations; interior: 4 NPI per
// thread).  (A ninth warp for the chains would cap registers at 168 -- three warps on one SM
// sub-partition -- and spill.)  The last thread issues the TMA refills.  One CTA barrier per row.
//
// Reductions: <a_{n+k}|a_{n+k}>, <a_{n+k}|a_{n+k+1}> for k = 0..3 (and the odd-N tail
// <a_{n+4}|a_{n+4}>) over owned sites, per lane, fixed order; written per lane group straight
// to the CTA's partial row.
#pragma once
#include "kpm_tri.cuh"

namespace kpm {

struct QuadGeom {
    int L0, L1;          // lattice extents
    int TX, TL, RG, G_L, PX;
    long long W;         // output rows = G_L * PX * L1
    int RP;
    int rows_total;      // partial-sum rows per slot (>= gridDim.x; extra rows are zeroed)
    double t, shift;
    const double2* phase;
    double* red[9];      // slots 2n .. 2n+7, (tail) 2n+8; red[8] nullable
    double2* outB;       // a_{n+3}
    double2* outC;       // a_{n+4}
};

constexpr int kThreadsQuad = 256;       // 8 warps: two per SM sub-partition, up to 255 registers
#ifndef KPM_SAQ
#define KPM_SAQ 10
#endif
#ifndef KPM_SPQ
#define KPM_SPQ 6
#endif
constexpr int kSAQ = KPM_SAQ;           // a_n ring: rows r1-2 .. r1+1 in use (eps of level 3's halo) + 6 ahead
constexpr int kSPQ = KPM_SPQ;           // a_{n-1} ring (5 ahead)

__host__ __device__ constexpr int quad_runs(int TL) { return 256 / TL; }  // runs per row
// a_{n-1} halo sites per side: 3, or 4 when 3 sites are not a multiple of 128 bytes (4-lane tiles:
// every TMA destination of a slot stays 128-byte aligned)
__host__ __device__ constexpr int quad_php(int TL) { return (3 * TL * 16) % 128 == 0 ? 3 : 4; }
// a_n slot: [4 halo][TX][4 halo] sites, then eps~ pieces [4 left][TX][4 right] (128-byte aligned);
// a_{n-1} slot [3][TX][3]; level rings keep the halo sites and the two ends of every run:
// level 1 [3 halo][2 per run][3 halo], level 2 [2][..][2], level 3 [1][..][1].
struct QuadLayout {
    int site, a_bytes, eps_l, eps_m, eps_r, p_bytes, b1_bytes, b2_bytes, b3_bytes;
    __host__ __device__ constexpr QuadLayout(int TX, int TL, bool onsite)
        : site(TL * 16),
          a_bytes(onsite ? (TX + 8) * TL * 16 + 128 + (TX * 8 + 127) / 128 * 128 + 128 : (TX + 8) * TL * 16),
          eps_l((TX + 8) * TL * 16),
          eps_m((TX + 8) * TL * 16 + 128),
          eps_r((TX + 8) * TL * 16 + 128 + (TX * 8 + 127) / 128 * 128),
          p_bytes(((TX + 2 * quad_php(TL)) * TL * 16 + 127) / 128 * 128),
          b1_bytes(((2 * quad_runs(TL) + 6) * TL * 16 + 127) / 128 * 128),
          b2_bytes(((2 * quad_runs(TL) + 4) * TL * 16 + 127) / 128 * 128),
          b3_bytes(((2 * quad_runs(TL) + 2) * TL * 16 + 127) / 128 * 128) {}
    // eps~ at tile x index lx in [-4, TX+3]
    __device__ __forceinline__ double eps(const unsigned char* slot, int lx, int TX) const {
        return *reinterpret_cast<const double*>(
            slot + (lx < 0 ? eps_l + (lx + 4) * 8 : (lx < TX ? eps_m + lx * 8 : eps_r + (lx - TX) * 8)));
    }
};

__host__ __device__ inline size_t quad_smem_bytes(int TX, int TL, bool onsite) {
    const QuadLayout S(TX, TL, onsite);
    return (size_t)kSAQ * S.a_bytes + (size_t)kSPQ * S.p_bytes + 3 * (size_t)S.b1_bytes + 3 * (size_t)S.b2_bytes +
           2 * (size_t)S.b3_bytes + (size_t)kThreadsQuad * 16 + (size_t)(TX + 8) * 16 + (kSAQ + kSPQ) * 8;
}

template <int TL, int TX, bool ONSITE, bool PEIERLS>
__global__ void __launch_bounds__(kThreadsQuad, 1)
    kpm_step_quad_kernel(const __grid_constant__ CUtensorMap mapA,    // a_n main box {2TL, TX, 1}
                         const __grid_constant__ CUtensorMap mapA4,   // a_n 4-site box {2TL, 4, 1}
                         const __grid_constant__ CUtensorMap mapP,    // a_{n-1} main box
                         const __grid_constant__ CUtensorMap mapP3,   // a_{n-1} halo box {2TL, PHP, 1}
                         const __grid_constant__ CUtensorMap mapE,    // eps~ box {TX, 1}
                         const __grid_constant__ CUtensorMap mapE4,   // eps~ box {4, 1}
                         const QuadGeom g, const int tail) {
    pdl_entry();
    constexpr int CONS = 256;
    constexpr int PRODUCER = CONS - 1;  // (chains: warps 0 and 1)
    constexpr int KSTEP = CONS / TL;  // runs per row
    constexpr int NPI = TX / KSTEP;   // sites per run
    static_assert(TX % KSTEP == 0 && NPI >= 1 && TL * 16 >= 64 && 4 * TL <= 32, "tile shape");
    constexpr int PHP = quad_php(TL);  // a_{n-1} halo sites per side in a slot (3 needed)
    constexpr int SITE = TL * 16;
    constexpr QuadLayout SL(TX, TL, ONSITE);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + kSAQ * SL.a_bytes;
    unsigned char* ringB1 = ringP + kSPQ * SL.p_bytes;
    unsigned char* ringB2 = ringB1 + 3 * SL.b1_bytes;
    unsigned char* ringB3 = ringB2 + 3 * SL.b2_bytes;
    double2* sred = reinterpret_cast<double2*>(ringB3 + 2 * SL.b3_bytes);  // [CONS]
    double2* sphase = sred + CONS;                                         // [TX + 8]: x0-4 .. x0+TX+3
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sphase + TX + 8);
    uint64_t* fullP = fullA + kSAQ;

    const int t = threadIdx.x;
    const long long w_begin = g.W * blockIdx.x / gridDim.x;
    const long long w_end = g.W * (blockIdx.x + 1) / gridDim.x;

    __shared__ LoadCursor cur_smem[2];
    __shared__ uint64_t pol_smem;
    LoadCursor& ca = cur_smem[0];
    LoadCursor& cp = cur_smem[1];
    auto issueA = [&](int slot) {  // next a_n row (4-site halos) into `slot`
        if (!ca.valid) return;
        const int row = ca.row, c0 = ca.c0, x0 = ca.x0, xl = ca.xl, xr = ca.xr;
        unsigned char* dst = ringA + slot * SL.a_bytes;
        mbar_expect_tx(fullA + slot, (TX + 8) * SITE + (ONSITE ? (TX + 8) * 8 : 0));
        tma_load(dst, &mapA4, fullA + slot, c0, xl, row);
        tma_load(dst + 4 * SITE, &mapA, fullA + slot, c0, x0, row);
        tma_load(dst + (TX + 4) * SITE, &mapA4, fullA + slot, c0, xr, row);
        if (ONSITE) {
            tma_load_2d(dst + SL.eps_l, &mapE4, fullA + slot, xl, row);
            tma_load_2d(dst + SL.eps_m, &mapE, fullA + slot, x0, row);
            tma_load_2d(dst + SL.eps_r, &mapE4, fullA + slot, xr, row);
        }
        ca.next(g, 8);
    };
    auto issueP = [&](int slot) {  // next a_{n-1} row (3-site halos) into `slot`
        if (!cp.valid) return;
        const int row = cp.row, c0 = cp.c0, x0 = cp.x0, xl = cp.xl, xr = cp.xr;
        unsigned char* dst = ringP + slot * SL.p_bytes;
        mbar_expect_tx(fullP + slot, (TX + 2 * PHP) * SITE);
        const uint64_t pol = pol_smem;
        tma_load_hint(dst, &mapP3, fullP + slot, c0, xl, row, pol);
        tma_load_hint(dst + PHP * SITE, &mapP, fullP + slot, c0, x0, row, pol);
        tma_load_hint(dst + (TX + PHP) * SITE, &mapP3, fullP + slot, c0, xr, row, pol);
        cp.next(g, 6, PHP);
    };
    if (t == PRODUCER) {
        for (int i = 0; i < kSAQ; ++i) mbar_init(fullA + i, 1);
        for (int i = 0; i < kSPQ; ++i) mbar_init(fullP + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&mapA);
        prefetch_tmap(&mapA4);
        prefetch_tmap(&mapP);
        prefetch_tmap(&mapP3);
        if (ONSITE) {
            prefetch_tmap(&mapE);
            prefetch_tmap(&mapE4);
        }
        pol_smem = policy_evict_first();
        ca.init(g, w_begin, w_end, 8);
        cp.init(g, w_begin, w_end, 6, PHP);
        for (int i = 0; i < kSAQ; ++i) issueA(i);
        for (int i = 0; i < kSPQ; ++i) issueP(i);
    }
    __syncthreads();

    // halo chain of this thread: distance 1 in warp 0, distances 2 and 3 in warp 1 (or none)
    const int chain = t < 2 * TL ? t : (t >= 32 && t < 32 + 4 * TL ? t - 32 + 2 * TL : -1);
    const int l = t % TL;
    const int k0 = t / TL;
    double2 acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = make_double2(0.0, 0.0);
    auto ld = [](const unsigned char* p) { return *reinterpret_cast<const double2*>(p); };
    auto st = [](unsigned char* p, double2 v) { *reinterpret_cast<double2*>(p) = v; };
    auto flush = [&](int lgf) {
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const double2 s = cta_lane_sum<TL, CONS>(acc[k], t, sred);  // (fixed-order shuffle tree)
            if (t < TL && g.red[k] != nullptr && (k < 8 || tail)) {
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
        for (int k = 0; k < 9; ++k) acc[k] = make_double2(0.0, 0.0);
    };
    auto step_val = [&](double2 x, double2 xm, double2 xp, double2 ym, double2 yp, double e, double2 ph, double2 p) {
        return hop_step<PEIERLS>(x, xm, xp, ym, yp, 2.0 * e, 2.0 * g.t, ph, p);
    };
    // slot offsets of tile x index lx: level 0 [-4, TX+3], level -1 [-3, TX+2]; level rings keep the
    // halo and the run ends: bix maps an interior run end to its packed index
    auto oA = [&](int lx, int ll) { return (lx + 4) * SITE + ll * 16; };
    auto oP = [&](int lx, int ll) { return (lx + PHP) * SITE + ll * 16; };
    auto bix = [&](int lx) { return lx < 0 ? lx : (lx >= TX ? 2 * KSTEP + (lx - TX) : 2 * (lx / NPI) + (lx % NPI != 0)); };
    auto oB1 = [&](int lx, int ll) { return (bix(lx) + 3) * SITE + ll * 16; };
    auto oB2 = [&](int lx, int ll) { return (bix(lx) + 2) * SITE + ll * 16; };
    auto oB3 = [&](int lx, int ll) { return (bix(lx) + 1) * SITE + ll * 16; };

    LoadCursor cs;
    cs.init(g, w_begin, w_end, 0);
    int ia = 0, ps = 0, cur_lg = -1, ipc = 0;  // a_n ring index at the segment start; a_{n-1} ring slot and index
    while (cs.valid) {
        const int lg = cs.lg, m0 = cs.m0, H = cs.H, x0 = cs.px * TX;
        if (cur_lg != -1 && lg != cur_lg) flush(cur_lg);
        cur_lg = lg;
        const long long g0 = (long long)(x0 + k0 * NPI) * g.RG + (long long)lg * TL + l;
        const long long gstep = (long long)g.RG;
        const long long growstep = (long long)g.L0 * g.RG;
        if (PEIERLS) {
            if (t < TX + 8) sphase[t] = scale2(2.0 * g.t, __ldg(g.phase + (x0 + t - 4 + 2 * g.L0) % g.L0));
            __syncthreads();
        }
        const int ia_seg = ia;
        int r3 = (m0 - 5 + 2 * g.L1) % g.L1;  // level-3 row of iteration 0 (r1 - 2)
        int r4 = (m0 - 6 + 2 * g.L1) % g.L1;  // level-4 row
        // a_n rows: index i <-> row m0-4+i; iteration q: r1 = m0-3+q <-> index q+1; rows r1-2 .. r1+1 in use
        // registers: levels 0-3 of the run, three rows each, roles rotating with q % 3
        double2 XA[3][NPI], XB[3][NPI], XC[3][NPI], XD[3][NPI];
        double E2[NPI], E3[NPI], E4[NPI];  // eps~ at rows r2, r3, r4 (interior)
        const int lx0 = k0 * NPI;
        double2 PH[NPI];  // 2t e^{i phi} of the run's sites (Landau gauge: a function of x only)
#pragma unroll
        for (int p = 0; p < NPI; ++p) PH[p] = PEIERLS ? sphase[lx0 + p + 4] : make_double2(0.0, 0.0);
        int s0 = ia_seg % kSAQ;  // slot of index q (row r1-1); index q+1 = r1, q+2 = r1+1, q-1 = r1-2
        // S (steady): all four levels computed and owned (q in [6, H+3)), compile-time
        auto row = [&](const int q, const int u, auto steady) {
            constexpr bool S = decltype(steady)::value;
            const int sA0 = s0;                                  // r1-1
            const int sA1 = sA0 + 1 == kSAQ ? 0 : sA0 + 1;       // r1
            const int sA2 = sA1 + 1 == kSAQ ? 0 : sA1 + 1;       // r1+1
            const int sAm = sA0 == 0 ? kSAQ - 1 : sA0 - 1;       // r1-2 (q >= 1)
            const int i0 = ia_seg + q;
            if (!S && q == 0) {
                mbar_wait(fullA + sA0, (uint32_t)((i0 / kSAQ) & 1));
                mbar_wait(fullA + sA1, (uint32_t)(((i0 + 1) / kSAQ) & 1));
            }
            mbar_wait(fullA + sA2, (uint32_t)(((i0 + 2) / kSAQ) & 1));
            mbar_wait(fullP + ps, (uint32_t)((ipc / kSPQ) & 1));
            ++ipc;
            const unsigned char* Am = ringA + sAm * SL.a_bytes;  // a_n row r1-2 (eps of level 3)
            const unsigned char* A0 = ringA + sA0 * SL.a_bytes;  // a_n row r1-1
            const unsigned char* A1 = ringA + sA1 * SL.a_bytes;  // a_n row r1
            const unsigned char* A2 = ringA + sA2 * SL.a_bytes;  // a_n row r1+1
            const unsigned char* Pq = ringP + ps * SL.p_bytes;  // a_{n-1} row r1
            unsigned char* B1n = ringB1 + u * SL.b1_bytes;                     // level 1 row r1
            const unsigned char* B1c = ringB1 + ((u + 2) % 3) * SL.b1_bytes;  // level 1 row r1-1 = r2
            const unsigned char* B1m = ringB1 + ((u + 1) % 3) * SL.b1_bytes;  // level 1 row r1-2
            unsigned char* B2n = ringB2 + u * SL.b2_bytes;                     // level 2 row r2
            const unsigned char* B2c = ringB2 + ((u + 2) % 3) * SL.b2_bytes;  // level 2 row r2-1 = r3
            const unsigned char* B2m = ringB2 + ((u + 1) % 3) * SL.b2_bytes;  // level 2 row r2-2
            unsigned char* B3n = ringB3 + (q & 1) * SL.b3_bytes;              // level 3 row r3
            const unsigned char* B3c = ringB3 + ((q & 1) ^ 1) * SL.b3_bytes;  // level 3 row r3-1 = r4
            const bool do2 = S || q >= 2, do3 = S || q >= 4, do4 = S || q >= 6;
            const bool own1 = S || (q >= 3 && q < H + 3), own2 = S || (q >= 4 && q < H + 4),
                       own3 = S || (q >= 5 && q < H + 5);
            if (chain >= 0) {
                // chain c of 2 TL per distance d: side c / TL, lane c % TL; (d = 1) levels 1-3 at x0-1 /
                // x0+TX, (d = 2) levels 1-2 at x0-2 / x0+TX+1, (d = 3) level 1 at x0-3 / x0+TX+2
                {
                    const int c = chain;
                    const int d = 1 + c / (2 * TL), side = (c / TL) & 1, hl = c % TL;
                    const int hx = side == 0 ? -d : TX - 1 + d;
                    const double2 ph = PEIERLS ? sphase[hx + 4] : make_double2(0.0, 0.0);
                    // level 1 at row r1
                    const double e1 = ONSITE ? SL.eps(A1, hx, TX) : g.shift;
                    const double2 hb = step_val(ld(A1 + oA(hx, hl)), ld(A1 + oA(hx - 1, hl)), ld(A1 + oA(hx + 1, hl)),
                                                ld(A0 + oA(hx, hl)), ld(A2 + oA(hx, hl)), e1, ph, ld(Pq + oP(hx, hl)));
                    st(B1n + oB1(hx, hl), hb);
                    if (d <= 2 && do2) {  // level 2 at row r2 = r1-1
                        const double e2 = ONSITE ? SL.eps(A0, hx, TX) : g.shift;
                        const double2 hc = step_val(ld(B1c + oB1(hx, hl)), ld(B1c + oB1(hx - 1, hl)),
                                                    ld(B1c + oB1(hx + 1, hl)), ld(B1m + oB1(hx, hl)), hb, e2, ph,
                                                    ld(A0 + oA(hx, hl)));
                        st(B2n + oB2(hx, hl), hc);
                        if (d == 1 && do3) {  // level 3 at row r3 = r1-2; "- a_{n+1}" at row r1-2 = B1m
                            const double e3 = ONSITE ? SL.eps(Am, hx, TX) : g.shift;
                            const double2 hd = step_val(ld(B2c + oB2(hx, hl)), ld(B2c + oB2(hx - 1, hl)),
                                                        ld(B2c + oB2(hx + 1, hl)), ld(B2m + oB2(hx, hl)), hc, e3, ph,
                                                        ld(B1m + oB1(hx, hl)));
                            st(B3n + oB3(hx, hl), hd);
                        }
                    }
                }
            }
            {
                double2(&am)[NPI] = XA[u];
                double2(&ac)[NPI] = XA[(u + 1) % 3];
                double2(&ap)[NPI] = XA[(u + 2) % 3];
                double2(&bm)[NPI] = XB[u];
                double2(&bc)[NPI] = XB[(u + 1) % 3];
                double2(&b)[NPI] = XB[(u + 2) % 3];
                double2(&cm)[NPI] = XC[u];
                double2(&cc)[NPI] = XC[(u + 1) % 3];
                double2(&c)[NPI] = XC[(u + 2) % 3];
                double2(&dm)[NPI] = XD[u];
                double2(&dc)[NPI] = XD[(u + 1) % 3];
                double2(&d)[NPI] = XD[(u + 2) % 3];
                double2* outB = g.outB + r3 * growstep + g0;
                double2* outC = g.outC + r4 * growstep + g0;
                if (!S && q == 0) {
#pragma unroll
                    for (int p = 0; p < NPI; ++p) {
                        am[p] = ld(A0 + oA(lx0 + p, l));
                        ac[p] = ld(A1 + oA(lx0 + p, l));
                    }
                }
#pragma unroll
                for (int p = 0; p < NPI; ++p) ap[p] = ld(A2 + oA(lx0 + p, l));
                double en[NPI];
                {  // level 1 at row r1
                    const double2 xl = ld(A1 + oA(lx0 - 1, l)), xr = ld(A1 + oA(lx0 + NPI, l));
#pragma unroll
                    for (int p = 0; p < NPI; ++p) {
                        const int lx = lx0 + p;
                        const double2 ph = PH[p];
                        const double e1 = ONSITE ? reinterpret_cast<const double*>(A1 + SL.eps_m)[lx] : g.shift;
                        en[p] = e1;
                        b[p] = step_val(ac[p], p == 0 ? xl : ac[p - 1], p == NPI - 1 ? xr : ac[p + 1], am[p], ap[p], e1,
                                        ph, ld(Pq + oP(lx, l)));
                        if (own1) {
                            dot_acc<PEIERLS>(acc[0], ac[p], ac[p]);
                            dot_acc<PEIERLS>(acc[1], ac[p], b[p]);
                        }
                    }
                    st(B1n + oB1(lx0, l), b[0]);
                    st(B1n + oB1(lx0 + NPI - 1, l), b[NPI - 1]);
                }
                if (do2) {  // level 2 at row r2 = r1-1: centre bc, y-neighbours bm, b; "- a_n" = am
                    const double2 xl = ld(B1c + oB1(lx0 - 1, l)), xr = ld(B1c + oB1(lx0 + NPI, l));
#pragma unroll
                    for (int p = 0; p < NPI; ++p) {
                        const double2 ph = PH[p];
                        c[p] = step_val(bc[p], p == 0 ? xl : bc[p - 1], p == NPI - 1 ? xr : bc[p + 1], bm[p], b[p],
                                        ONSITE ? E2[p] : g.shift, ph, am[p]);
                        if (own2) {
                            dot_acc<PEIERLS>(acc[2], bc[p], bc[p]);
                            dot_acc<PEIERLS>(acc[3], bc[p], c[p]);
                        }
                    }
                    st(B2n + oB2(lx0, l), c[0]);
                    st(B2n + oB2(lx0 + NPI - 1, l), c[NPI - 1]);
                }
                if (do3) {  // level 3 at row r3 = r1-2: centre cc, y-neighbours cm, c; "- a_{n+1}" = bm
                    const double2 xl = ld(B2c + oB2(lx0 - 1, l)), xr = ld(B2c + oB2(lx0 + NPI, l));
#pragma unroll
                    for (int p = 0; p < NPI; ++p) {
                        const double2 ph = PH[p];
                        d[p] = step_val(cc[p], p == 0 ? xl : cc[p - 1], p == NPI - 1 ? xr : cc[p + 1], cm[p], c[p],
                                        ONSITE ? E3[p] : g.shift, ph, bm[p]);
                        if (own3) {
                            __stcs(outB + p * gstep, d[p]);
                            dot_acc<PEIERLS>(acc[4], cc[p], cc[p]);
                            dot_acc<PEIERLS>(acc[5], cc[p], d[p]);
                        }
                    }
                    st(B3n + oB3(lx0, l), d[0]);
                    st(B3n + oB3(lx0 + NPI - 1, l), d[NPI - 1]);
                }
                if (do4) {  // level 4 at row r4 = r1-3: centre dc, y-neighbours dm, d; "- a_{n+2}" = cm
                    const double2 xl = ld(B3c + oB3(lx0 - 1, l)), xr = ld(B3c + oB3(lx0 + NPI, l));
#pragma unroll
                    for (int p = 0; p < NPI; ++p) {
                        const double2 ph = PH[p];
                        const double2 e = step_val(dc[p], p == 0 ? xl : dc[p - 1], p == NPI - 1 ? xr : dc[p + 1], dm[p],
                                                   d[p], ONSITE ? E4[p] : g.shift, ph, cm[p]);
                        __stcs(outC + p * gstep, e);
                        dot_acc<PEIERLS>(acc[6], dc[p], dc[p]);
                        dot_acc<PEIERLS>(acc[7], dc[p], e);
                        dot_acc<PEIERLS>(acc[8], e, e);  // (kept only with the tail)
                    }
                }
                if (ONSITE) {  // eps~ history (rows r2, r3, r4 of the next iteration)
#pragma unroll
                    for (int p = 0; p < NPI; ++p) {
                        E4[p] = E3[p];
                        E3[p] = E2[p];
                        E2[p] = en[p];
                    }
                }
            }
            __syncthreads();  // row q done: a_n row r1-2 and a_{n-1} row r1 are free; rings advance
            if (t == PRODUCER) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (S || q >= 1) issueA(sAm);
                issueP(ps);
            }
            s0 = sA1;
            ps = ps + 1 == kSPQ ? 0 : ps + 1;
            r3 = r3 + 1 == g.L1 ? 0 : r3 + 1;
            r4 = r4 + 1 == g.L1 ? 0 : r4 + 1;
        };
        for (int q0 = 0; q0 < H + 6; q0 += 3) {
            if (q0 >= 6 && q0 + 2 < H + 3) {
                row(q0, 0, std::true_type{});
                row(q0 + 1, 1, std::true_type{});
                row(q0 + 2, 2, std::true_type{});
            } else {
                row(q0, 0, std::false_type{});
                if (q0 + 1 < H + 6) row(q0 + 1, 1, std::false_type{});
                if (q0 + 2 < H + 6) row(q0 + 2, 2, std::false_type{});
            }
        }
        if (t == PRODUCER) {  // the segment's last three a_n rows are free too
            issueA((ia_seg + H + 5) % kSAQ);
            issueA((ia_seg + H + 6) % kSAQ);
            issueA((ia_seg + H + 7) % kSAQ);
        }
        ia = ia_seg + H + 8;
        cs.seg(g, 0);
    }
    if (cur_lg != -1) flush(cur_lg);
    const int lg_lo = (int)(w_begin / ((long long)g.PX * g.L1));
    const int lg_hi = w_end > w_begin ? (int)((w_end - 1) / ((long long)g.PX * g.L1)) : -1;  // inclusive
    const int per_lg = PEIERLS ? TL : 2 * TL;
    for (int k = 0; k < 9; ++k) {
        double* rowk = g.red[k];
        if (rowk == nullptr || (k == 8 && !tail)) continue;
        for (int v = t; v < g.RP; v += blockDim.x) {
            const int lgv = v / per_lg;
            if (lgv < lg_lo || lgv > lg_hi) rowk[(size_t)blockIdx.x * g.RP + v] = 0.0;
        }
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int v = t; v < g.RP; v += blockDim.x) rowk[(size_t)rr * g.RP + v] = 0.0;
    }
}

}  // namespace kpm
