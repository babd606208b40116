// kpm_tmak.cuh -- KS recursion steps per HBM pass (deep temporal blocking), 2D lattices.
//
// One launch advances the recursion (Eq 18) by KS steps,
//     a_{n+j} = 2 H~ a_{n+j-1} - a_{n+j-2},   j = 1 .. KS,
// reading a_n and a_{n-1} from HBM once and writing only a_{n+KS-1} and a_{n+KS}:
// 4 D R s bytes per KS steps (KS = 2 is kpm_tma2.cuh's case).
// The intermediate blocks a_{n+1} .. a_{n+KS-2} never leave the SM.
//
// Geometry.  A CTA marches a pencil of TX sites x TL lanes over y (rows).  "Level" j is
// the block a_{n+j}: level 0 = a_n and level -1 = a_{n-1} come from TMA, levels 1..KS are
// computed.  In the iteration for row r, level j is computed at row r - (j-1) (one row
// behind the level below it), on the tile x range widened by KS - j halo sites per side
// (halo sites are recomputed, not exchanged):
//     level j at row r-j+1 needs level j-1 at rows r-j, r-j+1, r-j+2 (x) and at row r-j+1
//     (x-1, x+1), and level j-2 at row r-j+1 (x).
// Every tile column (x, all TL lanes) is owned by ONE thread for all levels, so the rows a
// column needs of its own x come from registers (three rows per level, rolled), and only
// the x-neighbours (row r-j+1 of level j-1, computed in the previous iteration) come from
// shared memory: each level 1..KS-1 writes its row into a 2-slot ring.  One CTA barrier
// per row; the TMA refills of the slots a row released are issued by one thread right
// after that barrier (the barrier is the "slot empty" signal, an mbarrier transaction
// count the "slot full" one).
//
// Threads: NI = TX*TL/2 interior threads own two interior columns each (they also store
// the outputs and accumulate the inner products); NH = (KS-1)*TL halo threads own one left
// and one right halo column each (a column at distance d outside the tile computes levels
// 1..KS-d).
//
// Reductions (doubling identities, north_star): level j contributes <a_{n+j-1}|a_{n+j-1}>
// (moment slot 2(n+j-1)) and <a_{n+j-1}|a_{n+j}> (slot 2(n+j-1)+1) over owned sites; the
// odd-N tail adds <a_{n+KS}|a_{n+KS}> (slot 2(n+KS)).  Per lane, fixed order.
#pragma once
#include "kpm_tma2.cuh"

namespace kpm {

struct TmaKGeom {
    int L0, L1;          // lattice extents
    int TX, TL, RG, G_L, PX;
    long long W;         // output rows = G_L * PX * L1
    int RP;
    double t, shift;
    const double2* phase;
    double* red;         // partial rows: slot k of this launch at red + k * slot_stride
    long long slot_stride;
    int rows_total;      // partial-sum rows per slot (>= gridDim.x; extra rows are zeroed)
    double2* outB;       // a_{n+KS-1}
    double2* outC;       // a_{n+KS}
};

constexpr int kSAK = 5;  // a_n ring (rows r, r+1 in use, three in flight)
constexpr int kSPK = 3;  // a_{n-1} ring

template <int KS, int TL, int TX>
struct SlotKLayout {
    static constexpr int SITE = TL * 16;
    __host__ __device__ static constexpr int round128(int b) { return (b + 127) / 128 * 128; }
    // a_n slot: sites [-KS, TX+KS), then eps~ in three 128-byte aligned pieces [KS][TX][KS]
    static constexpr int A_VEC = (TX + 2 * KS) * SITE;
    static constexpr int EPS_L = A_VEC;
    static constexpr int EPS_M = EPS_L + 128;
    static constexpr int EPS_R = EPS_M + round128(TX * 8);
    static constexpr int A_ON = EPS_R + 128;
    static constexpr int P_BYTES = round128((TX + 2 * (KS - 1)) * SITE);
    // ring of level j (1..KS-1): sites [-(KS-j), TX+KS-j), 2 slots
    __host__ __device__ static constexpr int lev_row(int j) { return round128((TX + 2 * (KS - j)) * SITE); }
    __host__ __device__ static constexpr int lev_off(int j) {  // offset of level j's ring from the first ring
        int o = 0;
        for (int i = 1; i < j; ++i) o += 2 * lev_row(i);
        return o;
    }
    static constexpr int LEV_BYTES = lev_off(KS);
};

template <int KS, int TL, int TX, int NPI>
struct StepKThreads {
    static_assert(NPI == 2, "two columns per thread (the halo threads own a left and a right column)");
    static constexpr int NI = TX * TL / NPI;
    static constexpr int NH = (KS - 1) * TL;
    static constexpr int NT = NI + NH;
};

template <int KS, int TL, int TX, int NPI>
__host__ __device__ inline size_t stepk_smem_bytes(bool onsite, int RP) {
    using SL = SlotKLayout<KS, TL, TX>;
    const size_t a = onsite ? SL::A_ON : SL::A_VEC;
    return (size_t)kSAK * a + (size_t)kSPK * SL::P_BYTES + (size_t)SL::LEV_BYTES + (2 * KS + 1) * (size_t)RP * 8 +
           (size_t)StepKThreads<KS, TL, TX, NPI>::NI * 16 + (kSAK + kSPK) * 8 + 64;
}

template <int KS, int TL, int TX, int NPI, bool ONSITE, bool PEIERLS>
__global__ void __launch_bounds__(StepKThreads<KS, TL, TX, NPI>::NT, 1)
    kpm_stepk_tma_kernel(const __grid_constant__ CUtensorMap mapA,    // a_n main box {2TL, TX, 1}
                         const __grid_constant__ CUtensorMap mapAH,   // a_n halo box {2TL, KS, 1}
                         const __grid_constant__ CUtensorMap mapP,    // a_{n-1} main box
                         const __grid_constant__ CUtensorMap mapPH,   // a_{n-1} halo box {2TL, KS-1, 1}
                         const __grid_constant__ CUtensorMap mapE,    // eps~ box {TX, 1}
                         const __grid_constant__ CUtensorMap mapEH,   // eps~ box {KS, 1}
                         const TmaKGeom g, const int tail) {
    using SL = SlotKLayout<KS, TL, TX>;
    using TH = StepKThreads<KS, TL, TX, NPI>;
    constexpr int NI = TH::NI;
    constexpr int SITE = SL::SITE;
    constexpr int KSTEP = NI / TL;  // interior columns per pass
    constexpr int NACC = 2 * KS + 1;
    constexpr int A_BYTES = ONSITE ? SL::A_ON : SL::A_VEC;
    static_assert(KS >= 2 && KS <= 4, "KS in 2..4");
    static_assert(NI % 32 == 0, "interior threads fill whole warps");
    static_assert(TX % KSTEP == 0, "interior columns must fill whole passes");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + kSAK * A_BYTES;
    unsigned char* ringL = ringP + kSPK * SL::P_BYTES;
    double* sacc = reinterpret_cast<double*>(ringL + SL::LEV_BYTES);  // [NACC][RP]
    double2* sred = reinterpret_cast<double2*>(sacc + NACC * g.RP);   // [NI]
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sred + NI);
    uint64_t* fullP = fullA + kSAK;

    const int t = threadIdx.x;
    const long long w_begin = g.W * blockIdx.x / gridDim.x;
    const long long w_end = g.W * (blockIdx.x + 1) / gridDim.x;

    // ---- in-band producer (thread PRODUCER: the first halo thread, whose column computes one level)
    constexpr int PRODUCER = NI;
    __shared__ LoadCursor cur_smem[2];
    __shared__ uint64_t pol_smem;
    LoadCursor& ca = cur_smem[0];
    LoadCursor& cp = cur_smem[1];
    auto issueA = [&](int slot) {  // next a_n row: rows m0-KS .. m1+KS-1 of each segment
        if (!ca.valid) return;
        const int row = (ca.m0 - KS + ca.q + 4 * g.L1) % g.L1;
        const int c0 = 2 * ca.lg * TL, x0 = ca.px * TX;
        const int xl = (x0 - KS + g.L0) % g.L0, xr = (x0 + TX) % g.L0;
        unsigned char* dst = ringA + slot * A_BYTES;
        mbar_expect_tx(fullA + slot, (TX + 2 * KS) * SITE + (ONSITE ? (TX + 2 * KS) * 8 : 0));
        tma_load(dst, &mapAH, fullA + slot, c0, xl, row);
        tma_load(dst + KS * SITE, &mapA, fullA + slot, c0, x0, row);
        tma_load(dst + (TX + KS) * SITE, &mapAH, fullA + slot, c0, xr, row);
        if (ONSITE) {
            tma_load_2d(dst + SL::EPS_L, &mapEH, fullA + slot, xl, row);
            tma_load_2d(dst + SL::EPS_M, &mapE, fullA + slot, x0, row);
            tma_load_2d(dst + SL::EPS_R, &mapEH, fullA + slot, xr, row);
        }
        ca.next(g, 2 * KS);
    };
    auto issueP = [&](int slot) {  // next a_{n-1} row: rows m0-KS+1 .. m1+KS-2
        if (!cp.valid) return;
        const int row = (cp.m0 - KS + 1 + cp.q + 4 * g.L1) % g.L1;
        const int c0 = 2 * cp.lg * TL, x0 = cp.px * TX;
        const int xl = (x0 - (KS - 1) + g.L0) % g.L0, xr = (x0 + TX) % g.L0;
        unsigned char* dst = ringP + slot * SL::P_BYTES;
        mbar_expect_tx(fullP + slot, (TX + 2 * (KS - 1)) * SITE);
        const uint64_t pol = pol_smem;
        tma_load_hint(dst, &mapPH, fullP + slot, c0, xl, row, pol);
        tma_load_hint(dst + (KS - 1) * SITE, &mapP, fullP + slot, c0, x0, row, pol);
        tma_load_hint(dst + (TX + KS - 1) * SITE, &mapPH, fullP + slot, c0, xr, row, pol);
        cp.next(g, 2 * KS - 2);
    };
    if (t == 0) {
        for (int i = 0; i < kSAK; ++i) mbar_init(fullA + i, 1);
        for (int i = 0; i < kSPK; ++i) mbar_init(fullP + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&mapA);
        prefetch_tmap(&mapAH);
        prefetch_tmap(&mapP);
        prefetch_tmap(&mapPH);
        if (ONSITE) {
            prefetch_tmap(&mapE);
            prefetch_tmap(&mapEH);
        }
        pol_smem = policy_evict_first();
        ca.init(g, w_begin, w_end, 2 * KS);
        cp.init(g, w_begin, w_end, 2 * KS - 2);
        for (int i = 0; i < kSAK; ++i) issueA(i);
        for (int i = 0; i < kSPK; ++i) issueP(i);
    }
    for (int i = t; i < NACC * g.RP; i += blockDim.x) sacc[i] = 0.0;
    __syncthreads();

    // ---- this thread's columns: interior threads own columns t/TL and t/TL + KSTEP; halo thread
    // hc owns the left column -(KS-1)+hc and the right column TX+hc, which compute levels
    // 1..top (top = KS - distance outside the tile).  All levels are evaluated every row
    // (straight-line code; the two columns are independent chains the scheduler interleaves);
    // results outside a column's range or before a level's first row are never stored.
    const bool interior = t < NI;
    const int l = (interior ? t : t - NI) % TL;
    const int lo = l * 16;
    int lxs[2], top[2];
    if (interior) {
        lxs[0] = t / TL;
        lxs[1] = t / TL + KSTEP;
        top[0] = top[1] = KS;
    } else {
        const int hc = (t - NI) / TL;
        lxs[0] = hc - (KS - 1);
        lxs[1] = TX + hc;
        top[0] = hc + 1;
        top[1] = KS - 1 - hc;
    }

    double2 acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = make_double2(0.0, 0.0);
    auto ld = [](const unsigned char* p) { return *reinterpret_cast<const double2*>(p); };
    auto flush = [&](int lgf) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) {
            if (interior) sred[t] = acc[k];
            __syncthreads();
            if (t < TL) {
                double2 s = make_double2(0.0, 0.0);
                for (int j = t; j < NI; j += TL) s = add2(s, sred[j]);
                const int v = lgf * TL + t;
                if (PEIERLS) {
                    sacc[k * g.RP + v] += s.x;
                } else {
                    sacc[k * g.RP + 2 * v] += s.x;
                    sacc[k * g.RP + 2 * v + 1] += s.y;
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < NACC; ++k) acc[k] = make_double2(0.0, 0.0);
    };
    // 2 H~ x - p from the 4 neighbours (y neighbours carry the Peierls phase) and the site value
    auto step_val = [&](double2 x, double2 xm, double2 xp, double2 ym, double2 yp, double e, double2 ph, double2 p) {
        double2 nb = add2(xm, xp);
        if (PEIERLS) nb = add2(nb, add2(cmulc(ph, yp), cmul(ph, ym)));
        else nb = add2(nb, add2(ym, yp));
        const double2 h = fma2(e, x, scale2(g.t, nb));
        return make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));
    };

    LoadCursor cs;
    cs.init(g, w_begin, w_end, 0);
    int ia = 0, ip = 0, cur_lg = -1;
    while (cs.valid) {
        const int lg = cs.lg, m0 = cs.m0, H = cs.H, x0 = cs.px * TX;
        if (cur_lg != -1 && lg != cur_lg) flush(cur_lg);
        cur_lg = lg;
        // per column: levels 0..KS-1 at three rows (m2 = two rows back, m1 = one row back,
        // c = this row), eps~ of the rows of levels 2..KS, Peierls phase, output pointer
        double2 vm2[2][KS], vm1[2][KS], vc[2][KS];
        double es[2][KS];
        double2 ph[2];
        long long ocol[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            ph[p] = PEIERLS ? __ldg(g.phase + (x0 + lxs[p] + g.L0) % g.L0) : make_double2(0.0, 0.0);
            ocol[p] = (long long)(x0 + lxs[p]) * g.RG + (long long)lg * TL + l;
        }
        const long long growstep = (long long)g.L0 * g.RG;
        const int ia_seg = ia;
        const int NQ = H + 2 * KS - 2;
        int s1 = (ia_seg + 1) % kSAK;  // slot of a_n row r
        int ps = ip % kSPK;
        for (int q = 0; q < NQ; ++q) {
            const int s2 = s1 + 1 == kSAK ? 0 : s1 + 1;  // a_n row r+1
            const int r = m0 - KS + 1 + q;                // level-1 row (unwrapped)
            if (q == 0) {
                mbar_wait(fullA + ia_seg % kSAK, (uint32_t)((ia_seg / kSAK) & 1));
                mbar_wait(fullA + s1, (uint32_t)(((ia_seg + 1) / kSAK) & 1));
                const unsigned char* A0 = ringA + (ia_seg % kSAK) * A_BYTES;
                const unsigned char* A1 = ringA + s1 * A_BYTES;
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    vm2[p][0] = ld(A0 + (lxs[p] + KS) * SITE + lo);
                    vm1[p][0] = ld(A1 + (lxs[p] + KS) * SITE + lo);
                }
            }
            mbar_wait(fullA + s2, (uint32_t)(((ia_seg + q + 2) / kSAK) & 1));
            mbar_wait(fullP + ps, (uint32_t)((ip / kSPK) & 1));
            const unsigned char* A1 = ringA + s1 * A_BYTES;  // a_n row r
            const unsigned char* A2 = ringA + s2 * A_BYTES;  // a_n row r+1
            const unsigned char* Pq = ringP + ps * SL::P_BYTES;
            const int wslot = q & 1, rslot = wslot ^ 1;
            double e1[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const int lx = lxs[p];
                vc[p][0] = ld(A2 + (lx + KS) * SITE + lo);
                e1[p] = g.shift;
                if (ONSITE)
                    e1[p] = *reinterpret_cast<const double*>(
                        A1 + (lx < 0 ? SL::EPS_L + (lx + KS) * 8 : (lx < TX ? SL::EPS_M + lx * 8 : SL::EPS_R + (lx - TX) * 8)));
            }
#pragma unroll
            for (int j = 1; j <= KS; ++j) {
                const int row = r - (j - 1);
                const bool owned = interior && row >= m0 && row < m0 + H;
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const int lx = lxs[p];
                    double2 xm, xp, minus;
                    if (j == 1) {
                        xm = ld(A1 + (lx + KS - 1) * SITE + lo);
                        xp = ld(A1 + (lx + KS + 1) * SITE + lo);
                        minus = ld(Pq + (lx + KS - 1) * SITE + lo);
                    } else {
                        const unsigned char* Lr = ringL + SL::lev_off(j - 1) + rslot * SL::lev_row(j - 1);
                        xm = ld(Lr + (lx + KS - j) * SITE + lo);
                        xp = ld(Lr + (lx + KS - j + 2) * SITE + lo);
                        minus = vm2[p][j >= 2 ? j - 2 : 0];
                    }
                    const double e = ONSITE ? (j == 1 ? e1[p] : es[p][j >= 2 ? j - 2 : 0]) : g.shift;
                    const double2 x = vm1[p][j - 1];
                    const double2 y = step_val(x, xm, xp, vm2[p][j - 1], vc[p][j - 1], e, ph[p], minus);
                    if (j < KS) {
                        if (j <= top[p]) {
                            unsigned char* Lw = ringL + SL::lev_off(j) + wslot * SL::lev_row(j);
                            *reinterpret_cast<double2*>(Lw + (lx + KS - j) * SITE + lo) = y;
                        }
                        vc[p][j] = y;
                    }
                    if (owned) {
                        if (j >= KS - 1) __stcs((j == KS ? g.outC : g.outB) + ocol[p] + row * growstep, y);
                        dot_acc<PEIERLS>(acc[2 * (j - 1)], x, x);
                        dot_acc<PEIERLS>(acc[2 * (j - 1) + 1], x, y);
                        if (j == KS && tail) dot_acc<PEIERLS>(acc[2 * KS], y, y);
                    }
                }
            }
            // roll one row down
#pragma unroll
            for (int p = 0; p < 2; ++p) {
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    vm2[p][j] = vm1[p][j];
                    vm1[p][j] = vc[p][j];
                }
                if (ONSITE) {
#pragma unroll
                    for (int j = KS - 1; j > 0; --j) es[p][j] = es[p][j - 1];
                    es[p][0] = e1[p];
                }
            }
            __syncthreads();  // row done: a_n row r (and at q == 0 row r-1) and a_{n-1} row r are free
            if (t == PRODUCER) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (q == 0) issueA(ia_seg % kSAK);
                issueA(s1);
                issueP(ps);
            }
            ++ip;
            s1 = s2;
            ps = ps + 1 == kSPK ? 0 : ps + 1;
        }
        if (t == PRODUCER) issueA(s1);  // the segment's last a_n row
        ia = ia_seg + H + 2 * KS;
        cs.seg(g, 0);
    }
    if (cur_lg != -1) flush(cur_lg);
    __syncthreads();
    for (int k = 0; k < NACC; ++k) {
        if (k == 2 * KS && !tail) continue;
        double* rowk = g.red + (size_t)k * g.slot_stride;
        for (int v = t; v < g.RP; v += blockDim.x) rowk[(size_t)blockIdx.x * g.RP + v] = sacc[k * g.RP + v];
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int v = t; v < g.RP; v += blockDim.x) rowk[(size_t)rr * g.RP + v] = 0.0;
    }
}

}  // namespace kpm
