// kpm_tmak.cuh -- KS recursion steps per HBM pass (deep temporal blocking), 2D lattices.
//
// One launch advances the recursion (Eq 18) by KS steps,
//     a_{n+j} = 2 H~ a_{n+j-1} - a_{n+j-2},   j = 1 .. KS,
// reading a_n and a_{n-1} from HBM once and writing only a_{n+KS-1} and a_{n+KS}:
// 4 D R s bytes per KS steps (kpm_tma2.cuh is the KS = 2 case).
// The intermediate blocks a_{n+1} .. a_{n+KS-2} never leave the SM.
//
// Geometry.  A CTA marches a pencil of TX sites x TL lanes over y (rows).  "Level" j is
// the block a_{n+j}: level 0 = a_n and level -1 = a_{n-1} arrive by TMA, levels 1..KS are
// computed, each on the tile widened by KS - j halo sites per side (halo sites are
// recomputed, not exchanged).  In iteration q a new a_n row enters and level j computes
// the row two rows behind the newest row of level j-1:
//     level j at row y needs level j-1 at rows y-1, y, y+1 (own x), at row y (x-1, x+1),
//     and level j-2 at row y (own x)
// -- all produced in EARLIER iterations, so the KS levels of an iteration are independent
// (KS x 2 columns of instruction-level parallelism per thread; a one-row lag would chain
// them).  Every tile column (x, TL lanes) is owned by one thread for all levels: the rows
// of its own x come from registers (rolled), the x-neighbours and the level j-2 term come
// from per-level shared-memory row rings.  One CTA barrier per iteration; right after it
// one thread refills the released TMA slots (the barrier is the "slot empty" signal, an
// mbarrier transaction count the "slot full" one).
//
// Threads: NI = TX*TL/2 interior threads own two interior columns each (they also store the
// outputs and accumulate the inner products); NH = (KS-1)*TL halo threads own one left and
// one right halo column (a column at distance d outside the tile computes levels 1..KS-d).
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

constexpr int kSAK = 5;  // a_n ring: rows of loads q-2, q-1, q in use, two in flight
constexpr int kSPK = 3;  // a_{n-1} ring

template <int KS, int TL, int TX, bool ONSITE>
struct SlotKLayout {
    static constexpr int SITE = TL * 16;
    __host__ __device__ static constexpr int round128(int b) { return (b + 127) / 128 * 128; }
    // a_n slot: sites [-KS, TX+KS), then eps~ in three 128-byte aligned pieces [KSE][TX][KSE]
    // (KSE = KS rounded up to even: a TMA box row must be a multiple of 16 bytes)
    static constexpr int KSE = (KS + 1) / 2 * 2;
    static constexpr int A_VEC = (TX + 2 * KS) * SITE;
    static constexpr int EPS_L = A_VEC;
    static constexpr int EPS_M = EPS_L + 128;
    static constexpr int EPS_R = EPS_M + round128(TX * 8);
    static constexpr int A_BYTES = ONSITE ? EPS_R + 128 : A_VEC;
    static constexpr int P_BYTES = round128((TX + 2 * (KS - 1)) * SITE);
    // level j (1..KS-1) ring: sites [-(KS-j), TX+KS-j) (+ their eps~), lev_slots(j) rows
    __host__ __device__ static constexpr int lev_sites(int j) { return TX + 2 * (KS - j); }
    __host__ __device__ static constexpr int lev_eps(int j) { return lev_sites(j) * SITE; }
    __host__ __device__ static constexpr int lev_row(int j) {
        return round128(lev_sites(j) * SITE + (ONSITE ? lev_sites(j) * 8 : 0));
    }
    // read back 2 iterations later (x-neighbours of level j+1) and 4 later (level j+2's term)
    __host__ __device__ static constexpr int lev_slots(int j) { return j <= KS - 2 ? 5 : 3; }
    __host__ __device__ static constexpr int lev_off(int j) {
        int o = 0;
        for (int i = 1; i < j; ++i) o += lev_slots(i) * lev_row(i);
        return o;
    }
    static constexpr int LEV_BYTES = lev_off(KS);
};

template <int KS, int TL, int TX>
struct StepKThreads {
    static constexpr int NI = TX * TL / 2;
    static constexpr int NH = (KS - 1) * TL;
    static constexpr int NT = NI + NH;
};

template <int KS, int TL, int TX, bool ONSITE>
__host__ __device__ inline size_t stepk_smem_bytes(int RP) {
    using SL = SlotKLayout<KS, TL, TX, ONSITE>;
    return (size_t)kSAK * SL::A_BYTES + (size_t)kSPK * SL::P_BYTES + (size_t)SL::LEV_BYTES +
           (2 * KS + 1) * (size_t)RP * 8 + (size_t)StepKThreads<KS, TL, TX>::NI * 16 + (kSAK + kSPK) * 8 + 64;
}

template <int KS, int TL, int TX, bool ONSITE, bool PEIERLS>
__global__ void __launch_bounds__(StepKThreads<KS, TL, TX>::NT, 1)
    kpm_stepk_tma_kernel(const __grid_constant__ CUtensorMap mapA,    // a_n main box {2TL, TX, 1}
                         const __grid_constant__ CUtensorMap mapAH,   // a_n halo box {2TL, KS, 1}
                         const __grid_constant__ CUtensorMap mapP,    // a_{n-1} main box
                         const __grid_constant__ CUtensorMap mapPH,   // a_{n-1} halo box {2TL, KS-1, 1}
                         const __grid_constant__ CUtensorMap mapE,    // eps~ box {TX, 1}
                         const __grid_constant__ CUtensorMap mapEH,   // eps~ box {KSE, 1}
                         const TmaKGeom g, const int tail) {
    using SL = SlotKLayout<KS, TL, TX, ONSITE>;
    using TH = StepKThreads<KS, TL, TX>;
    constexpr int NI = TH::NI;
    constexpr int SITE = SL::SITE;
    constexpr int KSTEP = NI / TL;  // = TX / 2: the second column of an interior thread
    constexpr int NACC = 2 * KS + 1;
    constexpr int A_BYTES = SL::A_BYTES;
    static_assert(KS >= 2 && KS <= 4, "KS in 2..4");
    static_assert(NI % 32 == 0, "interior threads fill whole warps");
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

    // ---- in-band producer (thread PRODUCER: the first halo thread)
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
        mbar_expect_tx(fullA + slot, (TX + 2 * KS) * SITE + (ONSITE ? (TX + 2 * SL::KSE) * 8 : 0));
        tma_load(dst, &mapAH, fullA + slot, c0, xl, row);
        tma_load(dst + KS * SITE, &mapA, fullA + slot, c0, x0, row);
        tma_load(dst + (TX + KS) * SITE, &mapAH, fullA + slot, c0, xr, row);
        if (ONSITE) {
            tma_load_2d(dst + SL::EPS_L, &mapEH, fullA + slot, (x0 - SL::KSE + g.L0) % g.L0, row);
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

    // ---- this thread's columns: interior threads own columns t/TL and t/TL + TX/2; halo
    // thread hc owns the left column -(KS-1)+hc and the right column TX+hc, which compute
    // levels 1..top (top = KS - distance outside the tile).  All levels are evaluated in
    // every iteration (straight-line code); a level's values before its first row, after its
    // last row or outside its column range are never stored nor read back.
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
    // Shared-memory addressing: 32-bit offsets from smem.  Per column one invariant offset
    // colA (site lx of an a_n slot); level j-1's row is shifted by j-1 sites, the a_{n-1} row
    // by one.  Slot bases are uniform per iteration and advanced incrementally.
    auto ld = [&](uint32_t off) { return *reinterpret_cast<const double2*>(smem + off); };
    auto ldd = [&](uint32_t off) { return *reinterpret_cast<const double*>(smem + off); };
    const uint32_t offA = 0, offP = kSAK * A_BYTES, offL = offP + kSPK * SL::P_BYTES;
    uint32_t colA[2], colE[2], epsA[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int lx = lxs[p];
        colA[p] = (uint32_t)((lx + KS) * SITE + lo);
        colE[p] = (uint32_t)((lx + KS) * 8);
        epsA[p] = (uint32_t)(lx < 0 ? SL::EPS_L + (lx + SL::KSE) * 8 : (lx < TX ? SL::EPS_M + lx * 8 : SL::EPS_R + (lx - TX) * 8));
    }
    // ring slot of level j for iteration q - back (back = 0, 2, 4), from the counters q mod 5, q mod 3
    auto lev_base = [&](int j, int c5, int c3, int back) -> uint32_t {
        const int S = SL::lev_slots(j);
        int sl;
        if (S == 5) sl = back == 0 ? c5 : (back == 2 ? (c5 >= 2 ? c5 - 2 : c5 + 3) : (c5 >= 4 ? c5 - 4 : c5 + 1));
        else sl = back == 0 ? c3 : (back == 2 ? (c3 >= 2 ? c3 - 2 : c3 + 1) : (c3 >= 1 ? c3 - 1 : c3 + 2));
        return offL + (uint32_t)SL::lev_off(j) + (uint32_t)sl * (uint32_t)SL::lev_row(j);
    };

    LoadCursor cs;
    cs.init(g, w_begin, w_end, 0);
    int ia = 0, ip = 0, cur_lg = -1;
    while (cs.valid) {
        const int lg = cs.lg, m0 = cs.m0, H = cs.H, x0 = cs.px * TX;
        if (cur_lg != -1 && lg != cur_lg) flush(cur_lg);
        cur_lg = lg;
        // Registers per column: a_n at the last four rows (a0[0] = newest), levels 1..KS-1 at
        // their last three rows (v[j][0] = newest); Peierls phase; output offset.
        double2 a0[2][4], v[2][KS][3];
        double2 ph[2];
        long long ocol[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            ph[p] = PEIERLS ? __ldg(g.phase + (x0 + lxs[p] + g.L0) % g.L0) : make_double2(0.0, 0.0);
            ocol[p] = (long long)(x0 + lxs[p]) * g.RG + (long long)lg * TL + l;
        }
        const long long growstep = (long long)g.L0 * g.RG;
        const int ia_seg = ia;
        const int NA = H + 2 * KS;  // a_n rows of the segment (loads 0 .. NA-1)
        const int NQ = H + 3 * KS;  // iterations
        const int yb = m0 - KS - 1; // level j computes row yb + q - 2j + 1 in iteration q
        int sN = ia_seg % kSAK;                 // slot of a_n load q
        int sX = (ia_seg + kSAK - 2) % kSAK;    // slot of a_n load q-2
        int c5 = 0, c3 = 0;                     // q mod 5, q mod 3
        for (int q = 0; q < NQ; ++q) {
            const bool newA = q < NA;             // a_n load q enters
            const bool useP = q >= 3 && q <= NA;  // level 1 consumes a_{n-1} load q-3
            const int sP = ip % kSPK;
            if (newA) mbar_wait(fullA + sN, (uint32_t)(((ia_seg + q) / kSAK) & 1));
            if (useP) mbar_wait(fullP + sP, (uint32_t)((ip / kSPK) & 1));
            const uint32_t An = offA + (uint32_t)sN * A_BYTES;   // newest a_n row
            const uint32_t Ax = offA + (uint32_t)sX * A_BYTES;   // a_n at level 1's row
            const uint32_t Pq = offP + (uint32_t)sP * SL::P_BYTES;
            double2 anew[2], y[2][KS + 1];
            double e1[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                anew[p] = ld(An + colA[p]);
                e1[p] = ONSITE ? ldd(Ax + epsA[p]) : g.shift;
            }
#pragma unroll
            for (int j = 1; j <= KS; ++j) {
                const int row = yb + q - 2 * j + 1;
                const bool owned = interior && row >= m0 && row < m0 + H;
                const long long rowoff = (long long)row * growstep;
                const uint32_t Lx = j >= 2 ? lev_base(j - 1, c5, c3, 2) : 0u;  // level j-1 at this row
                const uint32_t Lm = j >= 3 ? lev_base(j - 2, c5, c3, 4) : 0u;  // level j-2 at this row
                const uint32_t Lw = j < KS ? lev_base(j, c5, c3, 0) : 0u;      // level j, written now
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    double2 xm, xp, x, ym, yp, minus;
                    double e;
                    if (j == 1) {
                        const uint32_t c = Ax + colA[p];
                        xm = ld(c - SITE);
                        xp = ld(c + SITE);
                        ym = a0[p][2];
                        x = a0[p][1];
                        yp = a0[p][0];
                        minus = ld(Pq + colA[p] - SITE);
                        e = e1[p];
                    } else {
                        const uint32_t c = Lx + colA[p] - (j - 1) * SITE;  // site lx of level j-1's row
                        xm = ld(c - SITE);
                        xp = ld(c + SITE);
                        ym = v[p][j - 1][2];
                        x = v[p][j - 1][1];
                        yp = v[p][j - 1][0];
                        minus = j == 2 ? a0[p][3] : ld(Lm + colA[p] - (j - 2) * SITE);
                        e = ONSITE ? ldd(Lx + SL::lev_eps(j - 1) + colE[p] - (j - 1) * 8) : g.shift;
                    }
                    y[p][j] = step_val(x, xm, xp, ym, yp, e, ph[p], minus);
                    if (j < KS && j <= top[p]) {
                        *reinterpret_cast<double2*>(smem + Lw + colA[p] - j * SITE) = y[p][j];
                        if (ONSITE && l == 0) *reinterpret_cast<double*>(smem + Lw + SL::lev_eps(j) + colE[p] - j * 8) = e;
                    }
                    if (owned) {
                        if (j >= KS - 1) __stcs((j == KS ? g.outC : g.outB) + (rowoff + ocol[p]), y[p][j]);
                        dot_acc<PEIERLS>(acc[2 * (j - 1)], x, x);
                        dot_acc<PEIERLS>(acc[2 * (j - 1) + 1], x, y[p][j]);
                        if (j == KS && tail) dot_acc<PEIERLS>(acc[2 * KS], y[p][j], y[p][j]);
                    }
                }
            }
            // roll: this iteration's values become the newest rows
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                a0[p][3] = a0[p][2];
                a0[p][2] = a0[p][1];
                a0[p][1] = a0[p][0];
                a0[p][0] = anew[p];
#pragma unroll
                for (int j = 1; j < KS; ++j) {
                    v[p][j][2] = v[p][j][1];
                    v[p][j][1] = v[p][j][0];
                    v[p][j][0] = y[p][j];
                }
            }
            __syncthreads();  // iteration done: a_n load q-2 and a_{n-1} load q-3 are free
            if (t == PRODUCER) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (q >= 2 && q - 2 < NA) issueA(sX);
                if (useP) issueP(sP);
            }
            if (useP) ++ip;
            sN = sN + 1 == kSAK ? 0 : sN + 1;
            sX = sX + 1 == kSAK ? 0 : sX + 1;
            c5 = c5 + 1 == 5 ? 0 : c5 + 1;
            c3 = c3 + 1 == 3 ? 0 : c3 + 1;
        }
        ia = ia_seg + NA;
        cs.seg(g, 0);
    }
    if (cur_lg != -1) flush(cur_lg);
    __syncthreads();
    for (int k = 0; k < NACC; ++k) {
        if (k == 2 * KS && !tail) continue;
        double* rowk = g.red + (size_t)k * g.slot_stride;
        for (int vv = t; vv < g.RP; vv += blockDim.x) rowk[(size_t)blockIdx.x * g.RP + vv] = sacc[k * g.RP + vv];
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int vv = t; vv < g.RP; vv += blockDim.x) rowk[(size_t)rr * g.RP + vv] = 0.0;
    }
}

}  // namespace kpm
