// kpm_tma2.cuh -- two recursion steps per HBM pass (temporal blocking), 2D lattices.
//
// One launch advances the recursion by two steps (Eq 18 twice):
//     a_{n+1} = 2 H~ a_n - a_{n-1},     a_{n+2} = 2 H~ a_{n+1} - a_n,
// reading a_n and a_{n-1} from HBM once and writing a_{n+1} and a_{n+2} once:
// 4 D R s bytes per two steps instead of 6 D R s.  The
// intermediate a_{n+1} lives only in a 3-row shared-memory ring.
//
// Tiling is kpm_tma.cuh's march (pencil of TX sites x TL lanes, marching over y),
// with wider halos because the second step needs a_{n+1} one site beyond the tile:
//   a_n     rows m0-2 .. m1+1, sites x0-2 .. x0+TX+1   (TMA: main box + two 2-site boxes)
//   a_{n-1} rows m0-1 .. m1,   sites x0-1 .. x0+TX     (TMA: main box + two 1-site boxes)
//   a_{n+1} rows m0-1 .. m1,   sites x0-1 .. x0+TX     (computed; halo sites/rows are
//                                                       recomputed, not stored)
//   a_{n+2} rows m0 .. m1-1,   sites x0 .. x0+TX-1     (stored)
// Outputs go to two other buffers (out of place): an in-place write could overwrite
// halo values a neighbouring CTA still has to read.
//
// Execution: 8 warps, all computing (2 warps per SM sub-partition leave 255 registers
// per thread; each thread owns 4 interior sites of a row and keeps its own a_n rows
// r-1..r+1, a_{n+1} rows r-2..r-1 and eps~ values rolling in registers, so a site costs
// 7 shared-memory loads).  Row q of a segment: every thread computes a_{n+1}(row r) at
// its sites and, at the same site one row lower, a_{n+2}(row r-1), whose a_{n+1}(row r)
// neighbour is the value it just computed -- so one CTA barrier per row suffices.  The
// two halo sites of a_{n+1} are recomputed by the last two site groups.  After the
// barrier one thread refills the two ring slots the row released with the next TMA
// loads of the CTA's load sequence (the barrier is the "slot empty" signal; "slot full"
// is an mbarrier transaction count).
//
// Reductions: <a_n|a_n>, <a_n|a_{n+1}>, <a_{n+1}|a_{n+1}>, <a_{n+1}|a_{n+2}> (and the
// odd-N tail <a_{n+2}|a_{n+2}>) over owned sites, per lane, fixed order.
#pragma once
#include "kpm_tma.cuh"

namespace kpm {

struct Tma2Geom {
    int L0, L1;          // lattice extents
    int TX, TL, RG, G_L, PX;
    long long W;         // output rows = G_L * PX * L1
    int RP;
    int rows_total;      // partial-sum rows per slot (>= gridDim.x; extra rows are zeroed)
    double t, shift;
    const double2* phase;
    double* red[5];      // slots 2n, 2n+1, 2n+2, 2n+3, (tail) 2n+4; red[4] nullable
    double2* outB;       // a_{n+1}
    double2* outC;       // a_{n+2}
};

constexpr int kThreads2 = 256;  // 8 warps
constexpr int kSB2 = 3;         // a_{n+1} ring (computed)
// a_n / a_{n-1} ring depths: 5 / 3 slots for the 1024-lane row tiles (one CTA per SM, ~190 KB);
// 12 / 8 for the small 4-lane x 64-site tile (two CTAs per SM, L2-resident blocks): rows are only
// 4 KB there, and the deeper rings keep more TMA loads in flight per CTA.
__host__ __device__ constexpr int ring2_a(int TL, int TX) { return TL * TX <= 256 ? 12 : 5; }
__host__ __device__ constexpr int ring2_p(int TL, int TX) { return TL * TX <= 256 ? 8 : 3; }

// a_n slot: [2 halo sites][TX sites][2 halo sites] then eps~ as three 128-byte aligned
// pieces (TMA destinations must be 128-byte aligned): [2 left][TX main][2 right].
// a_{n-1} slot: [PH halo sites][TX sites][PH halo sites], PH = 1 when a site is >= 128 bytes
// (TL >= 8 lanes), else 2 (TL = 4: the halo box is two sites wide so that the main box lands on
// a 128-byte boundary; the outer halo site is loaded but not used).
__host__ __device__ constexpr int p_halo(int TL) { return TL * 16 >= 128 ? 1 : 2; }
struct Slot2Layout {
    int site, a_bytes, eps_l, eps_m, eps_r, p_bytes, b_bytes;
    __host__ __device__ constexpr Slot2Layout(int TX, int TL, bool onsite)
        : site(TL * 16),
          a_bytes(onsite ? (TX + 4) * TL * 16 + 128 + (TX * 8 + 127) / 128 * 128 + 128 : (TX + 4) * TL * 16),
          eps_l((TX + 4) * TL * 16),
          eps_m((TX + 4) * TL * 16 + 128),
          eps_r((TX + 4) * TL * 16 + 128 + (TX * 8 + 127) / 128 * 128),
          p_bytes(((TX + 2 * p_halo(TL)) * TL * 16 + 127) / 128 * 128),
          b_bytes(((TX + 2) * TL * 16 + 127) / 128 * 128) {}
    // eps~ at tile x index lx in [-2, TX+1]
    __device__ __forceinline__ double eps(const unsigned char* slot, int lx, int TX) const {
        const double* e = reinterpret_cast<const double*>(
            slot + (lx < 0 ? eps_l + (lx + 2) * 8 : (lx < TX ? eps_m + lx * 8 : eps_r + (lx - TX) * 8)));
        return *e;
    }
};

__host__ __device__ inline size_t step2_smem_bytes(int TX, int TL, bool onsite, int RP) {
    const Slot2Layout S(TX, TL, onsite);
    const int SA = ring2_a(TL, TX), SP = ring2_p(TL, TX);
    return (size_t)SA * S.a_bytes + (size_t)SP * S.p_bytes + (size_t)kSB2 * S.b_bytes + 5 * (size_t)RP * 8 +
           (size_t)kThreads2 * 16 + (size_t)(TX + 2) * 16 + (SA + SP) * 8;
}

// Walks one CTA's segments (lane group, pencil, rows [m0, m0+H)) and, within a segment,
// its loads q = 0 .. H+extra-1: a_n rows m0-2+q (extra 4) or a_{n-1} rows m0-1+q (extra 2).
// Per segment it also precomputes what every load of the segment needs -- the wrapped row of
// load q (advanced with one compare per load), the tile's x0, its periodic halo columns x0-hw
// and x0+TX (hw = extra/2 sites) and the lane coordinate c0 -- so that a refill costs no integer
// division (ncu: the producer's divisions and modulos kept its warp ~250 instructions per row
// behind the others, and every warp waited for it at the next row barrier).
struct LoadCursor {
    long long w, w_end;
    int lg, px, m0, H, q, nq;
    int row, x0, xl, xr, c0;
    bool valid;
    template <class G>
    __device__ void seg(const G& g, int extra, int xh = -1) {
        valid = w < w_end;
        if (!valid) return;
        const long long col = w / g.L1;
        m0 = (int)(w - col * g.L1);
        const long long e = min(w_end, (col + 1) * (long long)g.L1);
        H = (int)(e - w);
        px = (int)(col % g.PX);
        lg = (int)(col / g.PX);
        w = e;
        q = 0;
        nq = H + extra;
        const int hw = extra / 2;  // halo rows per side
        row = m0 - hw;
        while (row < 0) row += g.L1;
        x0 = px * g.TX;
        xl = x0 - (xh < 0 ? hw : xh);  // halo sites per side along x
        while (xl < 0) xl += g.L0;
        xr = x0 + g.TX;
        while (xr >= g.L0) xr -= g.L0;
        c0 = 2 * lg * g.TL;
    }
    template <class G>
    __device__ void init(const G& g, long long b, long long e, int extra, int xh = -1) {
        w = b;
        w_end = e;
        seg(g, extra, xh);
    }
    template <class G>
    __device__ void next(const G& g, int extra, int xh = -1) {
        if (++row == g.L1) row = 0;
        if (++q >= nq) seg(g, extra, xh);
    }
};

// XW = 1: a ninth warp computes the two halo sites of a_{n+1} (and issues the TMA refills), so
// the eight interior warps carry equal work per row (with XW = 0 the two warps holding the halo
// sites ran 5 site passes per row against 4, and ncu showed 25% of warp time stalled on the
// per-row barrier).
template <int XW>
struct Threads2 {
    static constexpr int N = kThreads2 + 32 * XW;
};

template <int TL, int TX, bool ONSITE, bool PEIERLS, int MINB, int XW = 0>
__global__ void __launch_bounds__(Threads2<XW>::N, MINB)
    kpm_step2_tma_kernel(const __grid_constant__ CUtensorMap mapA,    // a_n main box {2TL, TX, 1}
                         const __grid_constant__ CUtensorMap mapA2,   // a_n 2-site box {2TL, 2, 1}
                         const __grid_constant__ CUtensorMap mapP,    // a_{n-1} main box
                         const __grid_constant__ CUtensorMap mapP1,   // a_{n-1} PH-site box {2TL, PH, 1}
                         const __grid_constant__ CUtensorMap mapE,    // eps~ box {TX, 1}
                         const __grid_constant__ CUtensorMap mapE2,   // eps~ box {2, 1}
                         const Tma2Geom g, const int tail) {
    pdl_entry();
    constexpr int CONS = kThreads2;
    constexpr int KSTEP = CONS / TL;              // tile sites per pass
    constexpr int NB = TX + 2;                    // a_{n+1} sites per row (with halo)
    constexpr int SITE = TL * 16;
    constexpr int PH = p_halo(TL);                // a_{n-1} halo sites per side in the slot
    constexpr Slot2Layout SL(TX, TL, ONSITE);
    constexpr int kSA2 = ring2_a(TL, TX), kSP2 = ring2_p(TL, TX);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + kSA2 * SL.a_bytes;
    unsigned char* ringB = ringP + kSP2 * SL.p_bytes;
    double* sacc = reinterpret_cast<double*>(ringB + kSB2 * SL.b_bytes);  // [5][RP]
    double2* sred = reinterpret_cast<double2*>(sacc + 5 * g.RP);           // [CONS]
    double2* sphase = sred + CONS;                                         // [TX + 2]
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sphase + TX + 2);
    uint64_t* fullP = fullA + kSA2;

    const int t = threadIdx.x;
    const long long w_begin = g.W * blockIdx.x / gridDim.x;
    const long long w_end = g.W * (blockIdx.x + 1) / gridDim.x;

    // ---- in-band producer state (thread 0 only; kept in shared memory, not registers)
    __shared__ LoadCursor cur_smem[2];
    __shared__ uint64_t pol_smem;
    LoadCursor& ca = cur_smem[0];
    LoadCursor& cp = cur_smem[1];
    auto issueA = [&](int slot) {  // next a_n row of the sequence into `slot`
        if (!ca.valid) return;
        const int row = ca.row, c0 = ca.c0, x0 = ca.x0, xl2 = ca.xl, xr2 = ca.xr;
        unsigned char* dst = ringA + slot * SL.a_bytes;
        mbar_expect_tx(fullA + slot, (TX + 4) * SITE + (ONSITE ? (TX + 4) * 8 : 0));
        tma_load(dst, &mapA2, fullA + slot, c0, xl2, row);
        tma_load(dst + 2 * SITE, &mapA, fullA + slot, c0, x0, row);
        tma_load(dst + (TX + 2) * SITE, &mapA2, fullA + slot, c0, xr2, row);
        if (ONSITE) {
            tma_load_2d(dst + SL.eps_l, &mapE2, fullA + slot, xl2, row);
            tma_load_2d(dst + SL.eps_m, &mapE, fullA + slot, x0, row);
            tma_load_2d(dst + SL.eps_r, &mapE2, fullA + slot, xr2, row);
        }
        ca.next(g, 4);
    };
    auto issueP = [&](int slot) {  // next a_{n-1} row of the sequence into `slot`
        if (!cp.valid) return;
        const int row = cp.row, c0 = cp.c0, x0 = cp.x0, xl1 = cp.xl, xr1 = cp.xr;
        unsigned char* dst = ringP + slot * SL.p_bytes;
        mbar_expect_tx(fullP + slot, (TX + 2 * PH) * SITE);
        const uint64_t pol = pol_smem;
        tma_load_hint(dst, &mapP1, fullP + slot, c0, xl1, row, pol);
        tma_load_hint(dst + PH * SITE, &mapP, fullP + slot, c0, x0, row, pol);
        tma_load_hint(dst + (TX + PH) * SITE, &mapP1, fullP + slot, c0, xr1, row, pol);
        cp.next(g, 2, PH);
    };
    if (t == 0) {
        for (int i = 0; i < kSA2; ++i) mbar_init(fullA + i, 1);
        for (int i = 0; i < kSP2; ++i) mbar_init(fullP + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&mapA);
        prefetch_tmap(&mapA2);
        prefetch_tmap(&mapP);
        prefetch_tmap(&mapP1);
        if (ONSITE) {
            prefetch_tmap(&mapE);
            prefetch_tmap(&mapE2);
        }
        pol_smem = policy_evict_first();
        ca.init(g, w_begin, w_end, 4);
        cp.init(g, w_begin, w_end, 2, PH);
        for (int i = 0; i < kSA2; ++i) issueA(i);
        for (int i = 0; i < kSP2; ++i) issueP(i);
    }
    for (int i = t; i < 5 * g.RP; i += blockDim.x) sacc[i] = 0.0;
    __syncthreads();

    const int l = t % TL;
    const int k0 = t / TL;
    const int lo = l * 16;
    double2 acc[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) acc[k] = make_double2(0.0, 0.0);
    auto ld = [](const unsigned char* p) { return *reinterpret_cast<const double2*>(p); };
    auto flush = [&](int lgf) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            double2 s = make_double2(0.0, 0.0);
            if (TL <= 4) {  // few lanes: 64+ values per lane -- shuffle tree (cta_lane_sum)
                s = cta_lane_sum<TL, CONS>(acc[k], t, sred);
            } else {
                if (t < CONS) sred[t] = acc[k];
                __syncthreads();
                if (t < TL)
                    for (int j = t; j < CONS; j += TL) s = add2(s, sred[j]);
                __syncthreads();
            }
            if (t < TL) {
                const int v = lgf * TL + t;
                if (PEIERLS) {
                    sacc[k * g.RP + v] += s.x;
                } else {
                    sacc[k * g.RP + 2 * v] += s.x;
                    sacc[k * g.RP + 2 * v + 1] += s.y;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[k] = make_double2(0.0, 0.0);
    };
    // 2 H~ x - p from the 4 neighbours (y neighbours carry the Peierls phase) and the site value
    auto step_val = [&](double2 x, double2 xm, double2 xp, double2 ym, double2 yp, double e, double2 ph, double2 p) {
        double2 nb = add2(xm, xp);
        if (PEIERLS) nb = add2(nb, add2(cmulc(ph, yp), cmul(ph, ym)));
        else nb = add2(nb, add2(ym, yp));
        const double2 h = fma2(e, x, scale2(g.t, nb));
        return make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));
    };

    // Work split per row: interior sites lx = k0 + p*KSTEP (p < NPI) -> a_{n+1} and a_{n+2};
    // the two halo sites of a_{n+1} (lx = -1, TX) -> the last two site groups; the TMA
    // refills -> thread PRODUCER (a warp without halo work).
    constexpr int NPI = TX / KSTEP;
    static_assert(TX % KSTEP == 0 && KSTEP >= 4, "interior sites must fill whole passes");
    // refills: one thread issues both (measured: splitting a_n / a_{n-1} refills over two warps
    // made c2 2% slower in sustained runs, 26.39 vs 25.85 ms, though one ncu launch was faster)
    constexpr int PRODUCER = XW ? CONS : 32;  // the halo warp's first thread, else thread 0 of warp 1
    constexpr int PRODUCER_P = PRODUCER;
    const bool halo_warp = XW && t >= CONS;
    const int hs = XW ? -1 : k0 - (KSTEP - 2);   // 0, 1: halo site of this thread, else < 0
    const int hlx = hs == 0 ? -1 : TX;           // its tile x index
    LoadCursor cs;  // segment iterator of the consumers (same sequence)
    cs.init(g, w_begin, w_end, 0);
    int ia = 0, ip = 0, cur_lg = -1;
    while (cs.valid) {
        const int lg = cs.lg, m0 = cs.m0, H = cs.H, x0 = cs.px * TX;
        if (cur_lg != -1 && lg != cur_lg) flush(cur_lg);
        cur_lg = lg;
        // global offset of (row 0, site x0 + k0, this lane); uniform per-pass step
        const long long g0 = (long long)(x0 + k0) * g.RG + (long long)lg * TL + l;
        const long long gstep = (long long)KSTEP * g.RG;
        const long long growstep = (long long)g.L0 * g.RG;
        if (PEIERLS) {
            if (t < NB) sphase[t] = __ldg(g.phase + (x0 + t - 1 + g.L0) % g.L0);
            __syncthreads();
        }
        const int ia_seg = ia;
        int sB = 0;                                   // ring slot of a_{n+1} row q
        int s0 = ia_seg % kSA2;                       // ring slot of a_n row r-1
        int ps = ip % kSP2;
        int rB = (m0 - 1 + g.L1) % g.L1;              // a_{n+1} row r
        int rC = (m0 - 2 + g.L1) % g.L1;              // a_{n+2} row r-1
        // values this thread needs again in later rows, kept in registers (per pass p):
        // a_n at rows r-1, r, r+1; a_{n+1} at rows r-2, r-1; eps~ at row r-1
        double2 am[NPI], ac[NPI], ap[NPI], bm[NPI], bc[NPI];
        double em[NPI];
        for (int q = 0; q < H + 2; ++q) {
            const int i0 = ia_seg + q;
            const int s1 = s0 + 1 == kSA2 ? 0 : s0 + 1;
            const int s2 = s1 + 1 == kSA2 ? 0 : s1 + 1;
            if (q == 0) {
                mbar_wait(fullA + s0, (uint32_t)((i0 / kSA2) & 1));
                mbar_wait(fullA + s1, (uint32_t)(((i0 + 1) / kSA2) & 1));
            }
            mbar_wait(fullA + s2, (uint32_t)(((i0 + 2) / kSA2) & 1));
            mbar_wait(fullP + ps, (uint32_t)((ip / kSP2) & 1));
            const unsigned char* A0 = ringA + s0 * SL.a_bytes;   // a_n row r-1
            const unsigned char* A1 = ringA + s1 * SL.a_bytes;   // a_n row r
            const unsigned char* A2 = ringA + s2 * SL.a_bytes;   // a_n row r+1
            const unsigned char* Pq = ringP + ps * SL.p_bytes;   // a_{n-1} row r
            unsigned char* Bq = ringB + sB * SL.b_bytes;         // a_{n+1} row r (written now)
            const int sBc = sB == 0 ? kSB2 - 1 : sB - 1;
            const unsigned char* Bc = ringB + sBc * SL.b_bytes;  // a_{n+1} row r-1
            const bool own_b = (q >= 1 && q <= H);
            const bool do_c = (q >= 2);
            double2* outB = g.outB + rB * growstep + g0;
            double2* outC = g.outC + rC * growstep + g0;
#pragma unroll
            for (int p = 0; p < NPI; ++p) {
                if (halo_warp) break;
                const int lx = k0 + p * KSTEP;       // interior site
                const int oa = (lx + 2) * SITE + lo;  // a_n slot index
                const int ob = (lx + 1) * SITE + lo;  // a_{n+1} slot index
                const int op = (lx + PH) * SITE + lo; // a_{n-1} slot index
                const double2 ph = PEIERLS ? sphase[lx + 1] : make_double2(0.0, 0.0);
                if (q == 0) {
                    am[p] = ld(A0 + oa);
                    ac[p] = ld(A1 + oa);
                    if (ONSITE) em[p] = reinterpret_cast<const double*>(A0 + SL.eps_m)[lx];
                }
                ap[p] = ld(A2 + oa);
                // first step: a_{n+1}(row r, lx)
                const double2 x = ac[p];
                const double e1 = ONSITE ? reinterpret_cast<const double*>(A1 + SL.eps_m)[lx] : g.shift;
                const double2 b = step_val(x, ld(A1 + oa - SITE), ld(A1 + oa + SITE), am[p], ap[p], e1, ph, ld(Pq + op));
                *reinterpret_cast<double2*>(Bq + ob) = b;
                if (own_b) {
                    __stcs(outB + p * gstep, b);
                    dot_acc<PEIERLS>(acc[0], x, x);
                    dot_acc<PEIERLS>(acc[1], x, b);
                    dot_acc<PEIERLS>(acc[2], b, b);
                }
                // second step: a_{n+2}(row r-1, lx); centre a_{n+1}(r-1) and y-neighbours
                // a_{n+1}(r-2), a_{n+1}(r) are this thread's own values
                if (do_c) {
                    const double e0 = ONSITE ? em[p] : g.shift;
                    const double2 c = step_val(bc[p], ld(Bc + ob - SITE), ld(Bc + ob + SITE), bm[p], b, e0, ph, am[p]);
                    __stcs(outC + p * gstep, c);
                    dot_acc<PEIERLS>(acc[3], bc[p], c);
                    if (tail) dot_acc<PEIERLS>(acc[4], c, c);
                }
                // roll the per-thread values one row down
                am[p] = ac[p];
                ac[p] = ap[p];
                bm[p] = bc[p];
                bc[p] = b;
                if (ONSITE) em[p] = e1;
            }
            if (hs >= 0) {  // halo a_{n+1} site (recomputed here, owned by the neighbouring pencil)
                const int oa = (hlx + 2) * SITE + lo;
                const int ob = (hlx + 1) * SITE + lo;
                const int op = (hlx + PH) * SITE + lo;
                const double2 ph = PEIERLS ? sphase[hlx + 1] : make_double2(0.0, 0.0);
                const double e1 = ONSITE ? SL.eps(A1, hlx, TX) : g.shift;
                const double2 b = step_val(ld(A1 + oa), ld(A1 + oa - SITE), ld(A1 + oa + SITE), ld(A0 + oa), ld(A2 + oa), e1,
                                           ph, ld(Pq + op));
                *reinterpret_cast<double2*>(Bq + ob) = b;
            }
            if (halo_warp) {  // the two halo sites x0-1, x0+TX of a_{n+1}, all lanes
                for (int j = t - CONS; j < 2 * TL; j += 32) {
                    const int hx = j < TL ? -1 : TX, hl = j % TL;
                    const int oa = (hx + 2) * SITE + hl * 16;
                    const int ob = (hx + 1) * SITE + hl * 16;
                    const int op = (hx + PH) * SITE + hl * 16;
                    const double2 ph = PEIERLS ? sphase[hx + 1] : make_double2(0.0, 0.0);
                    const double e1 = ONSITE ? SL.eps(A1, hx, TX) : g.shift;
                    const double2 b = step_val(ld(A1 + oa), ld(A1 + oa - SITE), ld(A1 + oa + SITE), ld(A0 + oa),
                                               ld(A2 + oa), e1, ph, ld(Pq + op));
                    *reinterpret_cast<double2*>(Bq + ob) = b;
                }
            }
            __syncthreads();  // row q done: slots of a_n row r-1 and a_{n-1} row r are free
            if (t == PRODUCER) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issueA(s0);
            }
            if (t == PRODUCER_P) {
                if (PRODUCER_P != PRODUCER) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issueP(ps);
            }
            ++ip;
            sB = sB + 1 == kSB2 ? 0 : sB + 1;
            s0 = s1;
            ps = ps + 1 == kSP2 ? 0 : ps + 1;
            rB = rB + 1 == g.L1 ? 0 : rB + 1;
            rC = rC + 1 == g.L1 ? 0 : rC + 1;
        }
        if (t == PRODUCER) {  // the segment's last two a_n rows are free too
            issueA((ia_seg + H + 2) % kSA2);
            issueA((ia_seg + H + 3) % kSA2);
        }
        ia = ia_seg + H + 4;
        cs.seg(g, 0);
    }
    if (cur_lg != -1) flush(cur_lg);
    __syncthreads();
    for (int k = 0; k < 5; ++k) {
        double* rowk = g.red[k];
        if (rowk == nullptr || (k == 4 && !tail)) continue;
        for (int v = t; v < g.RP; v += blockDim.x) rowk[(size_t)blockIdx.x * g.RP + v] = sacc[k * g.RP + v];
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int v = t; v < g.RP; v += blockDim.x) rowk[(size_t)rr * g.RP + v] = 0.0;
    }
}

}  // namespace kpm
