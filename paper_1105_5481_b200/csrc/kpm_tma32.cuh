// kpm_tma32.cuh -- two recursion steps per HBM pass (temporal blocking) for 3D lattices
// (c3, c5 hot path).
//
// One launch advances Eq 18 by two steps,
//     a_{n+1} = 2 H~ a_n - a_{n-1},     a_{n+2} = 2 H~ a_{n+1} - a_n,
// reading a_n and a_{n-1} from HBM once and writing a_{n+1} and a_{n+2} once: 4 D R s
// bytes per two steps instead of 6 D R s.  The doubling inner products of both steps
// (<a_n|a_n>, <a_n|a_{n+1}>, <a_{n+1}|a_{n+1}>, <a_{n+1}|a_{n+2}>, odd-N tail
// <a_{n+2}|a_{n+2}>) are reduced from registers, as in the single-step kernels.
//
// Tiling: a pencil of TX x TY sites x TL vector lanes marching over z (the 3D march of
// kpm_tma3.cuh), with the halos the second step needs:
//   a_n     sites x0-2 .. x0+TX+1, y0-2 .. y0+TY+1   dense [TY+4][TX+4] box per plane
//   a_{n-1} sites x0-1 .. x0+TX,   y0-1 .. y0+TY     dense [TY+2][TX+2] box per plane
//   a_{n+1} computed on the same [TY+2][TX+2] ring-1 region (the ring is recomputed, not
//           stored) into a 2-plane shared-memory ring; interior stored
//   a_{n+2} interior TX x TY, stored
// The x halos come from the x-row frame of periodic images (row pitch L0 + 4, xpad = 2:
// kpm_capi.cu), so every box is ONE TMA load of TY rows plus two row loads (2 rows for
// a_n, 1 row for a_{n-1} and eps~) at periodically wrapped y; eps~ comes from a copy in
// the same frame layout (boxes TX+4 wide from an even frame column: TMA faulted with an
// illegal instruction on 8-byte aligned box starts).  z neighbours are rolled in registers: the thread that computes
// a site of a_{n+1} keeps a_n of the planes below and above; interior sites are the first
// passes of the ring-1 enumeration, so the same thread also owns a_{n+1} of the planes
// around and a_n of the plane below, which the second step needs.
//
// March iteration q of a segment with output planes [m0, m0+H): a_{n+1} of plane
// zb = m0-1+q on the ring-1 region (needs a_n planes zb-1..zb+1 and a_{n-1} plane zb),
// then a_{n+2} of plane zb-1 (needs a_{n+1} planes zb-2..zb and a_n plane zb-1).  One CTA
// barrier per iteration; after it one thread refills the two released ring slots with
// the next TMA loads of the CTA's load sequence (in-band producer, as kpm_tma2.cuh).
// Outputs go to two other buffers (out of place): an in-place store could overwrite a
// halo value a neighbouring CTA has still to read.
#pragma once
#include "kpm_tma.cuh"

namespace kpm {

struct Tma32Geom {
    int L0, L1, L2;      // lattice extents
    int PX, PY;          // pencils along x, y
    int G_L;             // lane groups = RG / TL
    int RG, RP;
    long long W;         // rr: columns; contiguous: output planes (columns * L2)
    int rr;              // 1: whole columns round-robin over CTAs; 0: contiguous plane ranges
    int rows_total;      // partial-sum rows per slot (>= gridDim.x; extra rows are zeroed)
    int pfirst;          // 1: a_{n-1} boxes with the L2 evict-first policy
    int lg_fast;         // 1: columns enumerate lane groups fastest (all lanes of a pencil at once)
    double t, shift;
    double* red[5];      // slots 2n .. 2n+3, (tail) 2n+4; red[4] nullable
    double2* outB;       // a_{n+1} (frame layout)
    double2* outC;       // a_{n+2}
};

// NT threads per CTA (all computing, one CTA per SM): 512 (16 warps, <= 128 registers) --
// the ncu capture of the 256-thread variant showed 8 warps stalled on the per-plane barrier
// and shared-memory latency (DRAM 46% busy).
template <int TX, int TY, int TL, bool ONSITE, int NT>
struct Lay32 {
    static constexpr int SITE = TL * 16;
    static constexpr int AW = TX + 4, AH = TY + 4;   // a_n box
    static constexpr int BW = TX + 2, BH = TY + 2;   // a_{n-1}, a_{n+1}, eps~ boxes
    static constexpr int A_BOX = AH * AW * SITE;
    // eps~ rows are loaded AW wide from an even (16-byte aligned) frame column: sites x0-2 .. x0+TX+1
    static constexpr int EROW = (AW * 8 + 127) / 128 * 128;           // eps~ single row piece
    static constexpr int EMAIN = (TY * AW * 8 + 127) / 128 * 128;     // eps~ main piece
    static constexpr int E_TOP = A_BOX, E_MAIN = A_BOX + EROW, E_BOT = A_BOX + EROW + EMAIN;
    static constexpr int A_SLOT = ONSITE ? E_BOT + EROW : A_BOX;
    static constexpr int B_SLOT = (BH * BW * SITE + 127) / 128 * 128;
    static constexpr int NRING = BW * BH;            // ring-1 sites
    static constexpr int NINT = TX * TY;
    static constexpr int KSTEP = NT / TL;            // sites per pass
    static constexpr int NPI = NINT / KSTEP;         // interior passes
    static constexpr int NPH = (NRING - NINT + KSTEP - 1) / KSTEP;  // halo passes
    static constexpr uint32_t A_TX = A_BOX + (ONSITE ? BH * AW * 8 : 0);
    static constexpr uint32_t P_TX = BH * BW * SITE;
};

template <int TX, int TY, int TL, bool ONSITE, int NT, int KA, int KP>
__host__ __device__ inline size_t step32_smem_bytes(int RP) {
    using Y = Lay32<TX, TY, TL, ONSITE, NT>;
    return (size_t)KA * Y::A_SLOT + (size_t)KP * Y::B_SLOT + 2 * (size_t)Y::B_SLOT + 5 * (size_t)RP * 8 +
           (size_t)NT * 16 + (KA + KP) * 8;
}

// One CTA's load sequence: segments (column, planes [m0, m0+H)), loads q = 0 .. H+extra-1.
struct Cursor32 {
    long long w, w_end;
    int col_step;
    int lg, px, py, m0, H, q, nq;
    int z;  // wrapped plane of load q (m0 - extra/2 + q), advanced with one compare per load
    bool valid;
    __device__ void seg(const Tma32Geom& g, int extra) {
        valid = w < w_end;
        if (!valid) return;
        long long col;
        if (g.rr) {
            col = w;
            m0 = 0;
            H = g.L2;
            w += col_step;
        } else {
            col = w / g.L2;
            m0 = (int)(w - col * g.L2);
            const long long e = min(w_end, (col + 1) * (long long)g.L2);
            H = (int)(e - w);
            w = e;
        }
        int pencil;
        if (g.lg_fast) {
            pencil = (int)(col / g.G_L);
            lg = (int)(col - (long long)pencil * g.G_L);
        } else {
            pencil = (int)(col % ((long long)g.PX * g.PY));
            lg = (int)(col / ((long long)g.PX * g.PY));
        }
        px = pencil % g.PX;
        py = pencil / g.PX;
        q = 0;
        nq = H + extra;
        z = m0 - extra / 2;
        while (z < 0) z += g.L2;
    }
    __device__ void init(const Tma32Geom& g, int extra) {
        if (g.rr) {
            w = blockIdx.x;
            w_end = g.W;
            col_step = gridDim.x;
        } else {
            w = g.W * blockIdx.x / gridDim.x;
            w_end = g.W * (blockIdx.x + 1) / gridDim.x;
            col_step = 0;
        }
        seg(g, extra);
    }
    __device__ void next(const Tma32Geom& g, int extra) {
        if (++z == g.L2) z = 0;
        if (++q >= nq) seg(g, extra);
    }
};

template <int TX, int TY, int TL, bool ONSITE, int NT, int KA, int KP>
__global__ void __launch_bounds__(NT, 1)
    kpm_step32_tma_kernel(const __grid_constant__ CUtensorMap mapA,    // a_n {2TL, TX+4, TY, 1}
                          const __grid_constant__ CUtensorMap mapA2,   // a_n {2TL, TX+4, 2, 1}
                          const __grid_constant__ CUtensorMap mapP,    // a_{n-1} {2TL, TX+2, TY, 1}
                          const __grid_constant__ CUtensorMap mapP1,   // a_{n-1} {2TL, TX+2, 1, 1}
                          const __grid_constant__ CUtensorMap mapE,    // eps~ frame {TX+4, TY, 1}
                          const __grid_constant__ CUtensorMap mapE1,   // eps~ frame {TX+4, 1, 1}
                          const Tma32Geom g, const int tail) {
    using Y = Lay32<TX, TY, TL, ONSITE, NT>;
    constexpr int SITE = Y::SITE, KSTEP = Y::KSTEP, NPI = Y::NPI, NPH = Y::NPH, NP = NPI + NPH;
    static_assert(Y::NINT % KSTEP == 0, "interior sites fill whole passes");
    static_assert(TY >= 2 && TX % 2 == 0, "2-row halo boxes; 16-byte eps rows");
    constexpr int XP = 2;  // x-row frame width (kpm_capi.cu xpad)
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + KA * Y::A_SLOT;
    unsigned char* ringB = ringP + KP * Y::B_SLOT;
    double* sacc = reinterpret_cast<double*>(ringB + 2 * Y::B_SLOT);  // [5][RP]
    double2* sred = reinterpret_cast<double2*>(sacc + 5 * g.RP);       // [threads]
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sred + NT);
    uint64_t* fullP = fullA + KA;

    const int t = threadIdx.x;
    __shared__ Cursor32 cur_smem[2];
    Cursor32& ca = cur_smem[0];
    Cursor32& cp = cur_smem[1];
    __shared__ uint64_t pol_smem;
    const int L0f = g.L0 + 2 * XP;  // frame row pitch (sites)
    auto issueA = [&](int slot) {   // next a_n plane (m0-2+q) of the sequence
        if (!ca.valid) return;
        const int z = ca.z;
        const int c0 = 2 * ca.lg * TL, x0 = ca.px * TX, y0 = ca.py * TY;
        const int yt = (y0 - 2 + g.L1) % g.L1, yb = (y0 + TY) % g.L1;
        unsigned char* dst = ringA + slot * Y::A_SLOT;
        mbar_expect_tx(fullA + slot, Y::A_TX);
        // frame x of site x0-2 is x0 (XP = 2)
        tma_load(dst, &mapA2, fullA + slot, c0, x0, yt, z);
        tma_load(dst + 2 * Y::AW * SITE, &mapA, fullA + slot, c0, x0, y0, z);
        tma_load(dst + (TY + 2) * Y::AW * SITE, &mapA2, fullA + slot, c0, x0, yb, z);
        if (ONSITE) {
            const int et = (y0 - 1 + g.L1) % g.L1, eb = (y0 + TY) % g.L1;
            tma_load(dst + Y::E_TOP, &mapE1, fullA + slot, x0, et, z);
            tma_load(dst + Y::E_MAIN, &mapE, fullA + slot, x0, y0, z);
            tma_load(dst + Y::E_BOT, &mapE1, fullA + slot, x0, eb, z);
        }
        ca.next(g, 4);
    };
    auto issueP = [&](int slot) {  // next a_{n-1} plane (m0-1+q) of the sequence
        if (!cp.valid) return;
        const int z = cp.z;
        const int c0 = 2 * cp.lg * TL, x0 = cp.px * TX, y0 = cp.py * TY;
        const int yt = (y0 - 1 + g.L1) % g.L1, yb = (y0 + TY) % g.L1;
        unsigned char* dst = ringP + slot * Y::B_SLOT;
        mbar_expect_tx(fullP + slot, Y::P_TX);
        if (g.pfirst) {
            const uint64_t pol = pol_smem;
            tma_load_hint(dst, &mapP1, fullP + slot, c0, x0 + 1, yt, z, pol);
            tma_load_hint(dst + Y::BW * SITE, &mapP, fullP + slot, c0, x0 + 1, y0, z, pol);
            tma_load_hint(dst + (TY + 1) * Y::BW * SITE, &mapP1, fullP + slot, c0, x0 + 1, yb, z, pol);
        } else {
            tma_load(dst, &mapP1, fullP + slot, c0, x0 + 1, yt, z);
            tma_load(dst + Y::BW * SITE, &mapP, fullP + slot, c0, x0 + 1, y0, z);
            tma_load(dst + (TY + 1) * Y::BW * SITE, &mapP1, fullP + slot, c0, x0 + 1, yb, z);
        }
        cp.next(g, 2);
    };
    if (t == 0) {
        for (int i = 0; i < KA; ++i) mbar_init(fullA + i, 1);
        for (int i = 0; i < KP; ++i) mbar_init(fullP + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&mapA);
        prefetch_tmap(&mapA2);
        prefetch_tmap(&mapP);
        prefetch_tmap(&mapP1);
        if (ONSITE) {
            prefetch_tmap(&mapE);
            prefetch_tmap(&mapE1);
        }
        pol_smem = policy_evict_first();
        ca.init(g, 4);
        cp.init(g, 2);
        for (int i = 0; i < KA; ++i) issueA(i);
        for (int i = 0; i < KP; ++i) issueP(i);
    }
    for (int i = t; i < 5 * g.RP; i += blockDim.x) sacc[i] = 0.0;
    __syncthreads();

    // ---- this thread's sites: lane l of ring-1 sites k0 + p*KSTEP (interior first, then the ring)
    const int l = t % TL, k0 = t / TL, lo = l * 16;
    int oa[NP], ob[NP], oe[NP];
    bool valid[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        int lx, ly;
        const int k = k0 + p * KSTEP;
        valid[p] = true;
        if (p < NPI) {
            lx = k % TX;
            ly = k / TX;
        } else {
            int h = k - Y::NINT;
            valid[p] = h < Y::NRING - Y::NINT;
            if (!valid[p]) h = 0;
            if (h < TX + 2) { lx = h - 1; ly = -1; }                       // top row
            else if (h < 2 * (TX + 2)) { lx = h - (TX + 2) - 1; ly = TY; }  // bottom row
            else if (h < 2 * (TX + 2) + TY) { lx = -1; ly = h - 2 * (TX + 2); }
            else { lx = TX; ly = h - 2 * (TX + 2) - TY; }
        }
        oa[p] = ((ly + 2) * Y::AW + lx + 2) * SITE + lo;
        ob[p] = ((ly + 1) * Y::BW + lx + 1) * SITE + lo;
        oe[p] = ly < 0 ? Y::E_TOP + (lx + 2) * 8
                       : (ly >= TY ? Y::E_BOT + (lx + 2) * 8 : Y::E_MAIN + (ly * Y::AW + lx + 2) * 8);
    }

    double2 acc[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) acc[k] = make_double2(0.0, 0.0);
    auto ld = [](const unsigned char* p) { return *reinterpret_cast<const double2*>(p); };
    auto flush = [&](int lgf) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            sred[t] = acc[k];
            __syncthreads();
            if (t < TL) {
                double2 s = make_double2(0.0, 0.0);
                for (int j = t; j < NT; j += TL) s = add2(s, sred[j]);
                const int v = lgf * TL + t;
                sacc[k * g.RP + 2 * v] += s.x;
                sacc[k * g.RP + 2 * v + 1] += s.y;
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[k] = make_double2(0.0, 0.0);
    };
    // 2 H~ x - p from the six neighbours' sum
    auto step_val = [&](double2 x, double2 nb, double e, double2 p) {
        const double2 h = fma2(e, x, scale2(g.t, nb));
        return make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));
    };

    constexpr int PRODUCER = 32;  // thread 0 of warp 1
    Cursor32 cs;  // segment iterator of the consumers (same sequence)
    cs.init(g, 0);
    int ia = 0, ip = 0, cur_lg = -1;
    const long long zstride = (long long)g.L1 * L0f * g.RG;  // lanes per frame plane
    while (cs.valid) {
        const int lg = cs.lg, m0 = cs.m0, H = cs.H, x0 = cs.px * TX, y0 = cs.py * TY;
        if (cur_lg != -1 && lg != cur_lg) flush(cur_lg);
        cur_lg = lg;
        // global lane offsets (plane 0) of this thread's interior sites, and their x images
        long long go[NPI];
        int img[NPI];  // +1: also store at +L0 (x < 2); -1: at -L0 (x >= L0-2); 0: none
#pragma unroll
        for (int p = 0; p < NPI; ++p) {
            const int k = k0 + p * KSTEP, lx = k % TX, ly = k / TX;
            const int xs = x0 + lx;
            go[p] = ((long long)(y0 + ly) * L0f + xs + XP) * g.RG + (long long)lg * TL + l;
            img[p] = xs < XP ? 1 : (xs >= g.L0 - XP ? -1 : 0);
        }
        const long long imgoff = (long long)g.L0 * g.RG;
        const int ia_seg = ia;
        int sB = 0;                         // ring-B slot of a_{n+1} plane zb
        int s0 = ia_seg % KA;               // a_n slot of plane zb-1
        int ps = ip % KP;
        int zb = (m0 - 1 + g.L2) % g.L2;    // plane of a_{n+1} computed this iteration
        int zc = (m0 - 2 + g.L2) % g.L2;    // plane of a_{n+2}
        double2 am[NP], ac[NP], bm[NPI], bc[NPI];
        double em[NPI];
        for (int q = 0; q < H + 2; ++q) {
            const int i0 = ia_seg + q;
            const int s1 = s0 + 1 == KA ? 0 : s0 + 1;
            const int s2 = s1 + 1 == KA ? 0 : s1 + 1;
            if (q == 0) {
                mbar_wait(fullA + s0, (uint32_t)((i0 / KA) & 1));
                mbar_wait(fullA + s1, (uint32_t)(((i0 + 1) / KA) & 1));
            }
            mbar_wait(fullA + s2, (uint32_t)(((i0 + 2) / KA) & 1));
            mbar_wait(fullP + ps, (uint32_t)((ip / KP) & 1));
            const unsigned char* A0 = ringA + s0 * Y::A_SLOT;   // a_n plane zb-1
            const unsigned char* A1 = ringA + s1 * Y::A_SLOT;   // a_n plane zb
            const unsigned char* A2 = ringA + s2 * Y::A_SLOT;   // a_n plane zb+1
            const unsigned char* Pq = ringP + ps * Y::B_SLOT;   // a_{n-1} plane zb
            unsigned char* Bq = ringB + sB * Y::B_SLOT;         // a_{n+1} plane zb (written now)
            const unsigned char* Bc = ringB + (sB ^ 1) * Y::B_SLOT;  // a_{n+1} plane zb-1
            const bool own_b = (q >= 1 && q <= H);
            const bool do_c = (q >= 2);
            double2* outB = g.outB + (long long)zb * zstride;
            double2* outC = g.outC + (long long)zc * zstride;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (p >= NPI && !valid[p]) continue;
                const int o = oa[p];
                if (q == 0) {
                    am[p] = ld(A0 + o);
                    ac[p] = ld(A1 + o);
                }
                const double2 x = ac[p];
                const double2 zp = ld(A2 + o);
                double2 nb = add2(ld(A1 + o - SITE), ld(A1 + o + SITE));
                nb = add2(nb, add2(add2(ld(A1 + o - Y::AW * SITE), ld(A1 + o + Y::AW * SITE)), add2(am[p], zp)));
                const double e1 = ONSITE ? *reinterpret_cast<const double*>(A1 + oe[p]) : g.shift;
                const double2 b = step_val(x, nb, e1, ld(Pq + ob[p]));   // a_{n+1}(zb)
                *reinterpret_cast<double2*>(Bq + ob[p]) = b;
                if (p < NPI) {
                    if (own_b) {
                        double2* dst = outB + go[p];
                        __stcs(dst, b);
                        if (img[p]) __stcs(dst + img[p] * imgoff, b);
                        dot_acc<false>(acc[0], x, x);
                        dot_acc<false>(acc[1], x, b);
                        dot_acc<false>(acc[2], b, b);
                    }
                    if (do_c) {  // a_{n+2}(zb-1): centre bc, z neighbours bm and b, a_n(zb-1) = am
                        const int ib = ob[p];
                        double2 nc = add2(ld(Bc + ib - SITE), ld(Bc + ib + SITE));
                        nc = add2(nc, add2(add2(ld(Bc + ib - Y::BW * SITE), ld(Bc + ib + Y::BW * SITE)), add2(bm[p], b)));
                        const double e0 = ONSITE ? em[p] : g.shift;
                        const double2 c = step_val(bc[p], nc, e0, am[p]);
                        double2* dst = outC + go[p];
                        __stcs(dst, c);
                        if (img[p]) __stcs(dst + img[p] * imgoff, c);
                        dot_acc<false>(acc[3], bc[p], c);
                        if (tail) dot_acc<false>(acc[4], c, c);
                    }
                    bm[p] = bc[p];
                    bc[p] = b;
                    if (ONSITE) em[p] = e1;
                }
                am[p] = x;
                ac[p] = zp;
            }
            __syncthreads();  // plane done: a_n slot of zb-1, a_{n-1} slot of zb are free; B(zb) complete
            if (t == PRODUCER) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issueA(s0);
                issueP(ps);
            }
            ++ip;
            sB ^= 1;
            s0 = s1;
            ps = ps + 1 == KP ? 0 : ps + 1;
            zb = zb + 1 == g.L2 ? 0 : zb + 1;
            zc = zc + 1 == g.L2 ? 0 : zc + 1;
        }
        if (t == PRODUCER) {  // the segment's last two a_n planes are free too
            issueA((ia_seg + H + 2) % KA);
            issueA((ia_seg + H + 3) % KA);
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
