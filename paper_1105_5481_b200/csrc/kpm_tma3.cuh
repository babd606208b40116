// kpm_tma3.cuh -- 3D march kernel with a dense halo box per plane (c3, c5 hot path).
//
// Same arithmetic, schedule and mbarrier protocol as kpm_step_tma_kernel<3, ...> (one
// recursion step, Eq 18, fused with the doubling inner products), with the
// per-site work cut down for an issue-bound kernel (ncu: ~49% issue slots busy):
//  * Thanks to the x-row frame of periodic images (row pitch L0 + 4, kpm_capi.cu xpad), a
//    plane tile's x-halo is contiguous in HBM, so ONE TMA box of (TX+2) x TY sites plus two
//    (TX+2)-site row boxes (y-halo rows, periodically wrapped) fill a dense
//    [TY+2][TX+2][TL lanes] smem box: every neighbour is a fixed offset (+-1 site, +-(TX+2)
//    sites), no halo branches, no runtime div/mod (TX, TY, TL are template parameters).
//  * March-dimension (z) neighbours are rolled in registers: a site of plane m needs the
//    centre of plane m-1 (last iteration's centre) and of plane m+1 (one new LDS); the centre
//    itself is last iteration's plane-(m+1) value.  5 LDS per site instead of 7.
// Tiles: TX*TY*TL = 1024 lanes (16 KB) as before; 8 consumer warps + 1 producer warp.
#pragma once
#include "kpm_tma.cuh"

namespace kpm {

template <int TX, int TY, int TL, bool ONSITE>
struct Slot3 {
    static constexpr int SITE = TL * 16;
    static constexpr int ROW = (TX + 2) * SITE;            // one box row (x-halo included)
    static constexpr int VEC = (TY + 2) * ROW;             // [TY+2][TX+2] sites
    static constexpr int EPS = VEC;                        // eps~ [TY][TX] doubles after the box
    static constexpr int BYTES = (VEC + (ONSITE ? TX * TY * 8 : 0) + 127) / 128 * 128;
    static constexpr int TILE = TX * TY * SITE;            // a_{n-1} tile (no halo)
    static constexpr int SP = TL >= 32 ? 3 : kSP;          // a_{n-1} ring (32-lane tiles: smem)
};

template <int TX, int TY, int TL, bool ONSITE>
__host__ __device__ inline size_t step3_smem_bytes(int RP) {
    using S = Slot3<TX, TY, TL, ONSITE>;
    return (size_t)kSA * S::BYTES + (size_t)S::SP * S::TILE + 3 * (size_t)RP * 8 +
           3 * (size_t)kTmaConsumerWarps * 32 * 16 + (2 * kSA + 2 * S::SP) * 8;
}

template <int TX, int TY, int TL, bool ONSITE>
__global__ void __launch_bounds__(kTmaThreads, 1)
    kpm_step3_tma_kernel(const __grid_constant__ CUtensorMap mapBox,   // a_n: {2TL, TX+2, TY, 1}
                         const __grid_constant__ CUtensorMap mapRow,   // a_n: {2TL, TX+2, 1, 1}
                         const __grid_constant__ CUtensorMap mapP,     // a_{n-1}: {2TL, TX, TY, 1}
                         const __grid_constant__ CUtensorMap mapE,     // eps~: {TX, TY, 1}
                         const TmaGeom g, const int tail) {
    pdl_entry();
    using S = Slot3<TX, TY, TL, ONSITE>;
    constexpr int CONS = kTmaConsumerWarps * 32;
    constexpr int KSTEP = CONS / TL;                 // tile sites per pass
    constexpr int NPASS = TX * TY / KSTEP;
    static_assert((TX * TY) % KSTEP == 0 && KSTEP % TX == 0, "passes advance whole tile rows");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + kSA * S::BYTES;
    double* sacc = reinterpret_cast<double*>(ringP + S::SP * S::TILE);  // [3][RP]
    double2* sred = reinterpret_cast<double2*>(sacc + 3 * g.RP);     // [3][CONS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sred + 3 * CONS);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + kSA;
    uint64_t* fullP = emptyA + kSA;
    uint64_t* emptyP = fullP + S::SP;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSA; ++i) {
            mbar_init(fullA + i, 1);
            mbar_init(emptyA + i, kTmaConsumerWarps);
        }
        for (int i = 0; i < S::SP; ++i) {
            mbar_init(fullP + i, 1);
            mbar_init(emptyP + i, kTmaConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 3 * g.RP; i += blockDim.x) sacc[i] = 0.0;
    __syncthreads();

    if (warp == kTmaConsumerWarps) {
        // ---------------------------------------------------------------- producer
        if (lane == 0) {
            prefetch_tmap(&mapBox);
            prefetch_tmap(&mapRow);
            prefetch_tmap(&mapP);
            if (ONSITE) prefetch_tmap(&mapE);
            const uint64_t pol_first = policy_evict_first();
            const uint64_t pol_last = policy_evict_last();
            constexpr uint32_t bytesA = S::VEC + (ONSITE ? TX * TY * 8 : 0);
            long long ia = 0, ip = 0;
            Sched sq = sched_begin(g);
            Seg s;
            while (next_seg(g, sq, s)) {
                const int c0 = 2 * s.lg * TL;
                const int x0 = s.px * TX, y0 = s.py * TY;
                const int xb = x0 + g.xpad - 1;  // frame coordinates: the box starts one site left
                const int yt = (y0 - 1 + g.L1) % g.L1, yb = (y0 + TY) % g.L1;
                const int H = s.m1 - s.m0;
                for (int q = 0; q < H + 2; ++q) {
                    const int m = g.ghost ? g.zoff + s.m0 + q : (s.m0 - 1 + q + g.Lm) % g.Lm;
                    const int slot = (int)(ia % kSA);
                    if (ia >= kSA) mbar_wait(emptyA + slot, (uint32_t)(((ia / kSA) - 1) & 1));
                    unsigned char* dst = ringA + slot * S::BYTES;
                    mbar_expect_tx(fullA + slot, bytesA);
// a_n boxes with the L2 evict-last policy: the halo rows and columns a neighbouring pencil re-reads
                    // stay in L2 behind the streamed a_{n-1} / a_{n+1} (A/B: c3 1087 -> 1078 ms, c5 9013 -> 8818 ms)
                    tma_load_hint(dst, &mapRow, fullA + slot, c0, xb, yt, m, pol_last);
                    tma_load_hint(dst + S::ROW, &mapBox, fullA + slot, c0, xb, y0, m, pol_last);
                    tma_load_hint(dst + (TY + 1) * S::ROW, &mapRow, fullA + slot, c0, xb, yb, m, pol_last);
                    if (ONSITE) tma_load(dst + S::EPS, &mapE, fullA + slot, x0, y0, m - g.ghost);
                    ++ia;
                    if (q >= 1 && q - 1 < H) {
                        const int mp = g.zoff + s.m0 + q - 1 + g.ghost;
                        const int ps = (int)(ip % S::SP);
                        if (ip >= S::SP) mbar_wait(emptyP + ps, (uint32_t)(((ip / S::SP) - 1) & 1));
                        mbar_expect_tx(fullP + ps, S::TILE);
                        tma_load_hint(ringP + ps * S::TILE, &mapP, fullP + ps, c0, x0 + g.xpad, y0, mp, pol_first);
                        ++ip;
                    }
                }
            }
        }
    } else {
        // ---------------------------------------------------------------- consumers
        const int t = threadIdx.x;
        const int l = t % TL;
        const int k0 = t / TL;
        const int lx = k0 % TX, ly0 = k0 / TX;  // pass p: tile row ly0 + p * (KSTEP / TX)
        // smem byte offset of this thread's lane of site (lx, ly) inside a box slot
        auto boff = [&](int p) { return ((ly0 + p * (KSTEP / TX) + 1) * (TX + 2) + lx + 1) * S::SITE + l * 16; };
        double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
        long long ia = 0, ip = 0;
        Sched sq = sched_begin(g);
        Seg s;
        int cur_lg = -1;
        auto flush = [&](int lg) {
            sred[t] = acc0;
            sred[CONS + t] = acc1;
            sred[2 * CONS + t] = acc2;
            named_bar_sync(1, CONS);
            if (t < TL) {
                for (int k = 0; k < 3; ++k) {
                    double2 sum = make_double2(0.0, 0.0);
                    for (int j = t; j < CONS; j += TL) sum = add2(sum, sred[k * CONS + j]);
                    const int v = lg * TL + t;
                    sacc[k * g.RP + 2 * v] += sum.x;
                    sacc[k * g.RP + 2 * v + 1] += sum.y;
                }
            }
            named_bar_sync(1, CONS);
            acc0 = acc1 = acc2 = make_double2(0.0, 0.0);
        };
        auto ld = [](const unsigned char* p) { return *reinterpret_cast<const double2*>(p); };
        const long long zstride = (long long)g.L1 * (g.L0 + 2 * g.xpad);  // memory sites per plane
        while (next_seg(g, sq, s)) {
            if (cur_lg != -1 && s.lg != cur_lg) flush(cur_lg);
            cur_lg = s.lg;
            const int x0 = s.px * TX, y0 = s.py * TY;
            const int H = s.m1 - s.m0;
            const long long ia_seg = ia;
            // global lane offset of site (x0 + lx, y0 + ly0 + pass rows) in plane 0 (frame coordinates)
            const int xs = x0 + lx;
            const long long o0 = ((long long)(y0 + ly0) * (g.L0 + 2 * g.xpad) + xs + g.xpad) * g.RG + s.lg * TL + l;
            const long long prow = (long long)(KSTEP / TX) * (g.L0 + 2 * g.xpad) * g.RG;  // pass -> +rows
            const bool img_lo = xs < g.xpad, img_hi = xs >= g.L0 - g.xpad;
            // z neighbours roll in registers; the plane loop is unrolled by 2 so the two roles (plane m-1,
            // plane m) swap at compile time instead of by register moves, and the ring slots advance
            // incrementally (no 64-bit modulo per plane)
            double2 ZR[2][NPASS];
            int sa0 = (int)(ia_seg % kSA), ph0 = (int)((ia_seg / kSA) & 1);  // slot / parity of load i0
            int ps = (int)(ip % S::SP), pph = (int)((ip / S::SP) & 1);
            auto plane = [&](const int j, const int u) {
                double2(&zm)[NPASS] = ZR[u];
                double2(&zc)[NPASS] = ZR[u ^ 1];
                int sa1 = sa0 + 1, ph1 = ph0;
                if (sa1 == kSA) { sa1 = 0; ph1 ^= 1; }
                int sa2 = sa1 + 1, ph2 = ph1;
                if (sa2 == kSA) { sa2 = 0; ph2 ^= 1; }
                if (j == 0) {
                    mbar_wait(fullA + sa0, (uint32_t)ph0);
                    mbar_wait(fullA + sa1, (uint32_t)ph1);
                }
                mbar_wait(fullA + sa2, (uint32_t)ph2);
                mbar_wait(fullP + ps, (uint32_t)pph);
                const unsigned char* S0 = ringA + sa0 * S::BYTES;  // plane m-1
                const unsigned char* S1 = ringA + sa1 * S::BYTES;  // plane m
                const unsigned char* S2 = ringA + sa2 * S::BYTES;  // plane m+1
                const unsigned char* Pv = ringP + ps * S::TILE;
                const long long mo = (long long)(g.zoff + s.m0 + j + g.ghost) * zstride * g.RG;
#pragma unroll
                for (int pass = 0; pass < NPASS; ++pass) {
                    const int o = boff(pass);
                    if (j == 0) {
                        zm[pass] = ld(S0 + o);
                        zc[pass] = ld(S1 + o);
                    }
                    const double2 x = zc[pass];
                    const double2 zp = ld(S2 + o);
                    double2 nb = add2(ld(S1 + o - S::SITE), ld(S1 + o + S::SITE));
                    nb = add2(nb, add2(add2(ld(S1 + o - S::ROW), ld(S1 + o + S::ROW)), add2(zm[pass], zp)));
                    const int k = k0 + pass * KSTEP;
                    const double e = ONSITE ? reinterpret_cast<const double*>(S1 + S::EPS)[k] : g.shift;
                    const double2 h = fma2(e, x, scale2(g.t, nb));
                    const double2 p = *reinterpret_cast<const double2*>(Pv + k * S::SITE + l * 16);
                    const double2 y = make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));  // Eq (18)
                    double2* out = g.out + mo + o0 + pass * prow;
                    __stcs(out, y);
                    if (img_lo) __stcs(out + (long long)g.L0 * g.RG, y);   // periodic x images in the frame
                    if (img_hi) __stcs(out - (long long)g.L0 * g.RG, y);
                    if (g.peer_lo) {  // fused halo: the neighbours' ghost planes (row partition)
                        const int mb = g.zoff + s.m0 + j + g.ghost;
                        store_peers(g, mb, out, y);
                        if (img_lo) store_peers(g, mb, out + (long long)g.L0 * g.RG, y);
                        if (img_hi) store_peers(g, mb, out - (long long)g.L0 * g.RG, y);
                    }
                    dot_acc<false>(acc0, x, x);
                    dot_acc<false>(acc1, x, y);
                    if (tail) dot_acc<false>(acc2, y, y);
                    zm[pass] = zp;  // plane m+1 takes the slot of plane m-1: next plane's "zc"
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(emptyA + sa0);
                    mbar_arrive(emptyP + ps);
                }
                ++ip;
                sa0 = sa1;
                ph0 = ph1;
                if (++ps == S::SP) {
                    ps = 0;
                    pph ^= 1;
                }
            };
            for (int j = 0; j < H; j += 2) {
                plane(j, 0);
                if (j + 1 < H) plane(j + 1, 1);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(emptyA + (int)((ia_seg + H) % kSA));
                mbar_arrive(emptyA + (int)((ia_seg + H + 1) % kSA));
            }
            ia = ia_seg + H + 2;
        }
        if (cur_lg != -1) flush(cur_lg);
    }
    __syncthreads();
    for (int k = 0; k < 3; ++k) {
        double* rowk = k == 0 ? g.red0 : (k == 1 ? g.red1 : (tail ? g.red2 : nullptr));
        if (rowk == nullptr) continue;
        rowk += (size_t)g.row_off * g.RP;
        for (int v = threadIdx.x; v < g.RP; v += blockDim.x) rowk[(size_t)blockIdx.x * g.RP + v] = sacc[k * g.RP + v];
        for (int rr = blockIdx.x + gridDim.x; rr < g.rows_total; rr += gridDim.x)
            for (int v = threadIdx.x; v < g.RP; v += blockDim.x) rowk[(size_t)rr * g.RP + v] = 0.0;
    }
}

}  // namespace kpm
