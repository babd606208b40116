// kpm_tma.cuh -- TMA-fed, mbarrier-pipelined fused recursion step for 2D/3D lattices.
//
// Same arithmetic as kpm_step_kernel<StencilOp, STEP> (Eq 18 + the doubling inner
// products), organised for sm_100a's memory system instead of relying on L1/L2
// to catch neighbour re-reads:
//
//  * The lattice is cut into pencils along the slowest dimension ("march" dim:
//    y in 2D, z in 3D).  A pencil is a TX (x TY) tile of sites x TL vector lanes.
//    Each CTA owns a contiguous range of (lane group, pencil, plane) output
//    planes and marches through it.
//  * One producer thread issues cp.async.bulk.tensor (TMA) loads of each plane
//    tile of a_n -- main tile, the two x-halo columns and (3D) the two y-halo
//    rows at periodically wrapped coordinates, and the on-site tile eps~ -- into
//    a ring of S_A shared-memory slots, and of each a_{n-1} tile into a ring of
//    S_P slots; completion is signalled by mbarrier transaction counts.  Bytes in
//    flight per SM are set by the ring depth, not by registers.
//  * Consumer warps compute a_{n+1} = 2 H~ a_n - a_{n-1} for plane m from slots
//    m-1, m, m+1 (every a_n element comes from HBM once per pencil; in-plane
//    halos come from L2), stream a_{n+1} to global with evict-first stores over
//    a_{n-1}, and accumulate <a_n|a_n>, <a_n|a_{n+1}> per vector in registers.
//  * Reductions are per lane, flushed at segment ends into a CTA accumulator in
//    a fixed order, and written once per CTA -> deterministic.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "kpm_kernels.cuh"

namespace kpm {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Geometry of the tiled march (host-filled).
struct TmaGeom {
    int L0, L1, L2;   // lattice extents (L2 = 1 in 2D)
    int TX, TY;       // tile (TY = 1 in 2D)
    int TL;           // lanes (16-byte) per tile site
    int RG;           // lanes per site in the vector block
    int G_L;          // lane groups = RG / TL
    int PX, PY;       // pencils along x, y (PY = 1 in 2D)
    int Lm;           // march extent (L1 in 2D, L2 in 3D)
    long long W;      // total output planes = G_L * PX * PY * Lm
    int rr;           // 1: round-robin whole columns over CTAs; 0: contiguous plane ranges
    int rows_total;   // partial-sum rows of this launch (>= gridDim.x; extra rows are zeroed)
    int row_off;      // first partial-sum row of this launch (row partition: boundary/interior launches)
    int zoff;         // ghost mode: first slab plane of this launch (planes [zoff, zoff + Lm))
    int xpad;         // 3D: x-rows of the vector blocks carry a frame of xpad periodic images per side
    int ghost;        // 1: row partition -- vector buffers hold Lm + 2 planes (ghost, local..., ghost),
                      //    march neighbours are never wrapped; 0: periodic wrap
    int RP;           // padded vectors (partial row length)
    double t;         // t / a
    double shift;     // -b / a (no on-site array)
    const double2* phase;  // Peierls phases by x (2D only)
    double* red0;     // partial rows [grid][RP]
    double* red1;
    double* red2;     // odd-N tail, nullable
    double2* out;     // a_{n-1} in place -> a_{n+1} (global, lane layout)
    // Row partition, fused halo (in-process slab handles, kpm_moments_group): the step kernel
    // itself stores its first / last local plane of a_{n+1} into the lower / upper neighbour's
    // ghost plane of the same block (peer memory; nullptr = exchanged separately).  plane_lanes:
    // lanes of one buffer plane; nloc: local planes (the last one is buffer plane nloc).
    double2* peer_lo;
    double2* peer_hi;
    long long plane_lanes;
    int nloc;
    // round-robin 3D schedule: pencils in Z (Morton) order when zbx, zby >= 0 (PX = 2^zbx, PY = 2^zby),
    // so the 148 columns of one wave form a compact block and their y-halo rows are the neighbours'
    // main tiles, loaded a moment earlier (L2 hits) -- in row-major order a wave is 2-3 pencil rows
    // wide and the y-halos of its edge rows came from DRAM again (ncu r01: c5 1.10x, c3 1.05x)
    int zbx, zby;
};

// (px, py) of pencil `code` in Z order: bits of x and y interleaved from the least significant
__device__ __forceinline__ void zdecode(int code, int bx, int by, int& px, int& py) {
    px = py = 0;
    int ix = 0, iy = 0, b = 0;
    while (ix < bx || iy < by) {
        if (ix < bx) px |= ((code >> b++) & 1) << ix++;
        if (iy < by) py |= ((code >> b++) & 1) << iy++;
    }
}

// a_{n+1} value y stored at `o` of buffer plane m: its copies in the neighbours' ghost planes
__device__ __forceinline__ void store_peers(const TmaGeom& g, int m, const double2* o, double2 y) {
    if (g.peer_lo == nullptr) return;
    const long long inpl = o - (g.out + (long long)m * g.plane_lanes);
    if (m == 1) __stcs(g.peer_lo + inpl, y);
    if (m == g.nloc) __stcs(g.peer_hi + inpl, y);
}

constexpr int kTmaConsumerWarps = 8;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;
#ifndef KPM_SA
#define KPM_SA 5
#endif
// a_{n-1} ring depth 4: c3 1093 vs 1132 ms per call with 3 (same-box A/B; a_n ring 6: no change, 4: slower)
#ifndef KPM_SP
#define KPM_SP 4
#endif
constexpr int kSA = KPM_SA;  // a_n ring slots
constexpr int kSP = KPM_SP;  // a_{n-1} ring slots

// Shared-memory carve-up of one a_n slot: [main TY*TX][left TY][right TY][top TX][bottom TX][eps TX*TY doubles],
// every region starting on a 128-byte boundary (TMA destinations; with TL = 4 lanes a 1-site halo
// column is only 64 bytes).
struct SlotLayout {
    int site_bytes, main_off, left_off, right_off, top_off, bot_off, eps_off, bytes;
    __host__ __device__ static int up(int x) { return (x + 127) / 128 * 128; }
    __host__ __device__ SlotLayout(int NDIM, int TX, int TY, int TL, bool onsite) {
        site_bytes = TL * 16;
        main_off = 0;
        left_off = up(main_off + TX * TY * site_bytes);
        right_off = up(left_off + TY * site_bytes);
        top_off = up(right_off + TY * site_bytes);
        bot_off = up(top_off + (NDIM == 3 ? TX * site_bytes : 0));
        eps_off = up(bot_off + (NDIM == 3 ? TX * site_bytes : 0));
        int end = eps_off + (onsite ? TX * TY * 8 : 0);
        bytes = up(end);
    }
};

// Work schedule.  A "column" is one (lane group, pencil) marched over all Lm planes.
//  * contiguous (rr == 0): CTA c owns output planes [W c/G, W (c+1)/G) of the
//    column-major plane order -- used when there are fewer columns than CTAs (2D);
//  * round-robin (rr == 1): CTA c owns whole columns c, c+G, c+2G, ...; all CTAs
//    march spatially adjacent pencils through the same planes at the same time, so
//    the in-plane halos one CTA loads are the main tiles its neighbours load a moment
//    earlier or later -- L2 hits instead of DRAM re-reads (3D).
struct Seg {
    int lg, px, py, m0, m1;  // lane group, pencil, planes [m0, m1)
};
struct Sched {
    long long w, w_end;  // contiguous: plane cursor; round-robin: column cursor / count
};
__device__ __forceinline__ Sched sched_begin(const TmaGeom& g) {
    Sched q;
    if (g.rr) {
        q.w = blockIdx.x;
        q.w_end = g.W / g.Lm;
    } else {
        q.w = g.W * blockIdx.x / gridDim.x;
        q.w_end = g.W * (blockIdx.x + 1) / gridDim.x;
    }
    return q;
}
__device__ __forceinline__ bool next_seg(const TmaGeom& g, Sched& q, Seg& s) {
    if (q.w >= q.w_end) return false;
    long long col;
    if (g.rr) {
        col = q.w;
        s.m0 = 0;
        s.m1 = g.Lm;
        q.w += gridDim.x;
    } else {
        col = q.w / g.Lm;
        s.m0 = (int)(q.w - col * g.Lm);
        const long long seg_end = min(q.w_end, (col + 1) * (long long)g.Lm);
        s.m1 = s.m0 + (int)(seg_end - q.w);
        q.w = seg_end;
    }
    const int pencil = (int)(col % ((long long)g.PX * g.PY));
    s.lg = (int)(col / ((long long)g.PX * g.PY));
    if (g.rr && g.zbx >= 0) {
        zdecode(pencil, g.zbx, g.zby, s.px, s.py);
    } else {
        s.px = pencil % g.PX;
        s.py = pencil / g.PX;
    }
    return true;
}

template <int NDIM, bool ONSITE, bool PEIERLS>
__global__ void __launch_bounds__(kTmaThreads, 1)
    kpm_step_tma_kernel(const __grid_constant__ CUtensorMap mapA,     // a_n: main box
                        const __grid_constant__ CUtensorMap mapCol,   // a_n: x-halo column box
                        const __grid_constant__ CUtensorMap mapRow,   // a_n: y-halo row box (3D)
                        const __grid_constant__ CUtensorMap mapP,     // a_{n-1}: main box
                        const __grid_constant__ CUtensorMap mapE,     // eps~: tile box
                        const TmaGeom g, const int tail) {
    pdl_entry();
    constexpr int CONS = kTmaConsumerWarps * 32;
    extern __shared__ __align__(128) unsigned char smem[];
    const SlotLayout SL(NDIM, g.TX, g.TY, g.TL, ONSITE);
    const int tile_bytes = g.TX * g.TY * g.TL * 16;
    unsigned char* ringA = smem;
    unsigned char* ringP = ringA + kSA * SL.bytes;
    double* sacc = reinterpret_cast<double*>(ringP + kSP * tile_bytes);     // [3][RP]
    double2* sred = reinterpret_cast<double2*>(sacc + 3 * g.RP);            // [3][CONS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sred + 3 * CONS);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + kSA;
    uint64_t* fullP = emptyA + kSA;
    uint64_t* emptyP = fullP + kSP;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSA; ++i) {
            mbar_init(fullA + i, 1);
            mbar_init(emptyA + i, kTmaConsumerWarps);
        }
        for (int i = 0; i < kSP; ++i) {
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
            prefetch_tmap(&mapA);
            prefetch_tmap(&mapCol);
            prefetch_tmap(&mapP);
            if (NDIM == 3) prefetch_tmap(&mapRow);
            if (ONSITE) prefetch_tmap(&mapE);
            const uint64_t pol_first = policy_evict_first();
            const uint32_t bytesA = tile_bytes + 2 * g.TY * SL.site_bytes + (NDIM == 3 ? 2 * g.TX * SL.site_bytes : 0) +
                                    (ONSITE ? g.TX * g.TY * 8 : 0);
            long long ia = 0, ip = 0;  // load counters
            Sched sq = sched_begin(g);
            Seg s;
            while (next_seg(g, sq, s)) {
                const int c0 = 2 * s.lg * g.TL;
                const int x0 = s.px * g.TX, y0 = s.py * g.TY;
                // padded x-rows (3D): the halo columns are the frame, never wrapped
                const int xm = x0 + g.xpad;
                const int xl = g.xpad ? xm - 1 : (x0 - 1 + g.L0) % g.L0;
                const int xr = g.xpad ? xm + g.TX : (x0 + g.TX) % g.L0;
                const int yt = (y0 - 1 + g.L1) % g.L1, yb = (y0 + g.TY) % g.L1;
                const int H = s.m1 - s.m0;
                for (int q = 0; q < H + 2; ++q) {
                    // buffer plane of march coordinate m0-1+q
                    const int m = g.ghost ? g.zoff + s.m0 + q : (s.m0 - 1 + q + g.Lm) % g.Lm;
                    const int slot = (int)(ia % kSA);
                    if (ia >= kSA) mbar_wait(emptyA + slot, (uint32_t)(((ia / kSA) - 1) & 1));
                    unsigned char* dst = ringA + slot * SL.bytes;
                    mbar_expect_tx(fullA + slot, bytesA);
                    if (NDIM == 2) {
                        tma_load(dst + SL.main_off, &mapA, fullA + slot, c0, x0, m);
                        tma_load(dst + SL.left_off, &mapCol, fullA + slot, c0, xl, m);
                        tma_load(dst + SL.right_off, &mapCol, fullA + slot, c0, xr, m);
                        if (ONSITE) tma_load_2d(dst + SL.eps_off, &mapE, fullA + slot, x0, m - g.ghost);
                    } else {
                        tma_load(dst + SL.main_off, &mapA, fullA + slot, c0, xm, y0, m);
                        tma_load(dst + SL.left_off, &mapCol, fullA + slot, c0, xl, y0, m);
                        tma_load(dst + SL.right_off, &mapCol, fullA + slot, c0, xr, y0, m);
                        tma_load(dst + SL.top_off, &mapRow, fullA + slot, c0, xm, yt, m);
                        tma_load(dst + SL.bot_off, &mapRow, fullA + slot, c0, xm, yb, m);
                        if (ONSITE) tma_load(dst + SL.eps_off, &mapE, fullA + slot, x0, y0, m - g.ghost);
                    }
                    ++ia;
                    // a_{n-1} for output plane q-1, issued right behind the a_n plane it pairs with
                    if (q >= 1 && q - 1 < H) {
                        const int mp = g.zoff + s.m0 + q - 1 + g.ghost;
                        const int ps = (int)(ip % kSP);
                        if (ip >= kSP) mbar_wait(emptyP + ps, (uint32_t)(((ip / kSP) - 1) & 1));
                        mbar_expect_tx(fullP + ps, tile_bytes);
                        if (NDIM == 2) tma_load_hint(ringP + ps * tile_bytes, &mapP, fullP + ps, c0, x0, mp, pol_first);
                        else tma_load_hint(ringP + ps * tile_bytes, &mapP, fullP + ps, c0, xm, y0, mp, pol_first);
                        ++ip;
                    }
                }
            }
        }
    } else {
        // ---------------------------------------------------------------- consumers
        const int t = threadIdx.x;                 // 0 .. CONS-1
        const int l = t % g.TL;                    // lane within the tile
        const int k0 = t / g.TL;                   // first tile site of this thread
        const int kstep = CONS / g.TL;
        const int npass = g.TX * g.TY / kstep;
        double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
        long long ia = 0, ip = 0;
        Sched sq = sched_begin(g);
        Seg s;
        int cur_lg = -1;
        auto flush = [&](int lg) {
            // fixed-order CTA reduction of the per-thread partials for lane group lg
            sred[t] = acc0;
            sred[CONS + t] = acc1;
            sred[2 * CONS + t] = acc2;
            named_bar_sync(1, CONS);
            if (t < g.TL) {
                for (int k = 0; k < 3; ++k) {
                    double2 sum = make_double2(0.0, 0.0);
                    for (int j = t; j < CONS; j += g.TL) sum = add2(sum, sred[k * CONS + j]);
                    const int v = lg * g.TL + t;  // lane index within the site
                    if (PEIERLS) {
                        sacc[k * g.RP + v] += sum.x;
                    } else {
                        sacc[k * g.RP + 2 * v] += sum.x;
                        sacc[k * g.RP + 2 * v + 1] += sum.y;
                    }
                }
            }
            named_bar_sync(1, CONS);
            acc0 = acc1 = acc2 = make_double2(0.0, 0.0);
        };
        while (next_seg(g, sq, s)) {
            if (cur_lg != -1 && s.lg != cur_lg) flush(cur_lg);
            cur_lg = s.lg;
            const int x0 = s.px * g.TX, y0 = s.py * g.TY;
            const int H = s.m1 - s.m0;
            const long long ia_seg = ia;  // load index of plane q = 0 of this segment
            for (int j = 0; j < H; ++j) {
                const long long i0 = ia_seg + j, i1 = i0 + 1, i2 = i0 + 2;
                mbar_wait(fullA + (int)(i0 % kSA), (uint32_t)((i0 / kSA) & 1));
                mbar_wait(fullA + (int)(i1 % kSA), (uint32_t)((i1 / kSA) & 1));
                mbar_wait(fullA + (int)(i2 % kSA), (uint32_t)((i2 / kSA) & 1));
                const int ps = (int)(ip % kSP);
                mbar_wait(fullP + ps, (uint32_t)((ip / kSP) & 1));
                const unsigned char* S0 = ringA + (int)(i0 % kSA) * SL.bytes;  // plane m-1
                const unsigned char* S1 = ringA + (int)(i1 % kSA) * SL.bytes;  // plane m
                const unsigned char* S2 = ringA + (int)(i2 % kSA) * SL.bytes;  // plane m+1
                const double2* Pv = reinterpret_cast<const double2*>(ringP + ps * tile_bytes);
                const int m = g.zoff + s.m0 + j + g.ghost;  // buffer plane of the output
                auto lane_at = [&](const unsigned char* base, int off, int site) {
                    return reinterpret_cast<const double2*>(base + off)[site * g.TL + l];
                };
#pragma unroll 4
                for (int pass = 0; pass < npass; ++pass) {
                    const int k = k0 + pass * kstep;  // tile site
                    const int lx = k % g.TX, ly = k / g.TX;
                    const double2 x = lane_at(S1, SL.main_off, k);
                    const double2 xm = lx > 0 ? lane_at(S1, SL.main_off, k - 1) : lane_at(S1, SL.left_off, ly);
                    const double2 xp = lx < g.TX - 1 ? lane_at(S1, SL.main_off, k + 1) : lane_at(S1, SL.right_off, ly);
                    double2 nb = add2(xm, xp);
                    const double2 mprev = lane_at(S0, SL.main_off, k);  // march-dim neighbour -1
                    const double2 mnext = lane_at(S2, SL.main_off, k);  // march-dim neighbour +1
                    if (NDIM == 2) {
                        if (PEIERLS) {
                            // y is the march dim: H[s][s+e_y] = t e^{-i theta_x}, H[s][s-e_y] = t e^{+i theta_x}
                            const double2 ph = __ldg(g.phase + x0 + lx);
                            nb = add2(nb, add2(cmulc(ph, mnext), cmul(ph, mprev)));
                        } else {
                            nb = add2(nb, add2(mprev, mnext));
                        }
                    } else {
                        const double2 ym = ly > 0 ? lane_at(S1, SL.main_off, k - g.TX) : lane_at(S1, SL.top_off, lx);
                        const double2 yp = ly < g.TY - 1 ? lane_at(S1, SL.main_off, k + g.TX) : lane_at(S1, SL.bot_off, lx);
                        nb = add2(nb, add2(add2(ym, yp), add2(mprev, mnext)));
                    }
                    const double e = ONSITE ? reinterpret_cast<const double*>(S1 + SL.eps_off)[k] : g.shift;
                    const double2 h = fma2(e, x, scale2(g.t, nb));
                    const double2 p = Pv[k * g.TL + l];
                    const double2 y = make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));  // Eq (18)
                    const int xs = x0 + lx;
                    const long long site = NDIM == 2 ? (long long)m * g.L0 + xs
                                                     : ((long long)m * g.L1 + (y0 + ly)) * (g.L0 + 2 * g.xpad) + xs + g.xpad;
                    double2* o = g.out + site * g.RG + s.lg * g.TL + l;
                    __stcs(o, y);
                    store_peers(g, m, o, y);
                    if (NDIM == 3 && g.xpad) {  // periodic x images in the frame
                        if (xs < g.xpad) {
                            __stcs(o + (long long)g.L0 * g.RG, y);
                            store_peers(g, m, o + (long long)g.L0 * g.RG, y);
                        }
                        if (xs >= g.L0 - g.xpad) {
                            __stcs(o - (long long)g.L0 * g.RG, y);
                            store_peers(g, m, o - (long long)g.L0 * g.RG, y);
                        }
                    }
                    dot_acc<PEIERLS>(acc0, x, x);
                    dot_acc<PEIERLS>(acc1, x, y);
                    if (tail) dot_acc<PEIERLS>(acc2, y, y);
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(emptyA + (int)(i0 % kSA));
                    mbar_arrive(emptyP + ps);
                }
                ++ip;
            }
            // release the last two a_n planes of the segment
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
    // one row of partial sums per CTA (fixed order)
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
