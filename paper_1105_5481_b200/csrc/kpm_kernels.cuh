// kpm_kernels.cuh -- sm_100a kernels of the KPM moment recursion.
//
// Hot path: one fused kernel per recursion step
//     a_{n+1} = 2 H~ a_n - a_{n-1}          (Eq 18)
// written over a_{n-1} in place, with the two inner products the doubling
// identities need, <a_n|a_n> and <a_n|a_{n+1}>, reduced from the values already
// in registers (per vector, per CTA; fixed order, no atomics).  The first-step
// kernel regenerates the Rademacher start block on the fly (Eq 14-15, 17).
//
// Data layout: the vector block is interleaved [site][vector] with the vector
// index fastest, handled as 16-byte lanes (double2): a real lane holds two
// vectors, a complex128 lane one vector.  One stencil/ELL entry is applied to all
// R vectors of a site by the threads of one warp, so a warp reads a contiguous
// run of 16-byte lanes (coalesced, 128-bit).  The matrix is never stored for
// lattices (StencilOp): hopping t~ = t/a and the rescaled on-site energies
// eps~_i = (eps_i - b)/a (Eq 8) are applied arithmetically.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "kpm_rng.cuh"

namespace kpm {

// ------------------------------------------------------------ programmatic dependent launch
// Every kernel of a kpm_moments call is launched with programmatic stream serialization (PDL,
// kpm_capi.cu launch_k): it lets the NEXT kernel of the chain launch as soon as every CTA of this
// one has started (griddepcontrol.launch_dependents), and each kernel waits for its predecessor's
// completion and memory flush (griddepcontrol.wait) before touching global memory.  The launch
// latency of step n+1 thus overlaps step n.  Both are no-ops for a kernel launched without PDL.
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------ lane arithmetic
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 scale2(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 fma2(double s, double2 a, double2 c) {
    return make_double2(fma(s, a.x, c.x), fma(s, a.y, c.y));
}
// complex p * z
__device__ __forceinline__ double2 cmul(double2 p, double2 z) {
    return make_double2(fma(p.x, z.x, -p.y * z.y), fma(p.x, z.y, p.y * z.x));
}
// complex conj(p) * z
__device__ __forceinline__ double2 cmulc(double2 p, double2 z) {
    return make_double2(fma(p.x, z.x, p.y * z.y), fma(p.x, z.y, -p.y * z.x));
}
// acc += Re <a|b> per vector: real lane = two vectors, complex lane = one vector
template <bool CPLX>
__device__ __forceinline__ void dot_acc(double2& acc, double2 a, double2 b) {
    if (CPLX) {
        acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
    } else {
        acc.x = fma(a.x, b.x, acc.x);
        acc.y = fma(a.y, b.y, acc.y);
    }
}

// ------------------------------------------------------------ CTA reductions
// Fixed-order CTA sum of a per-thread double2 over the threads that share a vector lane
// (lane = t % TL, TL a power of two; t = the linear thread index, threads t >= NT contribute
// nothing).  TL < 32: a shuffle tree inside each warp (offsets 16, 8, .., TL: thread t % 32 < TL
// ends up with its warp's partial of lane t % TL), then the NT / 32 warp partials in warp order;
// TL >= 32: the NT / TL partials of a lane in thread order.  The order depends only on (TL, NT),
// so repeated launches give identical bits.  Threads t < TL receive their lane's CTA total.  All
// threads of the block must call it (it holds two __syncthreads); scratch: >= NT double2 of shared
// memory.  (The former loop -- one thread per lane adding the NT / TL values serially -- cost up to
// 64 dependent shared-memory round trips per sum: ~1/4 of a launch for 4-lane tiles.)
template <int TL, int NT>
__device__ __forceinline__ double2 cta_lane_sum(double2 v, int t, double2* scratch) {
    static_assert(TL >= 1 && (TL & (TL - 1)) == 0 && NT % 32 == 0, "lanes a power of two, whole warps");
    double2 s = make_double2(0.0, 0.0);
    if (TL < 32) {
#pragma unroll
        for (int off = 16; off >= TL; off >>= 1) {
            v.x += __shfl_down_sync(0xffffffffu, v.x, off);
            v.y += __shfl_down_sync(0xffffffffu, v.y, off);
        }
        if (t < NT && (t & 31) < TL) scratch[(t >> 5) * TL + (t & 31)] = v;
        __syncthreads();
        if (t < TL)
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) s = add2(s, scratch[w * TL + t]);
    } else {
        if (t < NT) scratch[t] = v;
        __syncthreads();
        if (t < TL)
#pragma unroll
            for (int j = 0; j < NT / TL; ++j) s = add2(s, scratch[j * TL + t]);
    }
    __syncthreads();
    return s;
}
// The same with the lane count known only at run time (a power of two <= 32, NT a multiple of 32).
template <int NT>
__device__ __forceinline__ double2 cta_lane_sum_rt(double2 v, int t, int TL, double2* scratch) {
    switch (TL) {
        case 1: return cta_lane_sum<1, NT>(v, t, scratch);
        case 2: return cta_lane_sum<2, NT>(v, t, scratch);
        case 4: return cta_lane_sum<4, NT>(v, t, scratch);
        case 8: return cta_lane_sum<8, NT>(v, t, scratch);
        case 16: return cta_lane_sum<16, NT>(v, t, scratch);
        default: return cta_lane_sum<32, NT>(v, t, scratch);
    }
}

// ------------------------------------------------------------ operators H~
struct StencilGeom {
    int L0, L1, L2;          // extents (sites = L0*L1*L2; the slowest used extent is local under KPM_PART_ROWS)
    int plane;               // L0*L1
    int ghost;               // 1: the slowest dimension is a slab with a ghost plane on each side
                             //    (row partition): its neighbours are never wrapped
    double t;                // t / a
    double shift;            // -b / a   (used when there is no on-site array)
    const double* eps;       // (eps_i - b)/a per site, or nullptr
    const double2* phase;    // Peierls: e^{i 2 pi phi x}, x = 0..L0-1
};

// Nearest-neighbour periodic lattice in NDIM dims (readings X12-X15).
template <int NDIM, bool ONSITE, bool PEIERLS>
struct StencilOp {
    StencilGeom g;
    template <class XF>
    __device__ __forceinline__ double2 apply(int s, const XF& X, double2 xs) const {
        const int x = s % g.L0;
        const bool wx = NDIM > 1 || !g.ghost;  // 1D slab: x is the slab dimension
        const int xm = (x == 0 && wx) ? s + g.L0 - 1 : s - 1;
        const int xp = (x == g.L0 - 1 && wx) ? s - g.L0 + 1 : s + 1;
        double2 nb = add2(X(xm), X(xp));
        if (NDIM >= 2) {
            const int q = s / g.L0;
            const int y = (NDIM == 2) ? q : q % g.L1;
            const bool wy = NDIM > 2 || !g.ghost;  // 2D slab: y is the slab dimension
            const int ym = (y == 0 && wy) ? s + g.plane - g.L0 : s - g.L0;
            const int yp = (y == g.L1 - 1 && wy) ? s - g.plane + g.L0 : s + g.L0;
            if (PEIERLS) {
                // H[s][s+e_y] = t e^{-i theta_x}, H[s][s-e_y] = t e^{+i theta_x}
                const double2 ph = __ldg(g.phase + x);
                nb = add2(nb, add2(cmulc(ph, X(yp)), cmul(ph, X(ym))));
            } else {
                nb = add2(nb, add2(X(ym), X(yp)));
            }
            if (NDIM == 3) {
                const int z = q / g.L1;
                const int vol = g.plane * g.L2;
                const int zm = (z == 0 && !g.ghost) ? s + vol - g.plane : s - g.plane;
                const int zp = (z == g.L2 - 1 && !g.ghost) ? s - vol + g.plane : s + g.plane;
                nb = add2(nb, add2(X(zm), X(zp)));
            }
        }
        const double e = ONSITE ? __ldg(g.eps + s) : g.shift;
        return fma2(e, xs, scale2(g.t, nb));
    }
};

// General sparse H~ in ELL form, row-major: row i holds kp >= K entries (K rounded up to a multiple
// of 4: one 16-byte load brings 4 column indices) -- [rows][kp] arrays, values pre-scaled by 1/a, the
// -b/a shift applied separately.  Padding: col = row, val = 0.  A tile of consecutive rows is one
// contiguous run of both arrays (one bulk copy each into shared memory, kpm_ell.cuh).
template <bool CPLX>
struct EllOp {
    int D, K;
    const int* col;       // [rows][kp]
    const double* val;    // real: double[rows][kp]; complex: double2[rows][kp]
    double shift;         // -b / a
    int kp;               // entries per stored row (row stride)
    template <class XF>
    __device__ __forceinline__ double2 apply(int s, const XF& X, double2 xs) const {
        double2 h = scale2(shift, xs);
        // chunks of 8 entries: all column indices and values first, then all gathers, then the
        // sums -- 8 independent loads in flight instead of a load->gather->fma chain per entry
        constexpr int CH = 8;
        for (int k0 = 0; k0 < K; k0 += CH) {
            int j[CH];
            double2 v[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int k = k0 + u;
                const size_t e = (size_t)s * kp + (k < K ? k : K - 1);
                j[u] = __ldg(col + e);
                v[u] = CPLX ? __ldg(reinterpret_cast<const double2*>(val) + e) : make_double2(__ldg(val + e), 0.0);
                if (k >= K) v[u] = make_double2(0.0, 0.0);
            }
            double2 xj[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) xj[u] = X(j[u]);
#pragma unroll
            for (int u = 0; u < CH; ++u) h = CPLX ? add2(h, cmul(v[u], xj[u])) : fma2(v[u].x, xj[u], h);
        }
        return h;
    }
};

// ------------------------------------------------------------ the fused step
enum Mode { FIRST_GEN = 0, FIRST_BUF = 1, STEP = 2, DIRECT_GEN = 3, DIRECT_BUF = 4 };

struct VecArgs {
    double2* P;            // STEP: a_{n-1} in, a_{n+1} out; FIRST: a_0 (out for GEN, in for BUF)
    double2* C;            // STEP: a_n in; FIRST: a_1 out
    const double2* Rbuf;   // DIRECT_BUF: start block r in lane layout
    int D;                 // sites on this GPU
    int RG;                // lanes per site
    int RP;                // padded vectors per site (real: 2*RG, complex: RG)
    long long R_loc;       // real vectors on this GPU (<= RP)
    unsigned long long key;// vector_key(seed)
    long long r_off;       // global index of this GPU's first vector
    long long D_total;     // global number of sites (RNG counter stride)
    long long i_off;       // global index of this GPU's site 0
    const long long* sites;// KPM_LOCAL: global site of each global vector (unit start vectors e_site), else nullptr
    const long long* gmap; // ELL row partition: global index of ghost site D + k (k < n_ghost), else nullptr
    int ghost;             // row partition: site indices j < 0 or >= D are ghost sites (wrap globally)
    int L0;                // x extent
    int xpad;              // 3D lattices: 2 -- vector blocks store each x-row with a 2-site frame of
                           // periodic images on both sides (row pitch L0 + 4); 0 otherwise
    // memory site of lattice site j (j may index a ghost plane, i.e. be < 0 or >= D)
    __device__ __forceinline__ long long mem(long long j) const {
        if (!xpad) return j;
        const long long row = j >= 0 ? j / L0 : -((-j + L0 - 1) / L0);
        return j + 2 * xpad * row + xpad;
    }
    double* red0;          // partial sums of moment slot 0: [gridDim.x][RP] (nullable)
    double* red1;          // slot 1
    double* red2;          // slot 2 (odd-N tail <a_{n+1}|a_{n+1}>)
};

// Store the lane of lattice site s (memory site ms), plus its periodic x images in the frame
// when s is within xpad sites of an x boundary (both images when L0 < 2 xpad).
__device__ __forceinline__ void store_site(const VecArgs& v, double2* buf, int s, long long ms, int rg, double2 val,
                                           bool streaming) {
    auto st = [&](long long m) {
        double2* p = buf + m * v.RG + rg;
        if (streaming) __stcs(p, val);
        else *p = val;
    };
    st(ms);
    if (v.xpad) {
        const int x = s % v.L0;
        if (x < v.xpad) st(ms + v.L0);
        if (x >= v.L0 - v.xpad) st(ms - v.L0);
    }
}

template <bool CPLX>
__device__ __forceinline__ double2 gen_lane(const VecArgs& v, int j, int rg) {
    long long ig = v.i_off + j;
    if (v.gmap) {
        if (j >= v.D) ig = __ldg(v.gmap + (j - v.D));  // ghost site of a general sparse row partition
    } else if (v.ghost) {
        ig = (ig % v.D_total + v.D_total) % v.D_total;  // ghost plane of a neighbouring slab
    }
    if (v.sites) {  // unit start vectors |r> = e_{site(r)} (local DoS)
        auto unit = [&](long long r) { return (r < v.R_loc && __ldg(v.sites + v.r_off + r) == ig) ? 1.0 : 0.0; };
        return CPLX ? make_double2(unit(rg), 0.0) : make_double2(unit(2LL * rg), unit(2LL * rg + 1));
    }
    const uint64_t i = (uint64_t)ig;
    if (CPLX) {
        const long long r = rg;
        return make_double2(r < v.R_loc ? rademacher(v.key, (uint64_t)(v.r_off + r) * v.D_total + i) : 0.0, 0.0);
    } else {
        const long long r = 2LL * rg;
        const double x0 = r < v.R_loc ? rademacher(v.key, (uint64_t)(v.r_off + r) * v.D_total + i) : 0.0;
        const double x1 = r + 1 < v.R_loc ? rademacher(v.key, (uint64_t)(v.r_off + r + 1) * v.D_total + i) : 0.0;
        return make_double2(x0, x1);
    }
}

// Block = (TR lanes) x (TS sites); grid = (site CTAs) x (lane groups).
// Sites are visited grid-stride so that, at any moment, all CTAs sweep one compact
// window of the lattice and the neighbour planes they re-read stay in L2; the
// a_{n-1} read and a_{n+1} write are cache-streaming (evict-first) so they do not
// displace those planes.
//
// PERSIST (the L2-resident persistent kernel, kpm_persist.cuh): vector blocks change during the
// kernel, so they are read through L2 only (ld.global.cg) -- the non-coherent L1 path of __ldg
// could return a value another SM overwrote in an earlier step.
template <bool PERSIST>
__device__ __forceinline__ double2 ld_vec(const double2* p) {
    return PERSIST ? __ldcg(p) : __ldg(p);
}
template <class OP, int MODE, bool CPLX, bool PERSIST = false>
__device__ __forceinline__ void step_body(const OP& op, const VecArgs& v, const int tail) {
    const int TR = blockDim.x, TS = blockDim.y;
    const int rg = blockIdx.y * TR + threadIdx.x;
    const bool active = rg < v.RG;
    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0;
    if (active) {
        for (int s = blockIdx.x * TS + threadIdx.y; s < v.D; s += gridDim.x * TS) {
            const long long ms = v.mem(s);
            const size_t idx = (size_t)ms * v.RG + rg;
            if (MODE == FIRST_GEN) {
                auto X = [&](int j) { return gen_lane<CPLX>(v, j, rg); };
                const double2 x = X(s);
                const double2 y = op.apply(s, X, x);   // a_1 = H~ a_0   (Eq 17)
                store_site(v, v.P, s, ms, rg, x, false);
                store_site(v, v.C, s, ms, rg, y, false);
                dot_acc<CPLX>(acc0, x, x);
                dot_acc<CPLX>(acc1, x, y);
                if (tail) dot_acc<CPLX>(acc2, y, y);
            } else if (MODE == FIRST_BUF) {
                auto X = [&](int j) { return ld_vec<PERSIST>(v.P + (size_t)v.mem(j) * v.RG + rg); };
                const double2 x = X(s);
                const double2 y = op.apply(s, X, x);
                store_site(v, v.C, s, ms, rg, y, false);
                dot_acc<CPLX>(acc0, x, x);
                dot_acc<CPLX>(acc1, x, y);
                if (tail) dot_acc<CPLX>(acc2, y, y);
            } else {
                auto X = [&](int j) { return ld_vec<PERSIST>(v.C + (size_t)v.mem(j) * v.RG + rg); };
                const double2 x = X(s);
                const double2 h = op.apply(s, X, x);
                const double2 p = PERSIST ? __ldcg(v.P + idx) : __ldcs(v.P + idx);
                const double2 y = make_double2(fma(2.0, h.x, -p.x), fma(2.0, h.y, -p.y));  // Eq 18
                store_site(v, v.P, s, ms, rg, y, !PERSIST);
                if (MODE == STEP) {
                    dot_acc<CPLX>(acc0, x, x);
                    dot_acc<CPLX>(acc1, x, y);
                    if (tail) dot_acc<CPLX>(acc2, y, y);
                } else if (MODE == DIRECT_GEN) {
                    dot_acc<CPLX>(acc0, gen_lane<CPLX>(v, s, rg), y);   // <r|a_{n+1}>  (Eq 19)
                } else {
                    dot_acc<CPLX>(acc0, __ldcs(v.Rbuf + idx), y);
                }
            }
        }
    }
    // CTA-level finish of the per-vector partial sums, fixed order over the TS site rows.
    // (blocks of 512 threads = TR lanes x TS site rows, TR a power of two <= 32; cta_lane_sum)
    extern __shared__ double2 sred[];
    const int tid = threadIdx.y * TR + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double* rowk = k == 0 ? v.red0 : (k == 1 ? v.red1 : (tail ? v.red2 : nullptr));
        if (rowk == nullptr) continue;  // (uniform over the CTA)
        const double2 s = cta_lane_sum_rt<512>(k == 0 ? acc0 : (k == 1 ? acc1 : acc2), tid, TR, sred);
        if (threadIdx.y == 0 && active) {
            double* row = rowk + (size_t)blockIdx.x * v.RP;
            if (CPLX) {
                row[rg] = s.x;
            } else {
                row[2 * rg] = s.x;
                row[2 * rg + 1] = s.y;
            }
        }
    }
}

template <class OP, int MODE, bool CPLX>
__global__ void __launch_bounds__(512) kpm_step_kernel(const OP op, const VecArgs v, const int tail) {
    pdl_entry();
    step_body<OP, MODE, CPLX>(op, v, tail);
}

// ------------------------------------------------------------ helpers
// Caller start vectors, vector-major [R_loc][D] real -> lane layout [D][RG] (memory sites of v).
template <bool CPLX>
__global__ void load_r0_kernel(const double* __restrict__ r0, double2* __restrict__ out, const VecArgs v) {
    pdl_entry();
    const int D = v.D, RG = v.RG;
    const long long R_loc = v.R_loc;
    const long long n = (long long)D * RG;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(e / RG), rg = (int)(e % RG);
        double2 val;
        if (CPLX) {
            val = make_double2(rg < R_loc ? r0[(size_t)rg * D + s] : 0.0, 0.0);
        } else {
            const long long r = 2LL * rg;
            val = make_double2(r < R_loc ? r0[(size_t)r * D + s] : 0.0, r + 1 < R_loc ? r0[(size_t)(r + 1) * D + s] : 0.0);
        }
        store_site(v, out, s, v.mem(s), rg, val, false);
    }
}

// Eq (8) on the diagonal, in place: eps~_i = (eps_i - b) / a (kpm_create_stencil).
__global__ void rescale_onsite_kernel(double* __restrict__ e, long long n, double b, double a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        e[i] = (e[i] - b) / a;
}

// dst[k][l] = src[idx[k]][l] over n sites of RG 16-byte lanes (row-partition ghost exchange).
__global__ void gather_lanes_kernel(const double2* __restrict__ src, const int* __restrict__ idx, long long n, int RG,
                                    double2* __restrict__ dst) {
    pdl_entry();
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * RG; e += (long long)gridDim.x * blockDim.x) {
        const long long k = e / RG;
        dst[e] = src[(long long)__ldg(idx + k) * RG + (e - k * RG)];
    }
}

// Sum the CTA partials of every moment slot in a fixed order:
// Sv[m][v] = sum_c partial[m][c][v] (per vector), S[m] = sum_v Sv[m][v].
// One block per slot m; its threads form CG groups x VB vector lanes (VB = the power of two >= R_loc,
// at most 32): group g sums the CTA rows c = g, g + CG, ... of vectors v0 + lane, then the groups are
// combined by a fixed shared-memory tree.  The partition depends only on (nCTA, R_loc), so repeated
// calls give identical bits.  (One thread per vector summing all CTA rows serially took 90 us per
// call at R_loc = 8 on c2.)
__global__ void finish_kernel(const double* __restrict__ partial, int nCTA, int RP, long long R_loc,
                              double* __restrict__ Sv, double* __restrict__ S) {
    pdl_entry();
    const int m = blockIdx.x;
    const double* base = partial + (size_t)m * nCTA * RP;
    int VB = 1;
    while (VB < R_loc && VB < 32) VB <<= 1;
    const int CG = blockDim.x / VB;
    const int lane = threadIdx.x % VB, grp = threadIdx.x / VB;
    __shared__ double red[256];
    double total = 0.0;  // thread 0: sum over v in order of chunks
    for (long long v0 = 0; v0 < R_loc; v0 += VB) {
        const long long v = v0 + lane;
        double s = 0.0;
        if (v < R_loc && grp < CG)
            for (int c = grp; c < nCTA; c += CG) s += base[(size_t)c * RP + v];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = CG / 2; w > 0; w >>= 1) {  // fixed tree over the groups
            if (grp < w) red[threadIdx.x] += red[threadIdx.x + w * VB];
            __syncthreads();
        }
        if (threadIdx.x < VB && v < R_loc) Sv[(size_t)m * R_loc + v] = red[threadIdx.x];
        if (threadIdx.x == 0)
            for (int j = 0; j < VB && v0 + j < R_loc; ++j) total += red[j];
        __syncthreads();
    }
    if (threadIdx.x == 0) S[m] = total;
}

// Doubling transform + normalisation (north_star; Eq 19 for direct):
// mu_0 = S_0 c, mu_1 = S_1 c, mu_{2n} = 2 S_{2n} c - mu_0, mu_{2n+1} = 2 S_{2n+1} c - mu_1.
// (explicitly rounded ops: no FMA contraction, so the host path of kpm_assemble gives the same bits)
__device__ __forceinline__ double assemble_one(const double* S, long long stride, int n, double c, int direct) {
    const double x = __dmul_rn(S[(size_t)n * stride], c);
    if (direct || n < 2) return x;
    return __dsub_rn(__dmul_rn(2.0, x), __dmul_rn((n & 1) ? S[stride] : S[0], c));
}

__global__ void assemble_kernel(const double* __restrict__ S, int N, double c, int direct, double* __restrict__ mu) {
    pdl_entry();
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) mu[n] = assemble_one(S, 1, n, c, direct);
}

// Per-vector moments: pv[v][n] from Sv[n][v].
__global__ void assemble_pervec_kernel(const double* __restrict__ Sv, int N, long long R_loc, double c, int direct,
                                       double* __restrict__ pv) {
    pdl_entry();
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= (long long)N * R_loc) return;
    const long long v = e / N;
    const int n = (int)(e % N);
    pv[e] = assemble_one(Sv + v, R_loc, n, c, direct);
}

// ------------------------------------------------------------ DoS (Eq 6), Green's function
// Damping factors g_n of Eq (6) (X8, X26):
//   0 Jackson, 1 none (g = 1), 2 Lorentz sinh(lam (1 - n/N)) / sinh(lam), 3 Fejer 1 - n/N.
__device__ __forceinline__ double damping(int n, int N, int kernel, double lam) {
    if (kernel == 0) {
        const double q = CUDART_PI / (N + 1);
        double sn, cn;
        sincospi((double)n / (N + 1), &sn, &cn);
        return ((N - n + 1) * cn + sn * (cos(q) / sin(q))) / (N + 1);
    }
    if (kernel == 2) return sinh(lam * (1.0 - (double)n / N)) / sinh(lam);
    if (kernel == 3) return 1.0 - (double)n / N;
    return 1.0;
}

// c_n = g_n mu_n (n = 0), 2 g_n mu_n (n >= 1); mu == nullptr gives g_n itself.
__global__ void dos_coeff_kernel(const double* __restrict__ mu, int N, int kernel, double lam, double* __restrict__ c) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const double g = damping(n, N, kernel, lam);
    c[n] = mu ? (n == 0 ? 1.0 : 2.0) * g * mu[n] : g;
}

// Statistics of the per-vector moments mu_n^(r) (KPM_PER_VECTOR, layout [R][N]): the
// sample mean over r (the estimate of Eq 16) and its standard error
// sqrt(sum_r (mu_n^(r) - mean_n)^2 / ((R - 1) R)), two passes in fp64 (X28).
// One thread per n; consecutive threads read consecutive n of one vector (coalesced).
__global__ void moment_stats_kernel(const double* __restrict__ pv, long long R, int N, double* __restrict__ mean,
                                    double* __restrict__ sem) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    double s = 0.0;
    for (long long r = 0; r < R; ++r) s += pv[r * N + n];
    const double m = s / (double)R;
    double q = 0.0;
    for (long long r = 0; r < R; ++r) {
        const double d = pv[r * N + n] - m;
        q = fma(d, d, q);
    }
    mean[n] = m;
    sem[n] = R > 1 ? sqrt(q / ((double)(R - 1) * (double)R)) : CUDART_NAN;
}

// rho(omega) = sum_n c_n T_n(x) / (pi a sqrt(1 - x^2)), x = (omega - b)/a, with
// T_n(x) = cos(n theta), theta = arccos x (Eq 3) evaluated term by term.  (The three-term
// recurrence, Eq 4-5, propagates a rounding error like n^2 eps near x = +-1 -- 1.8e-9 at
// n = 4096 -- while cos(n theta) errs by about n theta eps; X27.)  One thread per energy.
__global__ void dos_kernel(const double* __restrict__ c, int N, double a, double b, const double* __restrict__ omega,
                           long long K, double* __restrict__ rho) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= K) return;
    const double x = (omega[k] - b) / a;
    if (!(fabs(x) < 1.0)) {
        rho[k] = 0.0;
        return;
    }
    const double th = acos(x);
    double s = c[0];
    for (int n = 1; n < N; ++n) s = fma(c[n], cos((double)n * th), s);
    // x^2 explicitly rounded (no FMA contraction into 1 - x^2): the same bits as the oracle, whose
    // numpy arithmetic rounds x * x first -- near |x| = 1 the two roundings of 1 - x^2 differ relatively
    // by eps / (1 - x^2), far above the expansion's own error (X27)
    rho[k] = s / (CUDART_PI * a * sqrt(1.0 - __dmul_rn(x, x)));
}

// Retarded G(omega) = G~(x)/a (X24).  Inside (|x| < 1), theta = arccos x:
//   G~ = -i sum_n c_n e^{-i n theta} / sin(theta)
//   Re G~ = -sum_{n>=1} c_n sin(n theta) / sin(theta),  Im G~ = -sum_n c_n cos(n theta) / sin(theta)
// (term by term, as dos_kernel).  Outside: G~ = sum_n c_n t^n / (sgn(x) sqrt(x^2 - 1)),
// t = x - sgn(x) sqrt(x^2 - 1), |t| < 1 (Horner).  |x| = 1: NaN.  G is [K][2] (re, im).
__global__ void green_kernel(const double* __restrict__ c, int N, double a, double b, const double* __restrict__ omega,
                             long long K, double* __restrict__ G) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= K) return;
    const double x = (omega[k] - b) / a;
    double re, im;
    if (fabs(x) < 1.0) {
        const double th = acos(x);
        double sc = c[0], ss = 0.0;
        for (int n = 1; n < N; ++n) {
            double sn, cn;
            sincos((double)n * th, &sn, &cn);
            sc = fma(c[n], cn, sc);
            ss = fma(c[n], sn, ss);
        }
        const double st = sin(th);  // sin(arccos x), as the oracle
        re = -ss / st;
        im = -sc / st;
    } else if (fabs(x) > 1.0) {
        const double sg = x > 0 ? 1.0 : -1.0;
        const double sq = sqrt(__dmul_rn(x, x) - 1.0);  // x^2 rounded first, as the oracle (see dos_kernel)
        const double t = x - sg * sq;
        double s = 0.0;
        for (int n = N - 1; n >= 0; --n) s = fma(s, t, c[n]);
        re = s / (sg * sq);
        im = 0.0;
    } else {
        re = im = CUDART_NAN;
    }
    G[2 * k] = re / a;
    G[2 * k + 1] = im / a;
}

}  // namespace kpm
