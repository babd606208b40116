// kpm_capi.cu -- host side of the C ABI declared in include/kpm.h.
//
// Owns: validation, the upload of H~ (Eq 8), the device workspace plan, the
// launch sequence of one kpm_moments call (first step, M-1 fused steps, finish,
// assembly) and error reporting.  All arithmetic of the method runs in the
// kernels of kpm_kernels.cuh; this file only marshals.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/kpm.h"
#include "kpm_kernels.cuh"
#include "kpm_tma.cuh"
#include "kpm_tma2.cuh"
#include "kpm_tma3.cuh"
#include "kpm_tri.cuh"
#include "kpm_quad.cuh"
// Kernels that are parity-green but measured slower than the default plan:
// their templates are instantiated (launched) only under KPM_EXPERIMENTAL, i.e. in libkpm_exp.so,
// and reached through kpm_plan_opts.experimental.  The default libkpm.so contains none of them.
#include "kpm_tmak.cuh"
#include "kpm_tma32.cuh"
#include "kpm_persist.cuh"
#include "kpm_ell.cuh"
#include "kpm_first.cuh"
#include "kpm_small.cuh"
#include "kpm_dense.cuh"

namespace {

thread_local std::string g_err;

kpm_status fail(kpm_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define KPM_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(KPM_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                        cudaGetErrorString(e_));                                              \
    } while (0)

#define KPM_TRY(expr)                        \
    do {                                     \
        kpm_status s_ = (expr);              \
        if (s_ != KPM_OK) return s_;         \
    } while (0)

struct IpcComm;  // kpm_ipc.cuh (KPM_COMM_IPC)

enum Kind { KIND_STENCIL = 0, KIND_ELL = 1, KIND_DENSE = 2 };
constexpr int kThreads = 512;     // threads per CTA of the step kernels
constexpr size_t kAlign = 256;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

}  // namespace

struct kpm_handle_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int kind = KIND_STENCIL;
    int dtype = KPM_REAL64;
    double a = 1.0, b = 0.0;
    int64_t D = 0;
    // stencil
    int ndim = 1;
    int64_t L[3] = {1, 1, 1};
    double t_scaled = 0.0;
    double* d_eps = nullptr;      // (eps_i - b)/a
    double* d_epsf = nullptr;     // 3D: the same in the x-row frame layout [L2][L1][L0+4] (kpm_tma32.cuh)
    double2* d_phase = nullptr;   // e^{i 2 pi phi x}
    // ELL
    int K = 0;
    int32_t* d_col = nullptr;     // [ell_ld rows][ell_kp] (row-major)
    double* d_val = nullptr;      // [ell_ld rows][ell_kp] (x2 for complex)
    int64_t ell_ld = 0;           // stored rows: D rounded up to 2048 (whole tiles)
    int ell_kp = 0;               // stored entries per row: K rounded up to a multiple of 4
    // dense H~ (the paper's variant): Dp x Dp row-major, H / a, zero padded (kpm_dense.cuh)
    double* d_dense = nullptr;
    int64_t Dp = 0;
    // partition
    kpm_dist dist{KPM_PART_NONE, 0, 1, KPM_COMM_SELF, nullptr};
    // row partition (KPM_PART_ROWS): slab [z0, z0 + nloc) of the slowest dimension `slow`;
    // vector blocks hold nloc + 2 planes (ghost, local..., ghost); D counts local sites
    bool rows = false;
    int slow = 0;
    int64_t z0 = 0, nloc = 0, Lm_global = 0, plane = 1;
    int64_t D_total = 0;  // global number of sites (normalisation, RNG counters)
    // row partition of a general sparse H (KIND_ELL): local rows [z0, z0 + D),
    // then n_ghost ghost sites (the off-block columns the local rows reference, ascending global index,
    // hence grouped by owner rank).  ELL columns index that extended block.
    int64_t n_ghost = 0, n_send = 0;
    long long* d_gmap = nullptr;     // [n_ghost] global index of each ghost site (RNG counters of a_0)
    int32_t* d_ghost_src = nullptr;  // [n_ghost] row of the ghost inside its owner's block (in-process groups)
    int32_t* d_send = nullptr;       // [n_send] local rows the other ranks need, peer by peer, ascending
    std::vector<int64_t> roff, rcnt, soff, scnt;  // per peer: ghost / send list offsets and counts
    ncclComm_t nccl = nullptr;
    IpcComm* ipc = nullptr;  // KPM_COMM_IPC: shared segment, launch events, mapped peer workspaces
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    bool ws_own = true;
    // device facts
    int num_sms = 148;
    int l2_bytes = 0;
    // timing of the last call
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    // row partition, overlapped halo exchange: a second stream and two events (created on demand)
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_bnd = nullptr, ev_comm = nullptr;
    int step_launches = 0, total_launches = 0;
    int halo_copies = 0, fused_halo_launches = 0;  // row partition: plane copies / launches storing into peers
    double steps_bytes = 0.0;   // SURVEY.md 8(d) algorithmic bytes of the recursion steps of the last call
    double design_bytes = 0.0;  // compulsory DRAM bytes of the kernels that ran (each array once per launch)
    int smem_optin = 227 * 1024;  // cudaDevAttrMaxSharedMemoryPerBlockOptin
    kpm_plan_opts opts{};         // kpm_set_plan_opts (zero = default plan)
    bool dead = false;            // an NCCL failure aborted the communicator
};

namespace {

struct Plan {
    int N = 0, M = 0;
    long long R_loc = 0, r_off = 0;
    int RG = 0, RP = 0;
    int TR = 0, TS = 0, gx = 0, gy = 0;
    int nslots = 0;      // moment slots = N
    // TMA-pipelined step kernel (2D/3D stencils), see kpm_tma.cuh
    bool use_tma = false;
    int TL = 0, TX = 0, TY = 0, tma_grid = 0, tma_rr = 0;
    // row partition: boundary planes first, halo exchange on a comm stream while the interior
    // planes compute; partial rows [0, G) interior, [G, 2G) and [2G, 3G) boundary
    bool overlap = false;
    // 3D: dense halo box + z rolled in registers (kpm_tma3.cuh) for the instantiated tiles
    bool use_tma3 = false;
    size_t tma_smem = 0;
    // two steps per launch (temporal blocking, 2D), see kpm_tma2.cuh; needs 4 vector blocks
    bool use_tma2 = false, no_fused = false;
    size_t tma2_smem = 0;
    int TX2 = 0, tma2_minb = 1, tma2_grid = 0;  // two-step tile width, CTAs per SM, grid
    // three steps per launch (kpm_tri.cuh), same tile as the two-step kernel; needs 4 vector blocks
    bool use_tri = false;
    size_t tri_smem = 0;
    // four steps per launch (kpm_quad.cuh): its own tile, TLQ lanes x TXQ sites (512 lanes)
    bool use_quad = false;
    int TLQ = 0, TXQ = 0, quad_grid = 0;
    size_t quad_smem = 0;
    // two steps per launch for 3D lattices (kpm_tma32.cuh); needs 4 vector blocks
    bool use_tma32 = false;
    int TX32 = 0, TY32 = 0, TL32 = 0, tma32_grid = 0, tma32_rr = 0;
    size_t tma32_smem = 0;
    // KS steps per launch (deep temporal blocking, 2D), see kpm_tmak.cuh; needs 4 vector blocks
    bool use_tmak = false;
    int KSK = 0, TLK = 0, TXK = 0, tmak_grid = 0;
    size_t tmak_smem = 0;
    // whole recursion in one cooperative launch with the vector blocks L2-resident (kpm_persist.cuh)
    bool use_persist = false;
    // whole recursion in one launch with the vector blocks in shared memory (kpm_small.cuh)
    bool use_small = false;
    size_t small_smem = 0;
    size_t lane_bytes = 0;
    size_t ghost_lanes = 0;  // lanes of one ghost plane (row partition), else 0
    int xpad = 0;            // 3D stencils: x-row frame of periodic images (row pitch L0 + 2 xpad)
    size_t mem_sites = 0;    // memory sites of the local block (with frames, without ghost planes)
    size_t off_P = 0, off_C = 0, off_R = 0, off_X2 = 0, off_X3 = 0, off_part = 0, off_Sv = 0, off_S = 0, off_out = 0,
           off_sites = 0, off_send = 0, total = 0;
};

bool is_cplx(const kpm_handle_s* h) { return h->dtype == KPM_COMPLEX128; }

// ---- NCCL: the handle's communicator (KPM_COMM_NCCL), failures -> KPM_ERR_NCCL
//
// Communicators are shared: handles created from the same (ncclUniqueId, rank, world, device)
// reuse one ncclComm_t (reference counted), so creating a handle per call -- the end-to-end
// pattern, H uploaded every time -- does not pay ncclCommInitRank every time.
struct CommEntry {
    ncclComm_t comm = nullptr;
    int refs = 0;
    bool aborted = false;
};
std::mutex g_comm_mu;
std::map<std::string, CommEntry> g_comms;  // key: id bytes + rank/world/device
std::map<ncclComm_t, std::string> g_comm_key;

void comm_release(ncclComm_t c, bool abort) {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto k = g_comm_key.find(c);
    if (k == g_comm_key.end()) return;
    CommEntry& e = g_comms[k->second];
    if (abort && !e.aborted) {
        ncclCommAbort(c);  // release the peers that wait on this rank
        e.aborted = true;
    }
    if (--e.refs == 0) {
        if (!e.aborted) ncclCommDestroy(c);
        g_comms.erase(k->second);
        g_comm_key.erase(k);
    }
}

kpm_status nccl_fail(kpm_handle_s* h, ncclResult_t e, const char* what) {
    if (h->nccl) comm_release(h->nccl, true);
    h->nccl = nullptr;
    h->dead = true;
    return fail(KPM_ERR_NCCL, "%s: %s", what, ncclGetErrorString(e));
}
#define KPM_NCCL(h, call, what)                                  \
    do {                                                         \
        ncclResult_t e_ = (call);                                \
        if (e_ != ncclSuccess) return nccl_fail((h), e_, (what)); \
    } while (0)

// Asynchronous errors (a peer that died, a transport fault) surface only through
// ncclCommGetAsyncError; an in-flight collective would otherwise block the stream forever.
kpm_status nccl_poll(kpm_handle_s* h) {
    if (!h->nccl) return KPM_OK;
    ncclResult_t ae = ncclSuccess;
    KPM_NCCL(h, ncclCommGetAsyncError(h->nccl, &ae), "ncclCommGetAsyncError");
    if (ae != ncclSuccess && ae != ncclInProgress) return nccl_fail(h, ae, "asynchronous NCCL error");
    return KPM_OK;
}

}  // namespace
#include "kpm_ipc.cuh"
namespace {

// Wait for the handle's stream; with a communicator, poll its error state while waiting.
kpm_status sync_stream(kpm_handle_s* h) {
    if (!h->nccl) {
        KPM_CUDA(cudaStreamSynchronize(h->stream));
        return KPM_OK;
    }
    for (;;) {
        const cudaError_t q = cudaStreamQuery(h->stream);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) KPM_CUDA(q);
        KPM_TRY(nccl_poll(h));
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    return nccl_poll(h);
}

// One kernel of the kpm_moments chain on stream st, with programmatic stream serialization (PDL)
// unless the plan switches it off: the kernel may launch while its predecessor in the stream is
// still running and waits for it in pdl_entry() (kpm_kernels.cuh) before touching global memory.
template <class... Exp, class... Act>
kpm_status launch_k(kpm_handle_s* h, cudaStream_t st, void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem,
                    Act&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = h->opts.no_pdl ? 0 : 1;
    KPM_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...));
    h->total_launches++;
    return KPM_OK;
}

// Communicator of a KPM_COMM_NCCL partition, from the caller's broadcast ncclUniqueId (shared
// with earlier handles of the same id, rank, world and device).
kpm_status init_comm(kpm_handle_s* h, const kpm_dist* dist) {
    if (!dist || dist->partition == KPM_PART_NONE || dist->comm != KPM_COMM_NCCL) return KPM_OK;
    ncclUniqueId id;
    memcpy(&id, dist->nccl_id, sizeof id);
    std::string key(reinterpret_cast<const char*>(&id), sizeof id);
    char tail[64];
    snprintf(tail, sizeof tail, "/%d/%d/%d", dist->rank, dist->world, h->device);
    key += tail;
    KPM_CUDA(cudaSetDevice(h->device));
    std::lock_guard<std::mutex> lk(g_comm_mu);
    CommEntry& e = g_comms[key];
    if (e.aborted) return fail(KPM_ERR_NCCL, "the communicator of this nccl_id was aborted by an earlier failure");
    if (!e.comm) {
        const ncclResult_t r = ncclCommInitRank(&e.comm, dist->world, id, dist->rank);
        if (r != ncclSuccess) {
            g_comms.erase(key);
            return fail(KPM_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
        }
        g_comm_key[e.comm] = key;
    }
    e.refs++;
    h->nccl = e.comm;
    return KPM_OK;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting: remember, per (kernel,
// device), the largest size already set.  Thread-safe (handles may live on several threads/devices).
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, size_t> g_attr;
kpm_status set_smem(const void* kern, size_t smem, int device) {
    // (raised for any request above 32 KB: the 48 KB default covers dynamic AND static shared memory,
    // so a dynamic request of exactly 48 KB plus a kernel's static barriers failed to launch)
    if (smem <= 32 * 1024) return KPM_OK;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& done = g_attr[{kern, device}];
    if (done >= smem) return KPM_OK;
    KPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done = smem;
    return KPM_OK;
}

#ifdef KPM_EXPERIMENTAL
// Shared memory of the instantiated KS-step kernels (0 = not instantiated).
size_t stepk_smem(int ks, int tl, bool onsite, int RP) {
    using namespace kpm;
    if (ks == 4 && tl == 16) return onsite ? stepk_smem_bytes<4, 16, 32, true>(RP) : stepk_smem_bytes<4, 16, 32, false>(RP);
    if (ks == 4 && tl == 8) return onsite ? stepk_smem_bytes<4, 8, 64, true>(RP) : stepk_smem_bytes<4, 8, 64, false>(RP);
    if (ks == 3 && tl == 16) return onsite ? stepk_smem_bytes<3, 16, 32, true>(RP) : stepk_smem_bytes<3, 16, 32, false>(RP);
    if (ks == 3 && tl == 8) return onsite ? stepk_smem_bytes<3, 8, 64, true>(RP) : stepk_smem_bytes<3, 8, 64, false>(RP);
    return 0;
}

// Shared memory of the instantiated 3D two-step kernels (0 = not instantiated); KA, KP ring depths.
constexpr int kKA32 = 5, kKP32 = 4;
size_t step32_smem(int tx, int ty, int tl, bool onsite, int RP) {
    using namespace kpm;
    constexpr int NT = 512, KA = kKA32, KP = kKP32;  // (NT only sizes the reduction scratch)
    if (tx == 8 && ty == 8 && tl == 8)
        return onsite ? step32_smem_bytes<8, 8, 8, true, NT, KA, KP>(RP) : step32_smem_bytes<8, 8, 8, false, NT, KA, KP>(RP);
    if (tx == 16 && ty == 4 && tl == 8)
        return onsite ? step32_smem_bytes<16, 4, 8, true, NT, KA, KP>(RP) : step32_smem_bytes<16, 4, 8, false, NT, KA, KP>(RP);
    if (tx == 8 && ty == 4 && tl == 16)
        return onsite ? step32_smem_bytes<8, 4, 16, true, NT, KA, KP>(RP) : step32_smem_bytes<8, 4, 16, false, NT, KA, KP>(RP);
    if (tx == 16 && ty == 8 && tl == 8)  // larger plane tile, shallower rings
        return onsite ? step32_smem_bytes<16, 8, 8, true, NT, 3, 2>(RP) : step32_smem_bytes<16, 8, 8, false, NT, 3, 2>(RP);
    return 0;
}

// 3D two-step kernel (kpm_tma32.cuh): real 3D stencils on whole lattices (not slabs), tiles
// dividing the lattice, 4 vector blocks (the caller falls back to single steps otherwise).
void plan_tma32(const kpm_handle_s* h, Plan* p) {
    p->use_tma32 = false;
    // Experimental (opts.experimental = 1): correct (GPU parity tests) but measured slower than the
    // single-step dense-box kernel on c3 (2.64 ms per launch = 1.32 ms per step vs 1.02 ms).
    if (h->opts.experimental != 1) return;
    if (h->ndim != 3 || p->no_fused || h->rows || is_cplx(h)) return;
    const int RG = p->RG;
    int TX = 8, TY = 8, TL = 8;
    const int shape = h->opts.exp_param;  // 1 = 16x4x8, 2 = 8x4x16, 3 = 16x8x8
    if (shape == 1) { TX = 16; TY = 4; TL = 8; }
    if (shape == 2) { TX = 8; TY = 4; TL = 16; }
    if (shape == 3) { TX = 16; TY = 8; TL = 8; }
    if (RG % TL || h->L[0] % TX || h->L[1] % TY || h->L[0] < 2 || h->L[1] < 2) return;
    const size_t sm = step32_smem(TX, TY, TL, h->d_eps != nullptr, p->RP);
    if (!sm || sm > 227 * 1024) return;
    const long long cols = (long long)(RG / TL) * (h->L[0] / TX) * (h->L[1] / TY);
    p->TX32 = TX;
    p->TY32 = TY;
    p->TL32 = TL;
    p->tma32_smem = sm;
    // whole columns round-robin when there are enough of them (in-plane halos then hit L2)
    p->tma32_rr = (cols >= 4LL * h->num_sms && !h->opts.contiguous) ? 1 : 0;
    p->tma32_grid = (int)std::min<long long>(p->tma32_rr ? cols : cols * h->L[2], (long long)h->num_sms);
    p->use_tma32 = true;
}
#endif

// Tile choice for the TMA march: ~16 KB main tiles (TX*TY*TL = 1024 lanes), full passes
// of the 256 consumer threads, tiles dividing the lattice, lane groups dividing RG.
void plan_tma(const kpm_handle_s* h, uint32_t flags, Plan* p) {
    p->use_tma = false;
    if (h->kind != KIND_STENCIL || h->ndim < 2 || (flags & KPM_DIRECT) || h->opts.no_tma) return;
    const int RG = p->RG;
    int TL = 0;
    // 3D: 16 lanes (256 contiguous bytes per site) first -- c3 measured 1119 ms vs 1358 ms with 8 lanes
    // (DRAM locality of the TMA box rows; with the dense-box kernel, kpm_tma3.cuh)
    // 2D real: 16 lanes first -- c2 25.35 vs 26.13 ms per call with 32 (same box, A/B); 2D complex:
    // 32 first -- c4 3114 vs 3166-3274 ms with 16
    // 2D: 4 lanes per site when RG is not a multiple of 8 (e.g. c2 at 8 GPUs: R = 8 real vectors per
    // GPU, an L2-resident block -- SURVEY.md 8(e) P1 strong scaling)
    // 2D complex: 16 lanes (the three-step kernel: c4 2346 vs 2438 ms per call with 32; its halo is
    // 3 sites per side, so the wider 64-site tile pays)
    const int cands2r[4] = {16, 32, 8, 4}, cands2c[4] = {16, 32, 8, 4}, cands3[4] = {16, 32, 8, 0};
    for (int c : (h->ndim == 2 ? (is_cplx(h) ? cands2c : cands2r) : cands3))
        if (c && RG % c == 0) { TL = c; break; }
    const int tl_opt = h->opts.tma_lanes;  // pinned lanes per tile site (A/B, tests)
    if (tl_opt > 0 && RG % tl_opt == 0) TL = tl_opt;
    if (!TL) return;
    int TX, TY;
    if (h->ndim == 2) {
        TY = 1;
        TX = 1024 / TL;
        while (TX * TL > 256 && h->L[0] % TX) TX /= 2;
        if (h->L[0] % TX) return;
    } else {
        TY = 8;
        TX = std::max(1, 1024 / (TL * TY));
        while (TX * TY * TL > 256 && h->L[0] % TX) TX /= 2;
        while (TX * TY * TL > 256 && h->L[1] % TY) TY /= 2;
        if (h->L[0] % TX || h->L[1] % TY) return;
    }
    if ((TX * TY * TL) % (kpm::kTmaConsumerWarps * 32) != 0) return;
    if ((TX * 8) % 16 != 0) return;  // eps box inner dimension
    const kpm::SlotLayout SL(h->ndim, TX, TY, TL, h->d_eps != nullptr);
    const size_t tile = (size_t)TX * TY * TL * 16;
    p->tma_smem = kpm::kSA * (size_t)SL.bytes + kpm::kSP * tile + 3 * (size_t)p->RP * 8 +
                  3 * (size_t)kpm::kTmaConsumerWarps * 32 * 16 + (2 * kpm::kSA + 2 * kpm::kSP) * 8;
    if (p->tma_smem > 227 * 1024) return;
    const long long Lm = h->ndim == 2 ? h->L[1] : h->L[2];
    const long long W = (long long)(RG / TL) * (h->L[0] / TX) * (h->ndim == 3 ? h->L[1] / TY : 1) * Lm;
    p->TL = TL;
    p->TX = TX;
    p->TY = TY;
    p->tma_grid = (int)std::min<long long>(W, h->num_sms);
    p->use_tma3 = false;
    if (h->ndim == 3 && !h->opts.no_box3) {
        const bool on = h->d_eps != nullptr;
        size_t sm3 = 0;
        if (TX == 16 && TY == 8 && TL == 8) sm3 = on ? kpm::step3_smem_bytes<16, 8, 8, true>(p->RP) : kpm::step3_smem_bytes<16, 8, 8, false>(p->RP);
        if (TX == 8 && TY == 8 && TL == 16) sm3 = on ? kpm::step3_smem_bytes<8, 8, 16, true>(p->RP) : kpm::step3_smem_bytes<8, 8, 16, false>(p->RP);
        if (TX == 4 && TY == 8 && TL == 32) sm3 = on ? kpm::step3_smem_bytes<4, 8, 32, true>(p->RP) : kpm::step3_smem_bytes<4, 8, 32, false>(p->RP);
        if (sm3 && sm3 <= 227 * 1024) {
            p->use_tma3 = true;
            p->tma_smem = sm3;
        }
    }
    // 3D: whole columns round-robin when there are enough of them (in-plane halos then hit L2)
    const long long cols = W / Lm;
    p->tma_rr = (h->ndim == 3 && cols >= 4LL * p->tma_grid && !h->opts.contiguous) ? 1 : 0;
    p->use_tma = true;
    // two-step kernel: 2D lattices with L0 >= 4, same tiles, shared memory permitting
    // One CTA per SM with TX*TL = 1024 lanes per row tile (measured on c2: two co-resident
    // CTAs with half-width tiles were 5% slower).
    p->use_tma2 = false;
    if (h->ndim == 2 && !p->no_fused && !h->opts.no_two_step && h->L[0] >= 4 && h->L[1] >= 4) {
        const bool on = h->d_eps != nullptr;
        int tx1 = 1024 / TL, minb = 1;
        // 4 lanes per site: the 64-site tile (2 CTAs per SM) when the 256-site tile would leave a CTA
        // fewer than 32 rows to march (per-segment pipeline fill dominates short segments)
        if (TL == 4 && (h->L[0] % tx1 || (long long)(RG / TL) * (h->L[0] / tx1) * h->L[1] < 32LL * h->num_sms)) {
            tx1 = 64;
            minb = 2;
        }
        if (h->opts.two_step_ctas > 0) minb = std::min(h->opts.two_step_ctas, tx1 == 64 && TL == 4 ? 2 : 1);
        const size_t sm1 = kpm::step2_smem_bytes(tx1, TL, on, p->RP);
        const long long Lm2 = h->L[1];
        if (h->L[0] % tx1 == 0 && sm1 <= 227 * 1024) {
            p->TX2 = tx1;
            p->tma2_minb = minb;
            p->tma2_smem = sm1;
        }
        if (p->TX2) {
            const long long W2 = (long long)(RG / TL) * (h->L[0] / p->TX2) * Lm2;
            p->tma2_grid = (int)std::min<long long>(W2, (long long)p->tma2_minb * h->num_sms);
            p->use_tma2 = true;
            // three steps per launch: the same row tile, sites of >= 128 bytes (8+ lanes)
            const size_t smt = kpm::tri_smem_bytes(p->TX2, TL, on, p->RP);
            p->use_tri = !h->opts.no_three_step && TL >= 8 && TL <= 32 && TL * p->TX2 == 1024 && h->L[0] >= 8 &&
                         h->L[1] >= 6 && smt <= (size_t)h->smem_optin;
            p->tri_smem = smt;
            // four steps per launch: 8-lane x 64-site tiles (2 sites per thread run); 4-lane x 128-site
            // tiles when the lanes are not a multiple of 8 (small R per GPU)
            const int tlq = RG % 8 == 0 ? 8 : 4, txq = tlq == 8 ? 64 : 128;
            const size_t smq = kpm::quad_smem_bytes(txq, tlq, on);
            p->use_quad = !h->opts.no_four_step && RG % tlq == 0 && h->L[0] % txq == 0 && h->L[1] >= 8 &&
                          smq <= (size_t)h->smem_optin;
            if (p->use_quad) {
                p->TLQ = tlq;
                p->TXQ = txq;
                p->quad_smem = smq;
                const long long WQ = (long long)(RG / tlq) * (h->L[0] / txq) * Lm2;
                p->quad_grid = (int)std::min<long long>(WQ, (long long)h->num_sms);
            }
        }
    }
    // KS-step kernel: 2D lattices, row tiles of TXK * TLK = 512 lanes (kpm_tmak.cuh)
    p->use_tmak = false;
#ifdef KPM_EXPERIMENTAL
    // Experimental (opts.experimental = 2, exp_param = KS = 3 or 4): measured slower than the
    // two-step kernel on c2 and c4 ("deeper temporal blocking").
    const int ks = h->opts.experimental == 2 ? h->opts.exp_param : 0;
    if (h->ndim == 2 && !p->no_fused && ks >= 2) {
        const bool on = h->d_eps != nullptr;
        const int tlk = RG % 16 == 0 ? 16 : (RG % 8 == 0 ? 8 : 0);
        const int txk = tlk ? 512 / tlk : 0;
        const size_t sm = tlk ? stepk_smem(ks, tlk, on, p->RP) : 0;
        if (sm && h->L[0] % txk == 0 && h->L[0] >= 4 && sm <= 227 * 1024) {
            p->KSK = ks;
            p->TLK = tlk;
            p->TXK = txk;
            p->tmak_smem = sm;
            const long long WK = (long long)(RG / tlk) * (h->L[0] / txk) * h->L[1];
            p->tmak_grid = (int)std::min<long long>(WK, (long long)h->num_sms);
            p->use_tmak = true;
        }
    }
    plan_tma32(h, p);
#endif
}

kpm_status make_plan(const kpm_handle_s* h, int32_t N, int64_t R, uint32_t flags, bool with_r0, Plan* p,
                     bool no_fused = false) {
    if (N < 1) return fail(KPM_ERR_INVALID_ARG, "N must be >= 1 (got %d)", N);
    if (R < 1) return fail(KPM_ERR_INVALID_ARG, "R must be >= 1 (got %lld)", (long long)R);
    // vector shards: the vector partition, or the vector groups of a hybrid row partition
    const bool hybrid = h->dist.partition == KPM_PART_ROWS && h->dist.vworld > 1;
    const int world = h->dist.partition == KPM_PART_VECTORS ? h->dist.world : (hybrid ? h->dist.vworld : 1);
    const int rank = h->dist.partition == KPM_PART_VECTORS ? h->dist.rank : (hybrid ? h->dist.vrank : 0);
    p->N = N;
    p->M = N / 2;
    p->no_fused = no_fused;
    p->r_off = (long long)(R * rank / world);
    p->R_loc = (long long)(R * (rank + 1) / world) - p->r_off;
    if (p->R_loc < 1) return fail(KPM_ERR_INVALID_ARG, "rank %d of %d owns no vectors (R=%lld)", rank, world, (long long)R);
    p->RG = is_cplx(h) ? (int)p->R_loc : (int)((p->R_loc + 1) / 2);
    p->RP = is_cplx(h) ? p->RG : 2 * p->RG;
    if (h->kind == KIND_DENSE) {  // GEMM tiles: vectors padded to 64 (zero columns)
        p->RP = (int)((p->R_loc + kpm::kDBN - 1) / kpm::kDBN * kpm::kDBN);
        p->RG = p->RP / 2;
    }
    int tr = 1;
    while (tr < p->RG && tr < 32) tr <<= 1;
    p->TR = tr;
    p->TS = kThreads / tr;
    p->gy = (p->RG + tr - 1) / tr;
    const long long site_ctas = (h->D + p->TS - 1) / p->TS;
    p->gx = (int)std::min<long long>(site_ctas, 2LL * h->num_sms);
    // the staged ELL kernel (one 512-thread CTA per SM: 128 registers) walks its tiles grid-stride:
    // one wave of CTAs over the (gx, gy) grid instead of 2 gy waves
    if (h->kind == KIND_ELL && h->K > 0 && h->K <= kpm::kEllKMax && !h->opts.ell_generic)
        p->gx = (int)std::max<long long>(1, std::min<long long>(site_ctas, h->num_sms / std::max(1, p->gy)));
    plan_tma(h, flags, p);
    if (p->use_tma) p->gx = p->tma_grid;
    if (h->kind == KIND_DENSE) p->gx = (int)(h->Dp / kpm::kDBM);  // partial rows = M tiles
    p->small_smem = 2 * (size_t)h->D * p->TR * sizeof(double2);
    p->use_small = !h->rows && !(flags & KPM_DIRECT) && p->small_smem <= kpm::kSmallSmemMax && !h->opts.no_small &&
                   h->kind != KIND_DENSE;
    if (p->use_small) {
        p->use_tma = p->use_tma2 = p->use_tma32 = false;
        p->TS = kpm::kSmallThreads / p->TR;
        p->gx = p->TS;  // partial-sum rows per slot = thread rows of the single CTA
    }
    if (p->use_tma2) p->gx = std::max(p->gx, p->tma2_grid);  // partial rows per slot (max over kernels)
    if (p->use_tmak) p->gx = std::max(p->gx, p->tmak_grid);
    if (p->use_tma32) p->gx = std::max(p->gx, p->tma32_grid);
    p->nslots = N;
    if (h->rows) p->use_tma2 = p->use_tri = p->use_quad = p->use_tmak = p->use_tma32 = false;  // multi-step kernels need deep halos; not with slabs
    p->overlap = h->rows && p->use_tma && h->nloc >= 3 && h->dist.comm != KPM_COMM_LOCAL &&
                 h->dist.comm != KPM_COMM_IPC && !(flags & KPM_DIRECT) &&
                 !h->opts.no_overlap;
    if (p->overlap) p->gx = 3 * p->tma_grid;
    if (p->use_tmak && p->M - 1 < p->KSK) p->use_tmak = false;
    p->xpad = (h->kind == KIND_STENCIL && h->ndim == 3) ? 2 : 0;
    const size_t rows_of_x = (size_t)(h->D / h->L[0]);
    p->mem_sites = (size_t)h->D + 2 * (size_t)p->xpad * rows_of_x;
    if (h->kind == KIND_DENSE) p->mem_sites = (size_t)h->Dp;
    if (h->kind == KIND_ELL) p->mem_sites = (size_t)(h->D + h->n_ghost);  // ghost sites after the local rows
    const size_t plane_mem = (!h->rows || h->kind == KIND_ELL) ? 0
                             : p->xpad ? (size_t)(h->plane / h->L[0]) * (h->L[0] + 2 * p->xpad) : (size_t)h->plane;
    p->ghost_lanes = plane_mem * p->RG;
    p->lane_bytes = (p->mem_sites * p->RG + 2 * p->ghost_lanes) * sizeof(double2);
    // Persistent L2-resident mode (experimental, opts.experimental = 3): the whole recursion in one
    // cooperative launch, one 512-thread CTA per SM per lane-group row of the grid.  Measured on c2
    // with R = 8 (2 x 16.8 MB, L2-resident): 7.85 ms vs 7.42 ms for the per-step launches of round 1
    // -- the launch gaps it removes are smaller than what the grid barrier costs.
    p->use_persist = false;
#ifdef KPM_EXPERIMENTAL
    if (!p->use_small && h->kind != KIND_DENSE && !h->rows && !(flags & KPM_DIRECT) && p->M >= 2 &&
        p->gy <= h->num_sms && h->opts.experimental == 3) {
        p->use_persist = true;
        p->use_tma = p->use_tma2 = p->use_tma32 = p->use_tmak = p->use_tma3 = false;
        p->overlap = false;
        const long long site_ctas = (h->D + p->TS - 1) / p->TS;
        p->gx = (int)std::max<long long>(1, std::min<long long>(site_ctas, h->num_sms / p->gy));
    }
#endif
    size_t off = 0;
    p->off_P = off; off = align_up(off + p->lane_bytes);
    p->off_C = off; off = align_up(off + std::max(p->lane_bytes, with_r0 ? (size_t)p->R_loc * h->D * sizeof(double) : 0));
    p->off_R = off;
    if ((flags & KPM_DIRECT) && with_r0) off = align_up(off + p->lane_bytes);
    if (p->use_tri && (p->M - 1 < 3 || !p->use_tma2)) p->use_tri = false;
    if (p->use_quad && (p->M - 1 < 4 || !p->use_tma2)) p->use_quad = false;
    if (p->use_quad) p->gx = std::max(p->gx, p->quad_grid);
    if (p->use_tma2 && p->M - 1 < 2) p->use_tma2 = false;
    if (p->use_tma32 && p->M - 1 < 2) p->use_tma32 = false;
    if (p->use_tma2 || p->use_tmak || p->use_tma32) {  // out-of-place multi-step launches: two spare blocks
        p->off_X2 = off; off = align_up(off + p->lane_bytes);
        p->off_X3 = off; off = align_up(off + p->lane_bytes);
    }
    p->off_part = off; off = align_up(off + (size_t)std::max(N, 3) * p->gx * p->RP * sizeof(double));
    p->off_Sv = off; off = align_up(off + (size_t)N * p->R_loc * sizeof(double));
    p->off_S = off; off = align_up(off + (size_t)N * sizeof(double));
    p->off_out = off; off = align_up(off + (size_t)N * p->R_loc * sizeof(double));
    p->off_sites = off; off = align_up(off + ((flags & KPM_LOCAL) ? (size_t)R * sizeof(long long) : 0));
    p->off_send = off; off = align_up(off + (size_t)h->n_send * p->RG * sizeof(double2));
    p->total = off;
    if (h->D * (long long)p->RG > (1LL << 40)) return fail(KPM_ERR_INVALID_ARG, "problem too large");
    return KPM_OK;
}

// Workspace from the device's stream-ordered pool (release threshold raised at handle
// creation), so creating/destroying handles per call does not pay cudaMalloc/cudaFree.
kpm_status ensure_workspace(kpm_handle_s* h, size_t bytes) {
    if (h->ws_bytes >= bytes) return KPM_OK;
    if (!h->ws_own) return fail(KPM_ERR_OOM, "caller workspace has %zu bytes, need %zu", h->ws_bytes, bytes);
    void* p = nullptr;
    cudaError_t e;
    if (h->ipc) {  // CUDA IPC handles need a plain allocation (not the stream-ordered pool)
        if (h->ws) {
            cudaStreamSynchronize(h->stream);
            cudaFree(h->ws);
        }
        h->ws = nullptr;
        h->ws_bytes = 0;
        e = cudaMalloc(&p, bytes);
    } else {
        if (h->ws) cudaFreeAsync(h->ws, h->stream);
        h->ws = nullptr;
        h->ws_bytes = 0;
        e = cudaMallocAsync(&p, bytes, h->stream);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(KPM_ERR_OOM, "cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    h->ws = static_cast<char*>(p);
    h->ws_bytes = bytes;
    return KPM_OK;
}

// Launch one fused kernel of `mode` with operator op.
template <int MODE, bool CPLX, class OP>
kpm_status launch_step(kpm_handle_s* h, const Plan& p, const OP& op, const kpm::VecArgs& v, int tail) {
    dim3 block(p.TR, p.TS), grid(p.gx, p.gy);
    const size_t smem = 3 * (size_t)kThreads * sizeof(double2);
    return launch_k(h, h->stream, kpm::kpm_step_kernel<OP, MODE, CPLX>, grid, block, smem, op, v, tail);
}

template <bool CPLX, class OP>
kpm_status launch_mode(kpm_handle_s* h, const Plan& p, const OP& op, int mode, const kpm::VecArgs& v, int tail) {
    switch (mode) {
        case kpm::FIRST_GEN: return launch_step<kpm::FIRST_GEN, CPLX>(h, p, op, v, tail);
        case kpm::FIRST_BUF: return launch_step<kpm::FIRST_BUF, CPLX>(h, p, op, v, tail);
        case kpm::STEP: return launch_step<kpm::STEP, CPLX>(h, p, op, v, tail);
        case kpm::DIRECT_GEN: return launch_step<kpm::DIRECT_GEN, CPLX>(h, p, op, v, tail);
        default: return launch_step<kpm::DIRECT_BUF, CPLX>(h, p, op, v, tail);
    }
}

kpm::StencilGeom stencil_geom(const kpm_handle_s* h) {
    kpm::StencilGeom g;
    g.L0 = (int)h->L[0];
    g.L1 = (int)h->L[1];
    g.L2 = (int)h->L[2];
    g.plane = (int)(h->L[0] * h->L[1]);
    g.t = h->t_scaled;
    g.shift = -h->b / h->a;
    g.eps = h->d_eps;
    g.phase = h->d_phase;
    g.ghost = h->rows ? 1 : 0;
    return g;
}

// ELL recursion step with cp.async-prefetched row entries (kpm_ell.cuh).
template <bool CPLX>
kpm_status launch_ell_t(kpm_handle_s* h, const Plan& p, const kpm::VecArgs& v, int tail) {
    dim3 block(p.TR, p.TS), grid(p.gx, p.gy);
    const bool spw8 = h->ell_kp == 8 && kpm::ell_smem_bytes(kThreads, p.TS, h->K, CPLX, kpm::kEllSPW8) <= (size_t)h->smem_optin;
    const size_t smem = kpm::ell_smem_bytes(kThreads, p.TS, h->K, CPLX, spw8 ? kpm::kEllSPW8 : kpm::kEllSPW);
    const bool wide = (double)(h->D + h->n_ghost) * p.RG >= 2147483648.0;  // 32-bit element offsets otherwise
    auto pick = [&](auto w) {
        constexpr bool W = decltype(w)::value;
        switch (h->ell_kp) {
            case 4: return kpm::kpm_ell_step_kernel<CPLX, 4, W>;
            case 8: return spw8 ? kpm::kpm_ell_step_kernel<CPLX, 8, W, kpm::kEllSPW8> : kpm::kpm_ell_step_kernel<CPLX, 8, W>;
            case 12: return kpm::kpm_ell_step_kernel<CPLX, 12, W>;
            default: return kpm::kpm_ell_step_kernel<CPLX, 16, W>;
        }
    };
    auto kern = wide ? pick(std::true_type{}) : pick(std::false_type{});
    KPM_TRY(set_smem((const void*)kern, smem, h->device));
    const kpm::EllOp<CPLX> op{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp};
    return launch_k(h, h->stream, kern, grid, block, smem, op, v, tail);
}

template <bool CPLX, class OP>
kpm_status launch_small_t(kpm_handle_s* h, const Plan& p, const OP& op, const kpm::VecArgs& v, int from_buf, int N,
                          double* part) {
    auto kern = kpm::kpm_small_kernel<OP, CPLX>;
    KPM_TRY(set_smem((const void*)kern, p.small_smem, h->device));
    return launch_k(h, h->stream, kern, dim3(1, p.gy), dim3(p.TR, p.TS), p.small_smem, op, v, from_buf, N, part);
}

kpm_status launch_small(kpm_handle_s* h, const Plan& p, const kpm::VecArgs& v, int from_buf, int N, double* part) {
    using namespace kpm;
    if (h->kind == KIND_ELL) {
        if (is_cplx(h)) return launch_small_t<true>(h, p, EllOp<true>{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp}, v, from_buf, N, part);
        return launch_small_t<false>(h, p, EllOp<false>{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp}, v, from_buf, N, part);
    }
    const StencilGeom g = stencil_geom(h);
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_small_t<true>(h, p, StencilOp<2, true, true>{g}, v, from_buf, N, part);
        return launch_small_t<true>(h, p, StencilOp<2, false, true>{g}, v, from_buf, N, part);
    }
    switch (h->ndim * 2 + (on ? 1 : 0)) {
        case 2: return launch_small_t<false>(h, p, StencilOp<1, false, false>{g}, v, from_buf, N, part);
        case 3: return launch_small_t<false>(h, p, StencilOp<1, true, false>{g}, v, from_buf, N, part);
        case 4: return launch_small_t<false>(h, p, StencilOp<2, false, false>{g}, v, from_buf, N, part);
        case 5: return launch_small_t<false>(h, p, StencilOp<2, true, false>{g}, v, from_buf, N, part);
        case 6: return launch_small_t<false>(h, p, StencilOp<3, false, false>{g}, v, from_buf, N, part);
        default: return launch_small_t<false>(h, p, StencilOp<3, true, false>{g}, v, from_buf, N, part);
    }
}

#ifdef KPM_EXPERIMENTAL
template <class OP, bool CPLX>
kpm_status launch_persist_t(kpm_handle_s* h, const Plan& p, const OP& op, const kpm::VecArgs& v, int first_buf, int N,
                            long long slot, double* part) {
    auto kern = kpm::kpm_persist_kernel<OP, CPLX>;
    dim3 block(p.TR, p.TS), grid(p.gx, p.gy);
    const size_t smem = 3 * (size_t)kThreads * sizeof(double2);
    int per_sm = 0;
    KPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, p.TR * p.TS, smem));
    if ((long long)per_sm * h->num_sms < (long long)p.gx * p.gy)
        return fail(KPM_ERR_UNSUPPORTED, "persistent kernel: %d x %d CTAs not co-resident (%d per SM)", p.gx, p.gy, per_sm);
    kpm::VecArgs va = v;
    int M = p.M;
    void* args[] = {(void*)&op, (void*)&va, (void*)&N, (void*)&M, (void*)&first_buf, (void*)&slot, (void*)&part};
    KPM_CUDA(cudaLaunchCooperativeKernel((const void*)kern, grid, block, args, smem, h->stream));
    h->total_launches++;
    return KPM_OK;
}

template <bool CPLX, class OP>
kpm_status launch_persist_op(kpm_handle_s* h, const Plan& p, const OP& op, const kpm::VecArgs& v, int first_buf, int N,
                             long long slot, double* part) {
    return launch_persist_t<OP, CPLX>(h, p, op, v, first_buf, N, slot, part);
}

#endif

// Dispatch on the operator type of the handle.
kpm_status launch(kpm_handle_s* h, const Plan& p, int mode, const kpm::VecArgs& v, int tail) {
    using namespace kpm;
    // the staged ELL kernel when its tile (index + value panels of TS * kEllSPW rows, double
    // buffered) fits the device's opt-in shared memory; else the generic kernel
    if (h->kind == KIND_ELL && mode == STEP && h->K > 0 && h->K <= kEllKMax && !h->opts.ell_generic &&
        ell_smem_bytes(kThreads, p.TS, h->K, is_cplx(h)) <= (size_t)h->smem_optin)
        return is_cplx(h) ? launch_ell_t<true>(h, p, v, tail) : launch_ell_t<false>(h, p, v, tail);
    if (h->kind == KIND_ELL) {
        if (is_cplx(h)) return launch_mode<true>(h, p, EllOp<true>{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp}, mode, v, tail);
        return launch_mode<false>(h, p, EllOp<false>{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp}, mode, v, tail);
    }
    const StencilGeom g = stencil_geom(h);
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_mode<true>(h, p, StencilOp<2, true, true>{g}, mode, v, tail);
        return launch_mode<true>(h, p, StencilOp<2, false, true>{g}, mode, v, tail);
    }
    switch (h->ndim * 2 + (on ? 1 : 0)) {
        case 2: return launch_mode<false>(h, p, StencilOp<1, false, false>{g}, mode, v, tail);
        case 3: return launch_mode<false>(h, p, StencilOp<1, true, false>{g}, mode, v, tail);
        case 4: return launch_mode<false>(h, p, StencilOp<2, false, false>{g}, mode, v, tail);
        case 5: return launch_mode<false>(h, p, StencilOp<2, true, false>{g}, mode, v, tail);
        case 6: return launch_mode<false>(h, p, StencilOp<3, false, false>{g}, mode, v, tail);
        default: return launch_mode<false>(h, p, StencilOp<3, true, false>{g}, mode, v, tail);
    }
}

// First step of a 2D/3D stencil with a_0 generated once per element (kpm_first.cuh).
template <int NDIM, bool ONSITE, bool PEIERLS, bool CPLX>
kpm_status launch_first_t(kpm_handle_s* h, const kpm::VecArgs& v, const kpm::FirstGeom& g, int grid, size_t smem, int tail,
                          int from_buf) {
    auto kern = kpm::kpm_first_tile_kernel<NDIM, ONSITE, PEIERLS, CPLX>;
    KPM_TRY(set_smem((const void*)kern, smem, h->device));
    return launch_k(h, h->stream, kern, dim3(grid), dim3(kpm::kFirstThreads), smem, v, g, tail, from_buf);
}

kpm_status launch_first_tile(kpm_handle_s* h, const Plan& p, const kpm::VecArgs& v, int tail, int from_buf) {
    kpm::FirstGeom g{};
    const int nd = h->ndim;
    g.L0 = (int)h->L[0];
    g.L1 = (int)h->L[1];
    // lanes per tile: a power of two (it must divide the 512 threads), masked when RG is not a multiple
    g.TL = 1;
    while (g.TL * 2 <= std::min(nd == 3 ? 8 : 16, p.RG)) g.TL *= 2;
    g.TX = (int)std::min<int64_t>(nd == 3 ? 16 : 64, h->L[0]);
    g.TY = nd == 3 ? (int)std::min<int64_t>(16, h->L[1]) : 1;
    g.PX = (g.L0 + g.TX - 1) / g.TX;
    g.PY = nd == 3 ? (g.L1 + g.TY - 1) / g.TY : 1;
    g.G_L = (p.RG + g.TL - 1) / g.TL;
    g.Lm = (int)h->L[nd - 1];  // (the slab's planes under KPM_PART_ROWS)
    const long long cols = (long long)g.G_L * g.PX * g.PY;
    const int rows = p.gx;     // partial-sum rows per slot of this plan
    int nseg = cols >= 2LL * rows ? 1 : (int)((2LL * rows + cols - 1) / cols);
    int seg = (g.Lm + nseg - 1) / nseg;
    if (seg < 4) seg = std::min(4, g.Lm);
    g.SEG = seg;
    g.NSEG = (g.Lm + seg - 1) / seg;
    g.items = cols * g.NSEG;
    g.rows_total = rows;
    g.ghost = h->rows ? 1 : 0;
    g.t = h->t_scaled;
    g.shift = -h->b / h->a;
    g.eps = h->d_eps;
    g.phase = h->d_phase;
    const int grid = (int)std::min<long long>(g.items, rows);
    const size_t smem = kpm::first_smem_bytes(nd, g.TX, g.TY, g.TL, p.RP);
    if (smem > (size_t)h->smem_optin) return fail(KPM_ERR_UNSUPPORTED, "first-step tile does not fit shared memory");
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_first_t<2, true, true, true>(h, v, g, grid, smem, tail, from_buf);
        return launch_first_t<2, false, true, true>(h, v, g, grid, smem, tail, from_buf);
    }
    if (nd == 2) {
        if (on) return launch_first_t<2, true, false, false>(h, v, g, grid, smem, tail, from_buf);
        return launch_first_t<2, false, false, false>(h, v, g, grid, smem, tail, from_buf);
    }
    if (on) return launch_first_t<3, true, false, false>(h, v, g, grid, smem, tail, from_buf);
    return launch_first_t<3, false, false, false>(h, v, g, grid, smem, tail, from_buf);
}

#ifdef KPM_EXPERIMENTAL
kpm_status launch_persist(kpm_handle_s* h, const Plan& p, const kpm::VecArgs& v, int first_buf, int N, long long slot,
                          double* part) {
    using namespace kpm;
    if (h->kind == KIND_ELL) {
        if (is_cplx(h))
            return launch_persist_op<true>(h, p, EllOp<true>{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp}, v, first_buf, N,
                                           slot, part);
        return launch_persist_op<false>(h, p, EllOp<false>{(int)h->D, h->K, h->d_col, h->d_val, -h->b / h->a, h->ell_kp}, v, first_buf,
                                        N, slot, part);
    }
    const StencilGeom g = stencil_geom(h);
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_persist_op<true>(h, p, StencilOp<2, true, true>{g}, v, first_buf, N, slot, part);
        return launch_persist_op<true>(h, p, StencilOp<2, false, true>{g}, v, first_buf, N, slot, part);
    }
    switch (h->ndim * 2 + (on ? 1 : 0)) {
        case 2: return launch_persist_op<false>(h, p, StencilOp<1, false, false>{g}, v, first_buf, N, slot, part);
        case 3: return launch_persist_op<false>(h, p, StencilOp<1, true, false>{g}, v, first_buf, N, slot, part);
        case 4: return launch_persist_op<false>(h, p, StencilOp<2, false, false>{g}, v, first_buf, N, slot, part);
        case 5: return launch_persist_op<false>(h, p, StencilOp<2, true, false>{g}, v, first_buf, N, slot, part);
        case 6: return launch_persist_op<false>(h, p, StencilOp<3, false, false>{g}, v, first_buf, N, slot, part);
        default: return launch_persist_op<false>(h, p, StencilOp<3, true, false>{g}, v, first_buf, N, slot, part);
    }
}
#else
kpm_status launch_persist(kpm_handle_s*, const Plan&, const kpm::VecArgs&, int, int, long long, double*) {
    return fail(KPM_ERR_UNSUPPORTED, "persistent kernel: experimental build only (libkpm_exp.so)");
}
#endif

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(ptr);
    }
    return fn;
}

// Tensor map over the lane-layout vector block viewed as doubles [L2][L1][L0][2 RG]
// (rank 3 in 2D, 4 in 3D) with the given box.
kpm_status make_vec_map(const kpm_handle_s* h, const Plan& p, void* base, int bx, int by, int bz, CUtensorMap* m,
                        int tl = 0) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int rank = h->ndim + 1;
    cuuint64_t dims[4] = {(cuuint64_t)2 * p.RG, (cuuint64_t)h->L[0], (cuuint64_t)h->L[1], (cuuint64_t)h->L[2]};
    if (h->rows) dims[1 + h->slow] += 2;  // ghost planes
    if (p.xpad) dims[1] += 2 * p.xpad;    // x-row frames (3D)
    cuuint64_t pitch = (cuuint64_t)h->L[0] + 2 * p.xpad;
    cuuint64_t strides[3] = {(cuuint64_t)p.RG * 16, (cuuint64_t)p.RG * 16 * pitch, (cuuint64_t)p.RG * 16 * pitch * h->L[1]};
    cuuint32_t box[4] = {(cuuint32_t)(2 * (tl ? tl : p.TL)), (cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
    if (h->ndim == 2) box[2] = 1;
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled (vectors) failed: %d", (int)r);
    return KPM_OK;
}

kpm_status make_eps_map(const kpm_handle_s* h, const Plan& p, CUtensorMap* m) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int rank = h->ndim;
    cuuint64_t dims[3] = {(cuuint64_t)h->L[0], (cuuint64_t)h->L[1], (cuuint64_t)h->L[2]};
    cuuint64_t strides[2] = {(cuuint64_t)h->L[0] * 8, (cuuint64_t)h->L[0] * h->L[1] * 8};
    cuuint32_t box[3] = {(cuuint32_t)p.TX, (cuuint32_t)(h->ndim == 3 ? p.TY : 1), 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, h->d_eps, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled (eps) failed: %d", (int)r);
    return KPM_OK;
}

// Maps of one vector buffer in the a_n role (main, x-halo column, y-halo row) and the a_{n-1} role.
struct BufMaps {
    const void* base = nullptr;
    CUtensorMap A, Col, Row, P, Col2;  // main, 1-site column, row, (=main), 2-site column (2D)
    CUtensorMap A2;                    // main box of the two-step kernel (width TX2)
    CUtensorMap A3;                    // 3-site box of the three-step kernel
    CUtensorMap AQ, AQ4, AQ3;          // four-step kernel (TLQ lanes): main box TXQ, 4-site and 3-site boxes
    CUtensorMap AK, AKH, AKH1;         // KS-step kernel: main (TXK), KS-site and (KS-1)-site boxes, TLK lanes
    CUtensorMap Box3, Row3;            // 3D dense-box kernel: (TX+2) x TY box, (TX+2)-site row
    CUtensorMap A32, A32r, P32, P32r;  // 3D two-step kernel: (TX+4) x TY, (TX+4) x 2, (TX+2) x TY, (TX+2) x 1
};

kpm_status make_buf_maps(const kpm_handle_s* h, const Plan& p, void* base, BufMaps* bm) {
    bm->base = base;
    KPM_TRY(make_vec_map(h, p, base, p.TX, p.TY, 1, &bm->A));
    KPM_TRY(make_vec_map(h, p, base, 1, p.TY, 1, &bm->Col));
    KPM_TRY(make_vec_map(h, p, base, p.TX, 1, 1, &bm->Row));
    if (h->ndim == 2) KPM_TRY(make_vec_map(h, p, base, 2, 1, 1, &bm->Col2));
    if (p.use_tma2) KPM_TRY(make_vec_map(h, p, base, p.TX2, 1, 1, &bm->A2));
    if (p.use_tri) KPM_TRY(make_vec_map(h, p, base, 3, 1, 1, &bm->A3));
    if (p.use_quad) {
        KPM_TRY(make_vec_map(h, p, base, p.TXQ, 1, 1, &bm->AQ, p.TLQ));
        KPM_TRY(make_vec_map(h, p, base, 4, 1, 1, &bm->AQ4, p.TLQ));
        KPM_TRY(make_vec_map(h, p, base, kpm::quad_php(p.TLQ), 1, 1, &bm->AQ3, p.TLQ));
    }
    if (p.use_tma3) {
        KPM_TRY(make_vec_map(h, p, base, p.TX + 2, p.TY, 1, &bm->Box3));
        KPM_TRY(make_vec_map(h, p, base, p.TX + 2, 1, 1, &bm->Row3));
    }
    if (p.use_tma32) {
        KPM_TRY(make_vec_map(h, p, base, p.TX32 + 4, p.TY32, 1, &bm->A32, p.TL32));
        KPM_TRY(make_vec_map(h, p, base, p.TX32 + 4, 2, 1, &bm->A32r, p.TL32));
        KPM_TRY(make_vec_map(h, p, base, p.TX32 + 2, p.TY32, 1, &bm->P32, p.TL32));
        KPM_TRY(make_vec_map(h, p, base, p.TX32 + 2, 1, 1, &bm->P32r, p.TL32));
    }
    if (p.use_tmak) {
        KPM_TRY(make_vec_map(h, p, base, p.TXK, 1, 1, &bm->AK, p.TLK));
        KPM_TRY(make_vec_map(h, p, base, p.KSK, 1, 1, &bm->AKH, p.TLK));
        KPM_TRY(make_vec_map(h, p, base, p.KSK - 1, 1, 1, &bm->AKH1, p.TLK));
    }
    bm->P = bm->A;
    return KPM_OK;
}

// eps~ map with a given box width along x (2D: {bx, 1}; 3D: {bx, TY, 1})
kpm_status make_eps_map_w(const kpm_handle_s* h, const Plan& p, int bx, CUtensorMap* m) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)h->L[0], (cuuint64_t)h->L[1], (cuuint64_t)h->L[2]};
    cuuint64_t strides[2] = {(cuuint64_t)h->L[0] * 8, (cuuint64_t)h->L[0] * h->L[1] * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)(h->ndim == 3 ? p.TY : 1), 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, h->ndim, h->d_eps, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled (eps) failed: %d", (int)r);
    return KPM_OK;
}

template <int TL, int TX, bool ONSITE, bool PEIERLS, int MINB, int XW>
kpm_status launch_tma2_x(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                         const CUtensorMap& E2, const kpm::Tma2Geom& g, int tail) {
    auto kern = kpm::kpm_step2_tma_kernel<TL, TX, ONSITE, PEIERLS, MINB, XW>;
    KPM_TRY(set_smem((const void*)kern, p.tma2_smem, h->device));
    // a_{n-1} halo box: 1 site, or 2 when a site is under 128 bytes (kpm_tma2.cuh p_halo)
    const CUtensorMap& Ph = kpm::p_halo(TL) == 2 ? P.Col2 : P.Col;
    return launch_k(h, h->stream, kern, dim3(p.tma2_grid), dim3(kpm::Threads2<XW>::N), p.tma2_smem, A.A2, A.Col2, P.A2, Ph,
                    E, E2, g, tail);
}

// Halo warp (XW = 1, kpm_tma2.cuh) for complex128 (Peierls) lattices: c4 3178 vs 3387 ms per call;
// real lattices keep XW = 0 (c2 26.8 vs 25.9 ms: the 168-register cap of nine warps spills there).
// opts.halo_warp = 1 / 2 pins it on / off.
template <int TL, int TX, bool ONSITE, bool PEIERLS, int MINB>
kpm_status launch_tma2_t(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                         const CUtensorMap& E2, const kpm::Tma2Geom& g, int tail) {
    const bool xw = h->opts.halo_warp == 1 || (h->opts.halo_warp == 0 && PEIERLS);
    if (xw) return launch_tma2_x<TL, TX, ONSITE, PEIERLS, MINB, 1>(h, p, A, P, E, E2, g, tail);
    return launch_tma2_x<TL, TX, ONSITE, PEIERLS, MINB, 0>(h, p, A, P, E, E2, g, tail);
}

template <int TL, int TX, int MINB>
kpm_status launch_tma2_s(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                         const CUtensorMap& E2, const kpm::Tma2Geom& g, int tail) {
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_tma2_t<TL, TX, true, true, MINB>(h, p, A, P, E, E2, g, tail);
        return launch_tma2_t<TL, TX, false, true, MINB>(h, p, A, P, E, E2, g, tail);
    }
    if (on) return launch_tma2_t<TL, TX, true, false, MINB>(h, p, A, P, E, E2, g, tail);
    return launch_tma2_t<TL, TX, false, false, MINB>(h, p, A, P, E, E2, g, tail);
}

// instantiated tile shapes of the two-step kernel (TX * TL = 1024 lanes per row tile)
kpm_status launch_tma2(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                       const CUtensorMap& E2, const kpm::Tma2Geom& g, int tail) {
    if (p.TL == 64 && p.TX2 == 16) return launch_tma2_s<64, 16, 1>(h, p, A, P, E, E2, g, tail);
    if (p.TL == 32 && p.TX2 == 32) return launch_tma2_s<32, 32, 1>(h, p, A, P, E, E2, g, tail);
    if (p.TL == 16 && p.TX2 == 64) return launch_tma2_s<16, 64, 1>(h, p, A, P, E, E2, g, tail);
    if (p.TL == 8 && p.TX2 == 128) return launch_tma2_s<8, 128, 1>(h, p, A, P, E, E2, g, tail);
    if (p.TL == 4 && p.TX2 == 256) return launch_tma2_s<4, 256, 1>(h, p, A, P, E, E2, g, tail);
    if (p.TL == 4 && p.TX2 == 64) return launch_tma2_s<4, 64, 2>(h, p, A, P, E, E2, g, tail);
    return fail(KPM_ERR_UNSUPPORTED, "no two-step kernel for TL=%d TX=%d", p.TL, p.TX2);
}

template <int TL, int TX, bool ONSITE, bool PEIERLS>
kpm_status launch_tri_t(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                        const CUtensorMap& E4, const kpm::TriGeom& g, int tail) {
    // 8 warps, 4 consecutive interior sites per thread (a 16-warp variant with 2 sites per thread and a
    // 128-register cap spilled: c2 48.4 vs 20.2 ms per call, c4 no faster)
    auto kern = kpm::kpm_step_tri_kernel<TL, TX, ONSITE, PEIERLS, kpm::kThreadsTri>;
    KPM_TRY(set_smem((const void*)kern, p.tri_smem, h->device));
    return launch_k(h, h->stream, kern, dim3(p.tma2_grid), dim3(kpm::kThreadsTri), p.tri_smem, A.A2, A.A3, P.A2, P.Col2, E,
                    E4, g, tail);
}

template <int TL, int TX>
kpm_status launch_tri_s(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                        const CUtensorMap& E4, const kpm::TriGeom& g, int tail) {
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_tri_t<TL, TX, true, true>(h, p, A, P, E, E4, g, tail);
        return launch_tri_t<TL, TX, false, true>(h, p, A, P, E, E4, g, tail);
    }
    if (on) return launch_tri_t<TL, TX, true, false>(h, p, A, P, E, E4, g, tail);
    return launch_tri_t<TL, TX, false, false>(h, p, A, P, E, E4, g, tail);
}

template <int TL, int TX, bool ONSITE, bool PEIERLS>
kpm_status launch_quad_t(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                         const CUtensorMap& E4, const kpm::QuadGeom& g, int tail) {
    auto kern = kpm::kpm_step_quad_kernel<TL, TX, ONSITE, PEIERLS>;
    KPM_TRY(set_smem((const void*)kern, p.quad_smem, h->device));
    return launch_k(h, h->stream, kern, dim3(p.quad_grid), dim3(kpm::kThreadsQuad), p.quad_smem, A.AQ, A.AQ4, P.AQ, P.AQ3,
                    E, E4, g, tail);
}

kpm_status launch_quad(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                       const CUtensorMap& E4, const kpm::QuadGeom& g, int tail) {
    const bool on = h->d_eps != nullptr;
    if (p.TLQ == 8 && p.TXQ == 64) {
        if (is_cplx(h)) return on ? launch_quad_t<8, 64, true, true>(h, p, A, P, E, E4, g, tail) : launch_quad_t<8, 64, false, true>(h, p, A, P, E, E4, g, tail);
        return on ? launch_quad_t<8, 64, true, false>(h, p, A, P, E, E4, g, tail) : launch_quad_t<8, 64, false, false>(h, p, A, P, E, E4, g, tail);
    }
    if (p.TLQ == 4 && p.TXQ == 128) {  // 4-lane tiles (e.g. 8 real / 4 complex vectors per GPU)
        if (is_cplx(h)) return on ? launch_quad_t<4, 128, true, true>(h, p, A, P, E, E4, g, tail) : launch_quad_t<4, 128, false, true>(h, p, A, P, E, E4, g, tail);
        return on ? launch_quad_t<4, 128, true, false>(h, p, A, P, E, E4, g, tail) : launch_quad_t<4, 128, false, false>(h, p, A, P, E, E4, g, tail);
    }
    return fail(KPM_ERR_UNSUPPORTED, "no four-step kernel for TL=%d TX=%d", p.TLQ, p.TXQ);
}

// instantiated tile shapes of the three-step kernel (TX * TL = 1024 lanes per row tile)
kpm_status launch_tri(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                      const CUtensorMap& E4, const kpm::TriGeom& g, int tail) {
    if (p.TL == 32 && p.TX2 == 32) return launch_tri_s<32, 32>(h, p, A, P, E, E4, g, tail);
    if (p.TL == 16 && p.TX2 == 64) return launch_tri_s<16, 64>(h, p, A, P, E, E4, g, tail);
    if (p.TL == 8 && p.TX2 == 128) return launch_tri_s<8, 128>(h, p, A, P, E, E4, g, tail);
    return fail(KPM_ERR_UNSUPPORTED, "no three-step kernel for TL=%d TX=%d", p.TL, p.TX2);
}

#ifdef KPM_EXPERIMENTAL
template <int KS, int TL, int TX, bool ONSITE, bool PEIERLS>
kpm_status launch_tmak_t(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                         const CUtensorMap& EH, const kpm::TmaKGeom& g, int tail) {
    auto kern = kpm::kpm_stepk_tma_kernel<KS, TL, TX, ONSITE, PEIERLS>;
    KPM_TRY(set_smem((const void*)kern, p.tmak_smem, h->device));
    kern<<<p.tmak_grid, kpm::StepKThreads<KS, TL, TX>::NT, p.tmak_smem, h->stream>>>(A.AK, A.AKH, P.AK, P.AKH1, E, EH, g,
                                                                                     tail);
    KPM_CUDA(cudaGetLastError());
    h->total_launches++;
    return KPM_OK;
}

template <int KS, int TL, int TX>
kpm_status launch_tmak_s(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                         const CUtensorMap& EH, const kpm::TmaKGeom& g, int tail) {
    const bool on = h->d_eps != nullptr;
    if (is_cplx(h)) {
        if (on) return launch_tmak_t<KS, TL, TX, true, true>(h, p, A, P, E, EH, g, tail);
        return launch_tmak_t<KS, TL, TX, false, true>(h, p, A, P, E, EH, g, tail);
    }
    if (on) return launch_tmak_t<KS, TL, TX, true, false>(h, p, A, P, E, EH, g, tail);
    return launch_tmak_t<KS, TL, TX, false, false>(h, p, A, P, E, EH, g, tail);
}

// instantiated shapes of the KS-step kernel (see stepk_smem)
kpm_status launch_tmak(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                       const CUtensorMap& EH, const kpm::TmaKGeom& g, int tail) {
    if (p.KSK == 4 && p.TLK == 16) return launch_tmak_s<4, 16, 32>(h, p, A, P, E, EH, g, tail);
    if (p.KSK == 4 && p.TLK == 8) return launch_tmak_s<4, 8, 64>(h, p, A, P, E, EH, g, tail);
    if (p.KSK == 3 && p.TLK == 16) return launch_tmak_s<3, 16, 32>(h, p, A, P, E, EH, g, tail);
    if (p.KSK == 3 && p.TLK == 8) return launch_tmak_s<3, 8, 64>(h, p, A, P, E, EH, g, tail);
    return fail(KPM_ERR_UNSUPPORTED, "no KS-step kernel for KS=%d TL=%d", p.KSK, p.TLK);
}
#else
kpm_status launch_tmak(kpm_handle_s*, const Plan&, const BufMaps&, const BufMaps&, const CUtensorMap&, const CUtensorMap&,
                       const kpm::TmaKGeom&, int) {
    return fail(KPM_ERR_UNSUPPORTED, "KS-step kernel: experimental build only (libkpm_exp.so)");
}
#endif

// eps~ in the x-row frame layout [L2][L1][L0+4] with a box of bx x by sites (3D two-step kernel)
kpm_status make_epsf_map(const kpm_handle_s* h, int bx, int by, CUtensorMap* m) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t pitch = (cuuint64_t)h->L[0] + 4;
    cuuint64_t dims[3] = {pitch, (cuuint64_t)h->L[1], (cuuint64_t)h->L[2]};
    cuuint64_t strides[2] = {pitch * 8, pitch * h->L[1] * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, h->d_epsf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KPM_ERR_CUDA, "cuTensorMapEncodeTiled (eps frame) failed: %d", (int)r);
    return KPM_OK;
}

#ifdef KPM_EXPERIMENTAL
template <int TX, int TY, int TL, bool ONSITE, int NT, int KA = kKA32, int KP = kKP32>
kpm_status launch_tma32_t(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                          const CUtensorMap& E1, const kpm::Tma32Geom& g, int tail) {
    auto kern = kpm::kpm_step32_tma_kernel<TX, TY, TL, ONSITE, NT, KA, KP>;
    KPM_TRY(set_smem((const void*)kern, p.tma32_smem, h->device));
    kern<<<p.tma32_grid, NT, p.tma32_smem, h->stream>>>(A.A32, A.A32r, P.P32, P.P32r, E, E1, g, tail);
    KPM_CUDA(cudaGetLastError());
    h->total_launches++;
    return KPM_OK;
}

// instantiated shapes of the 3D two-step kernel (see step32_smem)
kpm_status launch_tma32(kpm_handle_s* h, const Plan& p, const BufMaps& A, const BufMaps& P, const CUtensorMap& E,
                        const CUtensorMap& E1, const kpm::Tma32Geom& g, int tail) {
    const bool on = h->d_eps != nullptr;
    if (p.TX32 == 8 && p.TY32 == 8 && p.TL32 == 8) {
        return on ? launch_tma32_t<8, 8, 8, true, 256>(h, p, A, P, E, E1, g, tail)
                  : launch_tma32_t<8, 8, 8, false, 256>(h, p, A, P, E, E1, g, tail);
    }
    if (p.TX32 == 16 && p.TY32 == 4 && p.TL32 == 8)
        return on ? launch_tma32_t<16, 4, 8, true, 256>(h, p, A, P, E, E1, g, tail) : launch_tma32_t<16, 4, 8, false, 256>(h, p, A, P, E, E1, g, tail);
    if (p.TX32 == 8 && p.TY32 == 4 && p.TL32 == 16)
        return on ? launch_tma32_t<8, 4, 16, true, 256>(h, p, A, P, E, E1, g, tail) : launch_tma32_t<8, 4, 16, false, 256>(h, p, A, P, E, E1, g, tail);
    if (p.TX32 == 16 && p.TY32 == 8 && p.TL32 == 8)
        return on ? launch_tma32_t<16, 8, 8, true, 256, 3, 2>(h, p, A, P, E, E1, g, tail)
                  : launch_tma32_t<16, 8, 8, false, 256, 3, 2>(h, p, A, P, E, E1, g, tail);
    return fail(KPM_ERR_UNSUPPORTED, "no 3D two-step kernel for %dx%dx%d", p.TX32, p.TY32, p.TL32);
}
#else
kpm_status launch_tma32(kpm_handle_s*, const Plan&, const BufMaps&, const BufMaps&, const CUtensorMap&, const CUtensorMap&,
                        const kpm::Tma32Geom&, int) {
    return fail(KPM_ERR_UNSUPPORTED, "3D two-step kernel: experimental build only (libkpm_exp.so)");
}
#endif

template <int TX, int TY, int TL, bool ONSITE>
kpm_status launch_tma3_t(kpm_handle_s* h, const Plan& p, const BufMaps& cur, const BufMaps& prev, const CUtensorMap& E,
                         const kpm::TmaGeom& g, int tail, int grid) {
    auto kern = kpm::kpm_step3_tma_kernel<TX, TY, TL, ONSITE>;
    KPM_TRY(set_smem((const void*)kern, p.tma_smem, h->device));
    return launch_k(h, h->stream, kern, dim3(grid), dim3(kpm::kTmaThreads), p.tma_smem, cur.Box3, cur.Row3, prev.P, E, g,
                    tail);
}

template <int NDIM, bool ONSITE, bool PEIERLS>
kpm_status launch_tma_t(kpm_handle_s* h, const Plan& p, const BufMaps& cur, const BufMaps& prev, const CUtensorMap& E,
                        const kpm::TmaGeom& g, int tail, int grid) {
    auto kern = kpm::kpm_step_tma_kernel<NDIM, ONSITE, PEIERLS>;
    KPM_TRY(set_smem((const void*)kern, p.tma_smem, h->device));
    return launch_k(h, h->stream, kern, dim3(grid), dim3(kpm::kTmaThreads), p.tma_smem, cur.A, cur.Col, cur.Row, prev.P, E,
                    g, tail);
}

kpm_status launch_tma(kpm_handle_s* h, const Plan& p, const BufMaps& cur, const BufMaps& prev, const CUtensorMap& E,
                      const kpm::TmaGeom& g, int tail, int grid = 0) {
    const bool on = h->d_eps != nullptr;
    if (!grid) grid = p.tma_grid;
    if (h->ndim == 2) {
        if (is_cplx(h)) {
            if (on) return launch_tma_t<2, true, true>(h, p, cur, prev, E, g, tail, grid);
            return launch_tma_t<2, false, true>(h, p, cur, prev, E, g, tail, grid);
        }
        if (on) return launch_tma_t<2, true, false>(h, p, cur, prev, E, g, tail, grid);
        return launch_tma_t<2, false, false>(h, p, cur, prev, E, g, tail, grid);
    }
    if (p.use_tma3) {
        if (p.TL == 16) return on ? launch_tma3_t<8, 8, 16, true>(h, p, cur, prev, E, g, tail, grid)
                                  : launch_tma3_t<8, 8, 16, false>(h, p, cur, prev, E, g, tail, grid);
        if (p.TL == 32) return on ? launch_tma3_t<4, 8, 32, true>(h, p, cur, prev, E, g, tail, grid)
                                  : launch_tma3_t<4, 8, 32, false>(h, p, cur, prev, E, g, tail, grid);
        return on ? launch_tma3_t<16, 8, 8, true>(h, p, cur, prev, E, g, tail, grid)
                  : launch_tma3_t<16, 8, 8, false>(h, p, cur, prev, E, g, tail, grid);
    }
    if (on) return launch_tma_t<3, true, false>(h, p, cur, prev, E, g, tail, grid);
    return launch_tma_t<3, false, false>(h, p, cur, prev, E, g, tail, grid);
}

kpm_status new_handle(int32_t device, const kpm_dist* dist, kpm_handle_s** out) {
    if (!out) return fail(KPM_ERR_INVALID_ARG, "out handle pointer is NULL");
    *out = nullptr;
    if (dist) {
        if (dist->partition != KPM_PART_NONE && dist->partition != KPM_PART_VECTORS && dist->partition != KPM_PART_ROWS)
            return fail(KPM_ERR_UNSUPPORTED, "partition %d not supported", dist->partition);
        if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)
            return fail(KPM_ERR_INVALID_ARG, "bad rank %d / world %d", dist->rank, dist->world);
        if (dist->partition != KPM_PART_NONE) {
            if (dist->comm != KPM_COMM_SELF && dist->comm != KPM_COMM_NCCL && dist->comm != KPM_COMM_LOCAL &&
                dist->comm != KPM_COMM_IPC)
                return fail(KPM_ERR_INVALID_ARG, "bad comm %d", dist->comm);
            if (dist->comm == KPM_COMM_IPC && !dist->ipc_name)
                return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_IPC needs ipc_name");
            if (dist->comm == KPM_COMM_NCCL && !dist->nccl_id)
                return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_NCCL needs nccl_id");
        }
        if (dist->partition == KPM_PART_ROWS) {
            if (dist->comm == KPM_COMM_SELF && dist->world != 1)
                return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_SELF needs world == 1");
            if (dist->vworld > 1 && (dist->vrank < 0 || dist->vrank >= dist->vworld))
                return fail(KPM_ERR_INVALID_ARG, "bad vector group %d of %d", dist->vrank, dist->vworld);
        }
    }
    int ndev = 0;
    KPM_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(KPM_ERR_INVALID_ARG, "device %d not present (%d devices)", device, ndev);
    KPM_CUDA(cudaSetDevice(device));
    auto* h = new kpm_handle_s();
    h->device = device;
    if (dist) h->dist = *dist;
    h->dist.nccl_id = nullptr;  // not kept
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&h->l2_bytes, cudaDevAttrL2CacheSize, device);
    cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;  // keep freed workspace in the pool for the next handle
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev_begin);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev_end);
    if (e != cudaSuccess) {
        kpm_destroy(h);
        return fail(KPM_ERR_CUDA, "stream/event creation failed: %s", cudaGetErrorString(e));
    }
    h->own_stream = true;
    if (dist && dist->partition != KPM_PART_NONE && dist->comm == KPM_COMM_IPC) {
        const kpm_status st = ipc_open(h, dist->ipc_name);
        if (st != KPM_OK) {
            const std::string msg = g_err;
            kpm_destroy(h);
            return fail(st, "%s", msg.c_str());
        }
    }
    h->dist.ipc_name = nullptr;  // not kept
    *out = h;
    return KPM_OK;
}

kpm_status check_ab(double a, double b) {
    if (!(a > 0.0) || !std::isfinite(a) || !std::isfinite(b))
        return fail(KPM_ERR_INVALID_ARG, "scale a must be finite and > 0, shift b finite (a=%g b=%g)", a, b);
    return KPM_OK;
}

kpm_status check_stencil(const kpm_stencil_desc* d) {
    if (!d) return fail(KPM_ERR_INVALID_ARG, "stencil descriptor is NULL");
    if (d->ndim < 1 || d->ndim > 3) return fail(KPM_ERR_INVALID_ARG, "ndim must be 1..3 (got %d)", d->ndim);
    for (int k = 0; k < 3; ++k) {
        if (k < d->ndim && d->L[k] < 2) return fail(KPM_ERR_INVALID_ARG, "L[%d] must be >= 2", k);
        if (k >= d->ndim && d->L[k] != 1) return fail(KPM_ERR_INVALID_ARG, "unused L[%d] must be 1", k);
    }
    const long long D = d->L[0] * d->L[1] * d->L[2];
    if (D >= (1LL << 31)) return fail(KPM_ERR_INVALID_ARG, "D = %lld sites exceeds 2^31 per GPU", D);
    if (!std::isfinite(d->t)) return fail(KPM_ERR_INVALID_ARG, "hopping t not finite");
    if (d->flux != 0.0) {
        if (d->ndim != 2) return fail(KPM_ERR_INVALID_ARG, "Peierls flux needs ndim == 2");
        const double q = d->flux * (double)d->L[0];
        if (!std::isfinite(q) || std::fabs(q - std::nearbyint(q)) > 1e-9)
            return fail(KPM_ERR_INVALID_ARG, "flux * L[0] must be an integer (got %.17g)", q);
    }
    return KPM_OK;
}


// One kpm_moments_ex call as a sequence of phases, so that several slab handles of a
// row partition (KPM_COMM_LOCAL) can be driven in lock step: begin() (plan, workspace,
// start block, first step), launch_next() (one recursion launch: one step, or two with
// the temporal-blocking kernel), fresh() (the block just produced, whose boundary planes
// go to the neighbours), collect() (fixed-order finish of the partial sums), output().
struct Run {
    kpm_handle_s* h = nullptr;
    Plan p;
    int32_t N = 0;
    int64_t R = 0;
    uint32_t flags = 0;
    const void* r0 = nullptr;
    const int64_t* local_sites = nullptr;  // KPM_LOCAL: host list of R global sites
    long long* d_sites = nullptr;
    bool cplx = false, direct = false;
    double2 *P = nullptr, *C = nullptr, *Rb = nullptr, *X2 = nullptr, *X3 = nullptr;  // interiors
    double *part = nullptr, *Sv = nullptr, *S = nullptr, *dout = nullptr;
    size_t slot = 0;
    kpm::VecArgs v{};
    BufMaps maps[4];
    int nmaps = 0;
    CUtensorMap mapE, mapE2, mapEf;  // eps~: single-step box, 2-site box, two-step main box
    CUtensorMap mapEK, mapEKH;       // eps~: KS-step main box (TXK), KS-site box
    kpm::TmaGeom tg{};
    kpm::Tma2Geom tg2{};
    kpm::TriGeom tgt{};
    kpm::QuadGeom tgq{};
    CUtensorMap mapE4;               // eps~: 4-site box (three- and four-step kernels)
    CUtensorMap mapEQ;               // eps~: TXQ box (four-step kernel)
    kpm::TmaKGeom tgk{};
    kpm::Tma32Geom tg32{};
    CUtensorMap mapE32, mapE32r;     // eps~ frame: (TX+4) x TY box, (TX+4) x 1 box (3D two-step kernel)
    double2 *cur = nullptr, *prev = nullptr, *spare0 = nullptr, *spare1 = nullptr;
    int n = 1, nsteps = 0;
    double vbytes = 0, ebytes = 0, mbytes = 0;

    double2* base_of(double2* interior) const { return interior - p.ghost_lanes; }
    const BufMaps& maps_of(const void* b) const {
        for (int i = 0; i < nmaps; ++i)
            if (maps[i].base == b) return maps[i];
        return maps[0];
    }

    kpm_status begin(kpm_handle_s* h_, int32_t N_, int64_t R_, uint64_t seed, const void* r0_, uint32_t flags_) {
        h = h_;
        N = N_;
        R = R_;
        flags = flags_;
        r0 = r0_;
        if (flags & KPM_LOCAL) {
            // unit start vectors e_site: r0 is the host list of R global sites (not a vector block)
            if (!r0) return fail(KPM_ERR_INVALID_ARG, "KPM_LOCAL needs the site list in r0");
            if (flags & (KPM_RAW_SUMS | KPM_DEVICE_IN))
                return fail(KPM_ERR_INVALID_ARG, "KPM_LOCAL: per-site host list only (no raw sums, no device r0)");
            const int64_t* st = static_cast<const int64_t*>(r0);
            for (int64_t i = 0; i < R_; ++i)
                if (st[i] < 0 || st[i] >= h->D_total)
                    return fail(KPM_ERR_INVALID_ARG, "KPM_LOCAL: site %lld out of range [0, %lld)", (long long)st[i],
                                (long long)h->D_total);
            local_sites = st;
            r0 = nullptr;
            flags |= KPM_PER_VECTOR;
        }
        if ((flags & KPM_PER_VECTOR) && (flags & KPM_RAW_SUMS))
            return fail(KPM_ERR_INVALID_ARG, "KPM_PER_VECTOR and KPM_RAW_SUMS are exclusive");
        KPM_CUDA(cudaSetDevice(h->device));
        KPM_TRY(make_plan(h, N, R, flags, r0 != nullptr, &p));
        if (ensure_workspace(h, p.total) != KPM_OK) {
            if (!p.use_tma2 && !p.use_tma32) return KPM_ERR_OOM;
            // four vector blocks do not fit: fall back to in-place single steps (two blocks)
            KPM_TRY(make_plan(h, N, R, flags, r0 != nullptr, &p, true));
            KPM_TRY(ensure_workspace(h, p.total));
        }
        v.sites = nullptr;
        if (local_sites) {
            d_sites = reinterpret_cast<long long*>(h->ws + p.off_sites);
            KPM_CUDA(cudaMemcpyAsync(d_sites, local_sites, (size_t)R * sizeof(long long), cudaMemcpyHostToDevice, h->stream));
            v.sites = d_sites;
        }
        cplx = is_cplx(h);
        direct = (flags & KPM_DIRECT) != 0;
        P = reinterpret_cast<double2*>(h->ws + p.off_P) + p.ghost_lanes;
        C = reinterpret_cast<double2*>(h->ws + p.off_C) + p.ghost_lanes;
        Rb = reinterpret_cast<double2*>(h->ws + p.off_R) + p.ghost_lanes;
        X2 = reinterpret_cast<double2*>(h->ws + p.off_X2) + p.ghost_lanes;
        X3 = reinterpret_cast<double2*>(h->ws + p.off_X3) + p.ghost_lanes;
        part = reinterpret_cast<double*>(h->ws + p.off_part);
        Sv = reinterpret_cast<double*>(h->ws + p.off_Sv);
        S = reinterpret_cast<double*>(h->ws + p.off_S);
        dout = reinterpret_cast<double*>(h->ws + p.off_out);
        slot = (size_t)p.gx * p.RP;  // doubles per moment slot of partials
        h->total_launches = 0;
        h->step_launches = 0;
        h->halo_copies = 0;
        h->fused_halo_launches = 0;
        h->steps_bytes = 0.0;
        h->design_bytes = 0.0;

        v.P = P;
        v.C = C;
        v.Rbuf = Rb;
        v.D = (int)h->D;
        v.RG = p.RG;
        v.RP = p.RP;
        v.R_loc = p.R_loc;
        v.key = kpm::vector_key(seed);
        v.r_off = p.r_off;
        v.D_total = h->D_total;
        v.i_off = h->rows ? h->z0 * h->plane : 0;
        v.ghost = h->rows ? 1 : 0;
        v.gmap = h->kind == KIND_ELL ? h->d_gmap : nullptr;
        v.L0 = (int)h->L[0];
        v.xpad = p.xpad;

        // a_0: generated in the first-step kernel, or the caller's block staged through C.
        int first_mode = kpm::FIRST_GEN;
        if (r0) {
            const size_t rbytes = (size_t)p.R_loc * h->D * sizeof(double);
            double* stage = reinterpret_cast<double*>(base_of(C));
            if (h->kind == KIND_DENSE) KPM_CUDA(cudaMemsetAsync(P, 0, p.lane_bytes, h->stream));
            KPM_CUDA(cudaMemcpyAsync(stage, r0, rbytes,
                                     (flags & KPM_DEVICE_IN) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
            const long long ne = h->D * (long long)p.RG;
            const int blocks = (int)std::min<long long>((ne + 255) / 256, 8LL * h->num_sms);
            const double* cstage = stage;
            if (cplx) KPM_TRY(launch_k(h, h->stream, kpm::load_r0_kernel<true>, dim3(blocks), dim3(256), 0, cstage, P, v));
            else KPM_TRY(launch_k(h, h->stream, kpm::load_r0_kernel<false>, dim3(blocks), dim3(256), 0, cstage, P, v));
            if (direct) KPM_CUDA(cudaMemcpyAsync(Rb, P, p.mem_sites * p.RG * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream));
            first_mode = kpm::FIRST_BUF;
        }
        if (first_mode == kpm::FIRST_BUF && h->rows) KPM_TRY(need_exchange(P));
        if (h->kind == KIND_DENSE) return begin_dense(first_mode);
        if (p.use_persist) {  // the whole recursion in one cooperative launch (kpm_persist.cuh)
            KPM_CUDA(cudaEventRecord(h->ev_begin, h->stream));
            KPM_TRY(launch_persist(h, p, v, first_mode == kpm::FIRST_BUF, N, (long long)slot, part));
            h->step_launches = 1;
            const double s_el = cplx ? 16.0 : 8.0;
            const double vb = (double)h->D * (double)p.R_loc * s_el;
            const double mb = h->kind == KIND_ELL ? (double)h->K * (double)h->D * (4.0 + s_el) : 0.0;
            h->steps_bytes = 2.0 * vb + (p.M - 1) * (3.0 * vb + (h->d_eps ? 8.0 * (double)h->D : 0.0) + mb);
            h->design_bytes = h->steps_bytes;
            nsteps = 0;
            n = 1;
            return KPM_OK;
        }
        if (p.use_small) {  // the whole recursion in one launch (kpm_small.cuh)
            KPM_CUDA(cudaEventRecord(h->ev_begin, h->stream));
            KPM_TRY(launch_small(h, p, v, first_mode == kpm::FIRST_BUF, N, part));
            h->step_launches = 1;
            nsteps = 0;
            n = 1;
            return KPM_OK;
        }
        // First step: a_0, a_1 = H~ a_0; S_0 = <a_0|a_0>, S_1 = <a_0|a_1> (Eq 17, 19).
        v.red0 = part;
        v.red1 = N > 1 ? part + slot : nullptr;
        v.red2 = (!direct && N == 3) ? part + 2 * slot : nullptr;
        // 2D/3D stencils: a_0 hashed once per element into a shared-memory plane ring
        // (kpm_first.cuh); else the generic grid-stride kernel
        if ((first_mode == kpm::FIRST_GEN || first_mode == kpm::FIRST_BUF) && h->kind == KIND_STENCIL && h->ndim >= 2 &&
            !h->opts.no_first_tile)
            KPM_TRY(launch_first_tile(h, p, v, v.red2 != nullptr, first_mode == kpm::FIRST_BUF));
        else
            KPM_TRY(launch(h, p, first_mode, v, v.red2 != nullptr));

        // Recursion launches (Eq 18).  Single-step launches write a_{n+1} over a_{n-1} in place;
        // two-step launches (kpm_tma2.cuh) read (a_n, a_{n-1}) and write (a_{n+1}, a_{n+2}) into
        // the two spare blocks, after which the pairs swap roles.
        nsteps = direct ? std::max(0, N - 2) : std::max(0, p.M - 1);
        memset(&mapE, 0, sizeof mapE);
        memset(&mapE2, 0, sizeof mapE2);
        memset(&mapE4, 0, sizeof mapE4);
        memset(&mapEQ, 0, sizeof mapEQ);
        memset(&mapEf, 0, sizeof mapEf);
        memset(&mapEK, 0, sizeof mapEK);
        memset(&mapEKH, 0, sizeof mapEKH);
        memset(&mapE32, 0, sizeof mapE32);
        memset(&mapE32r, 0, sizeof mapE32r);
        if (p.use_tma && nsteps > 0) {
            double2* bufs[4] = {P, C, X2, X3};
            nmaps = (p.use_tma2 || p.use_tmak || p.use_tma32) ? 4 : 2;
            for (int i = 0; i < nmaps; ++i) KPM_TRY(make_buf_maps(h, p, base_of(bufs[i]), &maps[i]));
            if (h->d_eps) {
                KPM_TRY(make_eps_map(h, p, &mapE));
                if (p.use_tma2) {
                    KPM_TRY(make_eps_map_w(h, p, 2, &mapE2));
                    KPM_TRY(make_eps_map_w(h, p, p.TX2, &mapEf));
                }
                if (p.use_tri || p.use_quad) KPM_TRY(make_eps_map_w(h, p, 4, &mapE4));
                if (p.use_quad) KPM_TRY(make_eps_map_w(h, p, p.TXQ, &mapEQ));
                if (p.use_tma32) {
                    KPM_TRY(make_epsf_map(h, p.TX32 + 4, p.TY32, &mapE32));
                    KPM_TRY(make_epsf_map(h, p.TX32 + 4, 1, &mapE32r));
                }
                if (p.use_tmak) {
                    KPM_TRY(make_eps_map_w(h, p, p.TXK, &mapEK));
                    KPM_TRY(make_eps_map_w(h, p, (p.KSK + 1) / 2 * 2, &mapEKH));
                }
            }
            tg.L0 = (int)h->L[0];
            tg.L1 = (int)h->L[1];
            tg.L2 = (int)h->L[2];
            tg.TX = p.TX;
            tg.TY = p.TY;
            tg.TL = p.TL;
            tg.RG = p.RG;
            tg.G_L = p.RG / p.TL;
            tg.PX = (int)(h->L[0] / p.TX);
            tg.PY = h->ndim == 3 ? (int)(h->L[1] / p.TY) : 1;
            tg.Lm = (int)(h->ndim == 2 ? h->L[1] : h->L[2]);
            tg.W = (long long)tg.G_L * tg.PX * tg.PY * tg.Lm;
            tg.rr = p.tma_rr;
            {
                auto log2i = [](int v) { int b = 0; while ((1 << b) < v) ++b; return (1 << b) == v ? b : -1; };
                const int bx = log2i(tg.PX), by = log2i(tg.PY);
                tg.zbx = (bx >= 0 && by >= 0 && h->ndim == 3 && !h->opts.no_zorder) ? bx : -1;
                tg.zby = tg.zbx >= 0 ? by : -1;
            }
            tg.ghost = h->rows ? 1 : 0;
            tg.RP = p.RP;
            tg.rows_total = p.gx;
            tg.row_off = 0;
            tg.zoff = 0;
            tg.peer_lo = tg.peer_hi = nullptr;  // fused halo: set per launch by kpm_moments_group
            tg.plane_lanes = (long long)p.ghost_lanes;
            tg.nloc = (int)h->nloc;
            tg.xpad = p.xpad;
            tg.t = h->t_scaled;
            tg.shift = -h->b / h->a;
            tg.phase = h->d_phase;
            tg2.L0 = tg.L0;
            tg2.L1 = tg.L1;
            tg2.TX = p.TX2;
            tg2.TL = p.TL;
            tg2.RG = p.RG;
            tg2.G_L = tg.G_L;
            tg2.PX = p.TX2 ? (int)(h->L[0] / p.TX2) : 0;
            tg2.W = (long long)tg.G_L * tg2.PX * tg.L1;
            tg2.RP = p.RP;
            tg2.rows_total = p.gx;
            tg2.t = tg.t;
            tg2.shift = tg.shift;
            tg2.phase = tg.phase;
            tgt.L0 = tg2.L0;
            tgt.L1 = tg2.L1;
            tgt.TX = tg2.TX;
            tgt.TL = tg2.TL;
            tgt.RG = tg2.RG;
            tgt.G_L = tg2.G_L;
            tgt.PX = tg2.PX;
            tgt.W = tg2.W;
            tgt.RP = tg2.RP;
            tgt.rows_total = p.gx;
            tgt.t = tg.t;
            tgt.shift = tg.shift;
            tgt.phase = tg.phase;
            tgq.L0 = tg2.L0;
            tgq.L1 = tg2.L1;
            tgq.TX = p.TXQ;
            tgq.TL = p.TLQ;
            tgq.RG = tg2.RG;
            tgq.G_L = p.TLQ ? p.RG / p.TLQ : 0;
            tgq.PX = p.TXQ ? (int)(h->L[0] / p.TXQ) : 0;
            tgq.W = (long long)tgq.G_L * tgq.PX * tg2.L1;
            tgq.RP = tg2.RP;
            tgq.rows_total = p.gx;
            tgq.t = tg.t;
            tgq.shift = tg.shift;
            tgq.phase = tg.phase;
            tgk.L0 = tg.L0;
            tgk.L1 = tg.L1;
            tgk.TX = p.TXK;
            tgk.TL = p.TLK;
            tgk.RG = p.RG;
            tgk.G_L = p.TLK ? p.RG / p.TLK : 0;
            tgk.PX = p.TXK ? (int)(h->L[0] / p.TXK) : 0;
            tgk.W = (long long)tgk.G_L * tgk.PX * tg.L1;
            tgk.RP = p.RP;
            tgk.t = tg.t;
            tgk.shift = tg.shift;
            tgk.phase = tg.phase;
            tgk.slot_stride = (long long)slot;
            tgk.rows_total = p.gx;
            if (p.use_tma32) {
                tg32.L0 = tg.L0;
                tg32.L1 = tg.L1;
                tg32.L2 = tg.L2;
                tg32.PX = (int)(h->L[0] / p.TX32);
                tg32.PY = (int)(h->L[1] / p.TY32);
                tg32.G_L = p.RG / p.TL32;
                tg32.RG = p.RG;
                tg32.RP = p.RP;
                const long long cols = (long long)tg32.G_L * tg32.PX * tg32.PY;
                tg32.rr = p.tma32_rr;
                tg32.W = p.tma32_rr ? cols : cols * tg32.L2;
                tg32.rows_total = p.gx;
                tg32.pfirst = 1;   // measured: evict-first a_{n-1} 5.3 GB vs 6.2 GB DRAM reads
                tg32.lg_fast = 0;
                tg32.t = tg.t;
                tg32.shift = tg.shift;
            }
        }
        cur = C;
        prev = P;
        spare0 = X2;
        spare1 = X3;
        n = 1;
        const double s_el = cplx ? 16.0 : 8.0;
        vbytes = (double)h->D * (double)p.R_loc * s_el;
        ebytes = h->d_eps ? 8.0 * (double)h->D : 0.0;
        mbytes = h->kind == KIND_ELL ? (double)h->K * (double)h->D * (4.0 + s_el) : 0.0;
        KPM_CUDA(cudaEventRecord(h->ev_begin, h->stream));
        return KPM_OK;
    }

    // Dense H~ (kpm_dense.cuh): a_0 materialised (generated here, or the caller's block already
    // loaded into P), then a_1 = H~ a_0 by the GEMM kernel with the fused sums S_0, S_1.
    kpm_status begin_dense(int first_mode) {
        if (direct) return fail(KPM_ERR_UNSUPPORTED, "KPM_DIRECT is not implemented for dense H");
        if (first_mode != kpm::FIRST_BUF) {
            const long long ne = h->Dp * (long long)p.RG;
            const int blocks = (int)std::min<long long>((ne + 255) / 256, 8LL * h->num_sms);
            KPM_TRY(launch_k(h, h->stream, kpm::dense_gen_kernel<false>, dim3(blocks), dim3(256), 0, v, (int)h->Dp, P));
        }
        v.red0 = part;
        v.red1 = part + slot;  // the partial buffer has >= 3 slots (slot 1 unused when N = 1)
        v.red2 = (N == 3) ? part + 2 * slot : nullptr;
        KPM_TRY(launch_dense(true, P, C, v.red0, v.red1, v.red2, v.red2 != nullptr));
        nsteps = std::max(0, p.M - 1);
        cur = C;
        prev = P;
        n = 1;
        vbytes = (double)h->Dp * (double)p.RP * 8.0;
        ebytes = 0.0;
        mbytes = 8.0 * (double)h->Dp * (double)h->Dp;
        KPM_CUDA(cudaEventRecord(h->ev_begin, h->stream));
        return KPM_OK;
    }
    kpm_status launch_dense(bool first, double2* A, double2* out, double* r0_, double* r1_, double* r2_, int tail) {
        kpm::DenseArgs g;
        g.H = h->d_dense;
        g.A = reinterpret_cast<const double*>(A);
        g.P = reinterpret_cast<double*>(out);
        g.Dp = (int)h->Dp;
        g.RP = p.RP;
        g.shift = -h->b / h->a;
        g.red0 = r0_;
        g.red1 = r1_;
        g.red2 = r2_;
        dim3 grid(p.RP / kpm::kDBN, (unsigned)(h->Dp / kpm::kDBM));
        KPM_TRY(set_smem((const void*)kpm::kpm_dense_step_kernel<true>, kpm::kDenseSmem, h->device));
        KPM_TRY(set_smem((const void*)kpm::kpm_dense_step_kernel<false>, kpm::kDenseSmem, h->device));
        if (first) return launch_k(h, h->stream, kpm::kpm_dense_step_kernel<true>, grid, dim3(kpm::kDThreads), kpm::kDenseSmem, g, tail);
        return launch_k(h, h->stream, kpm::kpm_dense_step_kernel<false>, grid, dim3(kpm::kDThreads), kpm::kDenseSmem, g, tail);
    }

    // Row partition, one recursion step with the halo exchange overlapped:
    // (1) the two boundary planes of a_{n+1} (slab planes 0 and nloc-1), (2) their send/recv
    // into the neighbours' ghost planes on the comm stream, concurrently with (3) the interior
    // planes 1..nloc-2; the next step's launches wait for (2) (event join).  The three launches
    // write disjoint partial-sum row ranges, summed by finish_kernel in a fixed order.
    bool comm_pending = false, exchanged_inline = false;
    kpm_status launch_overlapped(int tail) {
        if (!h->comm_stream) {
            KPM_CUDA(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
            KPM_CUDA(cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming));
            KPM_CUDA(cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
        }
        if (comm_pending) KPM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_comm, 0));  // ghosts of a_n arrived
        const long long cols = tg.W / tg.Lm;
        const int Lm_full = tg.Lm, G = p.tma_grid;
        const BufMaps& mc = maps_of(base_of(cur));
        const BufMaps& mp = maps_of(base_of(prev));
        auto sub = [&](int z0, int nz, int row_off) -> kpm_status {
            kpm::TmaGeom g2 = tg;
            g2.zoff = z0;
            g2.Lm = nz;
            g2.W = cols * nz;
            const int grid = (int)std::min<long long>(g2.W, (long long)h->num_sms);
            g2.rr = (h->ndim == 3 && cols >= 4LL * grid) ? 1 : 0;
            g2.row_off = row_off;
            g2.rows_total = G;
            return launch_tma(h, p, mc, mp, mapE, g2, tail, grid);
        };
        KPM_TRY(sub(0, 1, G));
        KPM_TRY(sub(Lm_full - 1, 1, 2 * G));
        KPM_CUDA(cudaEventRecord(h->ev_bnd, h->stream));
        KPM_CUDA(cudaStreamWaitEvent(h->comm_stream, h->ev_bnd, 0));
        KPM_TRY(exchange_on(prev, h->comm_stream));
        KPM_CUDA(cudaEventRecord(h->ev_comm, h->comm_stream));
        comm_pending = true;
        exchanged_inline = true;
        return sub(1, Lm_full - 2, 0);
    }
    // join the comm stream before the partial sums are read
    kpm_status join_comm() {
        if (comm_pending) KPM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_comm, 0));
        comm_pending = false;
        return KPM_OK;
    }

    // ghost planes of `X` must be refreshed before the next launch (recorded; done by the caller)
    double2* pending = nullptr;
    kpm_status need_exchange(double2* X) {
        pending = X;
        if (exchanged_inline) {  // the overlapped step already sent them
            exchanged_inline = false;
            return KPM_OK;
        }
        return exchange_hook ? exchange_hook(this) : KPM_OK;
    }
    kpm_status exchange_on(double2* X, cudaStream_t st);
    // General sparse row partition: pack the rows each peer needs, NCCL send/recv straight into
    // the ghost range of that peer (ghosts are grouped by owner).  World 1 has no ghosts.
    kpm_status exchange_ell(double2* X, cudaStream_t st) {
        if (h->dist.world == 1 || (h->n_ghost == 0 && h->n_send == 0)) return KPM_OK;
        if (h->dist.comm != KPM_COMM_NCCL || !h->nccl) return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_LOCAL handles need kpm_moments_group");
        double2* sendbuf = reinterpret_cast<double2*>(h->ws + p.off_send);
        if (h->n_send) {
            const long long ne = h->n_send * (long long)p.RG;
            const int blocks = (int)std::min<long long>((ne + 255) / 256, 8LL * h->num_sms);
            const double2* cX = X;
            const int* cidx = h->d_send;
            KPM_TRY(launch_k(h, st, kpm::gather_lanes_kernel, dim3(blocks), dim3(256), 0, cX, cidx, (long long)h->n_send, p.RG, sendbuf));
        }
        const size_t lb = (size_t)p.RG * sizeof(double2);
        ncclResult_t e = ncclGroupStart();
        for (int q = 0; q < h->dist.world && e == ncclSuccess; ++q) {
            if (h->scnt[q]) e = ncclSend(sendbuf + h->soff[q] * p.RG, h->scnt[q] * lb, ncclUint8, q, h->nccl, st);
            if (e == ncclSuccess && h->rcnt[q])
                e = ncclRecv(X + (h->D + h->roff[q]) * p.RG, h->rcnt[q] * lb, ncclUint8, q, h->nccl, st);
        }
        ncclResult_t e2 = ncclGroupEnd();
        if (e != ncclSuccess || e2 != ncclSuccess) return nccl_fail(h, e != ncclSuccess ? e : e2, "NCCL ghost exchange");
        return nccl_poll(h);
    }
    kpm_status (*exchange_hook)(Run*) = nullptr;

    bool more() const { return n <= nsteps; }
    // the vector partition's all-reduce of S runs inside the library (KPM_COMM_NCCL)
    bool vector_collective() const {
        return !h->rows && h->dist.partition == KPM_PART_VECTORS &&
               ((h->dist.comm == KPM_COMM_NCCL && h->nccl) || h->dist.comm == KPM_COMM_IPC) &&
               !(flags & (KPM_RAW_SUMS | KPM_PER_VECTOR));
    }
    double2* fresh() const { return cur; }

    kpm_status launch_next() {
        if (h->kind == KIND_DENSE) {  // Eq (18) as a GEMM with the fused epilogue, in place over a_{n-1}
            const bool tail = (N & 1) && n == nsteps;
            KPM_TRY(launch_dense(false, cur, prev, part + (size_t)(2 * n) * slot, part + (size_t)(2 * n + 1) * slot,
                                 tail ? part + (size_t)(2 * n + 2) * slot : nullptr, tail));
            h->steps_bytes += 3.0 * vbytes + mbytes;
            h->design_bytes += 3.0 * vbytes + mbytes;
            h->step_launches++;
            std::swap(cur, prev);
            ++n;
            return KPM_OK;
        }
        if (!direct && p.use_tmak && n + p.KSK - 1 <= nsteps) {
            // steps n .. n+KS-1: slots 2n .. 2n+2KS-1 (+ odd-N tail 2(n+KS))
            const int KS = p.KSK;
            const bool tail = (N & 1) && n + KS - 1 == nsteps;
            tgk.red = part + (size_t)(2 * n) * slot;
            tgk.outB = spare0;
            tgk.outC = spare1;
            KPM_TRY(launch_tmak(h, p, maps_of(base_of(cur)), maps_of(base_of(prev)), mapEK, mapEKH, tgk, tail));
            double2* oc = cur;
            double2* op = prev;
            cur = spare1;
            prev = spare0;
            spare0 = oc;
            spare1 = op;
            h->steps_bytes += KS * (3.0 * vbytes + ebytes);  // KS steps
            h->design_bytes += 4.0 * vbytes + ebytes;
            h->step_launches++;
            n += KS;
            return KPM_OK;
        }
        if (!direct && p.use_tma32 && n + 1 <= nsteps && !(n == 1 && (nsteps & 1))) {
            // steps n and n+1 (3D): slots 2n .. 2n+3 (+ odd-N tail 2n+4)
            const bool tail = (N & 1) && n + 1 == nsteps;
            for (int k = 0; k < 4; ++k) tg32.red[k] = part + (size_t)(2 * n + k) * slot;
            tg32.red[4] = tail ? part + (size_t)(2 * n + 4) * slot : nullptr;
            tg32.outB = spare0;
            tg32.outC = spare1;
            KPM_TRY(launch_tma32(h, p, maps_of(base_of(cur)), maps_of(base_of(prev)), mapE32, mapE32r, tg32, tail));
            double2* oc = cur;
            double2* op = prev;
            cur = spare1;
            prev = spare0;
            spare0 = oc;
            spare1 = op;
            h->steps_bytes += 2.0 * (3.0 * vbytes + ebytes);  // two steps
            h->design_bytes += 4.0 * vbytes + ebytes;        // a_n, a_{n-1} read, a_{n+1}, a_{n+2} written once
            h->step_launches++;
            n += 2;
            return KPM_OK;
        }
        // four-step launches (kpm_quad.cuh): the remainder of the step count goes first (a three-step
        // launch, a pair or a single step), then every launch advances four steps
        const int left = nsteps - n + 1;
        if (!direct && p.use_quad && left >= 4 && left % 4 == 0) {
            // steps n .. n+3: slots 2n .. 2n+7 (+ odd-N tail 2n+8)
            const bool tail = (N & 1) && n + 3 == nsteps;
            for (int k = 0; k < 8; ++k) tgq.red[k] = part + (size_t)(2 * n + k) * slot;
            tgq.red[8] = tail ? part + (size_t)(2 * n + 8) * slot : nullptr;
            tgq.outB = spare0;
            tgq.outC = spare1;
            KPM_TRY(launch_quad(h, p, maps_of(base_of(cur)), maps_of(base_of(prev)), mapEQ, mapE4, tgq, tail));
            double2* oc = cur;
            double2* op = prev;
            cur = spare1;
            prev = spare0;
            spare0 = oc;
            spare1 = op;
            h->steps_bytes += 4.0 * (3.0 * vbytes + ebytes);  // four steps
            h->design_bytes += 4.0 * vbytes + ebytes;         // a_n, a_{n-1} read, a_{n+3}, a_{n+4} written once
            h->step_launches++;
            n += 4;
            return KPM_OK;
        }
        // three-step launches (kpm_tri.cuh): the remainder of the step count goes first as one pair
        // or one single step, then every launch advances three steps
        if (!direct && p.use_tri && left >= 3 && (p.use_quad ? left % 4 == 3 : left % 3 == 0)) {
            // steps n, n+1, n+2: slots 2n .. 2n+5 (+ odd-N tail 2n+6)
            const bool tail = (N & 1) && n + 2 == nsteps;
            for (int k = 0; k < 6; ++k) tgt.red[k] = part + (size_t)(2 * n + k) * slot;
            tgt.red[6] = tail ? part + (size_t)(2 * n + 6) * slot : nullptr;
            tgt.outB = spare0;
            tgt.outC = spare1;
            KPM_TRY(launch_tri(h, p, maps_of(base_of(cur)), maps_of(base_of(prev)), mapEf, mapE4, tgt, tail));
            double2* oc = cur;
            double2* op = prev;
            cur = spare1;
            prev = spare0;
            spare0 = oc;
            spare1 = op;
            h->steps_bytes += 3.0 * (3.0 * vbytes + ebytes);  // three steps
            h->design_bytes += 4.0 * vbytes + ebytes;         // a_n, a_{n-1} read, a_{n+2}, a_{n+3} written once
            h->step_launches++;
            n += 3;
            return KPM_OK;
        }
        const bool pair = !direct && p.use_tma2 && n + 1 <= nsteps &&
                          (p.use_quad ? left % 4 == 2 : (p.use_tri ? left % 3 == 2 : !(n == 1 && (nsteps & 1))));
        if (pair) {
            // steps n and n+1: slots 2n .. 2n+3 (+ odd-N tail 2n+4)
            const bool tail = (N & 1) && n + 1 == nsteps;
            for (int k = 0; k < 4; ++k) tg2.red[k] = part + (size_t)(2 * n + k) * slot;
            tg2.red[4] = tail ? part + (size_t)(2 * n + 4) * slot : nullptr;
            tg2.outB = spare0;
            tg2.outC = spare1;
            KPM_TRY(launch_tma2(h, p, maps_of(base_of(cur)), maps_of(base_of(prev)), mapEf, mapE2, tg2, tail));
            double2* oc = cur;
            double2* op = prev;
            cur = spare1;
            prev = spare0;
            spare0 = oc;
            spare1 = op;
            h->steps_bytes += 2.0 * (3.0 * vbytes + ebytes);  // two steps
            h->design_bytes += 4.0 * vbytes + ebytes;        // a_n, a_{n-1} read, a_{n+1}, a_{n+2} written once
            h->step_launches++;
            n += 2;
            return KPM_OK;
        }
        v.C = cur;
        v.P = prev;
        if (direct) {
            v.red0 = part + (size_t)(n + 1) * slot;  // <r|a_{n+1}> -> mu_{n+1}
            v.red1 = v.red2 = nullptr;
            KPM_TRY(launch(h, p, r0 ? kpm::DIRECT_BUF : kpm::DIRECT_GEN, v, 0));
            h->steps_bytes += 3.0 * vbytes + ebytes + mbytes + (r0 ? vbytes : 0.0);
            h->design_bytes += 3.0 * vbytes + ebytes + mbytes + (r0 ? vbytes : 0.0);
        } else {
            v.red0 = part + (size_t)(2 * n) * slot;      // <a_n|a_n>     -> mu_{2n}
            v.red1 = part + (size_t)(2 * n + 1) * slot;  // <a_n|a_{n+1}> -> mu_{2n+1}
            const bool tail = (N & 1) && n == nsteps;    // odd N: <a_M|a_M> -> mu_{N-1}
            v.red2 = tail ? part + (size_t)(2 * n + 2) * slot : nullptr;
            if (p.use_tma && p.overlap) {
                tg.red0 = v.red0;
                tg.red1 = v.red1;
                tg.red2 = v.red2;
                tg.out = base_of(prev);
                KPM_TRY(launch_overlapped(tail));
            } else if (p.use_tma) {
                tg.red0 = v.red0;
                tg.red1 = v.red1;
                tg.red2 = v.red2;
                tg.out = base_of(prev);
                KPM_TRY(launch_tma(h, p, maps_of(base_of(cur)), maps_of(base_of(prev)), mapE, tg, tail));
            } else {
                KPM_TRY(launch(h, p, kpm::STEP, v, tail));
            }
            h->steps_bytes += 3.0 * vbytes + ebytes + mbytes;
            h->design_bytes += 3.0 * vbytes + ebytes + mbytes;
        }
        h->step_launches++;
        std::swap(cur, prev);
        ++n;
        return KPM_OK;
    }

    // Fixed-order finish of the CTA partials: Sv[m][v] and S[m] on the device.
    kpm_status collect() {
        KPM_TRY(join_comm());
        KPM_CUDA(cudaEventRecord(h->ev_end, h->stream));
        const double* cpart = part;
        return launch_k(h, h->stream, kpm::finish_kernel, dim3(N), dim3(256), 0, cpart, p.gx, p.RP, p.R_loc, Sv, S);
    }

    kpm_status output(void* out) {
        const bool dev_out = (flags & KPM_DEVICE_OUT) != 0;
        size_t out_bytes = 0;
        const double* src = nullptr;
        if (flags & KPM_RAW_SUMS) {
            src = S;
            out_bytes = (size_t)N * sizeof(double);
        } else if (flags & KPM_PER_VECTOR) {
            const long long ne = (long long)N * p.R_loc;
            const double* cSv = Sv;
            KPM_TRY(launch_k(h, h->stream, kpm::assemble_pervec_kernel, dim3((unsigned)((ne + 255) / 256)), dim3(256), 0, cSv,
                             N, p.R_loc, local_sites ? 1.0 : 1.0 / (double)h->D_total, (int)direct, dout));
            src = dout;
            out_bytes = (size_t)ne * sizeof(double);
        } else {
            const bool multi = h->dist.partition == KPM_PART_VECTORS && h->dist.world > 1;
            if (multi && !vector_collective())
                return fail(KPM_ERR_INVALID_ARG,
                            "multi-rank vector partition without KPM_COMM_NCCL: use KPM_RAW_SUMS, all-reduce, then kpm_assemble");
            // S holds the sums over all R vectors after the all-reduce, else over this rank's R_loc = R
            const double Rn = multi ? (double)R : (double)p.R_loc;
            const double* cS = S;
            KPM_TRY(launch_k(h, h->stream, kpm::assemble_kernel, dim3((N + 255) / 256), dim3(256), 0, cS, N,
                             1.0 / ((double)h->D_total * Rn), (int)direct, dout));
            src = dout;
            out_bytes = (size_t)N * sizeof(double);
        }
        KPM_CUDA(cudaMemcpyAsync(out, src, out_bytes, dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
        if (dev_out) return nccl_poll(h);
        KPM_TRY(sync_stream(h));
        if (!(flags & KPM_RAW_SUMS)) {
            const long long rows = (flags & KPM_PER_VECTOR) ? p.R_loc : 1;
            KPM_TRY(spectrum_guard(static_cast<const double*>(out), rows, N));
        }
        return KPM_OK;
    }

    static kpm_status spectrum_guard(const double* o, long long rows, int N) {
        // |T_n| <= 1 on [-1, 1] (Eq 3) => |mu_n| <= mu_0 when [b-a, b+a] encloses spec(H).
        for (long long r = 0; r < rows; ++r) {
            const double* m = o + r * N;
            for (int k = 0; k < N; ++k)
                if (!std::isfinite(m[k]) || std::fabs(m[k]) > std::fabs(m[0]) * (1.0 + 1e-8) + 1e-300)
                    return fail(KPM_ERR_SPECTRUM, "|mu_%d| = %g exceeds mu_0 = %g: [b-a, b+a] does not enclose the spectrum",
                                k, m[k], m[0]);
        }
        return KPM_OK;
    }

    size_t plane_bytes() const { return p.ghost_lanes * sizeof(double2); }
    // interior plane 0 and nloc-1, ghost planes below and above, of block X
    double2* first_plane(double2* X) const { return X; }
    double2* last_plane(double2* X) const { return X + (h->nloc - 1) * p.ghost_lanes; }
    double2* ghost_lo(double2* X) const { return X - p.ghost_lanes; }
    double2* ghost_hi(double2* X) const { return X + h->nloc * p.ghost_lanes; }
};

// Halo exchange of a single row-partitioned handle: world 1 (periodic wrap inside the
// slab) or NCCL send/recv with the two neighbouring ranks, on the handle's stream.
kpm_status Run::exchange_on(double2* X, cudaStream_t st) {
    if (h->kind == KIND_ELL) return exchange_ell(X, st);
    const size_t pb = plane_bytes();
    if (h->dist.comm == KPM_COMM_SELF) {
        KPM_CUDA(cudaMemcpyAsync(ghost_lo(X), last_plane(X), pb, cudaMemcpyDeviceToDevice, st));
        KPM_CUDA(cudaMemcpyAsync(ghost_hi(X), first_plane(X), pb, cudaMemcpyDeviceToDevice, st));
        return KPM_OK;
    }
    if (h->dist.comm != KPM_COMM_NCCL || !h->nccl) return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_LOCAL handles need kpm_moments_group");
    const int W = h->dist.world, rk = h->dist.rank;
    const int lo = (rk - 1 + W) % W, hi = (rk + 1) % W;
    ncclResult_t e = ncclGroupStart();
    if (e == ncclSuccess) e = ncclSend(first_plane(X), pb, ncclUint8, lo, h->nccl, st);
    if (e == ncclSuccess) e = ncclRecv(ghost_hi(X), pb, ncclUint8, hi, h->nccl, st);
    if (e == ncclSuccess) e = ncclSend(last_plane(X), pb, ncclUint8, hi, h->nccl, st);
    if (e == ncclSuccess) e = ncclRecv(ghost_lo(X), pb, ncclUint8, lo, h->nccl, st);
    ncclResult_t e2 = ncclGroupEnd();
    if (e != ncclSuccess || e2 != ncclSuccess) return nccl_fail(h, e != ncclSuccess ? e : e2, "NCCL halo exchange");
    return nccl_poll(h);
}

// Halo exchange of a single row-partitioned handle (world 1: a local wrap copy; NCCL:
// send/recv with the two neighbouring ranks), on the handle's stream.
kpm_status exchange_single(Run* r) { return r->exchange_on(r->pending, r->h->stream); }

// Halo exchange between the in-process slab handles of a KPM_COMM_LOCAL group: every
// rank pulls its two ghost planes from its neighbours' freshly written blocks once both
// neighbours' streams have reached this point.
kpm_status exchange_group(std::vector<Run>& runs, std::vector<cudaEvent_t>& evs) {
    const int W = (int)runs.size();
    for (int i = 0; i < W; ++i) {
        KPM_CUDA(cudaSetDevice(runs[i].h->device));
        KPM_CUDA(cudaEventRecord(evs[i], runs[i].h->stream));
    }
    if (runs[0].h->kind == KIND_ELL) {
        // every rank gathers its ghost sites, peer by peer, from the owners' fresh blocks
        // (same device: plain loads; see kpm_moments_group)
        for (int i = 0; i < W; ++i) {
            Run& r = runs[i];
            KPM_CUDA(cudaSetDevice(r.h->device));
            for (int q = 0; q < W; ++q) {
                if (!r.h->rcnt[q]) continue;
                KPM_CUDA(cudaStreamWaitEvent(r.h->stream, evs[q], 0));
                const long long n = r.h->rcnt[q], ne = n * r.p.RG;
                const int blocks = (int)std::min<long long>((ne + 255) / 256, 8LL * r.h->num_sms);
                kpm::gather_lanes_kernel<<<blocks, 256, 0, r.h->stream>>>(runs[q].pending, r.h->d_ghost_src + r.h->roff[q], n,
                                                                          r.p.RG, r.pending + (r.h->D + r.h->roff[q]) * r.p.RG);
                KPM_CUDA(cudaGetLastError());
                r.h->total_launches++;
            }
        }
        return KPM_OK;
    }
    for (int i = 0; i < W; ++i) {
        Run& r = runs[i];
        Run& rl = runs[(i - 1 + W) % W];
        Run& rh = runs[(i + 1) % W];
        KPM_CUDA(cudaSetDevice(r.h->device));
        KPM_CUDA(cudaStreamWaitEvent(r.h->stream, evs[(i - 1 + W) % W], 0));
        KPM_CUDA(cudaStreamWaitEvent(r.h->stream, evs[(i + 1) % W], 0));
        double2* X = r.pending;
        KPM_CUDA(cudaMemcpyPeerAsync(r.ghost_lo(X), r.h->device, rl.last_plane(rl.pending), rl.h->device, r.plane_bytes(),
                                     r.h->stream));
        KPM_CUDA(cudaMemcpyPeerAsync(r.ghost_hi(X), r.h->device, rh.first_plane(rh.pending), rh.h->device, r.plane_bytes(),
                                     r.h->stream));
        r.h->halo_copies += 2;
    }
    return KPM_OK;
}

// Random-vector partition over in-process handles (KPM_COMM_LOCAL): every rank's recursion is
// enqueued on its own stream (interleaved launch by launch, so the ranks progress together), then
// the raw sums are added on the host in rank order -- the in-process form of the one all-reduce
// of SURVEY.md 8(e) P1 -- and assembled with the global R.
kpm_status moments_group_vectors(kpm_handle* hs, int32_t nh, int32_t N, int64_t R, uint64_t seed, double* mu) {
    for (int i = 0; i < nh; ++i)
        if (!hs[i] || hs[i]->dist.partition != KPM_PART_VECTORS || hs[i]->dist.comm != KPM_COMM_LOCAL ||
            hs[i]->dist.rank != i || hs[i]->dist.world != nh)
            return fail(KPM_ERR_INVALID_ARG, "handle %d is not rank %d of a KPM_COMM_LOCAL vector partition of %d", i, i, nh);
    std::vector<Run> runs(nh);
    for (int i = 0; i < nh; ++i) KPM_TRY(runs[i].begin(hs[i], N, R, seed, nullptr, 0u));
    bool any = true;
    while (any) {
        any = false;
        for (int i = 0; i < nh; ++i)
            if (runs[i].more()) {
                KPM_CUDA(cudaSetDevice(hs[i]->device));
                KPM_TRY(runs[i].launch_next());
                any = true;
            }
    }
    std::vector<double> Ssum(N, 0.0), Si(N);
    for (int i = 0; i < nh; ++i) {
        KPM_CUDA(cudaSetDevice(hs[i]->device));
        KPM_TRY(runs[i].collect());
    }
    for (int i = 0; i < nh; ++i) {
        KPM_CUDA(cudaSetDevice(hs[i]->device));
        KPM_CUDA(cudaMemcpyAsync(Si.data(), runs[i].S, N * sizeof(double), cudaMemcpyDeviceToHost, hs[i]->stream));
        KPM_CUDA(cudaStreamSynchronize(hs[i]->stream));
        for (int k = 0; k < N; ++k) Ssum[k] += Si[k];  // fixed rank order
    }
    KPM_TRY(kpm_assemble(nullptr, Ssum.data(), N, hs[0]->D_total, R, 0u, mu));
    return Run::spectrum_guard(mu, 1, N);
}

}  // namespace

extern "C" {

const char* kpm_last_error(void) { return g_err.c_str(); }
const char* kpm_version(void) { return "kpm-b200 0.1 (sm_100a)"; }

void kpm_destroy(kpm_handle h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->ws_own && h->ws && !h->ipc) cudaFreeAsync(h->ws, h->stream);
    if (h->d_eps) cudaFreeAsync(h->d_eps, h->stream);
    if (h->d_phase) cudaFreeAsync(h->d_phase, h->stream);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->ws_own && h->ws && h->ipc) cudaFree(h->ws);
    ipc_close(h);
    cudaFree(h->d_epsf);
    cudaFree(h->d_col);
    cudaFree(h->d_val);
    cudaFree(h->d_gmap);
    cudaFree(h->d_ghost_src);
    cudaFree(h->d_send);
    cudaFree(h->d_dense);
    if (h->nccl) comm_release(h->nccl, false);
    if (h->ev_begin) cudaEventDestroy(h->ev_begin);
    if (h->ev_end) cudaEventDestroy(h->ev_end);
    if (h->ev_bnd) cudaEventDestroy(h->ev_bnd);
    if (h->ev_comm) cudaEventDestroy(h->ev_comm);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

kpm_status kpm_gershgorin_stencil(const kpm_stencil_desc* d, double eps, double* a, double* b) {
    KPM_TRY(check_stencil(d));
    if (!a || !b) return fail(KPM_ERR_INVALID_ARG, "a/b output pointers are NULL");
    // Every row: diagonal eps_i, off-diagonal moduli |t| on 2 ndim bonds.
    const long long D = d->L[0] * d->L[1] * d->L[2];
    double lo = 0.0, hi = 0.0;
    if (d->onsite) {
        lo = hi = d->onsite[0];
        for (long long i = 1; i < D; ++i) {
            lo = std::min(lo, d->onsite[i]);
            hi = std::max(hi, d->onsite[i]);
        }
    }
    const double radius = 2.0 * d->ndim * std::fabs(d->t);
    const double Eu = hi + radius + eps, El = lo - radius - eps;
    *a = (Eu - El) / 2.0;
    *b = (Eu + El) / 2.0;
    return KPM_OK;
}

kpm_status kpm_gershgorin_csr(int64_t D, const int64_t* rowptr, const int32_t* col, const void* val, int32_t dtype,
                              double eps, double* a, double* b) {
    if (D < 1 || !rowptr || !col || !val || !a || !b) return fail(KPM_ERR_INVALID_ARG, "bad CSR arguments");
    if (dtype != KPM_REAL64 && dtype != KPM_COMPLEX128) return fail(KPM_ERR_INVALID_ARG, "bad dtype %d", dtype);
    const double* v = static_cast<const double*>(val);
    double Eu = -INFINITY, El = INFINITY;
    for (int64_t i = 0; i < D; ++i) {
        double diag = 0.0, rad = 0.0;
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            const double re = dtype == KPM_REAL64 ? v[k] : v[2 * k];
            const double im = dtype == KPM_REAL64 ? 0.0 : v[2 * k + 1];
            if (col[k] == i) diag += re;
            else rad += std::hypot(re, im);
        }
        Eu = std::max(Eu, diag + rad);
        El = std::min(El, diag - rad);
    }
    Eu += eps;
    El -= eps;
    *a = (Eu - El) / 2.0;
    *b = (Eu + El) / 2.0;
    return KPM_OK;
}

kpm_status kpm_create_stencil(const kpm_stencil_desc* d, double a, double b, int32_t device, const kpm_dist* dist,
                              kpm_handle* out) {
    KPM_TRY(check_stencil(d));
    KPM_TRY(check_ab(a, b));
    kpm_handle_s* h = nullptr;
    KPM_TRY(new_handle(device, dist, &h));
    h->kind = KIND_STENCIL;
    h->dtype = d->flux != 0.0 ? KPM_COMPLEX128 : KPM_REAL64;
    h->a = a;
    h->b = b;
    h->ndim = d->ndim;
    for (int k = 0; k < 3; ++k) h->L[k] = d->L[k];
    h->D = d->L[0] * d->L[1] * d->L[2];
    h->D_total = h->D;
    h->t_scaled = d->t / a;
    kpm_status st = KPM_OK;
    int64_t site0 = 0;  // global index of local site 0
    if (dist && dist->partition == KPM_PART_ROWS) {
        h->rows = true;
        h->slow = d->ndim - 1;
        h->Lm_global = d->L[h->slow];
        h->plane = h->D / h->Lm_global;
        h->z0 = h->Lm_global * dist->rank / dist->world;
        h->nloc = h->Lm_global * (dist->rank + 1) / dist->world - h->z0;
        if (h->nloc < 1) st = fail(KPM_ERR_INVALID_ARG, "rank %d of %d owns no planes", dist->rank, dist->world);
        h->L[h->slow] = h->nloc;
        h->D = h->plane * h->nloc;
        site0 = h->z0 * h->plane;
    }
    if (st == KPM_OK && d->onsite) {
        // raw eps_i of this rank's sites to the device, then Eq (8) on the diagonal there:
        // eps~_i = (eps_i - b) / a (the same correctly rounded ops as a host loop)
        // (stream-ordered pool, like the workspace: a plain cudaFree at kpm_destroy cost up to 0.5 s on c3)
        cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&h->d_eps), h->D * sizeof(double), h->stream);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(h->d_eps, d->onsite + site0, h->D * sizeof(double), cudaMemcpyHostToDevice, h->stream);
        if (ce == cudaSuccess) {
            const int blocks = (int)std::min<long long>((h->D + 255) / 256, 16LL * h->num_sms);
            kpm::rescale_onsite_kernel<<<blocks, 256, 0, h->stream>>>(h->d_eps, (long long)h->D, b, a);
            ce = cudaGetLastError();
        }
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
        if (ce != cudaSuccess) st = fail(KPM_ERR_CUDA, "on-site upload: %s", cudaGetErrorString(ce));
#ifdef KPM_EXPERIMENTAL
        if (st == KPM_OK && h->ndim == 3 && !h->rows) {
            // x-row frame copy for the 3D two-step kernel: row pitch L0 + 4, two periodic images per side
            const size_t L0 = (size_t)h->L[0], rowsN = (size_t)(h->L[1] * h->L[2]), pf = (L0 + 4) * 8;
            ce = cudaMalloc(&h->d_epsf, rowsN * pf);
            if (ce == cudaSuccess) ce = cudaMemcpy2D(h->d_epsf + 2, pf, h->d_eps, L0 * 8, L0 * 8, rowsN, cudaMemcpyDeviceToDevice);
            for (int s2 = 0; s2 < 2 && ce == cudaSuccess; ++s2) {
                // frame x = s2 (site L0-2+s2) and frame x = L0+2+s2 (site s2)
                const size_t src_lo = (L0 - 2 + s2) % L0, src_hi = (size_t)s2 % L0;
                ce = cudaMemcpy2D(h->d_epsf + s2, pf, h->d_eps + src_lo, L0 * 8, 8, rowsN, cudaMemcpyDeviceToDevice);
                if (ce == cudaSuccess)
                    ce = cudaMemcpy2D(h->d_epsf + L0 + 2 + s2, pf, h->d_eps + src_hi, L0 * 8, 8, rowsN, cudaMemcpyDeviceToDevice);
            }
            if (ce != cudaSuccess) st = fail(KPM_ERR_CUDA, "on-site frame: %s", cudaGetErrorString(ce));
        }
#endif
    }
    if (st == KPM_OK && d->flux != 0.0) {
        std::vector<double2> ph(h->L[0]);
        for (int64_t x = 0; x < h->L[0]; ++x) {
            // theta = 2 pi phi x, reduced to 2 pi frac(phi x) before the cos/sin
            const double f = std::fmod(d->flux * (double)x, 1.0);
            ph[x] = make_double2(std::cos(2.0 * CUDART_PI * f), std::sin(2.0 * CUDART_PI * f));
        }
        cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&h->d_phase), h->L[0] * sizeof(double2), h->stream);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(h->d_phase, ph.data(), h->L[0] * sizeof(double2), cudaMemcpyHostToDevice, h->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
        if (ce != cudaSuccess) st = fail(KPM_ERR_CUDA, "phase upload: %s", cudaGetErrorString(ce));
    }
    if (st == KPM_OK) st = init_comm(h, dist);
    if (st != KPM_OK) {
        kpm_destroy(h);
        return st;
    }
    *out = h;
    return KPM_OK;
}

}  // extern "C"

namespace {

// Row partition of an ELL matrix (every rank passes the whole matrix):
// rank g keeps rows [r0, r1) = kpm_slab_range(D, g, W); the columns outside them become ghost
// sites after the local rows (ascending global index = grouped by owner rank, so each peer's
// ghosts are one contiguous receive range); the send lists are the other ranks' ghost sets
// restricted to [r0, r1), computed here from the same matrix (no communication).
struct EllPartition {
    int64_t r0 = 0, nl = 0;
    std::vector<int32_t> ghosts;  // global index of ghost k (ascending)
    std::vector<int32_t> gsrc;    // row of ghost k inside its owner's block
    std::vector<int32_t> send;    // local rows to send, peer by peer
    std::vector<int64_t> roff, rcnt, soff, scnt;
};

// c: [K][D] global columns (padding = the row itself)
kpm_status ell_partition(int64_t D, int64_t K, const int32_t* c, int g, int W, EllPartition* P) {
    if (W < 1 || g < 0 || g >= W) return fail(KPM_ERR_INVALID_ARG, "bad rank %d / world %d", g, W);
    std::vector<int64_t> r0s(W + 1);
    for (int q = 0; q <= W; ++q) r0s[q] = D * q / W;
    P->r0 = r0s[g];
    P->nl = r0s[g + 1] - P->r0;
    if (P->nl < 1) return fail(KPM_ERR_INVALID_ARG, "rank %d of %d owns no rows (D=%lld)", g, W, (long long)D);
    auto owner = [&](int64_t j) { return (int)(std::upper_bound(r0s.begin(), r0s.end(), j) - r0s.begin()) - 1; };
    auto ghosts_of = [&](int q) {  // sorted distinct columns of rank q's rows outside its range
        std::vector<int32_t> gs;
        for (int64_t k = 0; k < K; ++k)
            for (int64_t i = r0s[q]; i < r0s[q + 1]; ++i) {
                const int32_t j = c[k * D + i];
                if (j < r0s[q] || j >= r0s[q + 1]) gs.push_back(j);
            }
        std::sort(gs.begin(), gs.end());
        gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
        return gs;
    };
    P->ghosts = ghosts_of(g);
    P->roff.assign(W, 0);
    P->rcnt.assign(W, 0);
    P->soff.assign(W, 0);
    P->scnt.assign(W, 0);
    P->gsrc.resize(P->ghosts.size());
    for (size_t k = 0; k < P->ghosts.size(); ++k) {
        const int q = owner(P->ghosts[k]);
        if (P->rcnt[q] == 0) P->roff[q] = (int64_t)k;
        P->rcnt[q]++;
        P->gsrc[k] = (int32_t)(P->ghosts[k] - r0s[q]);
    }
    P->send.clear();
    for (int q = 0; q < W; ++q) {
        P->soff[q] = (int64_t)P->send.size();
        if (q != g)
            for (int32_t j : ghosts_of(q))
                if (j >= P->r0 && j < P->r0 + P->nl) P->send.push_back((int32_t)(j - P->r0));
        P->scnt[q] = (int64_t)P->send.size() - P->soff[q];
    }
    return KPM_OK;
}

// Turn handle h into rank dist->rank's block of the row partition; `c`, `v` ([K][D] global) are
// replaced by the local [K][r1-r0] arrays with extended-block columns.
kpm_status ell_rows_setup(kpm_handle_s* h, const kpm_dist* dist, std::vector<int32_t>& c, std::vector<double>& v,
                          int w) {
    const int W = dist->world, g = dist->rank;
    const int64_t D = h->D_total, K = h->K;
    EllPartition P;
    KPM_TRY(ell_partition(D, K, c.data(), g, W, &P));
    const int64_t r0 = P.r0, nl = P.nl;
    const std::vector<int32_t>& mine = P.ghosts;
    h->rows = true;
    h->slow = 0;
    h->plane = 1;
    h->z0 = r0;
    h->nloc = nl;
    h->Lm_global = D;
    h->D = nl;
    h->n_ghost = (int64_t)mine.size();
    h->roff = P.roff;
    h->rcnt = P.rcnt;
    h->soff = P.soff;
    h->scnt = P.scnt;
    std::vector<long long> gmap(mine.begin(), mine.end());
    const std::vector<int32_t>& gsrc = P.gsrc;
    const std::vector<int32_t>& send = P.send;
    h->n_send = (int64_t)send.size();
    // local ELL: rows [r0, r0+nl), columns -> extended block index
    std::vector<int32_t> cl((size_t)K * nl);
    std::vector<double> vl((size_t)K * nl * w);
    for (int64_t k = 0; k < K; ++k)
        for (int64_t i = 0; i < nl; ++i) {
            const int32_t j = c[k * D + r0 + i];
            int32_t jl;
            if (j >= r0 && j < r0 + nl) jl = (int32_t)(j - r0);
            else jl = (int32_t)(nl + (std::lower_bound(mine.begin(), mine.end(), j) - mine.begin()));
            cl[k * nl + i] = jl;
            for (int q = 0; q < w; ++q) vl[(k * nl + i) * w + q] = v[(k * D + r0 + i) * w + q];
        }
    c.swap(cl);
    v.swap(vl);
    cudaError_t ce = cudaSuccess;
    if (h->n_ghost) {
        ce = cudaMalloc(&h->d_gmap, gmap.size() * sizeof(long long));
        if (ce == cudaSuccess) ce = cudaMemcpy(h->d_gmap, gmap.data(), gmap.size() * sizeof(long long), cudaMemcpyHostToDevice);
        if (ce == cudaSuccess) ce = cudaMalloc(&h->d_ghost_src, gsrc.size() * sizeof(int32_t));
        if (ce == cudaSuccess)
            ce = cudaMemcpy(h->d_ghost_src, gsrc.data(), gsrc.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    }
    if (ce == cudaSuccess && h->n_send) {
        ce = cudaMalloc(&h->d_send, send.size() * sizeof(int32_t));
        if (ce == cudaSuccess) ce = cudaMemcpy(h->d_send, send.data(), send.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    }
    if (ce != cudaSuccess) return fail(KPM_ERR_CUDA, "row-partition lists: %s", cudaGetErrorString(ce));
    return KPM_OK;
}

}  // namespace

extern "C" {

kpm_status kpm_create_ell(int64_t D, int32_t K, const int32_t* col, const void* val, int32_t dtype, double a,
                          double b, int32_t device, const kpm_dist* dist, kpm_handle* out) {
    if (D < 1 || D >= (1LL << 31) || K < 0 || (K > 0 && (!col || !val)))
        return fail(KPM_ERR_INVALID_ARG, "bad ELL arguments (D=%lld K=%d)", (long long)D, K);
    if (dtype != KPM_REAL64 && dtype != KPM_COMPLEX128) return fail(KPM_ERR_INVALID_ARG, "bad dtype %d", dtype);
    KPM_TRY(check_ab(a, b));
    const int w = dtype == KPM_COMPLEX128 ? 2 : 1;
    std::vector<int32_t> c((size_t)K * D);
    std::vector<double> v((size_t)K * D * w);
    const double* vin = static_cast<const double*>(val);
    for (int64_t e = 0; e < (int64_t)K * D; ++e) {
        const int64_t i = e % D;
        const int32_t j = col[e];
        if (j < -1 || j >= D) return fail(KPM_ERR_INVALID_ARG, "ELL column %d out of range at entry %lld", j, (long long)e);
        c[e] = j < 0 ? (int32_t)i : j;  // padding -> (row, 0)
        for (int q = 0; q < w; ++q) v[e * w + q] = j < 0 ? 0.0 : vin[e * w + q] / a;
    }
    kpm_handle_s* h = nullptr;
    KPM_TRY(new_handle(device, dist, &h));
    h->kind = KIND_ELL;
    h->D_total = D;
    h->dtype = dtype;
    h->a = a;
    h->b = b;
    h->D = D;
    h->K = K;
    kpm_status st = KPM_OK;
    if (dist && dist->partition == KPM_PART_ROWS) st = ell_rows_setup(h, dist, c, v, w);
    if (st == KPM_OK && K > 0) {
        // device layout row-major [ld][KP]: ld = D rounded up to 2048 rows (the largest ELL tile),
        // KP = K rounded up to a multiple of 4, so a tile of rows is one contiguous, 16-byte aligned run
        // of each array (one bulk copy into shared memory, kpm_ell.cuh) and a row's indices are KP/4
        // 16-byte loads; padding entries are (row, 0), pad rows (0, 0) and are never used
        const int64_t Dl = h->D, ld = (Dl + 2047) / 2048 * 2048, KP = kpm::ell_kp(K);
        h->ell_ld = ld;
        h->ell_kp = (int)KP;
        std::vector<int32_t> cp((size_t)KP * ld, 0);
        std::vector<double> vp((size_t)KP * ld * w, 0.0);
        for (int64_t i = 0; i < Dl; ++i)
            for (int64_t k = 0; k < KP; ++k) {
                cp[i * KP + k] = k < K ? c[k * Dl + i] : (int32_t)i;
                for (int q = 0; q < w && k < K; ++q) vp[(i * KP + k) * w + q] = v[(k * Dl + i) * w + q];
            }
        cudaError_t ce = cudaMalloc(&h->d_col, cp.size() * sizeof(int32_t));
        if (ce == cudaSuccess) ce = cudaMalloc(&h->d_val, vp.size() * sizeof(double));
        if (ce == cudaSuccess) ce = cudaMemcpy(h->d_col, cp.data(), cp.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
        if (ce == cudaSuccess) ce = cudaMemcpy(h->d_val, vp.data(), vp.size() * sizeof(double), cudaMemcpyHostToDevice);
        if (ce != cudaSuccess) st = fail(KPM_ERR_CUDA, "ELL upload: %s", cudaGetErrorString(ce));
    }
    if (st == KPM_OK) st = init_comm(h, dist);
    if (st != KPM_OK) {
        kpm_destroy(h);
        return st;
    }
    *out = h;
    return KPM_OK;
}

kpm_status kpm_gershgorin_dense(int64_t D, const void* H, int32_t dtype, double eps, double* a, double* b) {
    if (D < 1 || !H || !a || !b) return fail(KPM_ERR_INVALID_ARG, "bad dense arguments");
    if (dtype != KPM_REAL64) return fail(KPM_ERR_UNSUPPORTED, "dense H: KPM_REAL64 only");
    const double* m = static_cast<const double*>(H);
    double Eu = -INFINITY, El = INFINITY;
    for (int64_t i = 0; i < D; ++i) {
        double rad = 0.0;
        for (int64_t j = 0; j < D; ++j)
            if (j != i) rad += std::fabs(m[i * D + j]);
        Eu = std::max(Eu, m[i * D + i] + rad);
        El = std::min(El, m[i * D + i] - rad);
    }
    Eu += eps;
    El -= eps;
    *a = (Eu - El) / 2.0;
    *b = (Eu + El) / 2.0;
    return KPM_OK;
}

kpm_status kpm_create_dense(int64_t D, const void* H, int32_t dtype, double a, double b, int32_t device,
                            const kpm_dist* dist, kpm_handle* out) {
    if (D < 1 || D > (1LL << 17) || !H) return fail(KPM_ERR_INVALID_ARG, "bad dense arguments (D=%lld)", (long long)D);
    if (dtype != KPM_REAL64) return fail(KPM_ERR_UNSUPPORTED, "dense H: KPM_REAL64 only");
    KPM_TRY(check_ab(a, b));
    if (dist && dist->partition == KPM_PART_ROWS)
        return fail(KPM_ERR_UNSUPPORTED, "row partition is implemented for lattice stencils only");
    const int64_t Dp = (D + kpm::kDBM - 1) / kpm::kDBM * kpm::kDBM;
    std::vector<double> hp((size_t)Dp * Dp, 0.0);
    const double* m = static_cast<const double*>(H);
    for (int64_t i = 0; i < D; ++i)
        for (int64_t j = 0; j < D; ++j) hp[(size_t)i * Dp + j] = m[i * D + j] / a;
    kpm_handle_s* h = nullptr;
    KPM_TRY(new_handle(device, dist, &h));
    h->kind = KIND_DENSE;
    h->D_total = D;
    h->D = D;
    h->Dp = Dp;
    h->dtype = dtype;
    h->a = a;
    h->b = b;
    cudaError_t ce = cudaMalloc(&h->d_dense, hp.size() * sizeof(double));
    if (ce == cudaSuccess) ce = cudaMemcpy(h->d_dense, hp.data(), hp.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        kpm_destroy(h);
        return fail(KPM_ERR_CUDA, "dense upload: %s", cudaGetErrorString(ce));
    }
    const kpm_status st = init_comm(h, dist);
    if (st != KPM_OK) {
        kpm_destroy(h);
        return st;
    }
    *out = h;
    return KPM_OK;
}

kpm_status kpm_create_csr(int64_t D, const int64_t* rowptr, const int32_t* col, const void* val, int32_t dtype,
                          double a, double b, int32_t device, const kpm_dist* dist, kpm_handle* out) {
    if (D < 1 || D >= (1LL << 31) || !rowptr || !col || !val) return fail(KPM_ERR_INVALID_ARG, "bad CSR arguments");
    if (dtype != KPM_REAL64 && dtype != KPM_COMPLEX128) return fail(KPM_ERR_INVALID_ARG, "bad dtype %d", dtype);
    if (rowptr[0] != 0) return fail(KPM_ERR_INVALID_ARG, "rowptr[0] must be 0");
    int32_t K = 0;
    for (int64_t i = 0; i < D; ++i) {
        const int64_t len = rowptr[i + 1] - rowptr[i];
        if (len < 0) return fail(KPM_ERR_INVALID_ARG, "rowptr not monotone at row %lld", (long long)i);
        K = std::max<int32_t>(K, (int32_t)len);
    }
    const int w = dtype == KPM_COMPLEX128 ? 2 : 1;
    const double* vin = static_cast<const double*>(val);
    std::vector<int32_t> c((size_t)K * D, -1);
    std::vector<double> v((size_t)K * D * w, 0.0);
    for (int64_t i = 0; i < D; ++i) {
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            const int64_t slot = k - rowptr[i];
            if (col[k] < 0 || col[k] >= D) return fail(KPM_ERR_INVALID_ARG, "CSR column %d out of range in row %lld", col[k], (long long)i);
            c[slot * D + i] = col[k];
            for (int q = 0; q < w; ++q) v[(slot * D + i) * w + q] = vin[k * w + q];
        }
    }
    return kpm_create_ell(D, K, c.data(), v.data(), dtype, a, b, device, dist, out);
}

kpm_status kpm_csr_partition(int64_t D, const int64_t* rowptr, const int32_t* col, int32_t rank, int32_t world,
                             int64_t counts[3], int64_t* ghosts, int64_t* send_rows, int64_t* peers) {
    if (D < 1 || D >= (1LL << 31) || !rowptr || !col || !counts) return fail(KPM_ERR_INVALID_ARG, "bad CSR arguments");
    if (rowptr[0] != 0) return fail(KPM_ERR_INVALID_ARG, "rowptr[0] must be 0");
    int64_t K = 0;
    for (int64_t i = 0; i < D; ++i) {
        if (rowptr[i + 1] < rowptr[i]) return fail(KPM_ERR_INVALID_ARG, "rowptr not monotone at row %lld", (long long)i);
        K = std::max<int64_t>(K, rowptr[i + 1] - rowptr[i]);
    }
    std::vector<int32_t> c((size_t)K * D);
    for (int64_t i = 0; i < D; ++i)
        for (int64_t k = 0; k < K; ++k) {
            const int64_t e = rowptr[i] + k;
            const int32_t j = e < rowptr[i + 1] ? col[e] : (int32_t)i;
            if (j < 0 || j >= D) return fail(KPM_ERR_INVALID_ARG, "CSR column %d out of range in row %lld", j, (long long)i);
            c[k * D + i] = j;
        }
    EllPartition P;
    KPM_TRY(ell_partition(D, K, c.data(), rank, world, &P));
    counts[0] = P.nl;
    counts[1] = (int64_t)P.ghosts.size();
    counts[2] = (int64_t)P.send.size();
    if (ghosts) std::copy(P.ghosts.begin(), P.ghosts.end(), ghosts);
    if (send_rows) std::copy(P.send.begin(), P.send.end(), send_rows);
    if (peers)
        for (int q = 0; q < world; ++q) {
            peers[4 * q] = P.roff[q];
            peers[4 * q + 1] = P.rcnt[q];
            peers[4 * q + 2] = P.soff[q];
            peers[4 * q + 3] = P.scnt[q];
        }
    return KPM_OK;
}

kpm_status kpm_set_stream(kpm_handle h, void* stream) {
    if (!h) return fail(KPM_ERR_INVALID_ARG, "NULL handle");
    KPM_CUDA(cudaSetDevice(h->device));
    // work already queued on the outgoing stream (the workspace may be freed or reused on the new one)
    KPM_CUDA(cudaStreamSynchronize(h->stream));
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    h->stream = static_cast<cudaStream_t>(stream);
    h->own_stream = false;
    return KPM_OK;
}

kpm_status kpm_workspace_size(kpm_handle h, int32_t N, int64_t R, uint32_t flags, size_t* bytes) {
    if (!h || !bytes) return fail(KPM_ERR_INVALID_ARG, "NULL argument");
    Plan p;
    KPM_TRY(make_plan(h, N, R, flags, true, &p));
    *bytes = p.total;
    return KPM_OK;
}

kpm_status kpm_set_workspace(kpm_handle h, void* dev_ptr, size_t bytes) {
    if (!h) return fail(KPM_ERR_INVALID_ARG, "NULL handle");
    if (dev_ptr && (reinterpret_cast<uintptr_t>(dev_ptr) % kAlign) != 0)
        return fail(KPM_ERR_INVALID_ARG, "workspace must be %zu-byte aligned", kAlign);
    KPM_CUDA(cudaSetDevice(h->device));
    if (h->ws_own && h->ws) cudaFreeAsync(h->ws, h->stream);
    cudaStreamSynchronize(h->stream);
    h->ws = static_cast<char*>(dev_ptr);
    h->ws_bytes = dev_ptr ? bytes : 0;
    h->ws_own = dev_ptr == nullptr;
    return KPM_OK;
}

// KPM_COMM_IPC (kpm_ipc.cuh): one kpm_moments_ex call of a rank.  Row partition: the first
// step's ghost planes are pulled from the neighbours' mapped blocks (peer copies), then every
// recursion launch stores its boundary planes into the neighbours' ghost planes (fused halo) and
// the next launch waits on the device for both neighbours' launch; if any rank's plan is not a
// TMA march (or opts.no_fused_halo), ghost planes are pulled by peer copies after every launch.
// Both partitions end with the rank-order sum of S (and Sv for rows) over all ranks.
kpm_status moments_ipc(kpm_handle_s* h, int32_t N, int64_t R, uint64_t seed, const void* r0, uint32_t flags,
                       void* out) {
    IpcComm& I = *h->ipc;
    if (h->rows && h->kind != KIND_STENCIL) return fail(KPM_ERR_UNSUPPORTED, "KPM_COMM_IPC row partitions: stencils only");
    Run run;
    kpm_status st = run.begin(h, N, R, seed, r0, flags);  // plan, workspace, first step (launch 0)
    if (st != KPM_OK) {
        I.seg->r[I.rank].failed.store(1);
        h->dead = true;
        return st;
    }
    auto body = [&]() -> kpm_status {
        const bool fused_ok = h->rows && run.p.use_tma && !run.p.overlap && !h->opts.no_fused_halo;
        KPM_TRY(ipc_publish(h, run.p, reinterpret_cast<char*>(run.P), reinterpret_cast<char*>(run.C),
                            reinterpret_cast<char*>(run.S), reinterpret_cast<char*>(run.Sv), run.nsteps, fused_ok));
        KPM_TRY(ipc_attach(h));
        bool fused = fused_ok;
        for (int q = 0; q < I.world; ++q) {
            const IpcRank& r = I.seg->r[q];
            if (r.N != N || r.steps != run.nsteps || (h->rows && r.R_loc != run.p.R_loc))
                return ipc_fail(h, "KPM_COMM_IPC: %s", "ranks called with different N / R");
            fused = fused && r.fused_ok;
        }
        if (!h->rows) {
            while (run.more()) KPM_TRY(run.launch_next());
            return KPM_OK;
        }
        int nb[2];
        const int nn = ipc_neighbours(I, nb);
        const int lo = nn ? nb[0] : I.rank, hi = nn ? nb[nn - 1] : I.rank;
        const IpcRank& rl = I.seg->r[lo];
        const size_t pb = run.plane_bytes();
        // a block of rank q (its P or C, as `mine` is this rank's P or C) in this process's address space
        auto blk = [&](int q, const double2* mine) -> char* {
            const IpcRank& r = I.seg->r[q];
            return I.peers[q].ws + (mine == run.P ? r.off_P : r.off_C);
        };
        auto pull = [&](double2* X) -> kpm_status {  // ghost planes of X from the neighbours' same block
            const char* lo_last = blk(lo, X) + (rl.nloc - 1) * (int64_t)pb;
            const char* hi_first = blk(hi, X);
            KPM_CUDA(cudaMemcpyAsync(run.ghost_lo(X), lo_last, pb, cudaMemcpyDefault, h->stream));
            KPM_CUDA(cudaMemcpyAsync(run.ghost_hi(X), hi_first, pb, cudaMemcpyDefault, h->stream));
            h->halo_copies += 2;
            return KPM_OK;
        };
        KPM_TRY(ipc_record(h));  // launch 0: the first step
        KPM_TRY(ipc_wait_neighbours(h));
        KPM_TRY(pull(run.fresh()));
        while (run.more()) {
            if (fused) {
                // the neighbours' ghost planes of the block this launch overwrites (a_{n-1} -> a_{n+1})
                run.tg.peer_lo = reinterpret_cast<double2*>(blk(lo, run.prev) + rl.nloc * (int64_t)pb);
                run.tg.peer_hi = reinterpret_cast<double2*>(blk(hi, run.prev) - (int64_t)pb);
            }
            KPM_TRY(run.launch_next());
            if (fused) h->fused_halo_launches++;
            KPM_TRY(ipc_record(h));
            KPM_TRY(ipc_wait_neighbours(h));
            if (!fused) KPM_TRY(pull(run.fresh()));
        }
        run.tg.peer_lo = run.tg.peer_hi = nullptr;
        return KPM_OK;
    };
    st = body();
    if (st == KPM_OK) st = run.collect();
    if (st == KPM_OK) st = sync_stream(h);
    // sums over the ranks (Eq 16): all final -> every rank adds all ranks' sums in rank order ->
    // all reads done -> each rank overwrites its own
    const bool sum_S = h->rows || run.vector_collective();
    const bool sum_Sv = h->rows;
    std::vector<double> S, Sv;
    if (st == KPM_OK) st = ipc_barrier(h);
    if (st == KPM_OK && sum_S) st = ipc_sum(h, [](const IpcRank& r) { return r.off_S; }, (size_t)N, S);
    if (st == KPM_OK && sum_Sv) st = ipc_sum(h, [](const IpcRank& r) { return r.off_Sv; }, (size_t)N * run.p.R_loc, Sv);
    if (st == KPM_OK) st = ipc_barrier(h);
    if (st != KPM_OK) {
        I.seg->r[I.rank].failed.store(1);
        h->dead = true;
        return st;
    }
    if (sum_S) KPM_CUDA(cudaMemcpyAsync(run.S, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    if (sum_Sv) KPM_CUDA(cudaMemcpyAsync(run.Sv, Sv.data(), Sv.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    return run.output(out);
}

kpm_status kpm_moments_ex(kpm_handle h, int32_t N, int64_t R, uint64_t seed, const void* r0, uint32_t flags,
                          void* out) {
    if (!h) return fail(KPM_ERR_INVALID_ARG, "NULL handle");
    if (!out) return fail(KPM_ERR_INVALID_ARG, "NULL output");
    if (h->dead)
        return h->ipc ? fail(KPM_ERR_COMM, "the handle's KPM_COMM_IPC partition failed in an earlier call")
                      : fail(KPM_ERR_NCCL, "the handle's communicator was aborted by an earlier NCCL failure");
    if (h->rows && h->dist.comm == KPM_COMM_LOCAL)
        return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_LOCAL slab handles run through kpm_moments_group");
    if (h->ipc) return moments_ipc(h, N, R, seed, r0, flags, out);
    Run run;
    if (h->rows) run.exchange_hook = exchange_single;
    KPM_TRY(run.begin(h, N, R, seed, r0, flags));
    if (h->rows) KPM_TRY(run.need_exchange(run.fresh()));
    while (run.more()) {
        KPM_TRY(run.launch_next());
        if (h->rows) KPM_TRY(run.need_exchange(run.fresh()));
    }
    KPM_TRY(run.collect());
    if (h->rows && h->dist.comm == KPM_COMM_NCCL) {
        // moment sums over all slabs: one all-reduce of S (and the per-vector Sv) over NCCL
        KPM_NCCL(h, ncclAllReduce(run.S, run.S, N, ncclFloat64, ncclSum, h->nccl, h->stream), "ncclAllReduce (S)");
        KPM_NCCL(h, ncclAllReduce(run.Sv, run.Sv, (size_t)N * run.p.R_loc, ncclFloat64, ncclSum, h->nccl, h->stream),
                 "ncclAllReduce (Sv)");
    } else if (run.vector_collective()) {
        // random-vector partition: the ONE collective of the method -- S[N]
        // summed over the ranks' vectors (Eq 16; Fig 3 step (3))
        KPM_NCCL(h, ncclAllReduce(run.S, run.S, N, ncclFloat64, ncclSum, h->nccl, h->stream), "ncclAllReduce (S)");
    }
    return run.output(out);
}

kpm_status kpm_moments_group(kpm_handle* hs, int32_t nh, int32_t N, int64_t R, uint64_t seed, double* mu) {
    if (!hs || nh < 1 || !mu) return fail(KPM_ERR_INVALID_ARG, "bad kpm_moments_group arguments");
    if (hs[0] && hs[0]->dist.partition == KPM_PART_VECTORS) return moments_group_vectors(hs, nh, N, R, seed, mu);
    for (int i = 0; i < nh; ++i) {
        if (!hs[i] || !hs[i]->rows || hs[i]->dist.comm != KPM_COMM_LOCAL || hs[i]->dist.rank != i ||
            hs[i]->dist.world != nh)
            return fail(KPM_ERR_INVALID_ARG, "handle %d is not rank %d of a KPM_COMM_LOCAL row partition of %d", i, i, nh);
        if (hs[i]->kind != hs[0]->kind || (hs[i]->kind == KIND_ELL && hs[i]->device != hs[0]->device))
            return fail(KPM_ERR_UNSUPPORTED, "in-process ELL row partitions: one kind, one device");
    }
    std::vector<Run> runs(nh);
    std::vector<cudaEvent_t> evs(nh, nullptr);
    kpm_status st = KPM_OK;
    for (int i = 0; i < nh && st == KPM_OK; ++i) {
        cudaSetDevice(hs[i]->device);
        if (cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming) != cudaSuccess) st = fail(KPM_ERR_CUDA, "event");
    }
    for (int i = 0; i < nh && st == KPM_OK; ++i) st = runs[i].begin(hs[i], N, R, seed, nullptr, 0u);
    auto exch = [&]() {
        for (auto& r : runs) r.pending = r.fresh();
        return exchange_group(runs, evs);
    };
    if (st == KPM_OK) st = exch();  // ghosts of a_1 (first-step kernel): plane copies
    // Fused halo (stencil slabs on one device, TMA march kernels): every recursion launch stores its
    // boundary planes straight into the neighbours' ghost planes of the same block (peer memory),
    // so between launches only stream ordering remains -- each rank's next launch waits for its two
    // neighbours' current one (their ghost writes into it, and their reads of the ghosts it
    // overwrites next).  opts.no_fused_halo = 1 (on hs[0]) keeps the copy exchange.
    bool fused = st == KPM_OK && !hs[0]->opts.no_fused_halo;
    for (int i = 0; i < nh && fused; ++i)
        fused = hs[i]->kind == KIND_STENCIL && runs[i].p.use_tma && !runs[i].p.overlap;
    // slabs on different GPUs: the kernels store into the neighbours' memory over NVLink, which
    // needs peer access in both directions (else: plane copies, cudaMemcpyPeerAsync)
    for (int i = 0; i < nh && fused; ++i) {
        for (int d : {(i - 1 + nh) % nh, (i + 1) % nh}) {
            const int a0 = hs[i]->device, a1 = hs[d]->device;
            if (a0 == a1) continue;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, a0, a1) != cudaSuccess || !ok) {
                fused = false;
                break;
            }
            cudaSetDevice(a0);
            const cudaError_t e = cudaDeviceEnablePeerAccess(a1, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) {
                cudaGetLastError();
                fused = false;
                break;
            }
        }
    }
    while (st == KPM_OK && runs[0].more()) {
        for (int i = 0; i < nh && fused; ++i) {
            Run& lo = runs[(i - 1 + nh) % nh];
            Run& hi = runs[(i + 1) % nh];
            runs[i].tg.peer_lo = lo.ghost_hi(lo.prev);
            runs[i].tg.peer_hi = hi.ghost_lo(hi.prev);
        }
        for (int i = 0; i < nh && st == KPM_OK; ++i) {
            if (cudaSetDevice(hs[i]->device) != cudaSuccess) st = fail(KPM_ERR_CUDA, "cudaSetDevice");
            if (st == KPM_OK) st = runs[i].launch_next();
            if (fused) hs[i]->fused_halo_launches++;
        }
        if (st != KPM_OK) break;
        if (!fused) {
            st = exch();
            continue;
        }
        for (int i = 0; i < nh && st == KPM_OK; ++i)
            if (cudaSetDevice(hs[i]->device) != cudaSuccess || cudaEventRecord(evs[i], hs[i]->stream) != cudaSuccess)
                st = fail(KPM_ERR_CUDA, "event record");
        for (int i = 0; i < nh && st == KPM_OK; ++i)
            if (cudaSetDevice(hs[i]->device) != cudaSuccess ||
                cudaStreamWaitEvent(hs[i]->stream, evs[(i - 1 + nh) % nh], 0) != cudaSuccess ||
                cudaStreamWaitEvent(hs[i]->stream, evs[(i + 1) % nh], 0) != cudaSuccess)
                st = fail(KPM_ERR_CUDA, "event wait");
    }
    std::vector<double> Ssum(N, 0.0), Si(N);
    for (int i = 0; i < nh && st == KPM_OK; ++i) {
        runs[i].tg.peer_lo = runs[i].tg.peer_hi = nullptr;
        cudaSetDevice(hs[i]->device);
        st = runs[i].collect();
        if (st != KPM_OK) break;
        cudaSetDevice(hs[i]->device);
        if (cudaMemcpyAsync(Si.data(), runs[i].S, N * sizeof(double), cudaMemcpyDeviceToHost, hs[i]->stream) != cudaSuccess ||
            cudaStreamSynchronize(hs[i]->stream) != cudaSuccess)
            st = fail(KPM_ERR_CUDA, "group sums copy failed");
        for (int k = 0; k < N; ++k) Ssum[k] += Si[k];  // fixed rank order
    }
    for (auto e : evs)
        if (e) cudaEventDestroy(e);
    if (st != KPM_OK) return st;
    KPM_TRY(kpm_assemble(nullptr, Ssum.data(), N, hs[0]->D_total, runs[0].p.R_loc, 0u, mu));
    return Run::spectrum_guard(mu, 1, N);
}

kpm_status kpm_nccl_unique_id(void* out128) {
    if (!out128) return fail(KPM_ERR_INVALID_ARG, "NULL output");
    ncclUniqueId id;
    ncclResult_t e = ncclGetUniqueId(&id);
    if (e != ncclSuccess) return fail(KPM_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(e));
    memcpy(out128, &id, sizeof id);
    return KPM_OK;
}

kpm_status kpm_ipc_unique_name(char out64[64]) {
    if (!out64) return fail(KPM_ERR_INVALID_ARG, "NULL output");
    std::random_device rd;
    const unsigned long long r = ((unsigned long long)rd() << 32) ^ rd();
    snprintf(out64, 64, "/kpm-%d-%016llx", (int)getpid(), r);
    return KPM_OK;
}

kpm_status kpm_slab_range(int64_t Lm, int32_t rank, int32_t world, int64_t* begin, int64_t* count) {
    if (Lm < 1 || world < 1 || rank < 0 || rank >= world || !begin || !count)
        return fail(KPM_ERR_INVALID_ARG, "bad kpm_slab_range arguments");
    *begin = Lm * rank / world;
    *count = Lm * (rank + 1) / world - *begin;
    return KPM_OK;
}

kpm_status kpm_moments(kpm_handle h, int32_t N, int64_t R, uint64_t seed, double* mu) {
    return kpm_moments_ex(h, N, R, seed, nullptr, 0u, mu);
}

kpm_status kpm_assemble(kpm_handle h, const double* S, int32_t N, int64_t D, int64_t R, uint32_t flags, double* mu) {
    if (!S || !mu || N < 1 || R < 1 || D < 1) return fail(KPM_ERR_INVALID_ARG, "bad kpm_assemble arguments");
    const int direct = (flags & KPM_DIRECT) ? 1 : 0;
    const double c = 1.0 / ((double)D * (double)R);
    if (!(flags & KPM_DEVICE_OUT)) {
        // host: the same transform as assemble_kernel (a6: N multiply-adds)
        for (int n = 0; n < N; ++n) {
            const double x = S[n] * c;
            mu[n] = (direct || n < 2) ? x : 2.0 * x - ((n & 1) ? S[1] * c : S[0] * c);
        }
        return KPM_OK;
    }
    if (!h) return fail(KPM_ERR_INVALID_ARG, "device kpm_assemble needs a handle (stream)");
    KPM_CUDA(cudaSetDevice(h->device));
    kpm::assemble_kernel<<<(N + 255) / 256, 256, 0, h->stream>>>(S, N, c, direct, mu);
    KPM_CUDA(cudaGetLastError());
    return KPM_OK;
}

kpm_status kpm_vector_range(int64_t R, int32_t rank, int32_t world, int64_t* begin, int64_t* count) {
    if (R < 1 || world < 1 || rank < 0 || rank >= world || !begin || !count)
        return fail(KPM_ERR_INVALID_ARG, "bad kpm_vector_range arguments");
    *begin = R * rank / world;
    *count = R * (rank + 1) / world - *begin;
    return KPM_OK;
}

}  // extern "C"

namespace {
// Eq (6) on the device: c_n from mu and the kernel, then rho (what = 0) or G (what = 1) at the
// K energies.  Host in/out; scratch from cudaMalloc (not on the hot path).
kpm_status expand(const char* fn, int what, const double* mu, int32_t N, int32_t kernel, double lam, double a,
                  double b, const double* omega, int64_t K, double* out, int32_t device) {
    if (!mu || !omega || !out || N < 1 || K < 0) return fail(KPM_ERR_INVALID_ARG, "%s: bad arguments", fn);
    if (kernel < KPM_KERNEL_JACKSON || kernel > KPM_KERNEL_FEJER) return fail(KPM_ERR_INVALID_ARG, "%s: bad kernel %d", fn, kernel);
    if (kernel == KPM_KERNEL_LORENTZ && !(lam > 0.0 && std::isfinite(lam)))
        return fail(KPM_ERR_INVALID_ARG, "%s: Lorentz kernel needs lambda > 0 (got %g)", fn, lam);
    KPM_TRY(check_ab(a, b));
    if (K == 0) return KPM_OK;
    KPM_CUDA(cudaSetDevice(device));
    const size_t outw = what == 1 ? 2 : 1;
    double* buf = nullptr;
    const size_t bytes = (2 * (size_t)N + (1 + outw) * (size_t)K) * sizeof(double);
    KPM_CUDA(cudaMalloc(&buf, bytes));
    double *dmu = buf, *dc = buf + N, *dom = buf + 2 * N, *dout = buf + 2 * N + K;
    cudaError_t e = cudaMemcpy(dmu, mu, N * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dom, omega, K * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        kpm::dos_coeff_kernel<<<(N + 255) / 256, 256>>>(dmu, N, kernel, lam, dc);
        if (what == 1) kpm::green_kernel<<<(unsigned)((K + 255) / 256), 256>>>(dc, N, a, b, dom, K, dout);
        else kpm::dos_kernel<<<(unsigned)((K + 255) / 256), 256>>>(dc, N, a, b, dom, K, dout);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, outw * K * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e != cudaSuccess) return fail(KPM_ERR_CUDA, "%s: %s", fn, cudaGetErrorString(e));
    return KPM_OK;
}
}  // namespace

extern "C" {

kpm_status kpm_dos(const double* mu, int32_t N, int32_t kernel, double a, double b, const double* omega, int64_t K,
                   double* rho, int32_t device) {
    return expand("kpm_dos", 0, mu, N, kernel, KPM_LORENTZ_DEFAULT_LAMBDA, a, b, omega, K, rho, device);
}

kpm_status kpm_dos_ex(const double* mu, int32_t N, int32_t kernel, double lambda, double a, double b,
                      const double* omega, int64_t K, double* rho, int32_t device) {
    return expand("kpm_dos_ex", 0, mu, N, kernel, lambda, a, b, omega, K, rho, device);
}

kpm_status kpm_green(const double* mu, int32_t N, int32_t kernel, double lambda, double a, double b,
                     const double* omega, int64_t K, double* G, int32_t device) {
    return expand("kpm_green", 1, mu, N, kernel, lambda, a, b, omega, K, G, device);
}

kpm_status kpm_damping(int32_t N, int32_t kernel, double lambda, double* g, int32_t device) {
    if (!g || N < 1) return fail(KPM_ERR_INVALID_ARG, "kpm_damping: bad arguments");
    if (kernel < KPM_KERNEL_JACKSON || kernel > KPM_KERNEL_FEJER) return fail(KPM_ERR_INVALID_ARG, "bad kernel %d", kernel);
    if (kernel == KPM_KERNEL_LORENTZ && !(lambda > 0.0 && std::isfinite(lambda)))
        return fail(KPM_ERR_INVALID_ARG, "Lorentz kernel needs lambda > 0");
    KPM_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    KPM_CUDA(cudaMalloc(&d, N * sizeof(double)));
    kpm::dos_coeff_kernel<<<(N + 255) / 256, 256>>>(nullptr, N, kernel, lambda, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(g, d, N * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(KPM_ERR_CUDA, "kpm_damping: %s", cudaGetErrorString(e));
    return KPM_OK;
}

kpm_status kpm_moment_stats(const double* mu_pv, int64_t R, int32_t N, double* mean, double* sem, int32_t device) {
    if (!mu_pv || !mean || !sem || R < 1 || N < 1) return fail(KPM_ERR_INVALID_ARG, "kpm_moment_stats: bad arguments");
    if ((size_t)R > SIZE_MAX / sizeof(double) / (size_t)N) return fail(KPM_ERR_INVALID_ARG, "kpm_moment_stats: R*N too large");
    KPM_CUDA(cudaSetDevice(device));
    const size_t in = (size_t)R * N * sizeof(double), out = (size_t)N * sizeof(double);
    double* d = nullptr;
    KPM_CUDA(cudaMalloc(&d, in + 2 * out));
    cudaError_t e = cudaMemcpy(d, mu_pv, in, cudaMemcpyHostToDevice);
    double* dm = d + (size_t)R * N;
    double* ds = dm + N;
    if (e == cudaSuccess) {
        kpm::moment_stats_kernel<<<(N + 127) / 128, 128>>>(d, (long long)R, N, dm, ds);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(mean, dm, out, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(sem, ds, out, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(KPM_ERR_CUDA, "kpm_moment_stats: %s", cudaGetErrorString(e));
    return KPM_OK;
}

kpm_status kpm_moments_local(kpm_handle h, int32_t N, const int64_t* sites, int64_t nsites, double* out) {
    if (!sites) return fail(KPM_ERR_INVALID_ARG, "kpm_moments_local: NULL sites");
    return kpm_moments_ex(h, N, nsites, 0, sites, KPM_LOCAL, out);
}

kpm_status kpm_last_timing(kpm_handle h, double* steps_ms, int32_t* step_launches, int32_t* total_launches) {
    if (!h) return fail(KPM_ERR_INVALID_ARG, "NULL handle");
    KPM_CUDA(cudaSetDevice(h->device));
    float ms = 0.f;
    if (steps_ms) {
        KPM_CUDA(cudaEventSynchronize(h->ev_end));
        KPM_CUDA(cudaEventElapsedTime(&ms, h->ev_begin, h->ev_end));
        *steps_ms = ms;
    }
    if (step_launches) *step_launches = h->step_launches;
    if (total_launches) *total_launches = h->total_launches;
    return KPM_OK;
}

kpm_status kpm_last_stats(kpm_handle h, int64_t stats[4]) {
    if (!h || !stats) return fail(KPM_ERR_INVALID_ARG, "NULL argument");
    stats[0] = h->step_launches;
    stats[1] = h->total_launches;
    stats[2] = h->halo_copies;
    stats[3] = h->fused_halo_launches;
    return KPM_OK;
}

kpm_status kpm_plan_info(kpm_handle h, int32_t N, int64_t R, uint32_t flags, int64_t info[12]) {
    if (!h || !info) return fail(KPM_ERR_INVALID_ARG, "NULL argument");
    Plan p;
    KPM_TRY(make_plan(h, N, R, flags, false, &p));
    info[0] = p.use_tma;
    info[1] = p.TL;
    info[2] = p.TX;
    info[3] = p.TY;
    info[4] = p.gx;
    info[5] = (int64_t)p.tma_smem;
    info[6] = p.RG;
    info[7] = p.tma_rr | ((p.use_tma2 || p.use_tma32) ? 2 : 0) | (p.overlap ? 4 : 0) | (p.use_tma3 ? 8 : 0) |
              (p.use_tma32 ? 16 : 0);
    info[8] = p.use_tma2 ? p.TX2 : (p.use_tma32 ? p.TX32 * 100 + p.TY32 : 0);
    info[9] = p.use_tma2 ? p.tma2_minb : 0;
    info[10] = p.use_tma2 ? p.tma2_grid : 0;
    info[11] = p.use_tmak ? p.KSK : (p.use_quad ? 4 : (p.use_tri ? 3 : 0));
    if (p.use_persist) info[7] |= 32;
    if (p.use_tri) info[7] |= 64;
    if (p.use_quad) info[7] |= 128;
    return KPM_OK;
}

kpm_status kpm_step_bytes(kpm_handle h, double* bytes) {
    if (!h || !bytes) return fail(KPM_ERR_INVALID_ARG, "NULL argument");
    *bytes = h->steps_bytes;
    return KPM_OK;
}

kpm_status kpm_step_traffic(kpm_handle h, double bytes[2]) {
    if (!h || !bytes) return fail(KPM_ERR_INVALID_ARG, "NULL argument");
    bytes[0] = h->steps_bytes;
    bytes[1] = h->design_bytes;
    return KPM_OK;
}

kpm_status kpm_set_plan_opts(kpm_handle h, const kpm_plan_opts* o) {
    if (!h) return fail(KPM_ERR_INVALID_ARG, "NULL handle");
    if (!o) {
        h->opts = kpm_plan_opts{};
        return KPM_OK;
    }
    const int32_t f[] = {o->no_small, o->no_tma,        o->no_two_step, o->no_box3,   o->tma_lanes,
                         o->halo_warp, o->ell_generic,  o->no_overlap,  o->no_fused_halo, o->contiguous,
                         o->experimental, o->exp_param, o->two_step_ctas, o->no_pdl, o->no_first_tile, o->no_three_step, o->no_zorder, o->no_four_step};
    for (int32_t x : f)
        if (x < 0) return fail(KPM_ERR_INVALID_ARG, "kpm_plan_opts: negative field");
    for (int32_t x : o->reserved)
        if (x != 0) return fail(KPM_ERR_INVALID_ARG, "kpm_plan_opts: reserved words must be 0");
    if (o->halo_warp > 2 || o->experimental > 3 || o->two_step_ctas > 2 || o->no_four_step > 1)
        return fail(KPM_ERR_INVALID_ARG, "kpm_plan_opts: value out of range");
#ifndef KPM_EXPERIMENTAL
    if (o->experimental) return fail(KPM_ERR_UNSUPPORTED, "experimental kernels are built into libkpm_exp.so only");
#endif
    h->opts = *o;
    return KPM_OK;
}

}  // extern "C"
