// kpm_ipc.cuh -- KPM_COMM_IPC: the ranks of a partition are processes on ONE node (one per
// GPU, or several sharing a GPU) that exchange halos and moment sums through CUDA IPC instead
// of NCCL ("NVLink in-kernel halo" across processes).
//
// Row partition (BJ.c5): every rank maps its neighbours' workspaces
// (cudaIpcOpenMemHandle; across GPUs the mapping is NVLink peer memory) and the TMA march
// kernels store the two boundary planes of a_{n+1} straight into the neighbours' ghost planes
// of the same block (TmaGeom::peer_lo / peer_hi, the in-process fused halo of
// kpm_moments_group), so no copy and no send/recv sits between two recursion steps.  What
// remains between launches is ordering: launch k+1 of a rank reads the ghost planes its
// neighbours' launch k wrote (RAW) and writes ghost planes its neighbours' launch k read
// (WAR), so it waits, on the device, for its two neighbours' launch k -- interprocess CUDA
// events (cudaEventInterprocess), recorded after every launch, a ring of kIpcEv per rank.  The
// host threads only run ahead: a rank waits on the host until its neighbour has RECORDED the
// event it needs (a counter in a POSIX shared-memory segment), never until the GPU reached it,
// and a slot is re-recorded only after both neighbours issued their waits on its previous use.
// No kernel ever spins on a flag, so ranks that time-share one GPU cannot deadlock it.
//
// Sums (Eq 16; Fig 3 step (3)): after the fixed-order finish
// every rank reads every rank's S[N] (and, for the row partition, Sv[N][R_loc]) from the mapped
// workspaces and adds them in rank order -- the same order on every rank, so every rank returns
// identical bits -- between two host barriers (all sums final / all reads done).
//
// Failure behaviour: a rank that fails inside a collective section raises a flag in the
// segment; the others stop waiting and return KPM_ERR_COMM, as they do after kIpcTimeoutS
// seconds without progress from a peer.  The handle is then dead (like an aborted NCCL
// communicator).
#pragma once
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <random>

namespace {

constexpr int kIpcMaxWorld = 64;
constexpr int kIpcEv = 8;               // event slots per rank: launches a neighbour may run ahead
constexpr double kIpcTimeoutS = 600.0;  // no progress from a peer for this long -> KPM_ERR_COMM

struct IpcRank {
    cudaIpcMemHandle_t ws;             // the rank's workspace allocation
    cudaIpcEventHandle_t ev[kIpcEv];   // its launch events
    int64_t ws_gen;                    // bumps when the workspace allocation changes
    int64_t ws_off;                    // workspace pointer - allocation base (bytes)
    int64_t off_P, off_C, off_S, off_Sv;  // bytes from the workspace pointer (P, C: interiors)
    int64_t ghost_lanes, nloc, R_loc, N, steps;
    int32_t device, fused_ok;
    std::atomic<int64_t> ready;    // call number whose fields above are published
    std::atomic<int64_t> rec;      // launch number whose event was recorded last
    std::atomic<int64_t> waited;   // launch number whose neighbours' events it has waited on
    std::atomic<int64_t> bar;      // host barriers passed
    std::atomic<int32_t> failed;   // the rank gave up: everybody stops waiting
};
struct IpcSeg {
    IpcRank r[kIpcMaxWorld];
};
static_assert(std::atomic<int64_t>::is_always_lock_free, "process-shared counters need lock-free atomics");

struct IpcPeer {
    int64_t gen = -1;           // ws_gen of the mapping below
    char* map = nullptr;        // cudaIpcOpenMemHandle result (allocation base); nullptr for self
    char* ws = nullptr;         // the peer's workspace pointer in this process
    bool ev_open = false;
    cudaEvent_t ev[kIpcEv] = {};
};

struct IpcComm {
    std::string name;
    IpcSeg* seg = nullptr;
    int rank = 0, world = 1;
    bool unlinked = false;
    cudaEvent_t ev[kIpcEv] = {};
    int64_t call = 0, seq = 0, bars = 0, ws_gen = 0;
    char* ws_pub = nullptr;  // workspace pointer published last
    std::vector<IpcPeer> peers;
};

kpm_status ipc_fail(kpm_handle_s* h, const char* fmt, const char* what) {
    if (h->ipc && h->ipc->seg) h->ipc->seg->r[h->ipc->rank].failed.store(1);
    h->dead = true;
    return fail(KPM_ERR_COMM, fmt, what);
}

// Spin (then sleep) until pred() holds; a failed peer or kIpcTimeoutS without success -> KPM_ERR_COMM.
template <class Pred>
kpm_status ipc_wait(kpm_handle_s* h, Pred pred, const char* what) {
    IpcComm& I = *h->ipc;
    const auto t0 = std::chrono::steady_clock::now();
    for (long it = 0;; ++it) {
        if (pred()) return KPM_OK;
        for (int q = 0; q < I.world; ++q)
            if (q != I.rank && I.seg->r[q].failed.load()) return ipc_fail(h, "KPM_COMM_IPC: a peer failed (%s)", what);
        if (it > 1000) {
            std::this_thread::sleep_for(std::chrono::microseconds(20));
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kIpcTimeoutS)
                return ipc_fail(h, "KPM_COMM_IPC: timed out waiting for a peer (%s)", what);
        }
    }
}

kpm_status ipc_open(kpm_handle_s* h, const char* name) {
    if (!name || name[0] != '/' || strlen(name) > 200) return fail(KPM_ERR_INVALID_ARG, "KPM_COMM_IPC needs ipc_name \"/...\"");
    if (h->dist.world > kIpcMaxWorld) return fail(KPM_ERR_UNSUPPORTED, "KPM_COMM_IPC: world > %d", kIpcMaxWorld);
    auto* I = new IpcComm();
    h->ipc = I;
    I->name = name;
    I->rank = h->dist.rank;
    I->world = h->dist.world;
    I->peers.resize(I->world);
    const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) return fail(KPM_ERR_COMM, "shm_open(%s): %s", name, strerror(errno));
    // every rank sizes the segment (same size); a fresh segment is zero-filled
    if (ftruncate(fd, sizeof(IpcSeg)) != 0) {
        close(fd);
        return fail(KPM_ERR_COMM, "ftruncate(%s): %s", name, strerror(errno));
    }
    void* m = mmap(nullptr, sizeof(IpcSeg), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return fail(KPM_ERR_COMM, "mmap(%s): %s", name, strerror(errno));
    I->seg = static_cast<IpcSeg*>(m);
    IpcRank& me = I->seg->r[I->rank];
    for (int i = 0; i < kIpcEv; ++i) {
        KPM_CUDA(cudaEventCreateWithFlags(&I->ev[i], cudaEventInterprocess | cudaEventDisableTiming));
        KPM_CUDA(cudaIpcGetEventHandle(&me.ev[i], I->ev[i]));
    }
    me.device = h->device;
    return KPM_OK;
}

void ipc_close(kpm_handle_s* h) {
    IpcComm* I = h->ipc;
    if (!I) return;
    for (int q = 0; q < (int)I->peers.size(); ++q) {
        IpcPeer& P = I->peers[q];
        if (P.map) cudaIpcCloseMemHandle(P.map);
        if (P.ev_open && q != I->rank)
            for (int i = 0; i < kIpcEv; ++i) cudaEventDestroy(P.ev[i]);
    }
    for (int i = 0; i < kIpcEv; ++i)
        if (I->ev[i]) cudaEventDestroy(I->ev[i]);
    if (I->seg) munmap(I->seg, sizeof(IpcSeg));
    if (!I->unlinked && I->rank == 0) shm_unlink(I->name.c_str());
    delete I;
    h->ipc = nullptr;
}

using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

// Publish this rank's workspace (IPC handle of its allocation) and the layout of this call.
kpm_status ipc_publish(kpm_handle_s* h, const Plan& p, const char* P, const char* C, const char* S, const char* Sv,
                       int64_t steps, bool fused_ok) {
    IpcComm& I = *h->ipc;
    IpcRank& me = I.seg->r[I.rank];
    if (h->ws != I.ws_pub) {
        static AddrRangeFn range = nullptr;
        if (!range) {
            void* fp = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return fail(KPM_ERR_CUDA, "cuMemGetAddressRange entry point not found");
            range = reinterpret_cast<AddrRangeFn>(fp);
        }
        CUdeviceptr base = 0;
        size_t sz = 0;
        if (range(&base, &sz, (CUdeviceptr)h->ws) != CUDA_SUCCESS) return fail(KPM_ERR_CUDA, "cuMemGetAddressRange failed");
        KPM_CUDA(cudaIpcGetMemHandle(&me.ws, reinterpret_cast<void*>(base)));
        me.ws_off = (int64_t)((CUdeviceptr)h->ws - base);
        me.ws_gen = ++I.ws_gen;
        I.ws_pub = h->ws;
    }
    me.off_P = P - h->ws;
    me.off_C = C - h->ws;
    me.off_S = S - h->ws;
    me.off_Sv = Sv - h->ws;
    me.ghost_lanes = (int64_t)p.ghost_lanes;
    me.nloc = h->nloc;
    me.R_loc = p.R_loc;
    me.N = p.N;
    me.steps = steps;
    me.fused_ok = fused_ok ? 1 : 0;
    me.ready.store(++I.call, std::memory_order_release);
    return KPM_OK;
}

// Map every rank's workspace (and open its events) once all ranks have published this call.
kpm_status ipc_attach(kpm_handle_s* h) {
    IpcComm& I = *h->ipc;
    for (int q = 0; q < I.world; ++q) {
        IpcRank& r = I.seg->r[q];
        KPM_TRY(ipc_wait(h, [&] { return r.ready.load(std::memory_order_acquire) >= I.call; }, "publish"));
        IpcPeer& P = I.peers[q];
        if (q == I.rank) {
            P.ws = h->ws;
            if (!P.ev_open) {
                for (int i = 0; i < kIpcEv; ++i) P.ev[i] = I.ev[i];
                P.ev_open = true;
            }
            continue;
        }
        if (r.ws_gen != P.gen) {
            if (P.map) cudaIpcCloseMemHandle(P.map);
            P.map = nullptr;
            void* m = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&m, r.ws, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return ipc_fail(h, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
            }
            P.map = static_cast<char*>(m);
            P.ws = P.map + r.ws_off;
            P.gen = r.ws_gen;
        }
        if (!P.ev_open) {
            for (int i = 0; i < kIpcEv; ++i) {
                const cudaError_t e = cudaIpcOpenEventHandle(&P.ev[i], r.ev[i]);
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    return ipc_fail(h, "cudaIpcOpenEventHandle: %s", cudaGetErrorString(e));
                }
            }
            P.ev_open = true;
        }
    }
    // the segment name is no longer needed once every rank has mapped it
    if (I.rank == 0 && !I.unlinked) {
        shm_unlink(I.name.c_str());
        I.unlinked = true;
    }
    return KPM_OK;
}

// the (one or two) neighbours of a slab: ranks rank-1 and rank+1, periodic
int ipc_neighbours(const IpcComm& I, int nb[2]) {
    if (I.world == 1) return 0;
    nb[0] = (I.rank - 1 + I.world) % I.world;
    nb[1] = (I.rank + 1) % I.world;
    return nb[0] == nb[1] ? 1 : 2;
}

// After a launch: record its event (slot seq % kIpcEv) once both neighbours have issued their
// waits on the slot's previous use.
kpm_status ipc_record(kpm_handle_s* h) {
    IpcComm& I = *h->ipc;
    const int64_t k = ++I.seq;
    int nb[2];
    const int nn = ipc_neighbours(I, nb);
    for (int j = 0; j < nn; ++j) {
        IpcRank& r = I.seg->r[nb[j]];
        KPM_TRY(ipc_wait(h, [&] { return r.waited.load(std::memory_order_acquire) >= k - kIpcEv; }, "event slot"));
    }
    KPM_CUDA(cudaEventRecord(I.ev[k % kIpcEv], h->stream));
    I.seg->r[I.rank].rec.store(k, std::memory_order_release);
    return KPM_OK;
}

// Before the next launch: the stream waits (on the device) for both neighbours' latest launch.
kpm_status ipc_wait_neighbours(kpm_handle_s* h) {
    IpcComm& I = *h->ipc;
    const int64_t k = I.seq;
    int nb[2];
    const int nn = ipc_neighbours(I, nb);
    for (int j = 0; j < nn; ++j) {
        IpcRank& r = I.seg->r[nb[j]];
        KPM_TRY(ipc_wait(h, [&] { return r.rec.load(std::memory_order_acquire) >= k; }, "neighbour launch"));
        KPM_CUDA(cudaStreamWaitEvent(h->stream, I.peers[nb[j]].ev[k % kIpcEv], 0));
    }
    I.seg->r[I.rank].waited.store(k, std::memory_order_release);
    return KPM_OK;
}

kpm_status ipc_barrier(kpm_handle_s* h) {
    IpcComm& I = *h->ipc;
    const int64_t g = ++I.bars;
    I.seg->r[I.rank].bar.store(g, std::memory_order_release);
    for (int q = 0; q < I.world; ++q) {
        IpcRank& r = I.seg->r[q];
        KPM_TRY(ipc_wait(h, [&] { return r.bar.load(std::memory_order_acquire) >= g; }, "barrier"));
    }
    return KPM_OK;
}

// Sum `count` doubles at byte offset off_of(rank) of every rank's workspace, in rank order, into
// `dst` (this rank's device buffer).  Called between the two barriers of ipc_allreduce.
template <class Off>
kpm_status ipc_sum(kpm_handle_s* h, Off off_of, size_t count, std::vector<double>& acc) {
    IpcComm& I = *h->ipc;
    std::vector<double> tmp(count);
    acc.assign(count, 0.0);
    for (int q = 0; q < I.world; ++q) {
        const char* src = I.peers[q].ws + off_of(I.seg->r[q]);
        KPM_CUDA(cudaMemcpy(tmp.data(), src, count * sizeof(double), cudaMemcpyDefault));
        for (size_t i = 0; i < count; ++i) acc[i] += tmp[i];  // fixed rank order on every rank
    }
    return KPM_OK;
}

}  // namespace
