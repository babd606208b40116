/*
 * kpm.h -- C ABI of the B200-native KPM moment engine (libkpm.so).
 *
 * The Kernel Polynomial Method (Zhang, Yamagiwa, Okumura, Yunoki, arxiv
 * 1105.5481; PAPER.md = /root/reference/PAPER.md): estimate the Chebyshev
 * moments of the density of states
 *     mu_n = (1/D) Tr T_n(H~)                               (Eq 13)
 * stochastically with R random vectors |r> (Eq 14-16) through
 * the vector recursion |a_0> = |r>, |a_1> = H~|a_0>,
 * |a_{n+1}> = 2 H~|a_n> - |a_{n-1}> (Eq 17-18), on the
 * rescaled Hamiltonian H~ = (H - b)/a (Eq 8-9; a = alpha_-,
 * b = alpha_+), using the doubling identities
 *     mu_{2n} = 2<a_n|a_n> - mu_0,   mu_{2n+1} = 2<a_{n+1}|a_n> - mu_1,
 * so that N moments cost floor(N/2) sparse-matrix x vector-block products.
 * The DoS is rebuilt from Jackson-damped moments by Eq (6).
 *
 * Conventions (all entry points):
 *  - Every call returns a kpm_status; nothing throws across the ABI.  On a
 *    non-OK status kpm_last_error() returns a thread-local message.  After
 *    KPM_ERR_CUDA the handle is unusable except for kpm_destroy.
 *  - Input arrays are caller-owned HOST arrays, copied during the call, unless
 *    a flag says "device".  Outputs are caller-allocated.  Device memory of a
 *    handle is owned by the handle (cudaMalloc), or by the caller through
 *    kpm_set_workspace (e.g. a torch tensor).
 *  - Work is ordered on the handle's CUDA stream (kpm_set_stream; default: a
 *    stream the handle creates).  Calls with host outputs synchronise it.
 *  - Determinism: for a given handle, (N, R, seed) and GPU model, repeated
 *    calls return bitwise-identical results (fixed-order reductions, no
 *    floating-point atomics).
 *  - Vectors are real Rademacher +-1 (Eq 14 asks only for real iid mean 0,
 *    variance 1; reading X1): xi_{r,i} = 1 - 2*(mix64(key ^ ctr) >> 63),
 *    key = mix64(seed + 0x9E3779B97F4A7C15), ctr = r * D + i over GLOBAL r and
 *    i, mix64 = the splitmix64 finaliser.  They are generated on the fly on the
 *    GPU; the set does not depend on the number of ranks.
 *  - Normalisation: mu_n = (1/(D R)) sum_r <r|T_n(H~)|r> (Eq 16, 19).
 *  - Layout on the device: the vector block is interleaved [site][vector]
 *    (vector index fastest) so one matrix/stencil entry serves all R vectors.
 */
#ifndef KPM_H_
#define KPM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kpm_handle_s* kpm_handle;
typedef int32_t kpm_status;

enum {
    KPM_OK = 0,
    KPM_ERR_INVALID_ARG = 1, /* bad size, a <= 0, non-finite a/b, flux*L0 not integer, ... */
    KPM_ERR_OOM = 2,         /* device allocation failed or workspace too small */
    KPM_ERR_CUDA = 3,        /* CUDA runtime error (sticky) */
    KPM_ERR_UNSUPPORTED = 4, /* valid request this build does not implement */
    KPM_ERR_SPECTRUM = 5,    /* |mu_n| > mu_0 (1 + 1e-8) or non-finite: [b-a, b+a] does not
                                enclose the spectrum (Eq 8 requires it).  Output still written. */
    KPM_ERR_NCCL = 6,        /* an NCCL call of the handle failed, or ncclCommGetAsyncError reported an
                                asynchronous error (a peer died, a network fault).  The communicator
                                has been aborted; the handle is unusable except for kpm_destroy. */
    KPM_ERR_COMM = 7         /* KPM_COMM_IPC: a peer rank failed, or made no progress for 600 s, or the
                                ranks' calls disagree (N, R); the shared segment or a CUDA IPC mapping
                                could not be set up.  The handle is unusable except for kpm_destroy. */
};

/* Element type of H and of the vector block. */
enum { KPM_REAL64 = 0, KPM_COMPLEX128 = 1 };

/* Damping kernel g_n of Eq (6) ("a kernel which satisfies the limit" Eq 7, PAPER.md:65-68;
 * formulas from the paper's ref [10]; X8, X26). */
enum {
    KPM_KERNEL_JACKSON = 0, /* g_n = [(N-n+1)cos(pi n/(N+1)) + sin(pi n/(N+1))cot(pi/(N+1))]/(N+1)
                                */
    KPM_KERNEL_NONE = 1,    /* g_n = 1 (truncated series, Eq 1) */
    KPM_KERNEL_LORENTZ = 2, /* g_n = sinh(lambda (1 - n/N)) / sinh(lambda), lambda > 0 (Green's
                               functions; kpm_dos uses lambda = KPM_LORENTZ_DEFAULT_LAMBDA) */
    KPM_KERNEL_FEJER = 3    /* g_n = 1 - n/N (Cesaro mean of the partial sums) */
};
#define KPM_LORENTZ_DEFAULT_LAMBDA 4.0

/* kpm_moments_ex flags. */
enum {
    KPM_PER_VECTOR = 1u, /* out = [R_local][N] per-vector moments (1/D)<r|T_n(H~)|r> instead of mu[N] */
    KPM_DIRECT = 2u,     /* the paper's own scheme, Eq (19): mu_n = <r|a_n>, N-1 products (validation) */
    KPM_DEVICE_OUT = 4u, /* out is a device pointer */
    KPM_RAW_SUMS = 8u,   /* out = raw sums S[N] over this rank's vectors, before normalisation and
                            the doubling transform (for a cross-rank all-reduce; see kpm_assemble) */
    KPM_DEVICE_IN = 16u, /* r0 is a device pointer */
    KPM_LOCAL = 32u      /* local moments: r0 is a HOST int64 list of R global site indices; the start
                            vectors are the unit vectors e_site (no randomness, seed ignored) and
                            out[R_local][N] = <site|T_n(H~)|site> (implies KPM_PER_VECTOR; no 1/D).
                            Not combinable with KPM_RAW_SUMS or KPM_DEVICE_IN. */
};

/* Nearest-neighbour lattice Hamiltonian (the paper's model, PAPER.md:229:
 * 3D cubic, 7 entries per row, zero diagonal, off-diagonal -1; periodic).
 * Sites are numbered i = x + L[0]*(y + L[1]*z).  Unused dims must have L = 1. */
typedef struct {
    int32_t ndim;          /* 1, 2 or 3 */
    int64_t L[3];          /* extents (each >= 2 for used dims) */
    double t;              /* hopping on every bond (paper: -1) */
    const double* onsite;  /* host [D] on-site energies eps_i (Anderson), or NULL (all 0) */
    double flux;           /* ndim == 2 only: Peierls flux per plaquette phi; the bond
                              (x,y)->(x,y+1) carries H[(x,y+1)][(x,y)] = t e^{+i 2 pi phi x}
                              (Landau gauge, X15).  phi*L[0] must be an integer.
                              phi != 0 makes H complex (KPM_COMPLEX128). */
} kpm_stencil_desc;

/* Partition of the work across ranks (one process per GPU).  NULL = one GPU. */
enum { KPM_PART_NONE = 0, KPM_PART_VECTORS = 1, KPM_PART_ROWS = 2 };
/* How the ranks of a partition combine moment sums (and, for KPM_PART_ROWS, exchange halos). */
enum {
    KPM_COMM_SELF = 0,  /* no library collective.  KPM_PART_ROWS: world == 1 (the slab is the whole
                           lattice; halos are local copies).  KPM_PART_VECTORS: with world > 1 the
                           caller combines the ranks' raw sums (KPM_RAW_SUMS, its own all-reduce,
                           kpm_assemble) -- kpm_moments then fails with KPM_ERR_INVALID_ARG */
    KPM_COMM_NCCL = 1,  /* one process per GPU; the handle owns an NCCL communicator made from
                           nccl_id.  KPM_PART_VECTORS: ONE ncclAllReduce of the raw sums S[N] after
                           the recursion (Eq 16 is a sum over the ranks' vectors; PAPER.md:120-128,
                           Fig 3 step (3) PAPER.md:179), so kpm_moments returns mu on every rank.
                           KPM_PART_ROWS: NCCL send/recv of halo planes + the same all-reduce. */
    KPM_COMM_LOCAL = 2, /* all ranks' handles in this process, driven by kpm_moments_group */
    KPM_COMM_IPC = 3    /* ranks are processes on ONE node (one per GPU, or several sharing a GPU), no
                           NCCL: the handle opens the POSIX shared-memory segment `ipc_name` (made
                           by kpm_ipc_unique_name on one rank and passed to all) and maps the other
                           ranks' workspaces with CUDA IPC (NVLink peer memory across GPUs).
                           KPM_PART_ROWS (stencils): the recursion kernels store their boundary
                           planes straight into the neighbours' ghost planes (fused halo, SURVEY.md
                           8(f) NEXT-4) and each launch waits on the device for the neighbours'
                           previous launch (interprocess CUDA events); both partitions end with
                           every rank summing all ranks' S[N] in rank order (Eq 16), so kpm_moments
                           returns identical mu on every rank.  Calls are collective.  Errors:
                           KPM_ERR_COMM. */
};
typedef struct {
    int32_t partition; /* KPM_PART_VECTORS: rank owns global vectors
                          [R*rank/world, R*(rank+1)/world) (Eq 16 is a sum over independent r).
                          KPM_PART_ROWS (stencils): rank owns the slab of the slowest lattice
                          dimension [Lm*rank/world, Lm*(rank+1)/world) (z in 3D, y in 2D, x in
                          1D) plus one ghost plane on each side, exchanged after every step
                          (periodic: rank 0 and rank world-1 are neighbours).
                          KPM_PART_ROWS (CSR / ELL): every rank passes the
                          WHOLE matrix; rank owns rows [D*rank/world, D*(rank+1)/world) plus ghost
                          copies of the off-block columns its rows reference, refreshed after
                          every step (kpm_csr_partition gives the lists). */
    int32_t rank;
    int32_t world;
    int32_t comm;            /* KPM_COMM_* (see above) */
    const void* nccl_id;     /* KPM_COMM_NCCL: the 128-byte ncclUniqueId from kpm_nccl_unique_id on
                                rank 0, the same on every rank.  Handles created from the same id (and
                                rank, world, device) share one communicator, which lives while any of
                                them does; their calls are collective and must be issued in the same
                                order on every rank. */
    int32_t vrank, vworld;   /* KPM_PART_ROWS only -- hybrid rows x vectors:
                                with vworld > 1 this row group runs only the global vectors
                                kpm_vector_range(R, vrank, vworld) (0 / 0 = all vectors).  The moment
                                sums are combined inside the row group (rank/world, comm); across the
                                vworld groups the caller sums the raw sums (KPM_RAW_SUMS, allowed for
                                row partitions) and calls kpm_assemble with the global R. */
    const char* ipc_name;    /* KPM_COMM_IPC: the shared-memory segment name ("/...", from
                                kpm_ipc_unique_name), the same on every rank; copied, not kept.
                                Rank 0 removes the name once every rank has mapped the segment. */
} kpm_dist;

/* 128-byte NCCL unique id for KPM_COMM_NCCL (call on rank 0, broadcast to the others). */
kpm_status kpm_nccl_unique_id(void* out128);
/* A fresh shared-memory segment name for KPM_COMM_IPC ("/kpm-<pid>-<random>", NUL-terminated,
 * at most 63 characters): call on one rank and pass the same string to every rank's kpm_dist. */
kpm_status kpm_ipc_unique_name(char out64[64]);

/* Slab of the row partition: planes [begin, begin + count) of an extent Lm.  Host only. */
kpm_status kpm_slab_range(int64_t Lm, int32_t rank, int32_t world, int64_t* begin, int64_t* count);

/* Row partition of a general sparse H (host only, no device): for rank `rank` of `world`,
 * counts[0] = local rows n (rows [D*rank/world, D*rank/world + n)), counts[1] = ghost sites
 * n_ghost (the distinct columns outside the block referenced by the block's rows), counts[2] =
 * rows to send n_send.  Optional outputs (NULL = skip; call once with NULL to size them):
 * ghosts int64[n_ghost] = global index of ghost k, ascending (so grouped by owner rank);
 * send_rows int64[n_send] = local row indices the other ranks need, peer by peer in rank
 * order, ascending within a peer; peers int64[4*world] = per peer q: (offset into ghosts,
 * count, offset into send_rows, count).  This is the plan kpm_create_csr/ell use for
 * KPM_PART_ROWS; errors: KPM_ERR_INVALID_ARG for malformed CSR or a rank that owns no rows. */
kpm_status kpm_csr_partition(int64_t D, const int64_t* rowptr, const int32_t* col, int32_t rank, int32_t world,
                             int64_t counts[3], int64_t* ghosts, int64_t* send_rows, int64_t* peers);

/* ---- creation (host -> device upload of H~; "the CPU copies the data to
 *      the VRAM") ------------------------------------------------------------------- */

/* H given as a lattice stencil.  a > 0 and b are the rescaling of Eq (8):
 * H~ = (H - b)/a.  device: CUDA ordinal.  dist may be NULL. */
kpm_status kpm_create_stencil(const kpm_stencil_desc* desc, double a, double b, int32_t device,
                              const kpm_dist* dist, kpm_handle* out);

/* H given in CSR ("CRS"): rowptr int64[D+1], col int32[nnz] (0 <= col < D),
 * val: double[nnz] (KPM_REAL64) or interleaved (re, im) double[2*nnz] (KPM_COMPLEX128).
 * H must be Hermitian (not checked).  Converted to ELL on the host. */
kpm_status kpm_create_csr(int64_t D, const int64_t* rowptr, const int32_t* col, const void* val,
                          int32_t dtype, double a, double b, int32_t device, const kpm_dist* dist,
                          kpm_handle* out);

/* H given in ELL: K entries per row, col int32[K][D] (-1 = padding), val [K][D] of dtype.
 * With dist->partition == KPM_PART_ROWS (both CSR and ELL), see kpm_dist and kpm_csr_partition:
 * KPM_COMM_SELF (world 1), KPM_COMM_NCCL (one process per GPU: the rows each peer needs are
 * packed and sent with ncclSend/ncclRecv straight into the peer's ghost range, then one
 * all-reduce of the moment sums) or KPM_COMM_LOCAL (in-process handles on ONE device, through
 * kpm_moments_group). */
kpm_status kpm_create_ell(int64_t D, int32_t K, const int32_t* col, const void* val, int32_t dtype,
                          double a, double b, int32_t device, const kpm_dist* dist,
                          kpm_handle* out);

/* H given DENSE (the paper's own variant: "when H is considered as a dense matrix,
 * the complexity of the part becomes O(D^2)"; H_SIZE experiments PAPER.md:241-253): row-major
 * D x D doubles (KPM_REAL64 only; complex -> KPM_ERR_UNSUPPORTED), Hermitian (not checked),
 * D <= 131072.  Stored on the device pre-scaled by 1/a and zero padded to a multiple of 64;
 * each recursion step is a DMMA (fp64 tensor-core) GEMM with the recursion and the moment sums
 * fused into its epilogue (kpm_dense.cuh).  Partitions: none or KPM_PART_VECTORS.
 * KPM_DIRECT is not implemented for dense H (KPM_ERR_UNSUPPORTED). */
kpm_status kpm_create_dense(int64_t D, const void* H, int32_t dtype, double a, double b, int32_t device,
                            const kpm_dist* dist, kpm_handle* out);

/* Gerschgorin bounds: E_upper = max_i (Re H_ii + sum_{j!=i} |H_ij|),
 * E_lower = min_i (...); eps pads both (0 = none); returns a = (Eu-El)/2, b = (Eu+El)/2. */
kpm_status kpm_gershgorin_stencil(const kpm_stencil_desc* desc, double eps, double* a, double* b);
kpm_status kpm_gershgorin_csr(int64_t D, const int64_t* rowptr, const int32_t* col,
                              const void* val, int32_t dtype, double eps, double* a, double* b);
kpm_status kpm_gershgorin_dense(int64_t D, const void* H, int32_t dtype, double eps, double* a, double* b);

/* ---- execution ------------------------------------------------------------------- */

/* Kernel-plan options of one handle.  All-zero = the default plan (the fastest measured kernel
 * for the problem shape).  The fields only restrict or pin the planner's choice -- for A/B
 * measurements and for tests that must reach one specific kernel; the moments are the same
 * (to rounding) under every plan.  They are per handle: the library reads no environment. */
typedef struct {
    int32_t no_small;      /* 1: never the single-launch shared-memory kernel (kpm_small.cuh) */
    int32_t no_tma;        /* 1: no TMA march kernels: generic grid-stride step kernel only */
    int32_t no_two_step;   /* 1: no two-steps-per-launch kernel (temporal blocking): single steps */
    int32_t no_box3;       /* 1: 3D lattices: the generic TMA march, not the dense-box kernel */
    int32_t tma_lanes;     /* lanes per tile site of the TMA march (0 = automatic); must divide the
                              lanes per site, else the automatic choice is kept */
    int32_t halo_warp;     /* two-step kernel: 0 = automatic, 1 = a ninth warp for the halo sites,
                              2 = no halo warp */
    int32_t ell_generic;   /* 1: ELL steps through the generic kernel, not kpm_ell_step_kernel */
    int32_t no_overlap;    /* 1: row partition: halo exchange after each step, not overlapped */
    int32_t no_fused_halo; /* 1: in-process slab groups: plane copies, not fused peer stores */
    int32_t contiguous;    /* 1: 3D march: contiguous plane ranges, not round-robin columns */
    int32_t experimental;  /* experimental kernels, compiled only into libkpm_exp.so (the default
                              libkpm.so answers KPM_ERR_UNSUPPORTED): 1 = 3D two-step kernel
                              (exp_param = tile shape 0..3), 2 = KS-steps-per-launch 2D kernel
                              (exp_param = KS, 3 or 4), 3 = persistent L2-resident kernel */
    int32_t exp_param;
    int32_t two_step_ctas; /* two-step kernel CTAs per SM (0 = automatic; 2 only for the 4-lane,
                              64-site tile, else 1) */
    int32_t no_pdl;        /* 1: plain stream-ordered launches instead of programmatic dependent
                              launches (PDL: the next kernel's prologue overlaps this one's tail) */
    int32_t no_first_tile; /* 1: first step by the generic grid-stride kernel (a_0 hashed per neighbour)
                              instead of the plane-ring tile kernel (2D/3D stencils) */
    int32_t no_three_step; /* 1: no three-steps-per-launch kernel for 2D lattices (kpm_tri.cuh: 4 D R s
                              bytes per three steps; tiles of >= 8 lanes): the two-step kernel */
    int32_t no_zorder;     /* 1: 3D round-robin march in row-major pencil order instead of Z order */
    int32_t no_four_step;  /* 1: no four-step launches for 2D lattices (kpm_quad.cuh, 8-lane x 64-site
                              tiles, the default where the lanes allow it): three steps per launch */
    int32_t reserved[2];   /* must be 0 */
} kpm_plan_opts;

/* Set (opts != NULL) or reset to the default (opts == NULL) the plan options of h.
 * KPM_ERR_INVALID_ARG for negative fields or non-zero reserved words; KPM_ERR_UNSUPPORTED for
 * an experimental kernel this build does not contain. */
kpm_status kpm_set_plan_opts(kpm_handle h, const kpm_plan_opts* opts);

/* Use this CUDA stream (a cudaStream_t; NULL = legacy default stream). */
kpm_status kpm_set_stream(kpm_handle h, void* stream);

/* Device bytes kpm_moments_ex needs for (N, R global, flags). */
kpm_status kpm_workspace_size(kpm_handle h, int32_t N, int64_t R, uint32_t flags, size_t* bytes);

/* Give the handle caller-owned device memory (>= kpm_workspace_size bytes, 256-B aligned).
 * The caller keeps it alive until kpm_destroy or the next kpm_set_workspace. NULL = own. */
kpm_status kpm_set_workspace(kpm_handle h, void* dev_ptr, size_t bytes);

/* mu[0..N-1] (host) from R random vectors drawn from `seed` (R = the GLOBAL number of vectors).
 * Partitions: KPM_PART_VECTORS with KPM_COMM_NCCL and KPM_PART_ROWS with KPM_COMM_NCCL return the
 * same mu on every rank (all ranks call collectively); KPM_PART_VECTORS with world > 1 and
 * KPM_COMM_SELF fails with KPM_ERR_INVALID_ARG (use kpm_moments_ex + KPM_RAW_SUMS + kpm_assemble). */
kpm_status kpm_moments(kpm_handle h, int32_t N, int64_t R, uint64_t seed, double* mu);

/* General form.  R is the GLOBAL number of vectors; this rank runs its share R_local.
 * r0: NULL = generate (see conventions); else this rank's start vectors, vector-major
 *     [R_local][D] of real doubles (host, or device with KPM_DEVICE_IN).
 * out: mu[N] (all ranks' vectors, as kpm_moments); or [R_local][N] with KPM_PER_VECTOR (this
 *      rank's vectors, no collective); or S[N] with KPM_RAW_SUMS (sums over THIS rank's vectors,
 *      before any collective, for callers that bring their own all-reduce); host, or device with
 *      KPM_DEVICE_OUT (then the call returns without synchronising the stream).
 * Errors: KPM_ERR_NCCL if the handle's collective failed (see KPM_ERR_NCCL). */
kpm_status kpm_moments_ex(kpm_handle h, int32_t N, int64_t R, uint64_t seed, const void* r0,
                          uint32_t flags, void* out);

/* Row partition with KPM_COMM_LOCAL: run kpm_moments for the `n` slab handles hs[0..n-1]
 * (rank i = hs[i], world n, any devices; CSR/ELL handles: one device) in lock step,
 * exchanging halo planes (ghost sites) between them after every step; mu[N] (host) is the
 * moment estimate of the whole matrix. */
kpm_status kpm_moments_group(kpm_handle* hs, int32_t n, int32_t N, int64_t R, uint64_t seed, double* mu);

/* Raw sums S[N] (summed over all ranks) -> mu[N]: mu_0 = S_0/(D R), mu_1 = S_1/(D R),
 * mu_{2n} = 2 S_{2n}/(D R) - mu_0, mu_{2n+1} = 2 S_{2n+1}/(D R) - mu_1; with KPM_DIRECT
 * mu_n = S_n/(D R).  D = number of sites, R = global number of vectors.
 * Default: S and mu are host arrays and the transform runs on the host (h may be NULL).
 * KPM_DEVICE_OUT: S and mu are device pointers; a kernel on h's stream does it. */
kpm_status kpm_assemble(kpm_handle h, const double* S, int32_t N, int64_t D, int64_t R, uint32_t flags,
                        double* mu);

/* The random-vector partition (KPM_PART_VECTORS): rank owns global vectors
 * [begin, begin + count) = [R*rank/world, R*(rank+1)/world).  Host only. */
kpm_status kpm_vector_range(int64_t R, int32_t rank, int32_t world, int64_t* begin, int64_t* count);

/* Eq (6) mapped back to omega (Eq 11-12; X9):
 *   rho(omega_k) = [g_0 mu_0 + 2 sum_{n=1}^{N-1} g_n mu_n T_n(x_k)] / (pi a sqrt(1 - x_k^2)),
 *   x_k = (omega_k - b)/a; rho = 0 for |x_k| >= 1.
 * Host mu[N], omega[K] -> host rho[K]; computed on `device`. */
kpm_status kpm_dos(const double* mu, int32_t N, int32_t kernel, double a, double b,
                   const double* omega, int64_t K, double* rho, int32_t device);

/* Eq (6) with any kernel: as kpm_dos, with the Lorentz parameter lambda (> 0; ignored by the
 * other kernels). */
kpm_status kpm_dos_ex(const double* mu, int32_t N, int32_t kernel, double lambda, double a, double b,
                      const double* omega, int64_t K, double* rho, int32_t device);

/* Retarded Green's function from the damped moments (the paper's "Green's functions",
 * PAPER.md:23; expansion of ref [10]; X24): G(omega) = (1/D) Tr 1/(omega + i0 - H)
 * for DoS moments (or <i|1/(omega + i0 - H)|i> for local moments), with x = (omega - b)/a,
 * c_0 = g_0 mu_0, c_n = 2 g_n mu_n:
 *   |x| < 1: G = -i sum_n c_n e^{-i n arccos x} / (a sqrt(1 - x^2))   (Im G = -pi rho)
 *   |x| > 1: G = sum_n c_n t^n / (a sgn(x) sqrt(x^2 - 1)), t = x - sgn(x) sqrt(x^2 - 1)  (real)
 *   |x| = 1: NaN.
 * Host mu[N], omega[K] -> host G[K][2] = (Re, Im); computed on `device`. */
kpm_status kpm_green(const double* mu, int32_t N, int32_t kernel, double lambda, double a, double b,
                     const double* omega, int64_t K, double* G, int32_t device);

/* Damping factors g[0..N-1] of `kernel` (host output; computed on `device`). */
kpm_status kpm_damping(int32_t N, int32_t kernel, double lambda, double* g, int32_t device);

/* Statistical error bars of the stochastic trace (Eq 16; SURVEY.md 8(f)
 * NEXT-1): from per-vector moments mu_pv (host, [R][N] row-major, the output of
 * kpm_moments_ex with KPM_PER_VECTOR after the doubling transform), writes mean[n] =
 * (1/R) sum_r mu_n^(r) (equal to kpm_moments up to rounding) and sem[n] = the standard error
 * of that mean, sqrt(sum_r (mu_n^(r) - mean[n])^2 / ((R-1) R)); sem = NaN for R = 1.
 * Computed on `device` (two passes, fp64).  Caller owns all buffers.  KPM_ERR_INVALID_ARG on
 * NULL pointers, R < 1 or N < 1; KPM_ERR_CUDA on a CUDA failure (outputs undefined). */
kpm_status kpm_moment_stats(const double* mu_pv, int64_t R, int32_t N, double* mean, double* sem, int32_t device);

/* Local moments mu_n^(i) = <i|T_n(H~)|i> of the global sites i = sites[0..nsites-1] (local DoS;
 * SURVEY.md 8(f) NEXT-1): kpm_moments_ex(h, N, nsites, 0, sites, KPM_LOCAL, out), out host
 * [nsites_local][N].  With KPM_PART_VECTORS the sites are split like vectors. */
kpm_status kpm_moments_local(kpm_handle h, int32_t N, const int64_t* sites, int64_t nsites, double* out);

/* ---- introspection ---------------------------------------------------------------- */

/* Device time (ms, CUDA events on the handle's stream) of the last kpm_moments_ex's
 * recursion-step launches (all steps after the first), their count, and the kernel
 * launches the call made in total. */
kpm_status kpm_last_timing(kpm_handle h, double* steps_ms, int32_t* step_launches,
                           int32_t* total_launches);

/* Execution plan kpm_moments_ex would use for (N, R, flags): info[0] = 1 if the
 * TMA-pipelined march kernel runs the recursion steps (2D/3D stencils), else 0;
 * info[1..3] = lanes per tile TL, tile TX, TY; info[4] = partial-sum rows per moment slot
 * (CTAs of the widest step kernel); info[5] = dynamic shared memory bytes of the step
 * kernel; info[6] = lanes per site; info[7] bit 0: whole (lane group, pencil) columns are
 * dealt round-robin to CTAs; bit 1: two recursion steps per launch (temporal blocking, 2D;
 * 4 vector blocks); bit 2: row partition with the halo exchange overlapped (boundary planes,
 * exchange on a comm stream, interior planes); bit 3: 3D dense-box march kernel; bit 4: 3D two-step
 * (experimental); bit 5: persistent (experimental); bit 6: three steps per launch (2D, kpm_tri.cuh);
 * info[8] = two-step tile width TX2; info[9] = two-step CTAs per SM; info[10] = two-step grid;
 * info[11] = recursion steps per launch of the deepest kernel in the plan beyond two (3 for the
 * three-step kernel; KS for the experimental KS-step kernel), else 0. */
kpm_status kpm_plan_info(kpm_handle h, int32_t N, int64_t R, uint32_t flags, int64_t info[12]);

/* Counters of the last kpm_moments_ex / kpm_moments_group call on this handle: stats[0] =
 * recursion-step launches, stats[1] = all kernel launches, stats[2] = halo plane copies (row
 * partition, copy exchange), stats[3] = recursion launches that stored their boundary planes
 * straight into the neighbours' ghost planes (fused halo, in-process slab groups). */
kpm_status kpm_last_stats(kpm_handle h, int64_t stats[4]);

/* Algorithmic HBM bytes of the recursion steps of the last kpm_moments_ex call, SURVEY.md 8(d):
 * per recursion step 3 D R s (read a_n, read a_{n-1}, write a_{n+1}; s = 8 fp64, 16 complex128)
 * + 8 D for a stored on-site array + K D (4 + s) for ELL -- whatever kernel ran (a two-step
 * launch counts two steps).  Divide by kpm_last_timing's steps_ms. */
kpm_status kpm_step_bytes(kpm_handle h, double* bytes);

/* bytes[0] = kpm_step_bytes; bytes[1] = the compulsory DRAM bytes of the kernels that ran: every
 * vector block, on-site array and ELL array a launch touches counted once per launch (a two-step
 * launch reads a_n, a_{n-1} and writes a_{n+1}, a_{n+2}: 4 D R s for two steps). */
kpm_status kpm_step_traffic(kpm_handle h, double bytes[2]);

void kpm_destroy(kpm_handle h); /* NULL-safe */
const char* kpm_last_error(void);
const char* kpm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KPM_H_ */
