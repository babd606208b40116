/*
 * oracle/kpm_oracle.c -- CPU ORACLE for the KPM moment recursion.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1105_5481_b200/), and the CUDA path never loads it.
 *
 * Plain, slow, obviously correct: CSR storage built here from the lattice
 * description, one vector at a time, fp64 throughout.  OpenMP parallelises
 * over the random vectors (the paper's own decomposition: "the total number
 * of threads ... is SR"); per-vector results are summed in the
 * fixed order r = 0..R-1.  With fewer vectors than threads the vectors run in
 * turn and each row loop / inner product is split over the threads instead
 * (SURVEY.md 8(d)); only then does the inner-product summation order depend on
 * the thread count (reading X18).
 *
 * Functions and the passage each follows:
 *   oracle_build_lattice_csr   O1: H of the periodic nearest-neighbour lattice
 *                              (Sec IV-A: 7 entries per row in 3D,
 *                              zero diagonal, off-diagonal -1), optional on-site
 *                              energies (Anderson, reading X14) and a Peierls
 *                              phase on y-bonds (reading X15).
 *   oracle_gershgorin          Eq (8)-(9): E_upper/E_lower from
 *                              Gerschgorin discs, alpha_+- = (Eu +- El)/2.
 *   oracle_moments_direct      O2: Eq (17)-(19), PAPER.md:130-138:
 *                              |r_0> = |r>, |r_1> = H~|r_0>,
 *                              |r_{n+2}> = 2 H~|r_{n+1}> - |r_n>,
 *                              mu_n = (1/D)(1/R) sum_r <r_0|r_n>.
 *   oracle_moments_doubling    O3: the doubling identities of BASELINE.json's
 *                              north_star: mu_{2n} = 2<a_n|a_n> - mu_0,
 *                              mu_{2n+1} = 2<a_{n+1}|a_n> - mu_1 (they follow
 *                              from T_{2n} = 2 T_n^2 - T_0 and
 *                              T_{2n+1} = 2 T_n T_{n+1} - T_1, Eq (3)).
 * H~ = (H - alpha_+)/alpha_- (Eq 8) is applied as written: y = (Hx - b x)/a.
 * Complex H (Peierls) keeps real start vectors (Eq 14 takes xi real) and
 * takes the real part of the inner products (reading X16).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Entries per row: one diagonal entry if on-site energies are given, plus a
 * +1 and a -1 neighbour in each of the ndim dimensions. */
int64_t oracle_lattice_nnz(int ndim, const int64_t *L, int has_onsite) {
    int64_t D = L[0] * L[1] * L[2];
    return D * (2 * ndim + (has_onsite ? 1 : 0));
}

/* Phase angle carried by the bond from site u = (ux, uy, uz) to u + e_d:
 * H[u + e_d][u] = t * exp(i theta), theta = 2 pi flux ux on y-bonds (d == 1),
 * 0 otherwise (Landau gauge, reading X15). */
static double bond_phase(int d, int64_t ux, double flux) {
    return (d == 1) ? 2.0 * M_PI * flux * (double)ux : 0.0;
}

int oracle_build_lattice_csr(int ndim, const int64_t *L, double t, const double *onsite,
                             double flux, int64_t *rowptr, int32_t *col, double *val_re,
                             double *val_im) {
    if (ndim < 1 || ndim > 3) return 1;
    int64_t D = L[0] * L[1] * L[2];
    int64_t nnz = 0;
    for (int64_t i = 0; i < D; i++) {
        rowptr[i] = nnz;
        int64_t c[3] = {i % L[0], (i / L[0]) % L[1], i / (L[0] * L[1])};
        if (onsite) {
            col[nnz] = (int32_t)i;
            val_re[nnz] = onsite[i];
            val_im[nnz] = 0.0;
            nnz++;
        }
        for (int d = 0; d < ndim; d++) {
            for (int s = +1; s >= -1; s -= 2) {
                int64_t n[3] = {c[0], c[1], c[2]};
                n[d] = (c[d] + s + L[d]) % L[d]; /* periodic (reading X12) */
                int64_t j = n[0] + L[0] * (n[1] + L[1] * n[2]);
                double complex h;
                if (s == +1) {
                    /* H[i][i+e_d] = conj(H[i+e_d][i]) = conj(t e^{i theta(i)}) */
                    h = conj(t * cexp(I * bond_phase(d, c[0], flux)));
                } else {
                    /* H[i][i-e_d] = H[(i-e_d)+e_d][i-e_d] = t e^{i theta(i-e_d)} */
                    h = t * cexp(I * bond_phase(d, n[0], flux));
                }
                col[nnz] = (int32_t)j;
                val_re[nnz] = creal(h);
                val_im[nnz] = cimag(h);
                nnz++;
            }
        }
    }
    rowptr[D] = nnz;
    return 0;
}

/* Gerschgorin: every eigenvalue lies in some disc
 * |z - H_ii| <= sum_{j != i} |H_ij|; E_upper = max_i (Re H_ii + radius_i),
 * E_lower = min_i (Re H_ii - radius_i); eps pads both sides (reading X6). */
void oracle_gershgorin(int64_t D, const int64_t *rowptr, const int32_t *col, const double *val_re,
                       const double *val_im, double eps, double *a, double *b) {
    double Eu = -INFINITY, El = INFINITY;
    for (int64_t i = 0; i < D; i++) {
        double diag = 0.0, radius = 0.0;
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; k++) {
            double complex h = val_re[k] + I * (val_im ? val_im[k] : 0.0);
            if (col[k] == i) diag += creal(h);
            else radius += cabs(h);
        }
        if (diag + radius > Eu) Eu = diag + radius;
        if (diag - radius < El) El = diag - radius;
    }
    Eu += eps;
    El -= eps;
    *a = (Eu - El) / 2.0; /* alpha_-, Eq (9) */
    *b = (Eu + El) / 2.0; /* alpha_+, Eq (9) */
}

typedef struct {
    int64_t D;
    const int64_t *rowptr;
    const int32_t *col;
    const double *val_re;
    const double *val_im;
    double a, b;
} csr_t;

/* Parallel decomposition: OpenMP over the R vectors (the paper's own
 * decomposition); when there are fewer vectors than threads, the vectors run one
 * after the other and each row loop / inner product below is split over the threads instead
 * ("rows" below = 1).  Only the summation order of the inner products changes with it (reading
 * X18: rounding order is free; X17's tolerance covers it). */
static int rows = 0;

/* y = H~ x = (H x - b x) / a, real H (Eq 8). */
static void apply_Ht_real(const csr_t *H, const double *x, double *y) {
#pragma omp parallel for schedule(static) if (rows)
    for (int64_t i = 0; i < H->D; i++) {
        double s = 0.0;
        for (int64_t k = H->rowptr[i]; k < H->rowptr[i + 1]; k++) s += H->val_re[k] * x[H->col[k]];
        y[i] = (s - H->b * x[i]) / H->a;
    }
}

/* y = H~ x = (H x - b x) / a, complex H (Eq 8). */
static void apply_Ht_cplx(const csr_t *H, const double complex *x, double complex *y) {
#pragma omp parallel for schedule(static) if (rows)
    for (int64_t i = 0; i < H->D; i++) {
        double complex s = 0.0;
        for (int64_t k = H->rowptr[i]; k < H->rowptr[i + 1]; k++)
            s += (H->val_re[k] + I * H->val_im[k]) * x[H->col[k]];
        y[i] = (s - H->b * x[i]) / H->a;
    }
}

static double dot_real(int64_t D, const double *u, const double *v) {
    double s = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : s) if (rows)
    for (int64_t i = 0; i < D; i++) s += u[i] * v[i];
    return s;
}

/* nx = 2 nx - p (Eq 18), real and complex */
static void recur_real(int64_t D, double *nx, const double *p) {
#pragma omp parallel for schedule(static) if (rows)
    for (int64_t i = 0; i < D; i++) nx[i] = 2.0 * nx[i] - p[i];
}
static void recur_cplx(int64_t D, double complex *nx, const double complex *p) {
#pragma omp parallel for schedule(static) if (rows)
    for (int64_t i = 0; i < D; i++) nx[i] = 2.0 * nx[i] - p[i];
}

/* Re <u|v> = Re sum_i conj(u_i) v_i */
static double redot_cplx(int64_t D, const double complex *u, const double complex *v) {
    double s = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : s) if (rows)
    for (int64_t i = 0; i < D; i++) s += creal(conj(u[i]) * v[i]);
    return s;
}

/* Sum the per-vector moments m[r][n] in the fixed order r = 0..R-1 and
 * normalise by 1/(D R) (Eq 19; reading X2).  pervec (optional) gets m/D. */
static void finish(int64_t D, int64_t R, int N, const double *m, double *mu, double *pervec) {
    for (int n = 0; n < N; n++) {
        double s = 0.0;
        for (int64_t r = 0; r < R; r++) s += m[r * N + n];
        mu[n] = s / ((double)D * (double)R);
    }
    if (pervec)
        for (int64_t k = 0; k < R * (int64_t)N; k++) pervec[k] = m[k] / (double)D;
}

/* O2: the paper's scheme, Eq (17)-(19): N-1 applications of H~ per vector.
 * r is (R, D) vector-major; mu gets N values; pervec (nullable) gets (R, N). */
int oracle_moments_direct(int64_t D, const int64_t *rowptr, const int32_t *col,
                          const double *val_re, const double *val_im, int is_complex, double a,
                          double b, int64_t R, const double *r, int N, double *mu,
                          double *pervec) {
    if (N < 1 || R < 1 || D < 1 || !(a > 0)) return 1;
    csr_t H = {D, rowptr, col, val_re, val_im, a, b};
    double *m = calloc((size_t)(R * N), sizeof(double));
    if (!m) return 2;
    rows = R < omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) if (!rows)
    for (int64_t q = 0; q < R; q++) {
        const double *rv = r + q * D;
        double *mq = m + q * N;
        if (!is_complex) {
            double *u0 = malloc(D * sizeof(double)), *u1 = malloc(D * sizeof(double)),
                   *u2 = malloc(D * sizeof(double));
            memcpy(u0, rv, D * sizeof(double));          /* |r_0> = |r>      (Eq 17) */
            mq[0] = dot_real(D, rv, u0);
            if (N > 1) {
                apply_Ht_real(&H, u0, u1);                /* |r_1> = H~|r_0>  (Eq 17) */
                mq[1] = dot_real(D, rv, u1);
            }
            for (int n = 2; n < N; n++) {
                apply_Ht_real(&H, u1, u2);                /* (Eq 18) */
                recur_real(D, u2, u0);
                mq[n] = dot_real(D, rv, u2);              /* <r_0|r_n> (Eq 19) */
                double *tmp = u0; u0 = u1; u1 = u2; u2 = tmp;
            }
            free(u0); free(u1); free(u2);
        } else {
            double complex *u0 = malloc(D * sizeof(double complex)),
                           *u1 = malloc(D * sizeof(double complex)),
                           *u2 = malloc(D * sizeof(double complex)),
                           *rc = malloc(D * sizeof(double complex));
            for (int64_t i = 0; i < D; i++) rc[i] = rv[i];
            memcpy(u0, rc, D * sizeof(double complex));
            mq[0] = redot_cplx(D, rc, u0);
            if (N > 1) {
                apply_Ht_cplx(&H, u0, u1);
                mq[1] = redot_cplx(D, rc, u1);
            }
            for (int n = 2; n < N; n++) {
                apply_Ht_cplx(&H, u1, u2);
                recur_cplx(D, u2, u0);
                mq[n] = redot_cplx(D, rc, u2);
                double complex *tmp = u0; u0 = u1; u1 = u2; u2 = tmp;
            }
            free(u0); free(u1); free(u2); free(rc);
        }
    }
    finish(D, R, N, m, mu, pervec);
    free(m);
    return 0;
}

/* O3: doubling form, floor(N/2) applications of H~ per vector (N >= 2):
 *   p = a_0 = r, c = a_1 = H~ r, s0 = <r|r>, s1 = <r|a_1>
 *   for n = 1, 2, ... while 2n < N:
 *       m_{2n}   = 2 <a_n|a_n> - s0              (c = a_n)
 *       stop if 2n + 1 >= N
 *       q = a_{n+1} = 2 H~ a_n - a_{n-1}          (Eq 18)
 *       m_{2n+1} = 2 <a_n|a_{n+1}> - s1
 *       p, c = c, q                                                        */
int oracle_moments_doubling(int64_t D, const int64_t *rowptr, const int32_t *col,
                            const double *val_re, const double *val_im, int is_complex, double a,
                            double b, int64_t R, const double *r, int N, double *mu,
                            double *pervec) {
    if (N < 1 || R < 1 || D < 1 || !(a > 0)) return 1;
    csr_t H = {D, rowptr, col, val_re, val_im, a, b};
    double *m = calloc((size_t)(R * N), sizeof(double));
    if (!m) return 2;
    rows = R < omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) if (!rows)
    for (int64_t q = 0; q < R; q++) {
        const double *rv = r + q * D;
        double *mq = m + q * N;
        if (!is_complex) {
            double *p = malloc(D * sizeof(double)), *c = malloc(D * sizeof(double)),
                   *nx = malloc(D * sizeof(double));
            memcpy(p, rv, D * sizeof(double));
            double s0 = dot_real(D, p, p);
            mq[0] = s0;
            if (N > 1) {
                apply_Ht_real(&H, p, c);
                double s1 = dot_real(D, p, c);
                mq[1] = s1;
                for (int n = 1; 2 * n < N; n++) {
                    mq[2 * n] = 2.0 * dot_real(D, c, c) - s0;
                    if (2 * n + 1 >= N) break;
                    apply_Ht_real(&H, c, nx);
                    recur_real(D, nx, p);
                    mq[2 * n + 1] = 2.0 * dot_real(D, c, nx) - s1;
                    double *tmp = p; p = c; c = nx; nx = tmp;
                }
            }
            free(p); free(c); free(nx);
        } else {
            double complex *p = malloc(D * sizeof(double complex)),
                           *c = malloc(D * sizeof(double complex)),
                           *nx = malloc(D * sizeof(double complex));
            for (int64_t i = 0; i < D; i++) p[i] = rv[i];
            double s0 = redot_cplx(D, p, p);
            mq[0] = s0;
            if (N > 1) {
                apply_Ht_cplx(&H, p, c);
                double s1 = redot_cplx(D, p, c);
                mq[1] = s1;
                for (int n = 1; 2 * n < N; n++) {
                    mq[2 * n] = 2.0 * redot_cplx(D, c, c) - s0;
                    if (2 * n + 1 >= N) break;
                    apply_Ht_cplx(&H, c, nx);
                    recur_cplx(D, nx, p);
                    mq[2 * n + 1] = 2.0 * redot_cplx(D, c, nx) - s1;
                    double complex *tmp = p; p = c; c = nx; nx = tmp;
                }
            }
            free(p); free(c); free(nx);
        }
    }
    finish(D, R, N, m, mu, pervec);
    free(m);
    return 0;
}
