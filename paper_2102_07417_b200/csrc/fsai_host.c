/* Host-side replay of the final FSAI row solves (setup data, NOT the solve path).
 *
 * The reference builds each FSAI row as (amgkit/smoothers.py:80-96):
 *     idx  = pattern_i ++ [i]                       (strictly-lower pattern, sorted)
 *     sub  = A[idx, idx]                            (_principal_submatrix, :152-165)
 *     c    = cho_factor(sub, lower=True)            (LAPACK dpotrf, see below)
 *     y    = cho_solve((c, True), e_last)           (LAPACK dpotrs 'L')
 *     g_i  = y / sqrt(y[-1])        or the Jacobi row 1/sqrt(a_ii) on failure
 * The final coefficients depend only on (A, final pattern, fallback flag), so
 * a frozen hierarchy need not store them: given the pattern this file
 * recomputes them with the SAME LAPACK routines scipy calls (their addresses
 * come from scipy.linalg.cython_lapack, i.e. scipy's bundled OpenBLAS), in the
 * same element order, and the caller verifies the result against the SHA-256
 * digest recorded from the reference's own arrays.
 *
 * Rows are independent; they are split over `nthreads` pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef void (*potrf_fn)(char *uplo, int *n, double *a, int *lda, int *info);
typedef void (*potrs_fn)(char *uplo, int *n, int *nrhs, double *a, int *lda, double *b, int *ldb, int *info);

typedef struct {
    potrf_fn potrf;
    potrs_fn potrs;
    int64_t n;
    const int64_t *a_off;
    const int32_t *a_col;
    const double *a_val;
    const int64_t *g_off;
    const int32_t *g_col;
    const uint8_t *fallback;
    double *g_val;
    int64_t r0, r1;
    int64_t failed;  /* rows whose local solve failed (value set to NaN) */
    int64_t bad_row; /* a row whose fallback flag contradicts its pattern, or -1 */
} job_t;

static double a_diag(const job_t *J, int64_t i) {
    for (int64_t e = J->a_off[i]; e < J->a_off[i + 1]; ++e)
        if (J->a_col[e] == (int32_t)i) return J->a_val[e];
    return 0.0;
}

static void *run(void *arg) {
    job_t *J = (job_t *)arg;
    int cap = 0;
    double *sub = NULL, *y = NULL;
    for (int64_t i = J->r0; i < J->r1; ++i) {
        const int64_t gs = J->g_off[i];
        const int m = (int)(J->g_off[i + 1] - gs);
        const int32_t *idx = J->g_col + gs;
        double *out = J->g_val + gs;
        if (J->fallback && J->fallback[i]) {
            /* smoothers.py:94-96: empty pattern, Jacobi row */
            if (m != 1) { J->bad_row = i; break; }
            out[0] = 1.0 / sqrt(a_diag(J, i));
            continue;
        }
        if (m > cap) {
            cap = m < 16 ? 16 : 2 * m;
            free(sub);
            free(y);
            sub = (double *)malloc(sizeof(double) * (size_t)cap * cap);
            y = (double *)malloc(sizeof(double) * (size_t)cap);
            if (!sub || !y) { J->bad_row = i; break; }
        }
        memset(sub, 0, sizeof(double) * (size_t)m * m);
        /* sub[t, u] = A(idx[t], idx[u]) stored ROW-major (t*m + u), as the
         * reference's C-ordered ndarray; idx is ascending (pattern < i). */
        for (int t = 0; t < m; ++t) {
            const int64_t r = idx[t];
            for (int64_t e = J->a_off[r]; e < J->a_off[r + 1]; ++e) {
                const int32_t c = J->a_col[e];
                int lo = 0, hi = m;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (idx[mid] < c) lo = mid + 1; else hi = mid;
                }
                if (lo < m && idx[lo] == c) sub[(int64_t)t * m + lo] = J->a_val[e];
            }
        }
        /* cho_factor(sub, lower=True) (scipy >= 1.15, _batched_linalg) factors
         * the C-ordered buffer in place as the Fortran UPPER factor U = L^T:
         * dpotrf('U') on the row-major buffer.  Measured bit-identical. */
        char up = 'U', lo_ = 'L';
        int n = m, lda = m, info = 0, nrhs = 1;
        J->potrf(&up, &n, sub, &lda, &info);
        if (info != 0) { /* LinAlgError -> the reference would have fallen back */
            for (int t = 0; t < m; ++t) out[t] = NAN;
            J->failed++;
            continue;
        }
        /* cho_solve((c, True), e) hands LAPACK a Fortran copy of the C-ordered
         * factor c and calls dpotrs('L'): transpose into column-major. */
        for (int t = 0; t < m; ++t)
            for (int u = 0; u < t; ++u) {
                const double v = sub[(int64_t)t * m + u];
                sub[(int64_t)t * m + u] = sub[(int64_t)u * m + t];
                sub[(int64_t)u * m + t] = v;
            }
        memset(y, 0, sizeof(double) * (size_t)m);
        y[m - 1] = 1.0;
        J->potrs(&lo_, &n, &nrhs, sub, &lda, y, &lda, &info);
        if (info != 0 || !(y[m - 1] > 0.0)) {
            for (int t = 0; t < m; ++t) out[t] = NAN;
            J->failed++;
            continue;
        }
        const double s = sqrt(y[m - 1]);
        for (int t = 0; t < m; ++t) out[t] = y[t] / s;
    }
    free(sub);
    free(y);
    return NULL;
}

/* Recomputes every row of G's values.  Rows flagged in `fallback` (may be
 * NULL) get the Jacobi value.  Returns the number of rows whose local solve
 * failed (their values are NaN: the reference would have fallen back on
 * them), or -1 - r when the fallback flag of row r contradicts its pattern
 * (a fallback row has only its diagonal) or memory ran out. */
int64_t amgh_fsai_values(void *potrf, void *potrs, int64_t n, const int64_t *a_off, const int32_t *a_col,
                         const double *a_val, const int64_t *g_off, const int32_t *g_col,
                         const uint8_t *fallback, double *g_val, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
    job_t *jobs = (job_t *)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        job_t *J = &jobs[t];
        J->potrf = (potrf_fn)potrf;
        J->potrs = (potrs_fn)potrs;
        J->n = n;
        J->a_off = a_off; J->a_col = a_col; J->a_val = a_val;
        J->g_off = g_off; J->g_col = g_col; J->fallback = fallback; J->g_val = g_val;
        J->r0 = n * t / nthreads;
        J->r1 = n * (t + 1) / nthreads;
        J->bad_row = -1;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run, &jobs[t]);
    run(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    int64_t failed = 0, bad = -1;
    for (int t = 0; t < nthreads; ++t) {
        failed += jobs[t].failed;
        if (bad < 0 && jobs[t].bad_row >= 0) bad = jobs[t].bad_row;
    }
    free(jobs);
    free(th);
    return bad >= 0 ? -1 - bad : failed;
}
