/* amgb200 -- B200-native solve phase of classical-AMG preconditioned CG.
 *
 * C ABI of libamgb200.so (the drop-in boundary).  Plain pointers and sizes
 * only; every entry point returns an int status (AMG_OK = 0) and leaves a
 * message for amg_last_error().
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/amgkit):
 *   amg_upload_matrix / amg_set_smoother / amg_upload_coarse / amg_set_cycle
 *       the data contract AmgHierarchy / Level / Smoother handed over by
 *       setup():  hierarchy.py:95-152 (Level a/p/pt, factor, factor_kind,
 *       config.nu1/nu2), smoothers.py:26-43 (kind, inv_diag, gmat, gmat_t,
 *       omega).
 *   amg_spmv          sparse.py:203-217      spmv(A, x)
 *   amg_smoother      smoothers.py:168-173   apply_smoother(sm, A, b, x0, steps)
 *   amg_coarse_solve  hierarchy.py:149-152   AmgHierarchy.coarse_solve(b)
 *   amg_vcycle        hierarchy.py:294-312   vcycle(h, y)
 *   amg_pcg           krylov.py:40-92        pcg(spmv(A0,.), b, vcycle(h,.), x0, config)
 *   amg_bicgstab      krylov.py:95-193       bicgstab(spmv(A0,.), b, vcycle(h,.), x0, config)
 * Error mapping (errors.py): AMG_E_DIM -> DimensionMismatchError,
 * AMG_E_NOT_SPD -> NotSpdError, everything else -> AmgError.
 *
 * Conventions: host arrays are borrowed for the duration of the call and
 * copied; the handle owns all device memory; outputs go to caller buffers,
 * host pointers when on_device == 0, device pointers (e.g. a torch tensor's
 * data_ptr()) when on_device == 1.  A handle is driven by one host thread.
 * There is no CPU fallback: without a usable GPU every call fails with
 * AMG_E_CUDA.
 *
 * Multi-GPU: one process per GPU.  Rank 0 makes an ncclUniqueId with
 * amg_nccl_unique_id and shares it (e.g. torch.distributed broadcast); every
 * rank creates its handle with (rank, nranks, id), declares the contiguous row
 * partition of every distributed level (amg_set_partition) and the first
 * REPLICATED level (amg_set_agglomeration; levels from there down are held
 * whole by every rank, the coarsest always is), then uploads its local
 * matrices as produced by the host planner (paper_2102_07417_b200/partition.py):
 * local rows, LOCAL column ids (owned columns first, then halo columns) and
 * the halo plan of each matrix (amg_set_halo: per-peer receive counts in halo
 * order, per-peer owned indices to send).  Row entries keep the reference
 * order, so distributed SpMV rows are bit-identical to single-GPU ones; dots
 * are per-rank partials all-gathered and summed in rank order.  With
 * nranks == 1 none of these calls is needed.
 */
#ifndef AMGB200_H
#define AMGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    AMG_OK = 0,
    AMG_E_ARG = 1,      /* invalid argument / call order        -> AmgError */
    AMG_E_DIM = 2,      /* shape mismatch                        -> DimensionMismatchError */
    AMG_E_NOT_SPD = 3,  /* PCG curvature <= 0                    -> NotSpdError */
    AMG_E_CUDA = 4,     /* CUDA runtime failure / no GPU         -> AmgError */
    AMG_E_NCCL = 5,     /* NCCL failure                          -> AmgError */
    AMG_E_STATE = 6,    /* handle not finalized / already final  -> AmgError */
    AMG_E_BREAKDOWN = 7 /* BiCGstab breakdown                    -> BreakdownError */
};

/* matrix slots of a level (Level.a, Level.p, Level.pt, Smoother.gmat, Smoother.gmat_t) */
enum { AMG_A = 0, AMG_P = 1, AMG_PT = 2, AMG_G = 3, AMG_GT = 4 };
/* smoother kinds (smoothers.py:45-50) */
enum { AMG_SMOOTHER_FSAI = 0, AMG_SMOOTHER_JACOBI = 1 };
/* coarsest factor kinds (hierarchy.py:123-147) */
enum { AMG_COARSE_CHOLESKY = 0, AMG_COARSE_LU = 1 };

typedef struct amg_handle amg_t;

typedef struct amg_stats {
    double solve_ms;          /* device time of the last amg_pcg (CUDA events), excl. H2D/D2H */
    double e2e_ms;            /* host wall time of the last amg_pcg call incl. copies */
    int64_t launches_per_iter;/* kernels launched per PCG iteration (graph body) */
    int64_t launches_last;    /* kernels launched by the last amg_pcg call */
    int64_t bytes_per_iter;   /* algorithmic bytes per PCG iteration (SURVEY 8(d) model) */
    int64_t flops_per_iter;   /* algorithmic flops per PCG iteration */
    int graph_mode;           /* 2 = device while-loop graph, 1 = batched graph launches, 0 = eager */
    int n_levels;
    int tail_level;           /* first level run by the cluster tail kernel (0 = none) */
    int cluster;              /* CTAs in the tail cluster */
} amg_stats_t;

/* Handle for one GPU.  nccl_unique_id: 128 bytes (NULL when nranks == 1). */
int amg_create(int device, int rank, int nranks, const void *nccl_unique_id, amg_t **out);
void amg_destroy(amg_t *h);
const char *amg_last_error(void);
int amg_get_version(void);

int amg_set_levels(amg_t *h, int n_levels);
/* starts[0..nranks]: rows [starts[r], starts[r+1]) of `level` belong to rank r. */
int amg_set_partition(amg_t *h, int level, const int64_t *starts);
/* Matrix `which` of `level` (this rank's rows when the level is distributed):
 * local_nrows rows, CSR offsets[0..local_nrows] (offsets[0] == 0), column ids
 * in [0, ncols) in the reference's stored order, values.  ncols is the
 * column-space size: global columns on one rank / replicated levels, owned +
 * halo columns of the local block otherwise. */
int amg_upload_matrix(amg_t *h, int level, int which, int64_t local_nrows, int64_t ncols,
                      const int64_t *offsets, const int32_t *cols, const double *vals);
/* Multi-GPU (see top): 128-byte ncclUniqueId for amg_create (rank 0). */
int amg_nccl_unique_id(void *out);
/* Halo plan of an uploaded local matrix: columns [n_own, n_own + n_halo) are
 * received, n_recv peers in order with recv_counts each; n_send peers get
 * send_counts[i] owned entries listed (concatenated) in send_idx. */
int amg_set_halo(amg_t *h, int level, int which, int64_t n_own, int64_t n_halo, int n_recv,
                 const int *recv_peers, const int64_t *recv_counts, int n_send, const int *send_peers,
                 const int64_t *send_counts, const int32_t *send_idx);
/* First replicated level (its partition says where each rank's restricted piece goes). */
int amg_set_agglomeration(amg_t *h, int level);
/* inv_diag: this rank's rows (Jacobi) or NULL (FSAI). */
int amg_set_smoother(amg_t *h, int level, int kind, double omega, const double *inv_diag, int64_t n);
/* Dense coarsest factor, n x n row-major: lower Cholesky factor (upper part
 * ignored) or LAPACK getrf LU with 0-based pivots `piv` (kind LU). Replicated on every rank. */
int amg_upload_coarse(amg_t *h, int n, const double *factor, int kind, const int32_t *piv);
int amg_set_cycle(amg_t *h, int nu1, int nu2);
int amg_finalize(amg_t *h);

/* Rows owned by this rank at `level` (vectors passed to the calls below are
 * this rank's slice). */
int64_t amg_local_rows(amg_t *h, int level);

/* y = M x for M = matrix `which` of `level`; x has the matrix's column space
 * (this rank's slice), y its row space. */
int amg_spmv(amg_t *h, int level, int which, const double *x, double *y, int on_device);
/* x = apply_smoother(level, b, x0, steps); x0 may be NULL (zeros). */
int amg_smoother(amg_t *h, int level, const double *b, const double *x0, double *x, int steps,
                 int on_device);
/* z = coarse_solve(y) on the coarsest level (replicated). */
int amg_coarse_solve(amg_t *h, const double *y, double *z, int on_device);
/* z = vcycle(h, y) from level 0. */
int amg_vcycle(amg_t *h, const double *y, double *z, int on_device);
/* z = vcycle(h, y, level) (hierarchy.py:294: the cycle restarted at `level`, vectors of that level's
 * size).  Levels below the first level of the cluster-tail kernel cannot be entered separately
 * (AMG_E_STATE) unless the tail is switched off (option "tail_nnz" = 0). */
int amg_vcycle_level(amg_t *h, int level, const double *y, double *z, int on_device);

/* PCG with the V-cycle preconditioner (krylov.py:40-92).  x0 may be NULL.
 * history: max_iters+1 doubles or NULL; *hist_len = entries written.
 * On AMG_E_NOT_SPD, *n_iter holds the failing iteration and
 * *curvature_at_fail the curvature. */
int amg_pcg(amg_t *h, const double *b, const double *x0, double rtol, int max_iters,
            int recompute_every, double *x_out, int *n_iter, double *relres, int *converged,
            double *history, int *hist_len, double *curvature_at_fail, int on_device);

/* Preconditioned BiCGstab (krylov.py:95-193): one restart on a vanishing
 * shadow product, true-residual checks; AMG_E_BREAKDOWN on a breakdown the
 * reference raises BreakdownError for (outputs hold the state at that point). */
int amg_bicgstab(amg_t *h, const double *b, const double *x0, double rtol, int max_iters,
                 int recompute_every, double *x_out, int *n_iter, double *relres, int *converged,
                 int *restarts, double *history, int *hist_len, int on_device);

int amg_get_stats(amg_t *h, amg_stats_t *out);
/* Diagnostics: launch the SpMV kernel of matrix `which` `reps` times back to
 * back on the handle's stream between CUDA events (operands resident in
 * HBM); *ms_per_launch = average device time of one launch. */
int amg_time_spmv(amg_t *h, int level, int which, int reps, double *ms_per_launch);
/* Diagnostics: the device layout the SpMV of matrix `which` of `level` runs on
 * (chosen at amg_finalize; every layout gives bit-identical rows). */
enum {
    AMG_LAYOUT_CSR = 0,       /* CSR, register / tile kernels */
    AMG_LAYOUT_PADDED = 1,    /* padded-aligned CSR (vector loads) */
    AMG_LAYOUT_PATTERN = 2,   /* padded values + stencil-pattern columns */
    AMG_LAYOUT_SELL = 3,      /* SELL-32 slices, stored columns */
    AMG_LAYOUT_SELL_PAT = 4,  /* SELL-32 slices, stencil-pattern columns */
    AMG_LAYOUT_SYMD = 5,      /* symmetric stencil: upper diagonals + pattern ids */
    AMG_LAYOUT_LEAVES = 6,    /* long rows, leaf list */
    AMG_LAYOUT_EMPTY = 7,
    AMG_LAYOUT_SELL_UNIFORM = 8, /* SELL-32, every slice the same width (short rows) */
    AMG_LAYOUT_SELL_SORTED = 9,  /* SELL-32 over rows sorted by length in windows (SELL-C-sigma) */
    AMG_LAYOUT_SPLIT = 10,       /* rows <= 16 entries as width-16 SELL-32, longer rows from a row list */
    AMG_LAYOUT_DICT = 11,        /* row-class dictionary: class id per row + (offsets, values) table */
    AMG_LAYOUT_WCSR = 12         /* CSR, one warp per 32 consecutive rows (coalesced entries, products in smem) */
};
int amg_matrix_layout(amg_t *h, int level, int which, int *layout);
/* Diagnostics (roofline numerator): *stored = bytes the SpMV kernel of the
 * chosen layout must stream per launch (values, column / pattern ids, row
 * metadata; padding slots it never loads are not counted), *vectors = 8 B per
 * column of x (read once) + 8 B per row of y (written once). */
int amg_matrix_bytes(amg_t *h, int level, int which, int64_t *stored, int64_t *vectors);
/* Tuning / diagnostics: 0 = auto. */
int amg_set_option(amg_t *h, const char *key, int64_t value);

/* ---- Device setup operators -------------------------------
 * The two operators a lean hierarchy cache replays on load, on the GPU and
 * bit-identical to the reference's scipy calls (same terms, same order, products
 * rounded before the add, exact zeros dropped):
 *   amg_device_galerkin : amgkit/sparse.py:256-282 galerkin_product(A, P, symmetrize)
 *                         = P^T A P [(R + R^T)/2], called at hierarchy.py:210
 *   amg_device_transpose: amgkit/sparse.py:220-224 transpose(A) (hierarchy.py:216,
 *                         smoothers.py:145)
 * Host CSR in (int64 offsets, int32 columns, f64 values: the reference dtypes,
 * sparse.py:67-69), result held on the device until fetched into caller buffers
 * sized from amg_csr_result_shape; canonical CSR out (sorted unique columns). */
typedef struct amg_csr_result amg_csr_result_t;
int amg_device_galerkin(int device, int64_t n, int64_t m, const int64_t *a_offsets, const int32_t *a_cols,
                        const double *a_vals, const int64_t *p_offsets, const int32_t *p_cols, const double *p_vals,
                        int symmetrize, amg_csr_result_t **out);
int amg_device_transpose(int device, int64_t nrows, int64_t ncols, const int64_t *offsets, const int32_t *cols,
                         const double *vals, amg_csr_result_t **out);
int amg_csr_result_shape(const amg_csr_result_t *r, int64_t *nrows, int64_t *ncols, int64_t *nnz);
int amg_csr_result_fetch(const amg_csr_result_t *r, int64_t *offsets, int32_t *cols, double *vals);
void amg_csr_result_free(amg_csr_result_t *r);

#ifdef __cplusplus
}
#endif

#endif /* AMGB200_H */
