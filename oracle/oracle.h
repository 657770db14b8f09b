/* oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11 + pthreads) of the reference's batched
 * Newton-Raphson power-flow path, used as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm.
 * The product (paper_2101_02270_b200/libgbnr.so) never links, loads or calls it.
 *
 * What it restates (file:line in /root/reference):
 *   orc_build_ybus      grid.hpp:195-243   (MATPOWER branch model, shunts)
 *   orc_amd             amd.hpp:29-157     (quotient-graph AMD, lowest-index ties)
 *   orc_plan_create     SPEC.md:185-188 (reduced J pattern), :292-300
 *                       (factorize_initial: left-looking G-P + threshold pivoting),
 *                       :301-309 (level schedule), sparse.hpp:237-267 (scatter lookup)
 *   orc_solve           SPEC.md:195-230 (compute_npm, update_jacobian,
 *                       update_voltage), :213-221 (nr_solve_batch), :310-318
 *                       (refactorize_batch = PAPER.md Alg. 2), :328-336 (fs_bs_batch)
 *   orc_branch_flows    SPEC.md:231-239 (calc_branch_flows)
 *   worker pool + mini-batches: SPEC.md:254-255, batch_tape.hpp:80-92
 *
 * Parity status: the substrate (Ybus, profiles, AMD ordering, CRS/CCS/scatter)
 * is pinned against the reference's own headers compiled into oracle/_ref
 * (fixtures in tests/golden/, made by tools/make_golden.py).  The NR/LU part has no
 * reference implementation; it is pinned against the published
 * IEEE case14 solution and an independent scipy/SuperLU MATPOWER newtonpf.
 *
 * Arithmetic contract shared with the CUDA path: IEEE binary64,
 * no FP contraction (-ffp-contract=off), explicit fma() exactly where written,
 * the sincos of orc_sincos, fixed per-element accumulation orders.
 */
#ifndef GBNR_ORACLE_H
#define GBNR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_plan orc_plan;

const char* orc_last_error(void);

void orc_sincos(double x, double* s, double* c);

int orc_build_ybus(int32_t n_bus, int32_t n_branch, const int32_t* f, const int32_t* t,
                   const double* r, const double* x, const double* b, const double* tap,
                   const double* shift_deg, const uint8_t* in_service, const double* gs,
                   const double* bs, double base_mva, int32_t* indptr, int32_t* indices,
                   int32_t* diag, double* y_re, double* y_im, int32_t* nnz_out);

int orc_amd(int32_t n, const int32_t* col_ptr, const int32_t* row_ix, int32_t* fwd);

int orc_plan_create(int32_t n_bus, const int32_t* indptr, const int32_t* indices,
                    const double* y_re, const double* y_im, int32_t ref, const int32_t* pv,
                    int32_t n_pv, const int32_t* pq, int32_t n_pq, const double* vm0,
                    const double* va0, double pivot_tol, orc_plan** out);
void orc_plan_destroy(orc_plan* p);

/* out[0..15]: nJ, nnzJ, nnzLU, nnzL(strict), nnzU(strict), D, flops_lu, levels_lu,
 * levels_fs, levels_bs, offdiag_pivots, npvpq, n_fill, max_col, max_udeps, 0 */
int orc_plan_stats(const orc_plan* p, int64_t* out);
/* row_fwd/col_fwd [nJ]: J index -> A index; col_ptr [nJ+1], row_ix [nnzLU]; level [nJ] */
int orc_plan_export(const orc_plan* p, int32_t* row_fwd, int32_t* col_fwd, int32_t* col_ptr,
                    int32_t* row_ix, int32_t* level);

/* Batched NR.  Batched arrays are element-major, task innermost:
 *   y_re/y_im [nnzY][n_ysets], p0/q0 [n_bus][n_ssets], vm0/va0 [n_bus][n_vsets],
 *   n_*sets in {1, n_tasks}; outputs vm/va [n_bus][n_tasks].
 * status: 0 converged, 1 diverged, 2 singular. */
int orc_solve(const orc_plan* p, int32_t n_tasks, const double* y_re, const double* y_im,
              int32_t n_ysets, const double* p0, const double* q0, int32_t n_ssets,
              const double* vm0, const double* va0, int32_t n_vsets, double tol,
              int32_t max_iter, double singular_tol, double* vm_out, double* va_out,
              int32_t* iterations, uint8_t* converged, int32_t* status, double* max_mismatch,
              int32_t n_threads);

/* One Jacobian + refactorization per task at the given voltages,
 * for the LU microbenchmark parity (BASELINE configs[2]).
 * lu_out [nnzLU][n_tasks]; flags [n_tasks] = 1 if a pivot was flagged. */
int orc_refactor(const orc_plan* p, int32_t n_tasks, const double* vm, const double* va,
                 double singular_tol, double* lu_out, uint8_t* flags, int32_t n_threads);

/* Single mismatch evaluation for F vector checks.
 * f_out [nJ][n_tasks] in J row order [P(pv;pq); Q(pq)]. */
int orc_mismatch(const orc_plan* p, int32_t n_tasks, const double* p0, const double* q0,
                 const double* vm, const double* va, double* f_out);

/* calc_branch_flows for voltages vm/va [n_bus][n_tasks];
 * adm [n_branch][8] = (ff, ft, tf, tt) as (re, im); outage [n_tasks] or NULL;
 * outputs [n_branch][n_tasks]. */
int orc_branch_flows(int32_t n_bus, int32_t n_branch, const int32_t* f, const int32_t* t,
                     const double* adm, int32_t n_tasks, const double* vm, const double* va,
                     const int32_t* outage, double* sf_re, double* sf_im, double* st_re, double* st_im);

#ifdef __cplusplus
}
#endif
#endif
