/* gbnr.h -- C ABI of the B200-native batched Newton-Raphson power-flow solver.
 *
 * Drop-in boundary for the reference's hot path.  The
 * reference has no FFI; its in-library boundary is
 *     nr_solve_batch(case, symbolic, tapes, cfg) -> TaskResult[]
 * fed by batch_runtime.initialize / run, with the inputs
 * built by grid_model (grid.hpp:208-344) and laid out as BatchTape
 * (batch_tape.hpp:6-9).  The paper's caller reaches the same solver from Python
 * through Cython with numpy buffers.  This header replaces
 * that boundary with plain pointers:
 *
 *   gbnr_plan_create   <- batch_runtime.initialize: Jacobian
 *                         pattern, amd_order (amd.hpp:29),
 *                         factorize_initial, build_level_schedule
 *                         (SPEC.md:301-309), build_scatter_lookup (sparse.hpp:237)
 *   gbnr_solve         <- nr_solve_batch + TaskResult (:382-385)
 *   gbnr_build_ybus    <- build_ybus (grid.hpp:208-243)
 *   gbnr_amd_order     <- amd_order (amd.hpp:29-157)
 *   gbnr_plan_stats    <- cmd_inspect counters
 *   gbnr_refactor      <- refactorize_batch, LU-only microbenchmark
 *   gbnr_solve_batches <- batch_runtime.run over mini-batches, pipelined
 *   gbnr_contingency_values <- ybus_values_with_outage / outage_islands_grid (grid.hpp:245-261)
 *   gbnr_branch_flows  <- calc_branch_flows
 *
 * Conventions
 *  - Batched arrays are element-major with the task index innermost
 *    (value(elem, task) at elem * n_tasks + task), exactly BatchTape.
 *    n_*sets in {1, n_tasks}: one shared set broadcast to all tasks, or one
 *    per task (ProfileBatch.n_sets, grid.hpp:292, :301-302).
 *  - Voltages are polar (|V| p.u., angle rad) as PolarVoltageBatch;
 *    Sbus = p0 + j q0 is the specified injection in p.u. (grid.hpp:326-327).
 *  - Unknown/equation order is MATPOWER's: [theta(pv;pq), |V|(pq)].
 *  - Return codes map core.hpp:32-65: 0 ok, 1 parse, 2 structural, 3 config,
 *    4 singular initial factorization, 5 CUDA.  No C++ exception crosses the
 *    ABI.  Per-task numerical failure goes to status_out, never to the return
 *    code (core.hpp:33-34).
 *  - A plan is immutable after creation; calls on one plan serialize.  A plan
 *    with n_devices > 1 holds one device plan per GPU and drives them from one
 *    host thread each inside gbnr_solve / gbnr_solve_batches; the split form
 *    (gbnr_stage / gbnr_run / gbnr_fetch), gbnr_refactor and gbnr_branch_flows
 *    use the first device.  A batch larger than a device's memory is solved in
 *    chunks (gbnr_options.chunk_tasks); results never depend on the sharding or
 *    the chunking (tasks are independent).
 *  - There is no CPU fallback: a plan created with device >= 0 runs only on the
 *    GPU; gbnr_solve on a host-only plan (device = -1) returns 3.
 */
#ifndef GBNR_H
#define GBNR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBNR_OK 0
#define GBNR_EPARSE 1
#define GBNR_ESTRUCT 2
#define GBNR_ECONFIG 3
#define GBNR_ESINGULAR 4
#define GBNR_ECUDA 5

/* per-task status (TaskResult.status) */
#define GBNR_CONVERGED 0
#define GBNR_DIVERGED 1
#define GBNR_SINGULAR 2
#define GBNR_FALLBACK_CONVERGED 3 /* converged after the second-chance factorization */

typedef struct gbnr_plan gbnr_plan;

typedef struct gbnr_options {
    double tol;            /* mismatch infinity-norm tolerance, p.u. (default 1e-8)   */
    int32_t max_iter;      /* Newton iterations (default 10, at most 30)             */
    double pivot_tol;      /* threshold partial pivoting (default 1e-3) */
    double singular_tol;   /* refactor pivot flag, relative (default 1e-14)          */
    int32_t device;        /* CUDA ordinal; -1 = host-only plan (symbolic only)      */
    int32_t ring_rows;     /* per-walker ring of step blocks, 256 B rows (0 = auto) */
    int32_t profile;       /* 1 = record per-phase CUDA-event timings               */
    int32_t stage_rows;    /* per-walker staging ring rows (0 = auto)              */
    int32_t prefetch;      /* steps a walk copy may run ahead (0 = 8)              */
    int32_t headroom;      /* ring residency margin in steps (0 = 1)               */
    int32_t walkers;       /* warps per tile walking disjoint subtrees (0 = 8, <= 8) */
    int32_t jacobian;      /* when the next Jacobian is built: 0 = inside the mismatch
                              sweep unless every active task of its 32-task warp is
                              predicted to converge at that check (a wrong guess adds
                              a Jacobian-only launch);
                              1 = always inside the sweep; 2 = always after the check
                              (the reference's order).  Results are identical.        */
    int32_t second_chance; /* 1 (default): every task whose frozen pivot collapsed is
                              re-planned alone with fresh pivoting at its current
                              voltages and continues; status 3
                              on convergence.  The re-plans run concurrently (host
                              threads, one stream each).  0 = off.  With a shared
                              Ybus, >5% of the tasks failing at their first solve
                              restarts the batch once from the worst task's pivots
                              (SPEC.md design decisions).                           */
    int32_t n_devices;     /* gbnr_solve / gbnr_solve_batches shard the tasks over this
                              many GPUs (0 or 1 = one): contiguous slices, one plan,
                              host thread and stream per device, results gathered
                              straight into the caller's buffers.  No collective.   */
    int32_t device_step;   /* device of shard i = device + i * device_step (default 1;
                              0 = every shard on `device`, e.g. tests on one GPU)    */
    int32_t chunk_tasks;   /* most tasks per device launch; larger slices are solved in
                              chunks (0 = automatic, from the free device memory)    */
    int32_t tile_width;    /* tasks per tile, even, 2..32 (0 = automatic: 24 when that
                              keeps every SM at three tiles where 32 would not fit two,
                              else 32; narrower tiles give each walk warp more shared
                              rows).  Results never depend on it.                    */
} gbnr_options;

void gbnr_default_options(gbnr_options* opt);
const char* gbnr_last_error(void);
const char* gbnr_version(void);

/* MATPOWER branch model Ybus (grid.hpp:195-243).  Branch endpoints are internal
 * 0-based bus indices.  indptr [n_bus+1]; indices/diag/y_re/y_im need capacity
 * n_bus + 2*n_branch; *nnz_out receives nnz. */
int gbnr_build_ybus(int32_t n_bus, int32_t n_branch, const int32_t* from, const int32_t* to,
                    const double* r, const double* x, const double* b, const double* tap,
                    const double* shift_deg, const uint8_t* in_service, const double* gs,
                    const double* bs, double base_mva, int32_t* indptr, int32_t* indices,
                    int32_t* diag, double* y_re, double* y_im, int32_t* nnz_out);

/* N-1 contingency value sets on the base pattern (ybus_values_with_outage,
 * grid.hpp:245-255): task t removes branch outage_branch[t] (-1 = base case);
 * y_re/y_im [nnzY][n_tasks] element-major in gbnr_build_ybus slot order, ready
 * for gbnr_solve with n_ysets = n_tasks.  islanded [n_tasks] (may be NULL) =
 * the outage splits the grid (outage_islands_grid, grid.hpp:257-261). */
int gbnr_contingency_values(int32_t n_bus, int32_t n_branch, const int32_t* from, const int32_t* to,
                            const double* r, const double* x, const double* b, const double* tap,
                            const double* shift_deg, const uint8_t* in_service, const double* gs,
                            const double* bs, double base_mva, const int32_t* outage_branch, int32_t n_tasks,
                            double* y_re, double* y_im, uint8_t* islanded);

/* Per-branch admittances adm [n_branch][8]: (ff, ft, tf, tt) as (re, im),
 * zero for out-of-service branches (branch_admittance, grid.hpp:195-206). */
int gbnr_branch_admittances(int32_t n_bus, int32_t n_branch, const int32_t* from, const int32_t* to,
                            const double* r, const double* x, const double* b, const double* tap,
                            const double* shift_deg, const uint8_t* in_service, const double* gs,
                            const double* bs, double base_mva, double* adm);

/* Fill-reducing ordering on a square CCS pattern (amd.hpp:29-157); fwd[old] = new. */
int gbnr_amd_order(int32_t n, const int32_t* col_ptr, const int32_t* row_ix, int32_t* fwd);

/* One-time symbolic analysis + device setup.  (y_re, y_im) are the Ybus values
 * of the representative task and (vm0, va0) its start voltages [n_bus]; they
 * fix the pivot sequence of the initial factorization. */
int gbnr_plan_create(int32_t n_bus, const int32_t* indptr, const int32_t* indices,
                     const double* y_re, const double* y_im, int32_t ref, const int32_t* pv,
                     int32_t n_pv, const int32_t* pq, int32_t n_pq, const double* vm0,
                     const double* va0, const gbnr_options* opt, gbnr_plan** out);
void gbnr_plan_destroy(gbnr_plan* plan);

/* out[16]: nJ, nnzJ, nnzLU, nnzL, nnzU, D (VMAD element updates), flops_lu,
 * levels_lu, levels_fs, levels_bs, offdiag_pivots, npvpq, n_fill, max_col,
 * max_udeps, nnzY */
int gbnr_plan_stats(const gbnr_plan* plan, int64_t* out);
/* row_fwd/col_fwd [nJ] (J index -> LU index), col_ptr [nJ+1], row_ix [nnzLU],
 * level [nJ]; any pointer may be NULL. */
int gbnr_plan_export(const gbnr_plan* plan, int32_t* row_fwd, int32_t* col_fwd, int32_t* col_ptr,
                     int32_t* row_ix, int32_t* level);

/* Batched Newton-Raphson, host buffers in and out (H2D, solve, D2H).
 *   y_re/y_im [nnzY][n_ysets] (NULL = the plan's set; n_ysets = n_tasks for
 *   per-task sets, e.g. N-1 contingencies from gbnr_contingency_values),
 *   p0/q0 [n_bus][n_ssets], vm0/va0 [n_bus][n_vsets],
 *   vm_out/va_out [n_bus][n_tasks], iterations/converged/status/max_mismatch [n_tasks].
 * iterations follow MATPOWER: 0 if V0 already converged, else the number of
 * linear solves; max_iter for diverged tasks. */
int gbnr_solve(gbnr_plan* plan, int32_t n_tasks, const double* y_re, const double* y_im,
               int32_t n_ysets, const double* p0, const double* q0, int32_t n_ssets,
               const double* vm0, const double* va0, int32_t n_vsets, double* vm_out,
               double* va_out, int32_t* iterations_out, uint8_t* converged_out,
               int32_t* status_out, double* max_mismatch_out);

/* Split form of gbnr_solve for device-resident measurement:
 * gbnr_stage copies inputs to the device, gbnr_run solves on them (blocking
 * until done), gbnr_fetch copies results back. */
int gbnr_stage(gbnr_plan* plan, int32_t n_tasks, const double* p0, const double* q0,
               int32_t n_ssets, const double* vm0, const double* va0, int32_t n_vsets);
int gbnr_run(gbnr_plan* plan);
int gbnr_fetch(gbnr_plan* plan, double* vm_out, double* va_out, int32_t* iterations_out,
               uint8_t* converged_out, int32_t* status_out, double* max_mismatch_out);

/* A sequence of batches through one call, pipelined: batch i+1's injections go
 * host->device on a copy stream and batch i-1's voltages device->host on another
 * while batch i solves (batch_runtime.run over mini-batches).
 * Every batch has n_tasks tasks with per-task injections p0[i]/q0[i]
 * [n_bus][n_tasks] and the shared start voltages vm0/va0 [n_bus]; outputs per
 * batch as gbnr_solve (any output array pointer may be NULL).  The injection
 * and voltage host buffers should be pinned for full overlap (the small
 * per-task results go through the plan's own pinned staging). */
int gbnr_solve_batches(gbnr_plan* plan, int32_t n_batches, int32_t n_tasks, const double* const* p0,
                       const double* const* q0, const double* vm0, const double* va0, double* const* vm_out,
                       double* const* va_out, int32_t* const* iterations_out, uint8_t* const* converged_out,
                       int32_t* const* status_out, double* const* max_mismatch_out);

/* calc_branch_flows on the voltages of the last solve of
 * `plan` (still on the device; GBNR_ECONFIG if that solve was sharded over
 * devices or chunked, i.e. the device no longer holds every task): S_from = V_f conj(Yff V_f + Yft V_t), S_to =
 * V_t conj(Ytf V_f + Ytt V_t) per branch and task, zero for the task's outaged
 * branch (outage_branch [n_tasks] or NULL); outputs [n_branch][n_tasks]
 * element-major (any may be NULL).  Computed for every task (diverged ones
 * included); status_out of the solve flags them. */
int gbnr_branch_flows(gbnr_plan* plan, int32_t n_branch, const int32_t* from, const int32_t* to,
                      const double* adm, const int32_t* outage_branch, double* sf_re, double* sf_im,
                      double* st_re, double* st_im);

/* Per-kernel device time of the last gbnr_run/gbnr_solve (CUDA events on the
 * solver stream).  out[24]: [0..4] ms of npm, jacobian, lu, fsbs, vupdate when
 * opt.profile=1 (events recorded around each launch, no host syncs); [5] ms of
 * the whole solve; [6..10] launches of those kernels; [12] Newton iterations
 * executed; [13] tasks; [14] sum over LU launches of task tiles with work
 * (32 tasks each); [15] sum over LU launches of active tasks; [16..18] tasks
 * converged / diverged / singular; [19] kernels launched by the solve. */
int gbnr_last_timing(const gbnr_plan* plan, double* out);

/* Tile-walk execution plans (the static TMA copy programs of the LU+FS, LU-only
 * and BS walks).  which: 0 forward LU+FS, 1 LU only, 2 backward.
 * out[20]: steps, walkers, phases, smem rows, page words, pages per walker,
 * barriers per walker, program words, events, ring-resident dependency rows,
 * fetched rows, ops, copies, shared-memory bytes per CTA, first walker's ring
 * rows and staging rows, steps and dependencies in global memory (blocks /
 * fetches too large for a walker's pool), global scratch rows per walker, 0. */
int gbnr_walk_info(const gbnr_plan* plan, int32_t which, int64_t* out);
/* Raw walk arrays for host-side replay (tests): part 0 program words (int32,
 * walker-major pages), 1 first page per walker (int32 [walkers+1]), 2 owner
 * (int32 [nJ]: phase-0 walker of each column, -1 = top), 3 tape_of_ccs (int32
 * [nnzLU]), 4 lslot (int32 [nJ]), 5 ucrs0 (int32 [nJ+1]). */
int gbnr_walk_export(const gbnr_plan* plan, int32_t which, int32_t part, void* dst);

/* LU-only microbenchmark / parity: the Jacobian at the staged
 * voltages (gbnr_stage) is scattered once into the A tape, then `reps` batched
 * refactorizations A -> LU run back to back (out of place, so every rep does
 * the full work); lu_out [nnzLU][n_tasks] (may be NULL), flags_out [n_tasks]
 * (pivot flagged, may be NULL), ms_out = mean device ms per refactorization
 * (CUDA events on the solver stream). */
int gbnr_refactor(gbnr_plan* plan, int32_t reps, double* lu_out, uint8_t* flags_out,
                  double* ms_out);

#ifdef __cplusplus
}
#endif
#endif
