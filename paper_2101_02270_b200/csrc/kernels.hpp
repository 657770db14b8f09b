// kernels.hpp -- device-side view of a plan and the kernel launchers.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "symbolic.hpp"
#include "walk.hpp"

namespace gbnr {

constexpr int kTile = 32;      // most tasks per tile = lanes of a warp (DevView::tw: the batch's tile width)
constexpr int kSuper = 8;      // tiles per super-tile = warps per block (2 KB access runs)
#ifndef GBNR_ROW_CHUNK
#define GBNR_ROW_CHUNK 4
#endif
constexpr int kRowChunk = GBNR_ROW_CHUNK;  // Ybus rows per warp in the NPM / Jacobian kernels

// Everything a kernel needs, by value (device pointers + sizes).  All per-task
// tapes are element-major: value(elem, task) at elem * bpad + task.
struct DevView {
    int32_t n, nJ, nnzY, n_rows, nnzLU, bpad, n_tiles, n_tasks;
    // tasks per tile (even, 2..32): lane l < tw of a tile's warps owns task
    // tile * tw + l; lanes >= tw shadow lane tw - 1 (same task, same addresses,
    // same values: their loads and stores are duplicates, never a second task)
    int32_t tw;
    // shared structure (read-only, L2-resident)
    const int32_t *yp, *yi;
    const double *yre, *yim;      // Ybus values: slot q of task t at q * y_ld + t * y_inc
    int32_t y_ld, y_inc;          // (1, 0): one shared set; (n_tasks, 1): per task (N-1)
    const int32_t *rows, *brow_p, *brow_q, *zcol_t, *zcol_v;
    const int32_t* lk;
    // per-task tapes [elem][bpad]
    double *vm, *va, *c, *s;
    const double *vm_in, *va_in;  // staged start voltages (kept for repeated runs):
    int32_t vin_ld, vin_inc;      //   bus b of task t at b * vin_ld + t * vin_inc ((1, 0) = shared)
    const double *p0, *q0;
    int32_t s_ld, s_inc;          // p0[bus * s_ld + task * s_inc]
    // tile-blocked tapes, one block per tile of tstride doubles:
    //   [A: tape_rows][LU: tape_rows][b: nJ rows] x tw lanes   (layouts: walk.hpp LuLayout)
    // A = the Jacobian columns, each followed by F_m; LU = the factors with y;
    // b = dx, row nJ-1-k for J column k (backward walk).
    double *A, *LU, *b;           // tile 0's tapes; tile t's at + t * tstride
    size_t tstride;
    int32_t tape_rows;            // nnzLU + 3 nJ
    const int32_t *fslot_p, *fslot_q;  // bus -> A-tape slot of its P / Q mismatch (-1: none)
    // per-task state
    int32_t *status, *iters;
    uint8_t *active, *flag;
    double* maxmis;                 // max-norm at the last check (inf before the first)
    double* mis_prev;               // max-norm one check earlier (inf before)
    double* mis0;                   // max-norm at V0 (representative re-derivation)
    uint8_t* jskip;                 // the last NPM skipped this task's speculative Jacobian
    unsigned long long* norm_bits;  // running max-norm (IEEE bits) of the current NPM
    int32_t *tile_active, *active_count;
    int32_t* it_dev;                // Newton iteration counter on the device
    int32_t* h_counts;              // mapped host memory: [0,32) active tasks, [32,64) active
                                    // tiles per iteration, [64,68) tasks per final status,
                                    // [96,128) active tasks whose Jacobian was not written
    double tol, singular_tol;
    int32_t max_iter;
    int32_t jpolicy;                // gbnr_options.jacobian
    int32_t dbg;                    // experiment switches (GBNR_DBG), 0 in production
    unsigned long long* prof;       // walker time breakdown (GBNR_PROF builds), else null
    // per-tile, per-walker global scratch of the forward walk's global steps (columns
    // too large for shared memory): walker w of tile t at (t * 8 + w) * scratch_rows rows
    double* scratch;
    int32_t scratch_rows;
};

// Device copy of a Walk (walk.hpp).
struct WalkView {
    const int32_t* stream;  // program words (walk.hpp kRec*), walker-major pages
    int32_t walkers, page_words, rows;
    int32_t tw;             // tile width the program's row budget was planned for
    int32_t once_tape;      // tape whose copies this walk reads exactly once (-1: none): L2 evict-first
    int32_t wpage0[17];     // first page of each walker's program (<= 16 walkers)
};

// Most backward-walk warps per CTA (its kernel's launch bound).  12 warps fit three
// CTAs per SM at 56 registers but ran no faster than 8 at 78 (profiles/r02q_bs_walkers.log).
constexpr int kBsWarps = 8;
#ifndef GBNR_LU_WARPS
#define GBNR_LU_WARPS 8
#endif
constexpr int kLuWarps = GBNR_LU_WARPS;  // most forward-walk warps per CTA (its kernel's launch bound)

size_t walk_smem_bytes(const WalkView& w);
void configure_kernels();
int walk_ctas_per_sm(size_t smem, int threads);  // resident LU-walk CTAs per SM
int bs_ctas_per_sm(size_t smem, int threads);    // resident backward-walk CTAs per SM
void launch_init(const DevView& v, cudaStream_t st);
// NPM + convergence + iteration bump; with jac, also the next Jacobian of every
// active task not predicted to converge at this check
void launch_npm(const DevView& v, bool jac, cudaStream_t st);
// Jacobian only: of every active task (all) or of those the last NPM skipped
void launch_jacobian(const DevView& v, bool all, cudaStream_t st);
void launch_status_count(const DevView& v, cudaStream_t st);
void launch_lu_walk(const DevView& v, const WalkView& w, bool fs, cudaStream_t st);
void launch_bs_walk(const DevView& v, const WalkView& w, cudaStream_t st);
void launch_vupdate(const DevView& v, cudaStream_t st);
void launch_broadcast(double* dst, const double* src, int32_t n, int32_t bpad, cudaStream_t st);
void launch_pack(double* dst, const double* src, int32_t n, int32_t n_tasks, int32_t bpad, cudaStream_t st);
void launch_flows(const DevView& v, int32_t nb, const int32_t* bf, const int32_t* bt, const double* adm,
                  const int32_t* outage, double* sfr, double* sfi, double* str, double* sti, cudaStream_t st);

}  // namespace gbnr
