// kernels.hpp -- device-side view of a plan and the kernel launchers.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "symbolic.hpp"

namespace gbnr {

constexpr int kTile = 32;  // tasks per task tile = lanes of a warp

// Everything a kernel needs, by value (device pointers + sizes).
struct DevView {
    int32_t n, nJ, nnzY, n_rows, nnzLU, nA, bpad, n_tiles;
    // shared structure (read-only, L2-resident)
    const int32_t *yp, *yi;
    const double *yre, *yim;
    const int32_t *rows, *brow_p, *brow_q, *zcol_t, *zcol_v;
    const int32_t* lk;
    const ColInfo* col;
    const int32_t* dep_wait;
    const Upd* upd;
    const int32_t* lu_sched;
    const RowInfo *lrow, *urow;
    const RowEnt *lent, *uent;
    const int32_t *fs_sched, *bs_sched;
    // per-task tapes, element-major [elem][bpad]
    double *vm, *va, *c, *s;
    const double *vm_in, *va_in;  // staged start voltages (kept for repeated runs)
    const double *p0, *q0;
    int32_t s_ld, s_inc;  // p0[bus * s_ld + task * s_inc]
    // per-tile tapes [tile][elem][32]
    double *A, *LU, *b;
    // per-task state
    int32_t *status, *iters;
    uint8_t *active, *flag;
    double* maxmis;
    int32_t *tile_active, *active_count;
    double tol, singular_tol;
    int32_t max_iter, n_tasks;
    long long* lu_stats;  // optional per-warp cycle breakdown (GBNR_LU_STATS=1)
};

struct LaunchCfg {
    int lu_warps = 8;   // warps per CTA in LU
    int fs_warps = 8;   // warps per CTA in FS-BS
    int row_warps = 8;  // warps per CTA in NPM / Jacobian
    int lu_cap = 32;    // smem working-column capacity (rows) per warp
};

void launch_init(const DevView& v, cudaStream_t st);
void launch_npm(const DevView& v, const LaunchCfg& c, int it, cudaStream_t st);
void launch_jacobian(const DevView& v, const LaunchCfg& c, cudaStream_t st);
void launch_lu(const DevView& v, const LaunchCfg& c, cudaStream_t st);
void launch_fsbs(const DevView& v, const LaunchCfg& c, int it, cudaStream_t st);
void launch_vupdate(const DevView& v, cudaStream_t st);
void launch_broadcast(double* dst, const double* src, int32_t n, int32_t bpad, cudaStream_t st);
size_t lu_smem_bytes(const LaunchCfg& c);
void configure_kernels(const LaunchCfg& c);

}  // namespace gbnr
