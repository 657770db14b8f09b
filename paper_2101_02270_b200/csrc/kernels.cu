// kernels.cu -- hand-written sm_100a FP64 kernels of one Newton-Raphson iteration.
//
// Layout.  Every per-task tape is element-major, exactly the
// reference's BatchTape (batch_tape.hpp:6-9): value(elem, task) at
// elem * bpad + task, bpad = 32 * n_tiles.  A *tile* is the 32 tasks of one
// warp (one lane per task, 256 B per warp access).  A thread block is 8 warps =
// 8 consecutive tiles (a *super-tile*, 256 tasks) that process the SAME
// structural element (bus row, LU column, triangular-solve row) in lockstep, so
// every global access of a block is a 2 KB contiguous run.  HBM only streams at
// copy speed for runs of >= 2 KB on B200 (tools/membench.cu: 256 B random
// runs reach 1.1 TB/s, 2 KB runs 6.7 TB/s), which is what this layout buys.
//
//   npm_kernel / conv_kernel   compute_npm + convergence (Alg. 1)
//   jacobian_kernel            update_jacobian into the A tape via the static lookup
//                              (signs per SURVEY App. B)
//   lu_level_kernel            refactorize_batch (Alg. 2 operation order)
//                              scheduled level by level (Alg. 3 stage 1):
//                              one launch per level, block = (super-tile, column)
//   tri_level_kernel           fs_bs_batch: pull-style rows per level,
//                              no atomics (deterministic)
//   vupdate_kernel             update_voltage + unit phasor refresh
// Scenarios are independent, so no kernel ever needs a grid-wide barrier; the
// level order is carried by stream order.
#include "../../include/gbnr.h"
#include "kernels.hpp"
#include "numerics.cuh"

#include <algorithm>

namespace gbnr {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double nan_as_inf_abs(double v) {
    const double a = fabs(v);
    return isnan(a) ? INFINITY : a;
}

// tile of warp `warp` in super-tile `st`, or -1 when out of range / finished
__device__ __forceinline__ int my_tile(const DevView& v, int st, int warp) {
    const int tile = st * kSuper + warp;
    return (tile < v.n_tiles && v.tile_active[tile] != 0) ? tile : -1;
}

// ---------------------------------------------------------------------------
// init: working voltages from the staged inputs, unit phasors, task state
// grid (ceil(n/32), n_super), block 256: warp = tile, 32 buses per block
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) init_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.y * kSuper + warp;
    if (tile >= v.n_tiles) return;
    const int t = tile * kTile + lane;
    const bool real = t < v.n_tasks;
    const int b1 = min(v.n, int(blockIdx.x + 1) * 32);
    for (int bus = blockIdx.x * 32; bus < b1; ++bus) {
        const size_t o = size_t(bus) * v.bpad + t;
        const double vm = real ? v.vm_in[o] : 1.0, va = real ? v.va_in[o] : 0.0;
        v.vm[o] = vm;
        v.va[o] = va;
        double s, c;
        gb_sincos(va, &s, &c);
        v.s[o] = s;
        v.c[o] = c;
    }
    if (blockIdx.x == 0) {
        v.status[t] = real ? GBNR_DIVERGED : -1;
        v.iters[t] = 0;
        v.active[t] = real ? 1 : 0;
        v.flag[t] = 0;
        v.maxmis[t] = real ? INFINITY : 0.0;
        v.norm_bits[t] = 0ull;
        const int cnt = __popc(__ballot_sync(kFull, real));
        if (lane == 0) v.tile_active[tile] = cnt;
        if (t == 0) *v.it_dev = 0;
    }
}

// ---------------------------------------------------------------------------
// NPM (Alg. 1, row-level parallelism PAPER.md:183): block (row chunk, super-tile),
// each warp sweeps the chunk's Ybus rows for its tile; partial max-norms merge
// with an exact integer atomicMax on the (non-negative) IEEE bits.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) npm_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = my_tile(v, blockIdx.y, warp);
    if (tile < 0) return;
    const int t = tile * kTile + lane;
    const size_t bp = v.bpad;
    double nrm = 0.0;
    const int r1 = min(v.n_rows, int(blockIdx.x + 1) * kRowChunk);
    for (int ri = blockIdx.x * kRowChunk; ri < r1; ++ri) {
        const int r = __ldg(v.rows + ri);
        double ire = 0.0, iim = 0.0;
        const int q1 = __ldg(v.yp + r + 1);
        for (int q = __ldg(v.yp + r); q < q1; ++q) {
            const int k = __ldg(v.yi + q);
            const double vmk = v.vm[k * bp + t];
            acc_current(__ldg(v.yre + q), __ldg(v.yim + q), vmk * v.c[k * bp + t],
                        vmk * v.s[k * bp + t], ire, iim);
        }
        const double vmr = v.vm[r * bp + t];
        const double vre = vmr * v.c[r * bp + t], vim = vmr * v.s[r * bp + t];
        double P, Q;
        injection(vre, vim, ire, iim, P, Q);
        const double fp = P - v.p0[size_t(r) * v.s_ld + size_t(t) * v.s_inc];
        v.b[size_t(__ldg(v.brow_p + r)) * bp + t] = fp;
        nrm = fmax(nrm, nan_as_inf_abs(fp));
        const int bq = __ldg(v.brow_q + r);
        if (bq >= 0) {
            const double fq = Q - v.q0[size_t(r) * v.s_ld + size_t(t) * v.s_inc];
            v.b[size_t(bq) * bp + t] = fq;
            nrm = fmax(nrm, nan_as_inf_abs(fq));
        }
    }
    atomicMax(v.norm_bits + t, static_cast<unsigned long long>(__double_as_longlong(nrm)));
}

// Convergence / status per task (MATPOWER iteration convention).
__global__ void __launch_bounds__(256) conv_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x * kSuper + warp;
    if (tile >= v.n_tiles) return;
    const int t = tile * kTile + lane;
    const int it = *v.it_dev;
    const double m = __longlong_as_double(static_cast<long long>(v.norm_bits[t]));
    v.norm_bits[t] = 0ull;
    bool act = v.tile_active[tile] != 0 && v.active[t] != 0;
    if (act) {
        v.maxmis[t] = m;
        if (m < v.tol) {
            v.status[t] = GBNR_CONVERGED;
            v.iters[t] = it;
            v.active[t] = 0;
            act = false;
        } else if (it >= v.max_iter) {
            v.status[t] = GBNR_DIVERGED;
            v.iters[t] = v.max_iter;
            v.active[t] = 0;
            act = false;
        }
    }
    const int cnt = __popc(__ballot_sync(kFull, act));
    if (lane == 0) {
        v.tile_active[tile] = cnt;
        if (cnt) {
            atomicAdd(v.active_count + it, cnt);     // active tasks after iteration it
            atomicAdd(v.active_count + 32 + it, 1);  // tiles with work left
        }
    }
}

__global__ void bump_kernel(DevView v) { *v.it_dev += 1; }

// ---------------------------------------------------------------------------
// Jacobian -> A tape (LU slot order; fill slots are never written and stay 0).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) jacobian_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = my_tile(v, blockIdx.y, warp);
    if (tile < 0) return;
    const int t = tile * kTile + lane;
    const bool act = v.active[t] != 0;
    if (blockIdx.x == 0) v.flag[t] = 0;  // pivot flags of this iteration's refactorization
    const size_t bp = v.bpad;
    const int r1 = min(v.n_rows, int(blockIdx.x + 1) * kRowChunk);
    for (int ri = blockIdx.x * kRowChunk; ri < r1; ++ri) {
        const int r = __ldg(v.rows + ri);
        const int q0 = __ldg(v.yp + r), q1 = __ldg(v.yp + r + 1);
        double ire = 0.0, iim = 0.0;
        for (int q = q0; q < q1; ++q) {
            const int k = __ldg(v.yi + q);
            const double vmk = v.vm[k * bp + t];
            acc_current(__ldg(v.yre + q), __ldg(v.yim + q), vmk * v.c[k * bp + t],
                        vmk * v.s[k * bp + t], ire, iim);
        }
        const double vmr = v.vm[r * bp + t];
        const double vre = vmr * v.c[r * bp + t], vim = vmr * v.s[r * bp + t];
        double P, Q;
        injection(vre, vim, ire, iim, P, Q);
        for (int q = q0; q < q1; ++q) {
            const int k = __ldg(v.yi + q);
            const double ck = v.c[k * bp + t], sk = v.s[k * bp + t], vmk = v.vm[k * bp + t];
            double zre, zim, j[4];
            jac_z(__ldg(v.yre + q), __ldg(v.yim + q), vre, vim, ck, sk, zre, zim);
            jac_entries(k == r, zre, zim, vmk, ck, sk, ire, iim, P, Q, j);
            const int4 l = __ldg(reinterpret_cast<const int4*>(v.lk) + q);
            if (act) {
                if (l.x >= 0) v.A[size_t(l.x) * bp + t] = j[0];
                if (l.y >= 0) v.A[size_t(l.y) * bp + t] = j[1];
                if (l.z >= 0) v.A[size_t(l.z) * bp + t] = j[2];
                if (l.w >= 0) v.A[size_t(l.w) * bp + t] = j[3];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// LU column engine (cp.async).  The working column x (len slot rows of the
// warp's 32 tasks) and a 32-row ring of L values live in shared memory; every
// global->shared move is an asynchronous 16 B-per-lane copy (two 256 B rows per
// warp instruction), so a warp keeps up to (len + 32) rows in flight without
// spending registers.  Update records sit in three 32-record register windows
// (consume / issue / prefetch) broadcast with shuffles.  The per-element
// operation order is exactly Alg. 2's, so results are bit-identical.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// lanes 0-15 copy row a, lanes 16-31 row b (a row = the 32 tasks of one slot)
__device__ __forceinline__ void cp_rows(double* da, const double* sa, double* db, const double* sb,
                                        int lane) {
    const int c = (lane & 15) * 2;
    if (lane < 16) {
        if (da) cp16(da + c, sa + c);
    } else {
        if (db) cp16(db + c, sb + c);
    }
}

constexpr int kRing = 32;  // ring rows = one record window

// issue the L-value copies of updates [u, u+8) into ring rows u % 32; the LU
// slot of update u+q sits in lane (u+q) % 32 of the issue window w
__device__ __forceinline__ void ring_issue(double* ring, const double* lu_t, size_t bp, int w, int u,
                                           int nu, int lane) {
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
        const int a = u + q, b = u + q + 1;
        const int la = __shfl_sync(kFull, w, a & 31), lb = __shfl_sync(kFull, w, b & 31);
        cp_rows(a < nu ? ring + (a & 31) * kTile : nullptr, lu_t + size_t(la) * bp,
                b < nu ? ring + (b & 31) * kTile : nullptr, lu_t + size_t(lb) * bp, lane);
    }
}

// One column j of Alg. 2 for the 32 tasks of a tile.  a_t / lu_t point at the
// tile's first task (no lane offset); x rows are 32 doubles.
__device__ __forceinline__ bool column_async(const DevView& v, double* xw, double* ring,
                                             const double* a_t, double* lu_t, int s0, int len,
                                             int dp, int u0, int nu, int lane) {
    const size_t bp = v.bpad;
    const int* ls = v.upd_ls + u0;
    const int* dk = v.upd_dk + u0;
    const int wls0 = __ldg(ls + lane);  // ls window 0 (prologue issue)
    int wdk = __ldg(dk + lane);         // dk window 0
    int wls = __ldg(ls + 32 + lane);    // ls window 1
    int wls_n = __ldg(ls + 64 + lane);  // ls window 2 (prefetch)
    int wdk_n = __ldg(dk + 32 + lane);  // dk window 1 (prefetch)
    const double* a_col = a_t + size_t(s0) * bp;
    for (int z = 0; z < len; z += 2)
        cp_rows(xw + z * kTile, a_col + size_t(z) * bp, z + 1 < len ? xw + (z + 1) * kTile : nullptr,
                a_col + size_t(z + 1) * bp, lane);
    cp_commit();
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        ring_issue(ring, lu_t, bp, wls0, g * 8, nu, lane);
        cp_commit();
    }
    cp_wait<4>();
    __syncwarp();
    double* xl = xw + lane;
    const double* rl = ring + lane;
    for (int u = 0; u < nu; u += 8) {
        cp_wait<3>();
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int d = __shfl_sync(kFull, wdk, (u + q) & 31);
            if (u + q < nu) {
                const int dst = d & 0xffff, kp = d >> 16;
                xl[dst * kTile] = fma(-xl[kp * kTile], rl[((u + q) & 31) * kTile], xl[dst * kTile]);
            }
        }
        __syncwarp();
        ring_issue(ring, lu_t, bp, wls, u + 32, nu, lane);
        cp_commit();
        if (((u + 8) & 31) == 0) {  // crossed into the next record window
            wdk = wdk_n;
            wls = wls_n;
            const int nb = u + 8 + 32;
            wdk_n = nb < nu ? __ldg(dk + nb + lane) : 0;
            wls_n = nb + 32 < nu ? __ldg(ls + nb + 32 + lane) : 0;
        }
    }
    cp_wait<0>();
    __syncwarp();
    // pivot check and normalization L = x * (1 / pivot)
    const double piv = xl[dp * kTile];
    double cmax = 0.0;
    for (int z = 0; z < len; ++z) cmax = fmax(cmax, fabs(xl[z * kTile]));
    const bool flagged = isfinite(cmax) && (piv == 0.0 || fabs(piv) < v.singular_tol * cmax);
    const double inv = 1.0 / piv;
    double* out = lu_t + size_t(s0) * bp + lane;
    for (int z = 0; z < len; ++z) {
        const double xv = xl[z * kTile];
        out[size_t(z) * bp] = z > dp ? xv * inv : xv;
    }
    return flagged;
}

// Long columns (len > CAPX): the working column stays in the LU tape (in place),
// L loads batched 8 at a time in registers.  Same operation order.
__device__ __forceinline__ bool column_inplace(const DevView& v, const double* a_t, double* lu_t,
                                               int s0, int len, int dp, int u0, int nu, int lane) {
    const size_t bp = v.bpad;
    const double* a = a_t + size_t(s0) * bp + lane;
    double* x = lu_t + size_t(s0) * bp + lane;
    const double* lut = lu_t + lane;
    for (int z0 = 0; z0 < len; z0 += 8) {
        double av[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) av[q] = z0 + q < len ? a[size_t(z0 + q) * bp] : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (z0 + q < len) x[size_t(z0 + q) * bp] = av[q];
    }
    const int* ls = v.upd_ls + u0;
    const int* dk = v.upd_dk + u0;
    for (int c = 0; c < nu; c += 32) {
        const int wl = __ldg(ls + c + lane), wd = __ldg(dk + c + lane);
        const int m = min(32, nu - c);
        for (int g = 0; g < m; g += 8) {
            double l[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int s = __shfl_sync(kFull, wl, (g + q) & 31);
                l[q] = g + q < m ? lut[size_t(s) * bp] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int d = __shfl_sync(kFull, wd, (g + q) & 31);
                if (g + q < m) {
                    const size_t dst = size_t(d & 0xffff) * bp, kp = size_t(d >> 16) * bp;
                    x[dst] = fma(-x[kp], l[q], x[dst]);
                }
            }
        }
    }
    const double piv = x[size_t(dp) * bp];
    double cmax = 0.0;
    for (int z = 0; z < len; ++z) cmax = fmax(cmax, fabs(x[size_t(z) * bp]));
    const bool flagged = isfinite(cmax) && (piv == 0.0 || fabs(piv) < v.singular_tol * cmax);
    const double inv = 1.0 / piv;
    for (int z = dp + 1; z < len; ++z) x[size_t(z) * bp] *= inv;
    return flagged;
}

// One launch per level: block (super-tile, column of the level), warp = tile.
// All U dependencies sit in earlier levels, complete by stream order.
template <int CAPX>
__global__ void __launch_bounds__(256) lu_level_kernel(DevView v, const int32_t* sched, int pos0) {
    extern __shared__ double sm_all[];  // per warp [CAPX + 32 ring][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = my_tile(v, blockIdx.x, warp);
    if (tile < 0) return;
    const int j = __ldg(sched + pos0 + blockIdx.y);
    const int4* ci = reinterpret_cast<const int4*>(v.col);
    const int4 c0 = __ldg(ci + 2 * j), c1 = __ldg(ci + 2 * j + 1);
    const int s0 = c0.x, len = c0.y & 0xffff, dp = c0.y >> 16;
    const double* a_t = v.A + size_t(tile) * kTile;
    double* lu_t = v.LU + size_t(tile) * kTile;
    bool flagged;
    if (len <= CAPX) {
        double* xw = sm_all + size_t(warp) * (CAPX + kRing) * kTile;
        flagged = column_async(v, xw, xw + CAPX * kTile, a_t, lu_t, s0, len, dp, c1.x, c1.y, lane);
    } else {
        flagged = column_inplace(v, a_t, lu_t, s0, len, dp, c1.x, c1.y, lane);
    }
    if (flagged) v.flag[size_t(tile) * kTile + lane] = 1;
}

// ---------------------------------------------------------------------------
// Warp-specialized TMA pipeline for the short columns of a level.
//
// Persistent blocks (one per SM) walk (column, super-tile) items round-robin.
// Warp 8 is the producer: with cp.async.bulk (the TMA engine, no registers, no
// per-lane addressing) it copies each item's A rows -- 2 KB = one super-tile's
// slice of a slot row -- into one of two x buffers, and the L rows every update
// of the item reads into a ring of 8-row stages, all completion-tracked by
// mbarriers (expect_tx).  Warps 0-7 are consumers, one per tile of the
// super-tile: they wait on the stage barriers, apply Alg. 2's updates in order
// out of shared memory, normalise, write the column back and release buffers.
// The producer runs up to a whole ring ahead across item boundaries, so HBM
// sees long streams of 2 KB requests with deep queues.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    while (!mbar_try(b, parity)) {
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

constexpr int kPipeStages = 6;  // ring stages of 8 rows
constexpr int kRowBytes = kSuper * kTile * 8;  // 2 KB: one super-tile's slice of a slot row
constexpr int kPipeThreads = (kSuper + 1) * 32;

constexpr int kPipeXRows = 48;  // x region: 4 x 12, 3 x 16 or 2 x 24 rows (per level)
struct PipeSmem {
    double x[kPipeXRows][kSuper * kTile];
    double ring[kPipeStages][8][kSuper * kTile];
    unsigned long long x_full[4], x_empty[4], r_full[kPipeStages], r_empty[kPipeStages];
};

__global__ void __launch_bounds__(kPipeThreads, 1) lu_pipe_kernel(DevView v, const int32_t* sched,
                                                                  int pos0, int ncols, int nxb) {
    extern __shared__ __align__(128) unsigned char pipe_raw[];
    PipeSmem& S = *reinterpret_cast<PipeSmem*>(pipe_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_st = (v.n_tiles + kSuper - 1) / kSuper, items = ncols * n_st;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(&S.x_full[i], 1);
            mbar_init(&S.x_empty[i], kSuper);
        }
        for (int i = 0; i < kPipeStages; ++i) {
            mbar_init(&S.r_full[i], 1);
            mbar_init(&S.r_empty[i], kSuper);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const size_t bp = v.bpad;
    const int4* ci = reinterpret_cast<const int4*>(v.col);
    int n_item = 0, stage = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int cidx = item / n_st, st = item - cidx * n_st;
        // skip super-tiles with nothing left to solve (same decision on every warp)
        bool any = false;
        for (int w = 0; w < kSuper; ++w) {
            const int tl = st * kSuper + w;
            any |= tl < v.n_tiles && v.tile_active[tl] != 0;
        }
        if (!any) continue;
        const int j = __ldg(sched + pos0 + cidx);
        const int4 c0 = __ldg(ci + 2 * j), c1 = __ldg(ci + 2 * j + 1);
        const int s0 = c0.x, len = c0.y & 0xffff, dp = c0.y >> 16, u0 = c1.x, nu = c1.y;
        const int xb = n_item % nxb;                    // x buffer of this item
        const unsigned xpar = (n_item / nxb) & 1;
        double (*xbuf)[kSuper * kTile] = S.x + xb * (kPipeXRows / nxb);
        const size_t col_off = size_t(st) * kSuper * kTile;  // first task of the super-tile
        if (warp == kSuper) {
            // ---------------- producer ----------------
            mbar_wait(&S.x_empty[xb], xpar ^ 1);
            if (lane == 0) mbar_expect_tx(&S.x_full[xb], unsigned(len) * kRowBytes);
            __syncwarp();
            if (lane < len) bulk_g2s(xbuf[lane], v.A + size_t(s0 + lane) * bp + col_off, kRowBytes, &S.x_full[xb]);
            const int* ls = v.upd_ls + u0;
            for (int u = 0; u < nu; u += 8, ++stage) {
                const int slot = stage % kPipeStages;
                const unsigned spar = (stage / kPipeStages) & 1;
                const int m = min(8, nu - u);
                const int lsv = lane < m ? __ldg(ls + u + lane) : 0;
                mbar_wait(&S.r_empty[slot], spar ^ 1);
                if (lane == 0) mbar_expect_tx(&S.r_full[slot], unsigned(m) * kRowBytes);
                __syncwarp();
                if (lane < m) bulk_g2s(S.ring[slot][lane], v.LU + size_t(lsv) * bp + col_off, kRowBytes, &S.r_full[slot]);
            }
        } else {
            // ---------------- consumers ----------------
            const int tile = st * kSuper + warp;
            const bool act = tile < v.n_tiles && v.tile_active[tile] != 0;
            const int* dk = v.upd_dk + u0;
            mbar_wait(&S.x_full[xb], xpar);
            double* xl = &xbuf[0][warp * kTile + lane];
            int wdk = __ldg(dk + lane);
            for (int u = 0; u < nu; u += 8, ++stage) {
                const int slot = stage % kPipeStages;
                const unsigned spar = (stage / kPipeStages) & 1;
                const int m = min(8, nu - u);
                mbar_wait(&S.r_full[slot], spar);
                if (act) {
                    const double* rl = &S.ring[slot][0][warp * kTile + lane];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int d = __shfl_sync(kFull, wdk, (u + q) & 31);
                        if (q < m) {
                            const int dst = d & 0xffff, kp = d >> 16;
                            xl[dst * (kSuper * kTile)] =
                                fma(-xl[kp * (kSuper * kTile)], rl[q * (kSuper * kTile)], xl[dst * (kSuper * kTile)]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.r_empty[slot]);
                if (((u + 8) & 31) == 0) wdk = u + 8 < nu ? __ldg(dk + u + 8 + lane) : 0;
            }
            if (act) {
                // pivot check and normalization L = x * (1 / pivot)
                const double piv = xl[dp * (kSuper * kTile)];
                double cmax = 0.0;
                for (int z = 0; z < len; ++z) cmax = fmax(cmax, fabs(xl[z * (kSuper * kTile)]));
                const bool flagged = isfinite(cmax) && (piv == 0.0 || fabs(piv) < v.singular_tol * cmax);
                const double inv = 1.0 / piv;
                double* out = v.LU + size_t(s0) * bp + size_t(tile) * kTile + lane;
                for (int z = 0; z < len; ++z) {
                    const double xv = xl[z * (kSuper * kTile)];
                    out[size_t(z) * bp] = z > dp ? xv * inv : xv;
                }
                if (flagged) v.flag[size_t(tile) * kTile + lane] = 1;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.x_empty[xb]);
        }
        ++n_item;
    }
}

// ---------------------------------------------------------------------------
// Warp-specialized TMA pipeline for one triangular-solve level (rows of L for
// FS, of U for BS).  Item = (row i, super-tile).  The producer warp copies,
// per item, a head slot {b(i) row, diag row (BS)} and, in 8-entry stages, the
// (LU(i,k) row, b(k) row) pairs of the row's entries; consumers accumulate in
// the fixed per-element order (k ascending for FS, descending for BS).
// ---------------------------------------------------------------------------
constexpr int kTriStages = 5;
constexpr int kTriHeads = 8;
struct TriSmem {
    double ring[kTriStages][8][2][kSuper * kTile];  // [stage][entry][LU row, b row]
    double head[kTriHeads][2][kSuper * kTile];      // [slot][b(i) row, diag row]
    unsigned long long r_full[kTriStages], r_empty[kTriStages], h_full[kTriHeads], h_empty[kTriHeads];
};

template <bool BACK>
__global__ void __launch_bounds__(kPipeThreads, 1) tri_pipe_kernel(DevView v, int pos0, int nrows) {
    extern __shared__ __align__(128) unsigned char tri_raw[];
    TriSmem& S = *reinterpret_cast<TriSmem*>(tri_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_st = (v.n_tiles + kSuper - 1) / kSuper, items = nrows * n_st;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kTriStages; ++i) {
            mbar_init(&S.r_full[i], 1);
            mbar_init(&S.r_empty[i], kSuper);
        }
        for (int i = 0; i < kTriHeads; ++i) {
            mbar_init(&S.h_full[i], 1);
            mbar_init(&S.h_empty[i], kSuper);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const size_t bp = v.bpad;
    const int32_t* sched = BACK ? v.bs_sched : v.fs_sched;
    const int4* rif = reinterpret_cast<const int4*>(BACK ? v.urow : v.lrow);
    const int4* enf = reinterpret_cast<const int4*>(BACK ? v.uent : v.lent);
    int n_item = 0, stage = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int r = item / n_st, st = item - r * n_st;
        bool any = false;
        for (int w = 0; w < kSuper; ++w) {
            const int tl = st * kSuper + w;
            any |= tl < v.n_tiles && v.tile_active[tl] != 0;
        }
        if (!any) continue;
        const int i = __ldg(sched + pos0 + r);
        const int4 ri = __ldg(rif + i);
        const int e0 = ri.x, ne = ri.y;
        const int hs = n_item % kTriHeads;
        const unsigned hpar = (n_item / kTriHeads) & 1;
        const size_t col_off = size_t(st) * kSuper * kTile;
        if (warp == kSuper) {
            // ---------------- producer ----------------
            mbar_wait(&S.h_empty[hs], hpar ^ 1);
            if (lane == 0) mbar_expect_tx(&S.h_full[hs], (BACK ? 2u : 1u) * kRowBytes);
            __syncwarp();
            if (lane == 0) bulk_g2s(S.head[hs][0], v.b + size_t(i) * bp + col_off, kRowBytes, &S.h_full[hs]);
            if (BACK && lane == 1)
                bulk_g2s(S.head[hs][1], v.LU + size_t(ri.z) * bp + col_off, kRowBytes, &S.h_full[hs]);
            for (int c = 0; c < ne; c += 8, ++stage) {
                const int slot = stage % kTriStages;
                const unsigned spar = (stage / kTriStages) & 1;
                const int m = min(8, ne - c);
                const int4 en = lane < m ? __ldg(enf + e0 + c + lane) : make_int4(0, 0, 0, 0);
                mbar_wait(&S.r_empty[slot], spar ^ 1);
                if (lane == 0) mbar_expect_tx(&S.r_full[slot], unsigned(2 * m) * kRowBytes);
                __syncwarp();
                if (lane < m) {
                    bulk_g2s(S.ring[slot][lane][0], v.LU + size_t(en.x) * bp + col_off, kRowBytes, &S.r_full[slot]);
                    bulk_g2s(S.ring[slot][lane][1], v.b + size_t(en.y) * bp + col_off, kRowBytes, &S.r_full[slot]);
                }
            }
        } else {
            // ---------------- consumers ----------------
            const int tile = st * kSuper + warp;
            const bool act = tile < v.n_tiles && v.tile_active[tile] != 0;
            const int off = warp * kTile + lane;
            mbar_wait(&S.h_full[hs], hpar);
            double acc = S.head[hs][0][off];
            for (int c = 0; c < ne; c += 8, ++stage) {
                const int slot = stage % kTriStages;
                const unsigned spar = (stage / kTriStages) & 1;
                const int m = min(8, ne - c);
                mbar_wait(&S.r_full[slot], spar);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < m) acc = fma(-S.ring[slot][q][0][off], S.ring[slot][q][1][off], acc);
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.r_empty[slot]);
            }
            if (BACK) acc = acc / S.head[hs][1][off];
            if (act) v.b[size_t(i) * bp + size_t(tile) * kTile + lane] = acc;
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.h_empty[hs]);
        }
        ++n_item;
    }
}

// ---------------------------------------------------------------------------
// Triangular solves, one launch per level: block (super-tile, row), warp =
// tile.  Pull-style rows: FS  y(i) = b(i) - sum_k L(i,k) y(k)  (k ascending),
// BS x(i) = (y(i) - sum_k U(i,k) x(k)) / U(i,i)  (k descending) -- the same
// per-element order as the column-oriented sequential FS/BS, no atomics.
// ---------------------------------------------------------------------------
template <bool BACK>
__global__ void __launch_bounds__(256) tri_level_kernel(DevView v, int pos0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = my_tile(v, blockIdx.x, warp);
    if (tile < 0) return;
    const size_t bp = v.bpad;
    const int i = __ldg((BACK ? v.bs_sched : v.fs_sched) + pos0 + blockIdx.y);
    const int4 ri = __ldg(reinterpret_cast<const int4*>(BACK ? v.urow : v.lrow) + i);
    const int4* enf = reinterpret_cast<const int4*>(BACK ? v.uent : v.lent);
    const double* __restrict__ lut = v.LU + size_t(tile) * kTile + lane;
    double* bt = v.b + size_t(tile) * kTile + lane;
    double acc = bt[size_t(i) * bp];
    const int e0 = ri.x, ne = ri.y;
    for (int c = 0; c < ne; c += 32) {
        const int4 en = c + lane < ne ? __ldg(enf + e0 + c + lane) : make_int4(0, 0, 0, 0);
        const int m = min(32, ne - c);
        for (int g = 0; g < m; g += 8) {
            double l[8], xb[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int sl = __shfl_sync(kFull, en.x, (g + q) & 31);
                const int k = __shfl_sync(kFull, en.y, (g + q) & 31);
                l[q] = g + q < m ? lut[size_t(sl) * bp] : 0.0;
                xb[q] = g + q < m ? bt[size_t(k) * bp] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (g + q < m) acc = fma(-l[q], xb[q], acc);
        }
    }
    if (BACK) acc = acc / lut[size_t(ri.z) * bp];
    bt[size_t(i) * bp] = acc;
}

// ---------------------------------------------------------------------------
// V update for active tasks: va -= dtheta, vm -= d|V|; refresh (cos, sin).
// block (32-bus chunk, super-tile), warp = tile.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) vupdate_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = my_tile(v, blockIdx.y, warp);
    if (tile < 0) return;
    const int t = tile * kTile + lane;
    if (!v.active[t]) return;
    if (v.flag[t]) {  // frozen pivot collapsed: stop, never update V
        if (blockIdx.x == 0) {
            v.status[t] = GBNR_SINGULAR;
            v.iters[t] = *v.it_dev;
            v.active[t] = 0;
        }
        return;
    }
    const size_t bp = v.bpad;
    const int b1 = min(v.n, int(blockIdx.x + 1) * 32);
    for (int bus = blockIdx.x * 32; bus < b1; ++bus) {
        const int zt = __ldg(v.zcol_t + bus);
        if (zt < 0) continue;
        const size_t o = size_t(bus) * bp + t;
        const double va = v.va[o] - v.b[size_t(zt) * bp + t];
        v.va[o] = va;
        const int zv = __ldg(v.zcol_v + bus);
        if (zv >= 0) v.vm[o] = v.vm[o] - v.b[size_t(zv) * bp + t];
        double s, c;
        gb_sincos(va, &s, &c);
        v.s[o] = s;
        v.c[o] = c;
    }
}

__global__ void broadcast_kernel(double* dst, const double* src, int32_t n, int32_t bpad) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < size_t(n) * bpad) dst[i] = src[i / bpad];
}

constexpr int kCapX = 24;     // lu_level_kernel: 8 x (24 + 32) x 256 B = 112 KB -> 2 blocks / SM
constexpr int kCapLong = 80;  // long-column levels: 8 x (80 + 32) x 256 B = 224 KB

unsigned n_super(const DevView& v) { return unsigned((v.n_tiles + kSuper - 1) / kSuper); }

int g_num_sms = 148;

}  // namespace

size_t lu_smem_bytes() { return size_t(kSuper) * (kCapX + kRing) * kTile * sizeof(double); }
static size_t long_smem_bytes() { return size_t(kSuper) * (kCapLong + kRing) * kTile * sizeof(double); }

void configure_kernels() {
    cudaFuncSetAttribute(lu_level_kernel<kCapX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(lu_smem_bytes()));
    cudaFuncSetAttribute(lu_level_kernel<kCapX>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(lu_level_kernel<kCapLong>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(long_smem_bytes()));
    cudaFuncSetAttribute(lu_level_kernel<kCapLong>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(lu_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PipeSmem)));
    cudaFuncSetAttribute(tri_pipe_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(TriSmem)));
    cudaFuncSetAttribute(tri_pipe_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(TriSmem)));
    cudaFuncSetAttribute(lu_pipe_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
}

void launch_init(const DevView& v, cudaStream_t st) {
    init_kernel<<<dim3(unsigned((v.n + 31) / 32), n_super(v)), 256, 0, st>>>(v);
}

void launch_npm(const DevView& v, cudaStream_t st) {
    npm_kernel<<<dim3(unsigned((v.n_rows + kRowChunk - 1) / kRowChunk), n_super(v)), 256, 0, st>>>(v);
    conv_kernel<<<n_super(v), 256, 0, st>>>(v);
    bump_kernel<<<1, 1, 0, st>>>(v);
}

void launch_jacobian(const DevView& v, cudaStream_t st) {
    jacobian_kernel<<<dim3(unsigned((v.n_rows + kRowChunk - 1) / kRowChunk), n_super(v)), 256, 0, st>>>(v);
}

// Level launch: wide levels use the persistent pipelined kernel (one block per
// SM); levels holding a column longer than the pipeline's 24-row working set
// use the one-item-per-block kernel with an 80-row working set; the rest the
// one-item kernel with 2 blocks per SM.
void launch_lu_short(const DevView& v, int pos0, int ncols, int maxlen, cudaStream_t st) {
    if (ncols <= 0) return;
    const size_t items = size_t(ncols) * n_super(v);
    const unsigned grid = unsigned(std::min<size_t>(items, size_t(g_num_sms)));
    const int nxb = maxlen <= 12 ? 4 : (maxlen <= 16 ? 3 : 2);  // x buffers in flight
    lu_pipe_kernel<<<grid, kPipeThreads, sizeof(PipeSmem), st>>>(v, v.lu_short, pos0, ncols, nxb);
}

void launch_lu_long(const DevView& v, int pos0, int ncols, int maxlen, cudaStream_t st) {
    if (ncols <= 0) return;
    if (maxlen > kCapX)
        lu_level_kernel<kCapLong><<<dim3(n_super(v), unsigned(ncols)), 256, long_smem_bytes(), st>>>(
            v, v.lu_long, pos0);
    else
        lu_level_kernel<kCapX><<<dim3(n_super(v), unsigned(ncols)), 256, lu_smem_bytes(), st>>>(
            v, v.lu_long, pos0);
}

void launch_tri_level(const DevView& v, bool back, int pos0, int nrows, cudaStream_t st) {
    if (nrows <= 0) return;
    const size_t items = size_t(nrows) * n_super(v);
    const unsigned grid = unsigned(std::min<size_t>(items, size_t(g_num_sms)));
    if (back)
        tri_pipe_kernel<true><<<grid, kPipeThreads, sizeof(TriSmem), st>>>(v, pos0, nrows);
    else
        tri_pipe_kernel<false><<<grid, kPipeThreads, sizeof(TriSmem), st>>>(v, pos0, nrows);
}

void launch_vupdate(const DevView& v, cudaStream_t st) {
    vupdate_kernel<<<dim3(unsigned((v.n + 31) / 32), n_super(v)), 256, 0, st>>>(v);
}

void launch_broadcast(double* dst, const double* src, int32_t n, int32_t bpad, cudaStream_t st) {
    const size_t tot = size_t(n) * bpad;
    broadcast_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(dst, src, n, bpad);
}

}  // namespace gbnr
